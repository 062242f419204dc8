timeout 600 python tools/timeline.py > gpurun_out/r2q_timeline_grid.txt 2>&1
timeout 900 python tools/timeline.py --full > gpurun_out/r2q_timeline_full.txt 2>&1
