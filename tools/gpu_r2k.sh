timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2k_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2k_gputests.log
timeout 600 python tools/sim_times.py --only online > gpurun_out/r2k_simtimes_online.log 2>&1
