timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2d_gputests.log
timeout 300 python tools/sim_times.py --only grid > gpurun_out/r2d_simtimes.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2d_bench.log 2>&1
