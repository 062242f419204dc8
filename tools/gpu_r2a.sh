set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 600 python tools/sim_times.py > gpurun_out/r2a_simtimes.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2a_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2a_bench.log 2>&1
