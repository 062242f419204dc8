# lean kernel first correctness + timing pass
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2b_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1
timeout 300 python tools/sim_times.py --only grid > gpurun_out/r2b_simtimes.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench.log 2>&1
