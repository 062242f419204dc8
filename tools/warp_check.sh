# parity + sweep time of the opt-in warp-per-simulation build (libsimsweep_warp.so, -DSIM_WARP_SMALL)
SIMSWEEP_LIB=paper_2411_07447_b200/libsimsweep_warp.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_warp.log 2>&1
echo "tests rc=$?" >> gpurun_out/gputests_warp.log
SIMSWEEP_LIB=paper_2411_07447_b200/libsimsweep_warp.so timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_warp.log 2>&1
