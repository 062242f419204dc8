timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/r2af_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2af_gputests.log
for l in ablibs/lib_v10.so ablibs/lib_v11.so; do SIMSWEEP_LIB=$l timeout 300 python tools/crit_times.py >> gpurun_out/r2af_ab.log 2>&1; done
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2af_bench_grid.json 2> gpurun_out/r2af_bench_grid.err
