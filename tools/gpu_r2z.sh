timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/r2z_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2z_gputests.log
SIMSWEEP_LIB=ablibs/lib_v3.so timeout 300 python tools/crit_times.py >> gpurun_out/r2z_ab.log 2>&1
SIMSWEEP_LIB=ablibs/lib_v5.so timeout 300 python tools/crit_times.py >> gpurun_out/r2z_ab.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2z_bench_grid.json 2> gpurun_out/r2z_bench_grid.err
SIMSWEEP_LEAN_SPEC=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2z_bench_grid_nospec.json 2>&1
timeout 900 python tools/timeline.py --full > gpurun_out/r2z_timeline_full.txt 2>&1
timeout 600 python tools/timeline.py > gpurun_out/r2z_timeline_grid.txt 2>&1
