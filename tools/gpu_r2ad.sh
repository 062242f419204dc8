timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/r2ad_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2ad_gputests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2ad_bench_grid.json 2> gpurun_out/r2ad_bench_grid.err
SIMSWEEP_LEAN_SPEC=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2ad_bench_grid_spec0.json 2>&1
SIMSWEEP_LEAN_SPEC=2 timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2ad_bench_grid_spec2.json 2>&1
timeout 900 python bench.py --workload full --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/r2ad_bench_full.json 2> gpurun_out/r2ad_bench_full.err
SIMSWEEP_LEAN_SPEC=0 timeout 900 python bench.py --workload full --steps 3 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2ad_bench_full_spec0.json 2>&1
timeout 600 python tools/timeline.py > gpurun_out/r2ad_timeline_grid.txt 2>&1
