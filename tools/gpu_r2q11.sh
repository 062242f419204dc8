# lean arena kernel: one family per SM, head / tail claims (long with short): GPU suite, full bench, timeline, A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/r2q11_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2q11_gputests.log
timeout 900 python bench.py --workload full --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/r2q11_bench_full.json 2> gpurun_out/r2q11_bench_full.err
timeout 900 python tools/timeline.py --full > gpurun_out/r2q11_timeline_full.txt 2>&1
SIMSWEEP_LIB=ablibs/lib_v1.so timeout 900 python bench.py --workload full --steps 5 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q11_bench_full_v1.json 2> gpurun_out/r2q11_bench_full_v1.err
