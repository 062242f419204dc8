# persistent lean arena kernel, one family per SM (vLLM-family instance + generic): GPU suite, A/B, benches, timeline
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/r2q9_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2q9_gputests.log
for l in ablibs/lib_v1.so paper_2411_07447_b200/libsimsweep.so; do SIMSWEEP_LIB=$l timeout 600 python tools/crit_times.py >> gpurun_out/r2q9_ab.log 2>&1; done
timeout 900 python bench.py --workload full --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/r2q9_bench_full.json 2> gpurun_out/r2q9_bench_full.err
timeout 900 python tools/timeline.py --full > gpurun_out/r2q9_timeline_full.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q9_bench_grid.json 2> gpurun_out/r2q9_bench_grid.err
