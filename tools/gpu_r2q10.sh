# persistent lean arena kernel: arena CTAs per SM (2 default; 1, 3) on the full-sweep bench, timeline at 2
mkdir -p gpurun_out
for sl in 2 1 3; do
  SIMSWEEP_GM_SLOTS=$sl timeout 900 python bench.py --workload full --steps 5 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q10_bench_full_s$sl.json 2> gpurun_out/r2q10_bench_full_s$sl.err
done
timeout 900 python tools/timeline.py --full > gpurun_out/r2q10_timeline_full.txt 2>&1
