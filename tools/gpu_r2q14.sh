# pairing-aware placement of the lean arena CTAs (the longest alone on an SM): GPU suite, full bench A/B, timeline
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r2q14_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2q14_gputests.log
for pr in 1 0; do
  SIMSWEEP_GM_PAIRING=$pr timeout 900 python bench.py --workload full --steps 5 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q14_bench_full_p$pr.json 2> gpurun_out/r2q14_bench_full_p$pr.err
done
timeout 900 python tools/timeline.py --full gpurun_out/r2q14_timeline.npz > gpurun_out/r2q14_timeline_full.txt 2>&1
