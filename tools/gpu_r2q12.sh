# bisect of the persistent lean arena kernel: v1 (generic, one CTA per simulation, carveout 15), A (noinline bodies,
# two families, head/tail), B (inline bodies, two families, head/tail), C (inline, one family, head/tail)
mkdir -p gpurun_out
for l in v1 A B C; do
  SIMSWEEP_GM_CARVEOUT=15 SIMSWEEP_LIB=ablibs/lib_$l.so timeout 900 python bench.py --workload full --steps 5 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q12_bench_full_$l.json 2> gpurun_out/r2q12_bench_full_$l.err
  SIMSWEEP_GM_CARVEOUT=15 SIMSWEEP_LIB=ablibs/lib_$l.so timeout 600 python tools/crit_times.py >> gpurun_out/r2q12_ab.log 2>&1
done
