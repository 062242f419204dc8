# sweep time + single-simulation times for several builds: bash tools/cmp_libs.sh lib1 lib2 ...
for lib in "$@"; do
  b=$(basename $lib .so)
  SIMSWEEP_LIB=$lib timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$b.log 2>&1
  SIMSWEEP_LIB=$lib timeout 200 python tools/probe.py --product > gpurun_out/probe_$b.log 2>&1
done
