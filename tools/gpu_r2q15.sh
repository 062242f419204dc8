# carveouts that let the shared-memory lean CTAs run beside the arena CTAs from t = 0 (full sweep); fewer lean CTAs
# per SM on the grid; the hist-remainder branch A/B on the grid's critical simulations
mkdir -p gpurun_out
for x in "100 15" "50 50" "60 60" "43 43"; do set -- $x
  SIMSWEEP_SMEM_CARVEOUT=$1 SIMSWEEP_GM_CARVEOUT=$2 timeout 900 python bench.py --workload full --steps 5 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q15_full_$1_$2.json 2> gpurun_out/r2q15_full_$1_$2.err
done
SIMSWEEP_SMEM_CARVEOUT=50 SIMSWEEP_GM_CARVEOUT=50 timeout 900 python tools/timeline.py --full > gpurun_out/r2q15_timeline_50.txt 2>&1
for x in 100 86 70; do
  SIMSWEEP_SMEM_CARVEOUT=$x timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q15_grid_$x.json 2> gpurun_out/r2q15_grid_$x.err
done
for l in head hw head hw; do SIMSWEEP_LIB=ablibs/lib_$l.so timeout 600 python tools/crit_times.py --grid >> gpurun_out/r2q15_ab.log 2>&1; done
