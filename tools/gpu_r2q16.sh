# grid bench vs the shared-memory lean CTAs' carveout (CTAs per SM: 100 % -> 5, 70 % -> 3, 60 % -> 2), alternated
mkdir -p gpurun_out
for x in 100 70 60 100 70 60; do
  SIMSWEEP_SMEM_CARVEOUT=$x timeout 900 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q16_grid_$x.json 2> gpurun_out/r2q16_grid_$x.err
  python -c "import json; d=json.loads(open('gpurun_out/r2q16_grid_$x.json').readline()); print($x, d['ms_per_step'])" >> gpurun_out/r2q16_grid.txt
done
