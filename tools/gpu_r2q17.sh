# grid bench at carveouts giving 1-2 lean CTAs per SM, and the full sweep at 60 % vs 100 %
mkdir -p gpurun_out
for x in 30 60 30 60; do
  SIMSWEEP_SMEM_CARVEOUT=$x timeout 900 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q17_grid_$x.json 2> gpurun_out/r2q17_grid_$x.err
  python -c "import json; d=json.loads(open('gpurun_out/r2q17_grid_$x.json').readline()); print('grid', $x, d['ms_per_step'])" >> gpurun_out/r2q17.txt
done
for x in 60 100 60 100; do
  SIMSWEEP_SMEM_CARVEOUT=$x timeout 900 python bench.py --workload full --steps 5 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q17_full_$x.json 2> gpurun_out/r2q17_full_$x.err
  python -c "import json; d=json.loads(open('gpurun_out/r2q17_full_$x.json').readline()); print('full', $x, d['ms_per_step'])" >> gpurun_out/r2q17.txt
done
