# lean shared-memory variants' carveout alone (block kernels at 100 %): full sweep and grid
mkdir -p gpurun_out
for x in 30 45 60 100 30; do
  SIMSWEEP_LEAN_CARVEOUT=$x timeout 900 python bench.py --workload full --steps 5 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q18_full_$x.json 2> gpurun_out/r2q18_full_$x.err
  python -c "import json; d=json.loads(open('gpurun_out/r2q18_full_$x.json').readline()); print('full', $x, d['ms_per_step'])" >> gpurun_out/r2q18.txt
done
for x in 30 45 100; do
  SIMSWEEP_LEAN_CARVEOUT=$x timeout 900 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q18_grid_$x.json 2> gpurun_out/r2q18_grid_$x.err
  python -c "import json; d=json.loads(open('gpurun_out/r2q18_grid_$x.json').readline()); print('grid', $x, d['ms_per_step'])" >> gpurun_out/r2q18.txt
done
