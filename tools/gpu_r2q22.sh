# full sweep: the arena carveout vs the lean kernel's (44 %, two per SM): can lean CTAs start beside arena CTAs?
mkdir -p gpurun_out
for g in 15 44 58 15 44; do
  SIMSWEEP_GM_CARVEOUT=$g timeout 900 python bench.py --workload full --steps 5 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q22_full_$g.json 2> gpurun_out/r2q22_full_$g.err
  python -c "import json; d=json.loads(open('gpurun_out/r2q22_full_$g.json').readline()); print('full gm', $g, d['ms_per_step'])" >> gpurun_out/r2q22.txt
done
SIMSWEEP_GM_CARVEOUT=44 timeout 900 python tools/timeline.py --full > gpurun_out/r2q22_timeline_44.txt 2>&1
