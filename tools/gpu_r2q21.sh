# A/B: vLLM-family lean instance with a different carveout than the generic one (disjoint SMs if the SM split must
# match): generic 2 per SM at 44 % or 58 %, VL 2 per SM at the other
mkdir -p gpurun_out
for x in "44 58" "58 44" "44 44"; do set -- $x
  SIMSWEEP_LEAN_CARVEOUT=$1 SIMSWEEP_VL_CARVEOUT=$2 SIMSWEEP_LIB=ablibs/lib_vl2.so timeout 900 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q21_grid_$1_$2.json 2> gpurun_out/r2q21_grid_$1_$2.err
  python -c "import json; d=json.loads(open('gpurun_out/r2q21_grid_$1_$2.json').readline()); print('grid vl', '$1 $2', d['ms_per_step'])" >> gpurun_out/r2q21.txt
done
SIMSWEEP_LIB=ablibs/lib_final.so timeout 900 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q21_grid_final.json 2> gpurun_out/r2q21_grid_final.err
python -c "import json; d=json.loads(open('gpurun_out/r2q21_grid_final.json').readline()); print('grid final', d['ms_per_step'])" >> gpurun_out/r2q21.txt
