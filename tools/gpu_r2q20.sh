# A/B: a vLLM-family instance of the lean n <= 1024 kernel (SIMSWEEP_VL) on the grid (two lean CTAs per SM)
mkdir -p gpurun_out
for l in final vl final vl; do
  SIMSWEEP_LIB=ablibs/lib_$l.so timeout 900 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2q20_grid_$l.json 2> gpurun_out/r2q20_grid_$l.err
  python -c "import json; d=json.loads(open('gpurun_out/r2q20_grid_$l.json').readline()); print('grid', '$l', d['ms_per_step'])" >> gpurun_out/r2q20.txt
done
for l in final vl; do SIMSWEEP_LIB=ablibs/lib_$l.so timeout 600 python tools/crit_times.py --grid >> gpurun_out/r2q20_ab.log 2>&1; done
SIMSWEEP_LIB=ablibs/lib_vl.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "grid or hand_traces or random_small or config1" --timeout 900 > gpurun_out/r2q20_vl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2q20_vl_tests.log
