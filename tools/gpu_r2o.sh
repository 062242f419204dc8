# round-2 re-entry: GPU suite, smoke, both bench lines, sanitizers, ncu evidence of the lean kernel
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2o_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2o_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2o_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2o_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2o_smoke.log
timeout 900 python bench.py > gpurun_out/r2o_bench_grid.json 2> gpurun_out/r2o_bench_grid.err
timeout 1200 python bench.py --workload full --steps 5 > gpurun_out/r2o_bench_full.json 2> gpurun_out/r2o_bench_full.err
for t in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_cases.py > gpurun_out/r2o_san_$t.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_san_$t.log
done
bash tools/profile_round.sh r2o
