# round-2 re-entry (after the container was re-created): GPU suite, smoke, both bench lines, ncu evidence at HEAD
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2q2_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2q2_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2q2_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2q2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2q2_smoke.log
timeout 900 python bench.py > gpurun_out/r2q2_bench_grid.json 2> gpurun_out/r2q2_bench_grid.err
timeout 1200 python bench.py --workload full --steps 5 > gpurun_out/r2q2_bench_full.json 2> gpurun_out/r2q2_bench_full.err
bash tools/profile_round.sh r2q2
