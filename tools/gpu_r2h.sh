# round-2 final evidence (lean occupancy: 2 per SM): GPU suite, smoke, both bench lines, ncu launch list + full capture (grid), and a
# full capture of the lean arena kernel inside the north-star sweep (DRAM / L2 of the 220 arenas)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2h_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2h_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2h_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2h_smoke.log
timeout 900 python bench.py > gpurun_out/r2h_bench_grid.json 2> gpurun_out/r2h_bench_grid.err
timeout 1200 python bench.py --workload full --steps 5 > gpurun_out/r2h_bench_full.json 2> gpurun_out/r2h_bench_full.err
bash tools/profile_round.sh r2h
timeout 900 ncu --set full --clock-control none -k regex:sim_lean_kernel -c 1 -o gpurun_out/r2h_gm_full \
  python bench.py --workload full --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-critical > gpurun_out/r2h_gm_full.log 2>&1
