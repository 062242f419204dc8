# round-2 closing check of the tree as committed: GPU suite, smoke, both bench lines
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2i_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2i_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2i_smoke.log
timeout 900 python bench.py > gpurun_out/r2i_bench_grid.json 2> gpurun_out/r2i_bench_grid.err
timeout 1200 python bench.py --workload full --steps 5 > gpurun_out/r2i_bench_full.json 2> gpurun_out/r2i_bench_full.err
