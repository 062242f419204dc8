nproc > gpurun_out/r2j_nproc.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2j_bench_grid.log 2>&1
timeout 1500 python bench.py --workload full --steps 3 --warmup 3 > gpurun_out/r2j_bench_full.log 2>&1
timeout 600 python tools/sim_times.py --only online > gpurun_out/r2j_simtimes_online.log 2>&1
