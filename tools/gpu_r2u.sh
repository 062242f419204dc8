timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/r2u_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2u_gputests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2u_bench_grid.json 2> gpurun_out/r2u_bench_grid.err
for c in "vllm-srf 256 1024" "sarathi-srf 1024 1024"; do timeout 120 python tools/one_sim.py $c 1024 3 >> gpurun_out/r2u_one.log 2>&1; done
timeout 300 python tools/one_sim.py --full "online-70B vllm-srf llama3-70b_a100x4_theoretical M=100000 azureconv s9" 2 >> gpurun_out/r2u_one.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sim_ -s 1 -c 1 -o gpurun_out/r2u_vllm256 python tools/one_sim.py vllm-srf 256 1024 1024 2 > gpurun_out/r2u_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_ -s 1 -c 1 -o gpurun_out/r2u_azure python tools/one_sim.py --full "online-70B vllm-srf llama3-70b_a100x4_theoretical M=100000 azureconv s9" 2 > gpurun_out/r2u_ncu2.log 2>&1
