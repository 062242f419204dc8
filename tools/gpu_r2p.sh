# race fixes check + single-simulation ncu captures of the two critical paths (grid, full sweep)
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_cases.py > gpurun_out/r2p_san_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_san_racecheck.log
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/r2p_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2p_gputests.log
python tools/one_sim.py sarathi-srf 1024 1024 1024 3 > gpurun_out/r2p_one_grid.log 2>&1
python tools/one_sim.py --full "online-70B vllm-srf llama3-70b_a100x4_theoretical M=100000 azureconv s9" 2 > gpurun_out/r2p_one_azure.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sim_ -s 1 -c 1 -o gpurun_out/r2p_grid_crit python tools/one_sim.py sarathi-srf 1024 1024 1024 2 > gpurun_out/r2p_ncu_grid.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_ -s 1 -c 1 -o gpurun_out/r2p_azure_crit python tools/one_sim.py --full "online-70B vllm-srf llama3-70b_a100x4_theoretical M=100000 azureconv s9" 2 > gpurun_out/r2p_ncu_azure.log 2>&1
cp paper_2411_07447_b200/libsimsweep.so gpurun_out/r2p_lib.so
