ncu --set full --import-source on --clock-control none -k regex:sim_lean -s 1 -c 1 -o gpurun_out/r2g_lean python tools/one_sim.py vllm-srf 128 1024 > gpurun_out/r2g_ncu.log 2>&1
