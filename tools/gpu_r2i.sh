timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2i_gputests.log
timeout 300 python tools/sim_times.py --only grid > gpurun_out/r2i_simtimes.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:sim_lean -s 1 -c 1 -o gpurun_out/r2i_lean python tools/one_sim.py vllm-srf 128 1024 > gpurun_out/r2i_ncu.log 2>&1
