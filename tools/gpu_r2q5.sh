# full-sweep timeline (profiling build) and the AzureConv critical simulation under ncu after the cost-table change
mkdir -p gpurun_out
timeout 900 python tools/timeline.py --full > gpurun_out/r2q5_timeline_full.txt 2>&1
s="online-70B vllm-srf llama3-70b_a100x4_theoretical M=100000 azureconv s9"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_lean -c 1 -o gpurun_out/r2q5_gm python tools/one_sim.py --full "$s" 1 > gpurun_out/r2q5_ncugm.log 2>&1
