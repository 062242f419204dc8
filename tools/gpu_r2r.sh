timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/r2r_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2r_gputests.log
python tools/one_sim.py --full "online-70B vllm-srf llama3-70b_a100x4_theoretical M=100000 azureconv s9" 2 > gpurun_out/r2r_one_azure.log 2>&1
python tools/one_sim.py --full "online-70B vllm-srf llama3-70b_h100x4_theoretical M=inf azureconv s0" 2 >> gpurun_out/r2r_one_azure.log 2>&1
timeout 900 python tools/timeline.py --full > gpurun_out/r2r_timeline_full.txt 2>&1
