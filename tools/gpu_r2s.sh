for s in "vllm-srf llama3-70b_h100x4_theoretical M=inf azureconv s0" "vllm llama3-70b_a100x4_linear M=inf azureconv s0" "vllm-srf llama3-70b_a100x4_theoretical M=inf azureconv s9" "vllm-srf llama3-70b_h100x4_linear M=inf azureconv s0"; do
  timeout 300 python tools/one_sim.py --full "online-70B $s" 2 >> gpurun_out/r2s_one.log 2>&1
done
timeout 900 python tools/timeline.py --full > gpurun_out/r2s_timeline_full.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "online or azure or large_window or 70b" > gpurun_out/r2s_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2s_gputests.log
