timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/r2t_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2t_gputests.log
for s in "vllm-srf llama3-70b_a100x4_linear M=inf azureconv s6" "vllm-srf llama3-70b_h100x4_theoretical M=inf azureconv s0" "vllm-srf llama3-70b_a100x4_theoretical M=100000 azureconv s9"; do
  timeout 300 python tools/one_sim.py --full "online-70B $s" 2 >> gpurun_out/r2t_one.log 2>&1
done
for cv in 100 50 10; do
  SIMSWEEP_GM_CARVEOUT=$cv timeout 900 python tools/timeline.py --full > gpurun_out/r2t_timeline_full_cv$cv.txt 2>&1
  SIMSWEEP_GM_CARVEOUT=$cv timeout 300 python tools/one_sim.py --full "online-70B vllm-srf llama3-70b_a100x4_theoretical M=100000 azureconv s9" 2 >> gpurun_out/r2t_one_cv$cv.log 2>&1
  SIMSWEEP_GM_CARVEOUT=$cv timeout 300 python tools/one_sim.py --full "online-8B sarathi-srf-hist azureconv s0" 2 >> gpurun_out/r2t_one_cv$cv.log 2>&1
done
