timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/r2w_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2w_gputests.log
for l in ablibs/lib_v1.so ablibs/lib_v2.so; do SIMSWEEP_LIB=$l timeout 300 python tools/crit_times.py >> gpurun_out/r2w_ab.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sim_ -s 1 -c 1 -o gpurun_out/r2w_sar1024 python tools/one_sim.py sarathi-srf 1024 1024 1024 2 > gpurun_out/r2w_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sim_ -s 1 -c 1 -o gpurun_out/r2w_vllm128 python tools/one_sim.py vllm-srf 128 1024 1024 2 > gpurun_out/r2w_ncu2.log 2>&1
