# ncu source-level captures of the critical simulations alone (lean kernel): per-region instruction counts
set -x
mkdir -p gpurun_out
i=0
for a in "vllm-srf 128 1024" "sarathi-srf 1024 1024" "vllm-srf 256 1024"; do
  timeout 300 python tools/one_sim.py $a 1024 2 >> gpurun_out/r2q3_one.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sim_lean -c 1 -o gpurun_out/r2q3_one$i python tools/one_sim.py $a 1024 1 > gpurun_out/r2q3_ncu$i.log 2>&1
  i=$((i+1))
done
s="online-70B vllm-srf llama3-70b_a100x4_theoretical M=100000 azureconv s9"
timeout 300 python tools/one_sim.py --full "$s" 2 >> gpurun_out/r2q3_one.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_lean -c 1 -o gpurun_out/r2q3_gm python tools/one_sim.py --full "$s" 1 > gpurun_out/r2q3_ncugm.log 2>&1
timeout 900 python tools/timeline.py --full > gpurun_out/r2q3_timeline_full.txt 2>&1
