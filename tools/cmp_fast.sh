for fm in -1 96 128 192; do
SIMSWEEP_LIB=paper_2411_07447_b200/libsimsweep_f$fm.so timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_f$fm.log 2>&1
done
bash tools/ncu_stall.sh paper_2411_07447_b200/libsimsweep_f-1.so paper_2411_07447_b200/libsimsweep_f128.so
SIMSWEEP_LIB=paper_2411_07447_b200/libsimsweep_f128.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
