timeout 900 python -m pytest tests/test_gpu_trace.py -x -q > gpurun_out/gputrace.log 2>&1; echo "rc=$?" >> gpurun_out/gputrace.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_new.log 2>&1
