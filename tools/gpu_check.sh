timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1
timeout 200 python tools/probe.py > gpurun_out/probe.log 2>&1
