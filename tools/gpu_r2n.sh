timeout 120 python tools/dbg_hist.py > gpurun_out/r2n_dbg.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2n_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2n_gputests.log
timeout 600 python tools/sim_times.py --only online > gpurun_out/r2n_simtimes_online.log 2>&1
