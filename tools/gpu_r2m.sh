python tools/dbg_hist.py > gpurun_out/r2m_dbg.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2m_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2m_gputests.log
