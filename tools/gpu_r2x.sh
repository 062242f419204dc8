timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/r2x_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2x_gputests.log
for l in ablibs/lib_v2.so ablibs/lib_v3.so ablibs/lib_force.so; do SIMSWEEP_LIB=$l timeout 300 python tools/crit_times.py --grid >> gpurun_out/r2x_ab.log 2>&1; done
