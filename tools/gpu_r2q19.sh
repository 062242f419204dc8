# A/B: the roofline terms' batch variables from a per-step shared vector (SIMSWEEP_TV) vs per-lane selects
mkdir -p gpurun_out
for l in final tv final tv; do SIMSWEEP_LIB=ablibs/lib_$l.so timeout 600 python tools/crit_times.py >> gpurun_out/r2q19_ab.log 2>&1; done
