# warp-stall breakdown (per issued instruction) of one sweep launch for several builds: bash tools/ncu_stall.sh lib1 lib2 ...
for lib in "$@"; do
  SIMSWEEP_LIB=$lib timeout 600 ncu --metrics regex:smsp__average_warps_issue_stalled_.*_per_issue_active.ratio,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:sim_ -s 1 -c 1 \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/stall_$(basename $lib .so).txt 2>&1
done
