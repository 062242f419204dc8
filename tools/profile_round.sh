# ncu evidence for profiles/: launch list of a short bench run (cold-cache, serialised) and one full capture
# of the sweep kernel.   bash tools/profile_round.sh TAG
TAG=${1:-r1}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_ -s 1 -c 1 -o gpurun_out/${TAG}_full \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_full.log 2>&1
