# compute-sanitizer racecheck / synccheck / memcheck over every kernel instance (incl. the roofline term table)
mkdir -p gpurun_out
timeout 300 python tools/sanitize_cases.py > gpurun_out/r2san_plain.log 2>&1; echo "rc=$?" >> gpurun_out/r2san_plain.log
for t in racecheck synccheck memcheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_cases.py > gpurun_out/r2san_$t.log 2>&1; echo "rc=$?" >> gpurun_out/r2san_$t.log
done
