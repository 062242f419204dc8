# One GPU call for a round's evidence: -m gpu suite, smoke, the default bench line, launch list + one ncu capture.
#   bash tools/round_check.sh TAG
TAG=${1:-r1}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1
bash tools/profile_round.sh $TAG
