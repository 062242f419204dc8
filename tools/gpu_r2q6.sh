# full-sweep timelines at several GM-arena carveouts (does a second arena CTA / a shared-memory CTA fit beside one?)
mkdir -p gpurun_out
for cv in 10 15 20 30 50; do
  SIMSWEEP_GM_CARVEOUT=$cv timeout 600 python tools/timeline.py --full > gpurun_out/r2q6_timeline_cv$cv.txt 2>&1
done
