"""Warp-stall samples of an .ncu-rep summed over line ranges of sim_step.cuh (phases of a step).
    python tools/ncu_ranges.py REP"""
import csv
import subprocess
import sys

COL = int(sys.argv[2]) if len(sys.argv) > 2 else 4  # 4 = stall samples, 7 = instructions executed
RANGES = [("setup", 1, 149), ("arrivals+groups", 150, 291), ("handle/preempt", 292, 364), ("warp_run", 365, 469),
          ("decode_group", 470, 607), ("warp_np", 608, 724), ("round driver", 725, 968), ("idle", 969, 991),
          ("process+cost", 992, 1158), ("events+steady", 1159, 1257), ("run list", 1258, 1323), ("metrics", 1324, 2000)]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
acc, fname, tot = {}, "?", 0.0
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    try:
        ln, s = int(r[0]), float(r[COL])
    except (ValueError, IndexError):
        continue
    tot += s
    key = fname
    if fname == "sim_step.cuh":
        key = next((n for n, a, b in RANGES if a <= ln <= b), "?")
    acc[key] = acc.get(key, 0.0) + s
for k, v in sorted(acc.items(), key=lambda x: -x[1]):
    print(f"{100 * v / tot:5.1f}%  {k}")
