"""Instructions executed (column 7) or stall samples (column 4) of an .ncu-rep, summed per region of a source
file (regions start at `auto NAME = [` lambdas and `// ---- (...)` section comments).
    python tools/ncu_regions.py REP [COL] [FILE]"""
import csv
import re
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
col = int(sys.argv[2]) if len(sys.argv) > 2 else 7
fname = sys.argv[3] if len(sys.argv) > 3 else "paper_2411_07447_b200/csrc/sim_warp.cuh"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
src = open(fname).read().split("\n")
regions, name = [], "head"
for line in src:
    m = re.match(r"\s+auto (\w+) = \[", line) or re.match(r"\s+// ---- (\(\d\)[^-:]*)", line)
    if m:
        name = m.group(1)[:32]
    regions.append(name)
base = fname.rsplit("/", 1)[-1]
agg, tot, cur = Counter(), 0.0, "?"
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].rsplit("/", 1)[-1]
        continue
    try:
        ln, v = int(r[0]), float(r[col])
    except (ValueError, IndexError):
        continue
    tot += v
    agg[regions[ln - 1] if cur == base and ln <= len(regions) else cur] += v
print(f"total {tot:.4g}")
for k, v in agg.most_common(20):
    print(f"{100 * v / max(tot, 1):5.1f}%  {k}")
