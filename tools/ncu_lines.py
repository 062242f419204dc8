"""Top CUDA source lines by warp-stall samples of an .ncu-rep (ncu --import-source on).
    python tools/ncu_lines.py REP [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, tot = [], "?", 0.0
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] in ("Function Name", "Line No") or r[0] == "":
        continue
    try:
        s = float(r[4])
    except (ValueError, IndexError):
        continue
    rows.append((s, f"{fname}:{r[0]}", r[1].strip()))
    tot += s
rows.sort(key=lambda x: -x[0])
for s, loc, src in rows[:top]:
    print(f"{100 * s / max(tot, 1):5.1f}% {loc:18s} {src[:120]}")
