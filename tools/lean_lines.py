"""Instructions executed and warp-stall samples of the lean kernel per sim_lean.cuh source line (inlined helpers
charged to the sim_lean.cuh line that calls them), from one ncu capture.

    python tools/lean_lines.py REP LIB KERNEL_SUBSTR [per_unit] [top]
REP = .ncu-rep (ncu --set full --import-source on); LIB = the libsimsweep.so that ran; per_unit divides the counts
(e.g. formed steps)."""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

rep, lib, kname = sys.argv[1], sys.argv[2], sys.argv[3]
unit = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data = rows[1], rows[2:]
ia, iss, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
base = int(data[0][ia], 16)
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
# each instruction is charged to its innermost sim_lean.cuh line: the line itself, or (code inlined from another file)
# the sim_lean.cuh line of the nearest call site in the inline chain printed before it
on, cur, off2line, chain = False, None, {}, []
for l in dis.split("\n"):
    if l.startswith("//---------------------"):
        on = kname in l
        continue
    if not on:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
    if m:
        chain.append(m)
        continue
    m2 = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m2:
        if chain:
            cur = None
            for c in chain:
                if c.group(1).endswith("sim_lean.cuh"):
                    cur = int(c.group(2))
                    break
                if c.group(3) and c.group(3).endswith("sim_lean.cuh"):
                    cur = int(c.group(4))
                    break
            chain = []
        off2line[int(m2.group(1), 16)] = cur
src = open(os.environ.get("LEAN_SRC") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                                    "paper_2411_07447_b200", "csrc", "sim_lean.cuh")).read().split("\n")
S, E, B = collections.Counter(), collections.Counter(), collections.Counter()
ts = te = 0
for r in data:
    ln = off2line.get(int(r[ia], 16) - base)
    s, e = int(r[iss]), int(r[iex])
    S[ln] += s
    E[ln] += e
    B[ln] += 16 if e > 0 else 0
    ts += s
    te += e
print(f"total: {te / unit:.0f} instructions and {ts} stall samples per unit; hot code {sum(B.values()) / 1024:.1f} KB")
print(" samp%  instr/unit  hotKB  line  source")
for ln, s in sorted(S.items(), key=lambda x: -x[1])[:top]:
    txt = src[ln - 1].strip()[:90] if ln else "?"
    print(f"{100 * s / max(ts, 1):5.1f} {E[ln] / unit:10.1f} {B[ln] / 1024:6.2f} {ln!s:>5}  {txt}")
