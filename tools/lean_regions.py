"""Instructions executed and warp-stall samples of the lean kernel, per code region.
    python tools/lean_regions.py SASS_CSV NVDISASM_G_TXT [full_steps]
SASS_CSV = `ncu -i REP --page source --csv --print-source sass`; NVDISASM_G_TXT = `nvdisasm -g -c` of the same cubin."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ia, iss, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
base = int(data[0][ia], 16)
steps = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
on, cur, off2line = False, None, {}
for l in open(sys.argv[2]).read().split("\n"):
    if l.startswith("//---------------------"):
        on = "sim_lean_kernelILi1024" in l
        continue
    if not on:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        f, ln = m.group(1).rsplit("/", 1)[-1], int(m.group(2))
        cur = ("sim_lean.cuh", ln) if f == "sim_lean.cuh" else (f, ln, cur[1] if cur and cur[0] == "sim_lean.cuh" else (cur[2] if cur and len(cur) > 2 else 0))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        off2line[int(m.group(1), 16)] = cur
src = open("paper_2411_07447_b200/csrc/sim_lean.cuh").read().split("\n")
keys = [("auto warp_np", "warp_np"), ("auto nth_head", "nth_head"), ("auto decode_group", "decode_group"),
        ("// apply: evict", "evict"), ("if (pfirst) {", "dispatch"), ("---- (3)", "compensate"),
        ("// the prefill entries:", "process_prefill"), ("// decode completions:", "completion_scan"),
        ("// the new decodes join", "new_decodes"), ("// a9: lane k", "cost"), ("// event times", "events"),
        ("// this step's victims", "victims"), ("---- (4)", "steady"), ("---- (5)", "compact"),
        ("if (nmov > 0)", "srf_merge"), ("// the oldest unfinished", "lo"), ("---- a11", "epilogue"),
        ("---- (1)", "arrivals"), ("if (w_dirty)", "wcount")]
marks = sorted((i, n) for i, l in enumerate(src, 1) for k, n in keys if k in l)


def reg(ln):
    nm = "prologue"
    for a, n in marks:
        if ln >= a:
            nm = n
    return nm


S, E = collections.Counter(), collections.Counter()
L = collections.Counter()
ts = te = 0
for r in data:
    k = off2line.get(int(r[ia], 16) - base)
    rg = "?" if k is None else (reg(k[1]) if k[0] == "sim_lean.cuh" else (reg(k[2]) if len(k) > 2 and k[2] else k[0]))
    s, e = int(r[iss]), int(r[iex])
    S[rg] += s
    E[rg] += e
    ts += s
    te += e
    if k is not None:
        L[k[1] if k[0] == "sim_lean.cuh" else (k[2] if len(k) > 2 else 0)] += s
print(f"total instructions {te} ({te / steps:.1f} per step), samples {ts}")
for k, v in S.most_common():
    print(f"{k:16s} samples {100 * v / ts:5.1f}%  instr {E[k]:9d} ({E[k] / steps:6.1f}/step)")
print("--- top lines by samples")
for ln, v in L.most_common(25):
    print(f"{100 * v / ts:5.1f}% {ln:5d} {src[ln - 1].strip()[:100] if ln else ''}")
