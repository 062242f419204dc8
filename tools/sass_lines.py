"""Instruction count per source line (and per line range) of one kernel in `nvdisasm -g -c` output.
    python tools/sass_lines.py all.txt KERNEL_SUBSTRING"""
import collections
import re
import sys

txt = open(sys.argv[1]).read().split("\n")
key = sys.argv[2]
on = False
cur = "?"
cnt = collections.Counter()
for l in txt:
    if l.startswith("//---------------------"):
        on = key in l
        continue
    if not on:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1).rsplit('/', 1)[-1]}:{m.group(2)}"
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        cnt[cur] += 1
tot = sum(cnt.values())
print("total", tot)
RANGES = [(a, b, n) for n, a, b in [("head", 1, 200), ("arrivals/groups", 150, 300)]]
src = open("paper_2411_07447_b200/csrc/sim_step.cuh").read().split("\n")
fun = {}
name = "?"
for i, l in enumerate(src, 1):
    m = re.match(r"\s+auto (\w+) = \[", l) or re.match(r"\s+// ---- (.*)", l)
    if m:
        name = m.group(1)[:40]
    fun[i] = name
agg = collections.Counter()
for k, v in cnt.items():
    f, _, ln = k.partition(":")
    agg[fun.get(int(ln), "?") if f == "sim_step.cuh" and ln.isdigit() else f] += v
for k, v in agg.most_common(30):
    print(f"{v:7d} {100 * v / tot:5.1f}%  {k}")
print("--- top lines")
for k, v in cnt.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    f, _, ln = k.partition(":")
    s = src[int(ln) - 1].strip()[:90] if f == "sim_step.cuh" and ln.isdigit() else ""
    print(f"{v:6d} {k:22s} {s}")
