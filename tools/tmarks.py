"""Where a full step spends its cycles: clock marks of thread 0 over one simulation (trace build,
-DSIMSWEEP_TRACE), averaged per consecutive mark pair.   python tools/tmarks.py PRESET I O [W]"""
import ctypes
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_07447_b200 import build  # noqa: E402

lib = build.LIB.replace(".so", "_trace.so")
if not os.path.exists(lib) or "--rebuild" in sys.argv:
    subprocess.run([build.NVCC] + build.FLAGS + ["-DSIMSWEEP_TRACE", "-o", lib] + build.SRC, check=True)
os.environ["SIMSWEEP_LIB"] = lib
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_07447_b200 import simsweep, workloads  # noqa: E402

L = simsweep.lib()
L.sim_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]
nm, I, O = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
W = int(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[4].isdigit() else 1024
cm = [simsweep.load_cost_models()["llama3-8b_a100_linear"]]
ds = simsweep.DeviceSweep([simsweep.preset_config(nm, 100_000)], [workloads.fixed(I, O, W)], cm)
ds.launch()
torch.cuda.synchronize()
cnt = np.zeros(1, np.int32)
n = 1 << 21
buf = np.zeros(2 * n, np.uint32)
L.sim_trace_read(buf.ctypes.data, n, cnt.ctypes.data)
m = min(int(cnt[0]), n)
ids, clk = buf[0: 2 * m: 2].astype(np.int64), buf[1: 2 * m: 2].astype(np.int64)
d = (clk[1:] - clk[:-1]) % (1 << 32)
agg = defaultdict(lambda: [0, 0])
for a, b, x in zip(ids[:-1], ids[1:], d):
    agg[(int(a), int(b))][0] += 1
    agg[(int(a), int(b))][1] += int(x)
tot = int(d.sum())
steps = int(ds.fetch().results["steps"][0])
print(f"{nm} {I}/{O} W={W}: {m} marks, {steps} steps, {tot} cycles, loop tops {int((ids == 1).sum())}")
for (a, b), (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"  {a:3d} -> {b:3d}  n={c:7d}  avg={s / c:8.1f}  share={100 * s / tot:5.1f}%")
