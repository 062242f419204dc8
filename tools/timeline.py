"""Per-simulation start/end timeline of one grid sweep (profiling build): is the sweep bound by its
critical path or by aggregate work?   python tools/timeline.py [--full] [out.npz]"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_07447_b200 import build
os.environ["SIMSWEEP_LIB"] = os.environ.get("PROBE_LIB") or build.LIB.replace(".so", "_prof.so")
import numpy as np, torch
from paper_2411_07447_b200 import simsweep, sweep
L = simsweep.lib()
L.sim_debug_read.argtypes = [ctypes.c_void_p, ctypes.c_int32]
full = "--full" in sys.argv
sys.argv = [a for a in sys.argv if a != "--full"]
cfgs, wls, cms, labels = sweep.full_sweep() if full else sweep.grid_sweep()
order = sweep.partition_lpt(sweep.estimate(cfgs, wls), 1)[0]
ds = simsweep.DeviceSweep(cfgs, wls, cms, order=np.asarray(order, np.int32))
ds.launch(); torch.cuda.synchronize(); ds.launch(); torch.cuda.synchronize()
prof = np.zeros((len(cfgs), 24), np.int64)
L.sim_debug_read(prof.ctypes.data, len(cfgs))
res = ds.fetch().results
t0 = prof[:, 14].min()
st = (prof[:, 14] - t0) / 1e6
en = (prof[:, 15] - t0) / 1e6
du = en - st
sm = prof[:, 9]
print("max simulations per SM over the sweep:", np.bincount(sm).max(), "SMs used:", len(np.unique(sm)))
ev = sorted([(s, 1) for s in st] + [(e, -1) for e in en])
cur = mx = 0
for _, d in ev:
    cur += d
    mx = max(mx, cur)
print("max concurrently running simulations:", mx)
print(f"sweep makespan {en.max():.2f} ms; sum of sim durations {du.sum():.1f} ms; "
      f"mean concurrency {du.sum() / en.max():.0f}; longest sim {du.max():.2f} ms")
idx = np.argsort(-en)[:25]
print("latest-finishing simulations:  label  start  duration  end  steps  launch-rank  est")
est = sweep.estimate(cfgs, wls)
rank = {c: r for r, c in enumerate(order)}
for i in idx:
    print(f"  {labels[i]!s:32s} {st[i]:7.2f} {du[i]:7.2f} {en[i]:7.2f} {int(res['steps'][i]):7d} {rank[i]:5d} {est[i]:9.0f}")
import collections
cls = collections.Counter()
for i in range(len(cfgs)):
    lb = labels[i]
    key = f"{lb[0]} {lb[1].split()[0]} {lb[1].split()[1] if lb[0] == 'online-70B' else ''} {lb[2].split()[0] if full else ''}"
    cls[key] += du[i]
print("sum of simulation durations by class (ms):")
for k, v in cls.most_common(20):
    print(f"  {k:70s} {v:10.1f}")
bins = [0, 1, 5, 10, 20, 40, 80, 160, 320, 640, 1280]
print(f"start-time histogram {bins} ms:", np.histogram(st, bins=bins)[0])
print("longest-duration simulations:  label  start  duration  end  steps  launch-rank  est")
for i in np.argsort(-du)[:25]:
    print(f"  {labels[i]!s:32s} {st[i]:7.2f} {du[i]:7.2f} {en[i]:7.2f} {int(res['steps'][i]):7d} {rank[i]:5d} {est[i]:9.0f}")
if len(sys.argv) > 1:  # save per-simulation start/duration/steps for offline comparison
    np.savez(sys.argv[1], st=st, du=du, steps=np.asarray(res["steps"]), labels=np.asarray([str(l) for l in labels]))
