import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2411_07447_b200 import simsweep, workloads
W = lambda I, O: workloads.Workload(np.array(I, np.int32), np.array(O, np.int32), np.zeros(len(I)), "h")
cm = simsweep.unit_cost()
for ms in range(1, 8):
    c = simsweep.make_config(0, 0, 0, 2, C=1000, M=1000, max_steps=ms)
    r = simsweep.sim_sweep([c], [W([10]*5, [3]*5)], [cm])
    print("max_steps", ms, r.status(0), int(r.results["steps"][0]), r.request_times(0)[1].tolist())
for M in (1000, 2000, 100000):
    c = simsweep.make_config(0, 0, 0, 2, C=1000, M=M)
    r = simsweep.sim_sweep([c], [W([10]*5, [3]*5)], [cm])
    print("M", M, r.status(0), int(r.results["steps"][0]))
    c = simsweep.make_config(0, 0, 0, 1, C=1000, M=M)
    r = simsweep.sim_sweep([c], [W([10]*5, [3]*5)], [cm])
    print("srf M", M, r.status(0), int(r.results["steps"][0]))
