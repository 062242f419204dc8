"""Per-simulation GPU times of the north-star sweep's classes, each simulation launched ALONE (one CTA): the
critical-path candidates of the full sweep.  Prints one line per simulation: steps, ms, us/step.

    python tools/sim_times.py [--lib path] [--only grid|online|hetero]
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def cases(which):
    from paper_2411_07447_b200 import simsweep, workloads

    out = []
    if which in ("all", "grid"):
        for nm in ("vllm-srf", "vllm", "sarathi", "sarathi-srf", "vllm-hy-srf", "sarathi-nocp-srf", "sarathi-cs"):
            for (I, O) in ((128, 1024), (256, 1024), (1, 1024), (1024, 1024), (64, 1024)):
                out.append((f"{nm} I={I} O={O}", simsweep.preset_config(nm, 100_000), workloads.fixed(I, O, 1024),
                            ["llama3-8b_a100_linear"]))
        out.append(("vllm-srf 128/1024 K=4", simsweep.preset_config("vllm-srf", 100_000, cost=(0, 1, 2, 3)),
                    workloads.fixed(128, 1024, 1024), ["llama3-8b_a100_linear", "llama3-8b_h100_linear",
                                                       "llama3-70b_a100x4_linear", "llama3-70b_h100x4_linear"]))
    if which in ("all", "online"):
        for wname, wl in (("longform", workloads.longform(0)), ("azureconv", workloads.azureconv(0))):
            for nm in ("vllm", "sarathi"):
                for sfx in ("", "-srf", "-srf-hist"):
                    out.append((f"{wname} {nm}{sfx} 8B/A100", simsweep.preset_config(nm + sfx, 100_000, S=131072), wl,
                                ["llama3-8b_a100_linear"]))
            for cm in ("llama3-70b_a100x4_linear", "llama3-70b_h100x4_theoretical"):
                for sfx in ("", "-srf"):
                    for M in (100_000, -1):
                        out.append((f"{wname} vllm{sfx} {cm} M={M}", simsweep.preset_config("vllm" + sfx, M, S=131072),
                                    wl, [cm]))
    if which in ("all", "hetero"):
        for gname, wl in (("sharegpt", workloads.sharegpt(0)), ("tableqa-long", workloads.table_qa(0, long_context=True)),
                          ("text2sql", workloads.text_to_sql(0)), ("mix LILO+SILO", workloads.mix(("LILO", "SILO"), 1024, 0))):
            for nm in ("rank-org", "rank-i", "rank-o"):
                out.append((f"{gname} {nm}", simsweep.preset_config(nm, 100_000), wl, ["llama3-8b_a100_linear"]))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="all")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2411_07447_b200 import simsweep

    pcms = simsweep.load_cost_models()
    s = torch.cuda.Stream()
    print(f"{'simulation':48s} {'status':10s} {'steps':>8s} {'ms':>9s} {'us/step':>8s}")
    tot = 0.0
    for label, c, wl, names in cases(args.only):
        c = simsweep.SimConfig.from_buffer_copy(c)
        c.workload = 0
        c.n_cost = len(names)
        for k in range(len(names)):
            c.cost[k] = k
        ds = simsweep.DeviceSweep([c], [wl], [pcms[n] for n in names])
        ds.launch(s)  # warm
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ds.launch(s)
        e1.record(s)
        s.synchronize()
        ms = e0.elapsed_time(e1)
        r = ds.fetch()
        st = int(r.results["steps"][0])
        tot += ms
        print(f"{label:48s} {r.status(0):10s} {st:8d} {ms:9.2f} {1000 * ms / max(st, 1):8.2f}", flush=True)
    print(f"sum of alone times: {tot:.1f} ms")


if __name__ == "__main__":
    main()
