"""Derive the frozen cost-model data file ``data/cost_models.json``.

The paper does not print its calibrated coefficients or GPU constants
(reading Q23).  This one-off script freezes
them from public model dimensions and datasheet peaks:

* theoretical mode (Eq. 3) needs only the dims and peaks;
* linear mode ("linear cost models with all variables in
  Table 3") gets its coefficients from a non-negative least-squares fit to a
  synthetic profiler = Eq. 3 per operator x an inefficiency factor
  (matmul 1.25x, attention 3x; SPEC S:218 -- the paper's Fig. "Roofline
  analysis" shows attention "distant from the roofline").

The output is INPUT DATA, consumed identically by the oracle and the CUDA
path (like a workload); neither side runs this script.  Run:
    python tools/derive_cost_models.py > data/cost_models.json
"""
from __future__ import annotations

import json
import math
import sys

import numpy as np
from scipy.optimize import nnls

MODELS = {
    # public architecture dims (not in the paper): h, f, H, N_Q, N_KV, layers
    "llama2-7b": dict(h=4096, f=11008, H=128, NQ=32, NKV=32, layers=32),
    "llama3-8b": dict(h=4096, f=14336, H=128, NQ=32, NKV=8, layers=32),
    "llama3-70b": dict(h=8192, f=28672, H=128, NQ=64, NKV=8, layers=80),
}
HARDWARE = {
    # dense bf16 FLOP/s, HBM B/s, NVLink B/s per direction (public datasheets)
    "a100": dict(flops=312e12, bw=2.039e12, link_bw=300e9),
    "h100": dict(flops=989e12, bw=3.35e12, link_bw=450e9),
}
SETUPS = [
    ("llama3-8b", "a100", 1),
    ("llama3-8b", "h100", 1),
    ("llama3-70b", "a100", 4),
    ("llama3-70b", "h100", 4),
    ("llama2-7b", "a100", 1),
    ("llama2-7b", "h100", 1),
]
E = 2  # bytes per element (fp16/bf16)
EFF_MATMUL = 1.25
EFF_ATTN = 3.0


def _lat(F, RW, flops, bw):
    return max(F / flops, E * RW / bw)


def profile_non_attention(N, d, flops, bw, link_bw, tp):
    h, f, H, NQ, NKV = d["h"], d["f"], d["H"], d["NQ"], d["NKV"]
    qkv = _lat(2 * N * h * (NQ + 2 * NKV) * H, h * (NQ + 2 * NKV) * H + N * h + N * (NQ + 2 * NKV) * H, flops, bw)
    o = _lat(2 * N * h * h, h * h + 2 * N * h, flops, bw)
    gu = _lat(2 * N * h * 2 * f, 2 * h * f + N * h + 2 * N * f, flops, bw)
    dn = _lat(2 * N * f * h, f * h + N * f + N * h, flops, bw)
    t = EFF_MATMUL * (qkv + o + gu + dn)
    if tp > 1:
        t += 2 * (E * 2 * N * h * (tp - 1) / tp) / link_bw
    return t


def profile_prefill_attention(reqs, d, flops, bw):
    H, NQ, NKV = d["H"], d["NQ"], d["NKV"]
    F = sum(4 * H * NQ * c * (c + m) for c, m in reqs)
    RW = sum(2 * H * NQ * c + 2 * NQ * c * (c + m) + 2 * H * NKV * math.ceil(c / H) * (c + m) for c, m in reqs)
    return EFF_ATTN * _lat(F, RW, flops, bw)


def profile_decode_attention(ms, d, flops, bw):
    H, NQ, NKV = d["H"], d["NQ"], d["NKV"]
    F = sum(4 * H * NQ * (1 + m) for m in ms)
    RW = sum(2 * H * NQ + 2 * NQ * (1 + m) + 2 * H * NKV * (1 + m) for m in ms)
    return EFF_ATTN * _lat(F, RW, flops, bw)


def r2(y, yhat):
    ss_res = float(((y - yhat) ** 2).sum())
    ss_tot = float(((y - y.mean()) ** 2).sum())
    return 1.0 - ss_res / ss_tot


def fit_setup(model, hw, tp):
    d = MODELS[model]
    p = HARDWARE[hw]
    flops, bw, link_bw = p["flops"] * tp, p["bw"] * tp, p["link_bw"]
    rng = np.random.default_rng(0)
    # non-attention: t = a0 + a1 N, N in [1, 4096]
    Ns = np.unique(np.concatenate([np.arange(1, 65), np.geomspace(1, 8192, 200).astype(int)]))
    X = np.stack([np.ones_like(Ns, dtype=float), Ns.astype(float)], 1)
    y = np.array([profile_non_attention(int(N), d, flops, bw, link_bw, tp) for N in Ns])
    a, _ = nnls(X, y)
    r2_non = r2(y, X @ a)
    # prefill attention: features (1, sum c^2, sum m c, sum c, sum m) over random batches
    rows, ys = [], []
    for _ in range(600):
        k = int(rng.integers(1, 9))
        reqs = [(int(rng.integers(1, 4097)), int(rng.integers(0, 8193))) for _ in range(k)]
        rows.append([1.0, sum(c * c for c, _ in reqs), sum(m * c for c, m in reqs), sum(c for c, _ in reqs), sum(m for _, m in reqs)])
        ys.append(profile_prefill_attention(reqs, d, flops, bw))
    X = np.array(rows, dtype=float)
    y = np.array(ys)
    sc = X.max(0)
    b, _ = nnls(X / sc, y)
    b = b / sc
    r2_p = r2(y, X @ b)
    # decode attention: features (1, sum m, n_d)
    rows, ys = [], []
    for _ in range(600):
        k = int(rng.integers(1, 1025))
        ms = rng.integers(0, 4096, size=k)
        rows.append([1.0, float(ms.sum()), float(k)])
        ys.append(profile_decode_attention([int(x) for x in ms], d, flops, bw))
    X = np.array(rows, dtype=float)
    y = np.array(ys)
    sc = X.max(0)
    dd, _ = nnls(X / sc, y)
    dd = dd / sc
    r2_d = r2(y, X @ dd)
    lin = [float(a[0]), float(a[1])] + [float(x) for x in b] + [float(x) for x in dd]
    # round to 6 significant digits so the frozen file is human-checkable
    lin = [float(f"{v:.6g}") for v in lin]
    return lin, dict(non_attention=r2_non, prefill_attention=r2_p, decode_attention=r2_d)


def main():
    out = {"_comment": "Frozen by tools/derive_cost_models.py (DESIGN.md reading Q23). lin = per-layer "
           "[a0,a1 | b0,b1,b2,b3,b4 | d0,d1,d2] seconds: t = a0 + a1*N + [n_p>0](b0 + b1*sum_p c^2 + "
           "b2*sum_p m*c + b3*sum_p c + b4*sum_p m) + [n_d>0](d0 + d1*sum_d m + d2*n_d).",
           "models": MODELS, "hardware": HARDWARE, "bytes_per_element": E,
           "efficiency": {"matmul": EFF_MATMUL, "attention": EFF_ATTN}, "cost_models": []}
    for model, hw, tp in SETUPS:
        d = MODELS[model]
        p = HARDWARE[hw]
        lin, fit = fit_setup(model, hw, tp)
        base = dict(model=model, hw=hw, tp=tp, layers=d["layers"], h=d["h"], f=d["f"], H=d["H"],
                    NQ=d["NQ"], NKV=d["NKV"], e=E, flops=p["flops"] * tp, bw=p["bw"] * tp, link_bw=p["link_bw"])
        out["cost_models"].append(dict(name=f"{model}_{hw}{'x%d' % tp if tp > 1 else ''}_linear", mode=0, lin=lin,
                                       r2=fit, **base))
        out["cost_models"].append(dict(name=f"{model}_{hw}{'x%d' % tp if tp > 1 else ''}_theoretical", mode=1,
                                       lin=[0.0] * 10, **base))
    json.dump(out, sys.stdout, indent=1)
    sys.stdout.write("\n")


if __name__ == "__main__":
    main()
