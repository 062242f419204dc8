"""Seeded synthetic workload generators (shared input module).

This module is the ONLY code shared by the CPU oracle (``oracle/``) and the
CUDA path (``paper_2411_07447_b200``).  It holds none of the method's
arithmetic: it only draws request lengths and arrival times.  Every array it
returns is sorted by ``(T, id)`` ("ordered by the arrival
times"; reading Q1) and satisfies ``I + O - 1 <= S``
(PAPER.md:27).

Workload recipes:

* ``fixed(I, O, W)`` -- the analysis grid, all requests identical, T = 0
  (Sec. "Multi-Batch Cases with Preemption").
* ``longform(seed)`` -- LongForm-like: N = 2 000, evenly spaced arrivals over
  [0, 100) s, I ~ lognormal(mean 250) clipped to [1, 8 400],
  O ~ lognormal(mean 380) clipped to [1, 3 800].
* ``azureconv(seed)`` -- AzureConv-like: N = 19 700 over 1 h, Poisson arrivals,
  I ~ lognormal(mean 1 200) clipped to [1, 14 100], O ~ lognormal(mean 200)
  clipped to [1, 1 000].
* ``sharegpt / table_qa / text_to_sql`` -- length mixes of PAPER.md:27.
* ``mix(groups, W, seed)`` -- App. D SISO/SILO/LISO/LILO pairs
  (PAPER.md:1081-1088).

Lognormal parameterisation: mu = ln(mean) - sigma^2/2 with sigma = 1 (the
paper gives only means and maxima; this is a stated proposal).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Workload:
    """One workload: parallel arrays sorted by (T, id)."""

    I: np.ndarray  # int32 input lengths, >= 1
    O: np.ndarray  # int32 output lengths, >= 1
    T: np.ndarray  # float64 arrival times (s), non-decreasing
    name: str = ""

    @property
    def n(self) -> int:
        return int(self.I.shape[0])

    def scaled_O(self, o_scale: int, S: int) -> "Workload":
        """O x o_scale ("output length scale of 2x"), clamped so
        that I + O - 1 <= S."""
        O = np.minimum(self.O.astype(np.int64) * int(o_scale), S - self.I.astype(np.int64) + 1)
        return Workload(self.I.copy(), O.astype(np.int32), self.T.copy(), f"{self.name}-Ox{o_scale}")


def _pack(I, O, T, name) -> Workload:
    I = np.ascontiguousarray(np.asarray(I, dtype=np.int32))
    O = np.ascontiguousarray(np.asarray(O, dtype=np.int32))
    T = np.ascontiguousarray(np.asarray(T, dtype=np.float64))
    assert I.shape == O.shape == T.shape
    assert (I >= 1).all() and (O >= 1).all()
    assert (np.diff(T) >= 0).all(), "arrival times must be sorted"
    return Workload(I, O, T, name)


def _lognormal_int(rng: np.random.Generator, mean: float, lo: int, hi: int, n: int, sigma: float = 1.0):
    mu = np.log(mean) - 0.5 * sigma * sigma
    x = rng.lognormal(mu, sigma, size=n)
    return np.clip(np.rint(x), lo, hi).astype(np.int64)


def _clip_to_context(I: np.ndarray, O: np.ndarray, S: int):
    """Enforce I + O - 1 <= S by shortening O, then I."""
    I = np.minimum(I, S)
    O = np.minimum(O, S - I + 1)
    return I, np.maximum(O, 1)


def fixed(I: int, O: int, W: int) -> Workload:
    """Fixed-I/O analysis workload, all arrivals at T = 0."""
    return _pack(np.full(W, I), np.full(W, O), np.zeros(W), f"fixed-I{I}-O{O}-W{W}")


def grid_values(max_len: int = 1024):
    """I, O in {1, 2, 4, ..., 1024} ("vary the values from 1 to 1024")."""
    v, out = 1, []
    while v <= max_len:
        out.append(v)
        v *= 2
    return out


def longform(seed: int, N: int = 2000, S: int = 131072) -> Workload:
    rng = np.random.default_rng(seed)
    I = _lognormal_int(rng, 250.0, 1, 8400, N)
    O = _lognormal_int(rng, 380.0, 1, 3800, N)
    I, O = _clip_to_context(I, O, S)
    T = 100.0 * np.arange(N, dtype=np.float64) / N  # evenly spaced (reading Q32)
    return _pack(I, O, T, f"longform-s{seed}")


def azureconv(seed: int, N: int = 19700, S: int = 131072, horizon_s: float = 3600.0) -> Workload:
    rng = np.random.default_rng(seed)
    I = _lognormal_int(rng, 1200.0, 1, 14100, N)
    O = _lognormal_int(rng, 200.0, 1, 1000, N)
    I, O = _clip_to_context(I, O, S)
    gaps = rng.exponential(horizon_s / N, size=N)
    T = np.cumsum(gaps) - gaps[0]
    return _pack(I, O, T, f"azureconv-s{seed}")


def sharegpt(seed: int, W: int = 1024, S: int = 4096) -> Workload:
    rng = np.random.default_rng(seed)
    I = _lognormal_int(rng, 70.0, 1, S, W)
    O = _lognormal_int(rng, 215.0, 1, S, W)
    I, O = _clip_to_context(I, O, S)
    return _pack(I, O, np.zeros(W), f"sharegpt-s{seed}")


def table_qa(seed: int, W: int = 1024, S: int = 4096, long_context: bool = False) -> Workload:
    rng = np.random.default_rng(seed)
    I = _lognormal_int(rng, 1024.0 if long_context else 70.0, 1, S, W)
    O = rng.integers(1, 10, size=W).astype(np.int64)  # U{1..9}: "less than 10 tokens"
    I, O = _clip_to_context(I, O, S)
    return _pack(I, O, np.zeros(W), f"tableqa{'-long' if long_context else ''}-s{seed}")


def text_to_sql(seed: int, W: int = 1024, S: int = 4096, long_context: bool = False) -> Workload:
    rng = np.random.default_rng(seed)
    I = _lognormal_int(rng, 1024.0 if long_context else 70.0, 1, S, W)
    O = np.maximum(np.rint(rng.normal(50.0, 15.0, size=W)), 1).astype(np.int64)
    I, O = _clip_to_context(I, O, S)
    return _pack(I, O, np.zeros(W), f"text2sql{'-long' if long_context else ''}-s{seed}")


_L1 = (8, 16)
_L2 = (512, 1024)
_GROUPS = {
    "SISO": (_L1, _L1),
    "SILO": (_L1, _L2),
    "LISO": (_L2, _L1),
    "LILO": (_L2, _L2),
}


def mix(groups=("LILO", "SILO"), W: int = 1024, seed: int = 0) -> Workload:
    """App. D: W/2 requests from each of two groups, I and O drawn
    independently from the group's sets, shuffled."""
    assert len(groups) == 2 and W % 2 == 0
    rng = np.random.default_rng(seed)
    Is, Os = [], []
    for gname in groups:
        li, lo = _GROUPS[gname]
        Is.append(rng.choice(li, size=W // 2))
        Os.append(rng.choice(lo, size=W // 2))
    I = np.concatenate(Is)
    O = np.concatenate(Os)
    perm = rng.permutation(W)
    return _pack(I[perm], O[perm], np.zeros(W), f"mix-{'+'.join(groups)}-W{W}-s{seed}")


def random_small(seed: int, W: int, max_len: int = 16, online: bool = False, S: int = 64) -> Workload:
    """Tiny random workloads for invariant / parity sweeps."""
    rng = np.random.default_rng(seed)
    I = rng.integers(1, max_len + 1, size=W)
    O = rng.integers(1, max_len + 1, size=W)
    I, O = _clip_to_context(I, O, S)
    if online:
        T = np.sort(rng.integers(0, 4 * W, size=W).astype(np.float64) * 0.25)
    else:
        T = np.zeros(W)
    return _pack(I, O, T, f"random-s{seed}-W{W}")
