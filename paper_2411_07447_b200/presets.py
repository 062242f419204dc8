"""Scheduler presets by name (configuration, not arithmetic).

Rows of PAPER.md:39-57 (Table "Schedulers used in the multi-batch analysis")
and the taxonomy of PAPER.md:1593-1610 (Table 2), plus the App. D ranking
schedulers.  Names follow SPEC S:325.

    preset       GroupRequests order            hybrid chunked  C
    vllm         {R_w, R_r}     prefill-first     no     no     S (4096)
    sarathi      {R_r^d,R_r^p,R_w} decode-first   yes    yes    512
    sarathi-cs   decode-first                     yes    yes    S
    sarathi-nocp decode-first                     yes    no     S
    vllm-hy      prefill-first                    yes    no     S
    sarathi-nohy decode-first                     no     no     S
    rank-org / rank-i / rank-o  one group by (T,id) / (I,T,id) / (O,T,id);
                 hybrid on, chunking off, C = S (reading Q20)
    orca         {R_r, R_w} decode-first          yes    no     S    reserve S, preemption-free
                 (Table 2; reading Q40)

Suffixes: ``-srf`` (SRF replacement), ``-srf-hist``
(SRF + histogram deferral), ``-pf`` (the preemption-free
``*^pf`` variant: reserve I + O - 1 at admission, never preempt; Table 2
PAPER.md:1606, 1619).  Default replacement is NRF (Table 2 "Newest request
first") with the initial reserve r.I (s = I + g on refills).
"""
from __future__ import annotations

ORDER_PREFILL_FIRST = 0
ORDER_DECODE_FIRST = 1
ORDER_RANK_ORG = 2
ORDER_RANK_I = 3
ORDER_RANK_O = 4

REPL_NRF = 0
REPL_SRF = 1
REPL_SRF_HIST = 2
REPL_PF = 3

RESERVE_SEQ = 0      # s = I + g (Table 2 "r.I")
RESERVE_PEAK = 1     # I + O - 1 (*^pf)
RESERVE_CONTEXT = 2  # S (Orca)

# name -> (order, hybrid, chunked, C or None meaning C = S)
_BASE = {
    "vllm": (ORDER_PREFILL_FIRST, 0, 0, None),
    "sarathi": (ORDER_DECODE_FIRST, 1, 1, 512),
    "sarathi-cs": (ORDER_DECODE_FIRST, 1, 1, None),
    "sarathi-nocp": (ORDER_DECODE_FIRST, 1, 0, None),
    "vllm-hy": (ORDER_PREFILL_FIRST, 1, 0, None),
    "sarathi-nohy": (ORDER_DECODE_FIRST, 0, 0, None),
    "rank-org": (ORDER_RANK_ORG, 1, 0, None),
    "rank-i": (ORDER_RANK_I, 1, 0, None),
    "rank-o": (ORDER_RANK_O, 1, 0, None),
    "orca": (ORDER_DECODE_FIRST, 1, 0, None),
}

GRID_PRESETS = ["vllm", "sarathi", "sarathi-cs", "sarathi-nocp", "vllm-hy", "sarathi-nohy"]


def names():
    out = []
    for b in _BASE:
        out += [b] if b == "orca" else [b, b + "-srf", b + "-srf-hist", b + "-pf"]
    return out


def preset(name: str, S: int = 4096) -> dict:
    """-> dict(order, hybrid, chunked, replacement, reserve, C, S)."""
    repl, reserve = REPL_NRF, RESERVE_SEQ
    base = name
    if name.endswith("-srf-hist"):
        repl, base = REPL_SRF_HIST, name[: -len("-srf-hist")]
    elif name.endswith("-srf"):
        repl, base = REPL_SRF, name[: -len("-srf")]
    elif name.endswith("-pf"):
        repl, reserve, base = REPL_PF, RESERVE_PEAK, name[: -len("-pf")]
    if base not in _BASE or (base == "orca" and base != name):
        raise KeyError(f"unknown preset {name!r}; known: {names()}")
    if base == "orca":
        repl, reserve = REPL_PF, RESERVE_CONTEXT
    order, hybrid, chunked, C = _BASE[base]
    return dict(order=order, hybrid=hybrid, chunked=chunked, replacement=repl, reserve=reserve,
                C=int(C if C is not None else S), S=int(S))
