"""Seeded random configurations with the alternative-reading knobs on (shared by the oracle and GPU tests)."""
import numpy as np

import oracle as o
from paper_2411_07447_b200 import workloads

ORDERS = ["prefill_first", "decode_first", "rank_org", "rank_i", "rank_o"]
REPLS = ["nrf", "srf", "srf_hist"]


def random_knob_case(seed):
    rng = np.random.default_rng(50_000 + seed)
    W = int(rng.integers(1, 30))
    online = bool(rng.integers(0, 2))
    wl = workloads.random_small(50_000 + seed, W, max_len=int(rng.integers(2, 24)), online=online, S=96)
    order = ORDERS[int(rng.integers(0, 5))]
    repl = REPLS[int(rng.integers(0, 3))]
    chunked = int(rng.integers(0, 2))
    hybrid = int(rng.integers(0, 2)) if order in ("prefill_first", "decode_first") else 1
    peak = int((wl.I.astype(int) + wl.O - 1).max())
    C = int(rng.integers(1, 3 * peak + 1)) if chunked else int(rng.integers(peak, 3 * peak + 1))
    wm = int(rng.integers(0, 6)) if rng.random() < 0.5 else 0
    M = -1 if rng.random() < 0.1 else int(rng.integers(peak + wm, 4 * peak + wm + 1))
    bits = (o.KNOB_HOL if rng.random() < 0.6 else 0) | (o.KNOB_NRF_ARRIVAL if repl == "nrf" and rng.random() < 0.5 else 0)
    bits |= o.KNOB_SRF_VISIT_ADMISSION if repl != "nrf" and rng.random() < 0.5 else 0
    knobs = dict(knobs=bits, max_seqs=int(rng.integers(1, 6)) if rng.random() < 0.5 else 0,
                 kv_watermark=wm if M >= 0 else 0)
    if repl != "srf_hist" and rng.random() < 0.4:  # paged KV (Q15 alternative): capacity floor(M / b) blocks
        b = int(rng.integers(2, 9))
        knobs["kv_block"] = b
        if M >= 0:
            need = -(-peak // b) + -(-wm // b)  # blocks of the largest peak plus the watermark
            M = max(M, need * b + int(rng.integers(0, 3 * b)))
    cfg = o.make_config(order, hybrid, chunked, repl, C=C, M=M, S=96, **knobs)
    return wl, cfg, (C, M, hybrid), knobs
