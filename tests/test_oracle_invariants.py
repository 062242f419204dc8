"""Oracle pins: an independent log verifier (tests/verifier.py) re-derives every
request's trajectory from the oracle's trace and checks Eq. (4)-(7), the
conservation law and the paper's invariants on randomized configurations
(SPEC acceptance criterion 1), plus mutation tests proving the verifier fails.
"""
import copy

import numpy as np
import pytest

import oracle as o
from paper_2411_07447_b200 import workloads
from verifier import verify

ORDERS = ["prefill_first", "decode_first", "rank_org", "rank_i", "rank_o"]
REPLS = ["nrf", "srf", "srf_hist"]


def random_case(seed):
    rng = np.random.default_rng(seed)
    W = int(rng.integers(1, 25))
    online = bool(rng.integers(0, 2))
    wl = workloads.random_small(seed, W, max_len=int(rng.integers(2, 17)), online=online, S=64)
    order = ORDERS[int(rng.integers(0, 5))]
    repl = REPLS[int(rng.integers(0, 3))]
    chunked = int(rng.integers(0, 2))
    hybrid = int(rng.integers(0, 2)) if order in ("prefill_first", "decode_first") else 1
    peak = int((wl.I.astype(int) + wl.O - 1).max())
    C = int(rng.integers(1, 3 * peak + 1)) if chunked else int(rng.integers(peak, 3 * peak + 1))
    M = -1 if rng.random() < 0.15 else int(rng.integers(peak, 4 * peak + 1))
    return wl, o.make_config(order, hybrid, chunked, repl, C=C, M=M, S=64), (C, M, hybrid)


@pytest.mark.parametrize("seed", range(200))
def test_random_configs_verify(seed):
    wl, cfg, (C, M, hybrid) = random_case(seed)
    r = o.run(cfg, wl.I, wl.O, wl.T, o.load_cost_models()["llama3-8b_a100_theoretical"], trace=True)
    assert r.status == "ok"
    outs = dict(t_first=list(r.t_first[0]), t_done=list(r.t_done[0]), n_preempt=list(r.n_preempt),
                refill=list(r.refill))
    viol = verify(r.steps_list, list(wl.I), list(wl.O), list(wl.T), C, M, outs, hybrid=bool(hybrid),
                  replacement=REPLS[int(cfg.replacement)])
    assert viol == []
    assert r.steps == len(r.steps_list) and r.steps >= int(wl.O.max())
    assert r.preemptions == int(r.n_preempt.sum())
    assert r.processed_tokens == int((wl.I.astype(int) + wl.O - 1).sum() + r.refill.sum())
    if M < 0:
        assert r.preemptions == 0  # Infinite M


def test_infinite_M_never_preempts():
    for seed in range(40):
        wl, cfg, _ = random_case(1000 + seed)
        cfg.M = -1
        r = o.run(cfg, wl.I, wl.O, wl.T, o.unit_cost())
        assert r.status == "ok" and r.preemptions == 0


def _valid_trace():
    cfg = o.make_config("prefill_first", 0, 0, "nrf", C=4096, M=12)
    r = o.run(cfg, [1, 1, 5], [6, 6, 4], [0.0] * 3, o.unit_cost(), trace=True)
    return r.steps_list


def test_verifier_accepts_valid_and_rejects_mutations():
    st = _valid_trace()
    args = ([1, 1, 5], [6, 6, 4], [0.0] * 3, 7, 12)
    assert verify(st, *args) == []
    # Sigma c = C + 1 injected: C = 7 is exceeded by step 7's refill of 7 plus one token
    bad = copy.deepcopy(st)
    bad[6]["entries"] = [(2, 1, 8, 0)]
    assert any("C =" in x or "exceeds available" in x for x in verify(bad, *args))
    # refill one token short but the next step claims a decode (bad generation)
    bad = copy.deepcopy(st)
    bad[6]["entries"] = [(2, 1, 6, 0)]
    assert verify(bad, *args) != []
    # dropped preemption event
    bad = copy.deepcopy(st)
    bad[2]["events"] = []
    assert verify(bad, *args) != []
    # memory bound violated: tighten M
    assert any("KV holdings" in x for x in verify(st, [1, 1, 5], [6, 6, 4], [0.0] * 3, 4096, 11))


def test_verifier_checks_victim_order():
    # two victims in one step: NRF evicts the newest admission first (Table 2); swapping the
    # two events (or reading them under SRF's key where the m order differs) is a violation
    for repl in ("nrf", "srf"):
        I, O = [2, 6, 7, 1, 2], [2, 3, 3, 2, 7]
        cfg = o.make_config("prefill_first", 0, 0, repl, C=4096, M=11)
        r = o.run(cfg, I, O, [0.0] * 5, o.unit_cost(), trace=True)
        st = r.steps_list
        args = (I, O, [0.0] * 5, 4096, 11)
        assert verify(st, *args, replacement=repl) == []
        multi = [k for k, x in enumerate(st) if len(x["events"]) >= 2]
        assert multi, repl
        bad = copy.deepcopy(st)
        k = multi[0]
        bad[k]["events"] = bad[k]["events"][::-1]
        assert any("lower retention" in x for x in verify(bad, *args, replacement=repl)), repl
