"""Independent schedule-log verifier (test infrastructure).

Re-derives every request's trajectory from a step trace ALONE and checks the
CSP constraints of PAPER.md:352-407 (Termination, Non-decreasing sequence
length, Eq. (4) memory management, Eq. (5) tokens to process, Eq. (6) token
generation, Eq. (7) batch constraints) plus the conservation law
``sum_j sum_{B_j} c = sum_i (I_i + O_i - 1) + sum refill``,
B <= W, clock monotonicity and arrival causality.

It shares no code with either the oracle or the CUDA path; it only reads the
trace format documented in DESIGN.md ("Trace format").

trace: list of dict(step, U, tok, start, d, entries=[(id, phase, c, m_before)],
                    events=[(id, m_discarded)])
"""
from __future__ import annotations


def verify(steps, I, O, T, C, M, K_out=None, hybrid=True, reserve="seq", S=None, kv_block=1, replacement=None):
    """Returns a list of violation strings (empty = valid).

    reserve: the Table 2 "Initial KV reserve" taken at (re)admission:
    "seq" = s = I + g, "peak" = I + O - 1, "context" = S.  With "peak"/"context" the
    scheduler is preemption-free: any preemption event is a violation.

    K_out: optional dict(t_first=[...], t_done=[...], n_preempt=[...], refill=[...])
    to cross-check the reported per-request outputs against the trace.

    replacement: "nrf", "srf" or "srf_hist" also checks WHICH requests were preempted, in order
    (PAPER.md:1644-1646): when v is preempted, no running request outside the step's batch has
    a lower retention than v (NRF: later admission; SRF: smaller m, ties later admission).  Admission order
    is re-derived from the trace (a request's (re)admission is its first entry while not running).
    """
    n = len(I)
    v = []
    m = [0] * n
    g = [0] * n
    res = [0] * n
    running = [False] * n
    done = [False] * n
    npre = [0] * n
    refill = [0] * n
    t_first = [None] * n
    t_done = [None] * n
    total_c = 0
    prev_end = None
    seq = [0] * n
    nseq = 0

    def lower(a, b):  # retention of a below that of b
        if replacement == "nrf":
            return seq[a] > seq[b]
        return m[a] < m[b] or (m[a] == m[b] and seq[a] > seq[b])
    for st in steps:
        j, ents, evs = st["step"], st["entries"], st["events"]
        start, d = st["start"], st["d"]
        if not (1 <= len(ents) <= n):
            v.append(f"step {j}: |B|={len(ents)} outside [1, W]")
        if not d > 0:
            v.append(f"step {j}: non-positive duration {d}")
        if prev_end is not None:
            if start < prev_end:
                v.append(f"step {j}: start {start} before previous end {prev_end}")
            elif start != prev_end and not any(T[i] == start for i in range(n)):
                v.append(f"step {j}: clock jumped to {start} which is no arrival time")
        prev_end = start + d
        # preemption events (Eq. 4: m := 0 when e = 1); refill keeps g
        inB = {e[0] for e in ents}
        for (i, md) in evs:
            if replacement is not None and running[i]:
                for r in range(n):
                    if r != i and running[r] and r not in inB and lower(r, i):
                        v.append(f"step {j}: preempted {i} while {r} (running, not in the batch) has lower retention")
                        break
            if reserve != "seq":
                v.append(f"step {j}: preemption of {i} under a preemption-free reserve")
            if not running[i]:
                v.append(f"step {j}: preempted request {i} was not running")
            if md != m[i]:
                v.append(f"step {j}: preempted {i} discarded {md} but held m={m[i]}")
            refill[i] += m[i]
            npre[i] += 1
            m[i] = 0
            res[i] = 0
            running[i] = False
        sum_c = 0
        seen = set()
        phases = set()
        for (i, ph, c, mb) in ents:
            if i in seen:
                v.append(f"step {j}: request {i} twice in batch")
            seen.add(i)
            if done[i]:
                v.append(f"step {j}: completed request {i} scheduled")
            if T[i] > start:
                v.append(f"step {j}: request {i} scheduled before its arrival")
            s = I[i] + g[i]
            if c < 1:
                v.append(f"step {j}: request {i} c={c} < 1")
            if mb != m[i]:
                v.append(f"step {j}: request {i} m_before={mb} but tracked m={m[i]}")
            if c > s - m[i]:  # Eq. (5)
                v.append(f"step {j}: request {i} c={c} exceeds available {s - m[i]}")
            if ph == 0 and not (c == 1 and m[i] == s - 1):
                v.append(f"step {j}: decode entry {i} with c={c}, m={m[i]}, s={s}")
            phases.add(ph)
            if not running[i]:  # (re)admission reserves the initial reserve
                running[i] = True
                nseq += 1
                seq[i] = nseq
                res[i] = s if reserve == "seq" else (I[i] + O[i] - 1 if reserve == "peak" else S)
            sum_c += c
        if not hybrid and len(phases) > 1:
            v.append(f"step {j}: hybrid batch while hybrid batching is off")
        if sum_c > C:  # Eq. (7)
            v.append(f"step {j}: sum c = {sum_c} > C = {C}")
        if st.get("tok") is not None and st["tok"] != sum_c:
            v.append(f"step {j}: reported tok {st['tok']} != sum c {sum_c}")
        cmap = {i: c for (i, _, c, _) in ents}
        b = max(kv_block, 1)  # paged KV (Q15 alternative): holdings in blocks of b tokens, capacity floor(M / b)
        U = sum(-(-max(res[i], m[i] + cmap.get(i, 0)) // b) for i in range(n) if running[i])
        if st.get("U") is not None and st["U"] != U:
            v.append(f"step {j}: reported U {st['U']} != recomputed {U}")
        if M >= 0 and U > M // b:  # Eq. (7) memory
            v.append(f"step {j}: KV holdings {U} > M = {M // b}")
        end = start + d
        for (i, ph, c, mb) in ents:
            s = I[i] + g[i]
            gen = c == s - m[i]  # Eq. (6)
            m[i] += c
            total_c += c
            if gen:
                g[i] += 1
                if t_first[i] is None:
                    t_first[i] = end
                if g[i] == O[i]:
                    done[i] = True
                    running[i] = False
                    t_done[i] = end
                if g[i] > O[i]:
                    v.append(f"step {j}: request {i} generated more than O")
    for i in range(n):
        if g[i] != O[i]:  # Termination
            v.append(f"request {i}: generated {g[i]} != O = {O[i]}")
    expect = sum(I[i] + O[i] - 1 for i in range(n)) + sum(refill)
    if total_c != expect:
        v.append(f"conservation: sum c = {total_c} != sum(I+O-1) + refill = {expect}")
    if K_out is not None:
        for i in range(n):
            if K_out["n_preempt"][i] != npre[i]:
                v.append(f"request {i}: n_preempt {K_out['n_preempt'][i]} != trace {npre[i]}")
            if K_out["refill"][i] != refill[i]:
                v.append(f"request {i}: refill {K_out['refill'][i]} != trace {refill[i]}")
            if t_first[i] is not None and K_out["t_first"][i] != t_first[i]:
                v.append(f"request {i}: t_first {K_out['t_first'][i]} != trace {t_first[i]}")
            if t_done[i] is not None and K_out["t_done"][i] != t_done[i]:
                v.append(f"request {i}: t_done {K_out['t_done'][i]} != trace {t_done[i]}")
    return v
