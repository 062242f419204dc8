// ORACLE -- test infrastructure only (see oracle.h).  Plain, slow, literal.
//
// Follows Algorithm 1 and the text of GetNextBatch
// steps (1)-(4) step by step, with the readings of
// DESIGN.md "Readings" (Q-numbers cited inline).  Everything is explicit
// vectors, stable sorts and linear scans; no blocking, fusion or reordering.
// Time is the only floating-point quantity (fp64, built -ffp-contract=off).
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <queue>
#include <vector>

namespace {

enum Status { NOT_ARRIVED, WAITING, RUNNING, DONE };
enum Phase { PH_NONE = -1, PH_DECODE = 0, PH_PREFILL = 1 };

struct Req {
  int64_t id = 0, I = 0, O = 0;
  double T = 0.0;
  int st = NOT_ARRIVED;
  int64_t m = 0;         // r.m: processed tokens = KVs cached (Table 1)
  int64_t g = 0;         // generated tokens so far
  int64_t reserved = 0;  // KVs reserved at (re)admission (Table 2 "Initial KV reserve")
  bool filled = false;   // current (re)fill completed -> decode phase (Q17)
  int64_t seq = 0;       // admission sequence number, set at every (re)admission (Q6)
  bool has_first = false;
  double t_first[4] = {0, 0, 0, 0};
  double t_done[4] = {0, 0, 0, 0};
  int64_t n_preempt = 0, refill = 0;
  bool preempted_now = false;  // preempted during the current step (Q9)
  bool in_batch = false;
};

// s = I + g: all input and generated tokens (CSP variable s)
int64_t seq_len(const Req& r) { return r.I + r.g; }
// tokens available to process: s - m (Eq. 5)
int64_t avail(const Req& r) { return seq_len(r) - r.m; }
// Phase: prefill iff waiting or running with an incomplete (re)fill (Q17)
int phase_of(const Req& r) { return (r.st == WAITING || !r.filled) ? PH_PREFILL : PH_DECODE; }
// KVs held in the cache (Q13): running requests hold max(reserved, m) -- counted in blocks of b tokens under the
// Q15 alternative (paged KV), b = 1 otherwise
int64_t blocks(int64_t x, int64_t b) { return (x + b - 1) / b; }
int64_t held(const Req& r, int64_t b) { return r.st == RUNNING ? blocks(std::max(r.reserved, r.m), b) : 0; }

// true iff a is retained longer than b under the replacement policy.
// NRF: "newest request first" is preempted first (Table 2), newest
//      = most recently (re)admitted (Q6).
// SRF: "prioritizes running long requests (having large m) and preempts short
//      requests"; ties: later admission is preempted first (Q7).
// PF: never preempts; its running order is admission order, as NRF (Q39).
// retention priority (Q3, Q6, Q7): NRF keeps the earlier ADMITTED request (or, with the Q6 alternative, the
// earlier ARRIVAL: (T, id) = index order), SRF the one with more cached KVs
bool retained_longer(const Req& a, const Req& b, int repl, bool by_arrival = false) {
  if (by_arrival) return a.id < b.id;
  if (repl == OR_NRF || repl == OR_PF) return a.seq < b.seq;
  if (a.m != b.m) return a.m > b.m;
  return a.seq < b.seq;
}

int bucket_of(int64_t x) {  // floor(log2 x), x >= 1
  int b = 0;
  while ((int64_t(1) << (b + 1)) <= x) b++;
  return b > 17 ? 17 : b;
}

// nearest-rank p90 over a bucketed row: smallest bucket whose cumulative count
// reaches ceil(0.9 n); predict the bucket's upper edge 2^(b+1) - 1 (Q31)
int64_t p90_edge(const int64_t* row, int64_t n) {
  int64_t target = (9 * n + 9) / 10;  // = ceil(9n/10)
  int64_t cum = 0;
  for (int b = 0; b < 18; b++) {
    cum += row[b];
    if (cum >= target) return (int64_t(1) << (b + 1)) - 1;
  }
  return (int64_t(1) << 18) - 1;
}

int64_t hist_predict(const int32_t* H, int64_t I) {
  int bi = bucket_of(I);
  int64_t row[18], n = 0;
  for (int b = 0; b < 18; b++) {
    row[b] = H[bi * 18 + b];
    n += row[b];
  }
  if (n >= 8) return p90_edge(row, n);
  int64_t col[18];
  n = 0;
  for (int b = 0; b < 18; b++) {
    col[b] = 0;
    for (int a = 0; a < 18; a++) col[b] += H[a * 18 + b];
    n += col[b];
  }
  if (n >= 8) return p90_edge(col, n);
  return 256;  // prior
}

struct Entry {
  int64_t id, c, m_before;
  int phase;
};

// ---- cost model (Sec. "Cost Models for Batch Times") ----

// Eq. (1): FLOPs = 4 c (c+m) B H N_Q ; Eq. (2): RW = 2cHN_Q + 2c(c+m)BN_Q + 2 ceil(c/H) (c+m) B H N_KV
void attention_cost(int64_t c, int64_t m, int64_t B, int64_t H, int64_t NQ, int64_t NKV, int64_t* F, int64_t* RW) {
  *F = 4 * c * (c + m) * B * H * NQ;
  int64_t ceil_c_H = (c + H - 1) / H;
  *RW = 2 * c * H * NQ + 2 * c * (c + m) * B * NQ + 2 * ceil_c_H * (c + m) * B * H * NKV;
}

// (c x in)(in x out): "2cfh FLOPs, loading fh model parameters and cf inputs, and storing ch outputs"
void matmul_cost(int64_t c, int64_t in, int64_t out, int64_t* F, int64_t* RW) {
  *F = 2 * c * in * out;
  *RW = in * out + c * in + c * out;
}

// Eq. (3): max(FLOPs / GPU_FLOPS, RW / GPU_bandwidth), RW in bytes = e * elements (Q26)
double roofline(int64_t F, int64_t RW_elems, const oracle_cost_t& cm) {
  double tc = (double)F / cm.flops;
  double tm = (double)(RW_elems * (int64_t)cm.e) / cm.bw;
  return std::fmax(tc, tm);
}

double batch_time(const oracle_cost_t& cm, const std::vector<Entry>& B) {
  // "we sum the costs of non-attention operators and the attentions, either prefill- or
  // decode-attention based on the request phase. For hybrid batches, both"
  int64_t N = 0;
  for (const Entry& e : B) N += e.c;
  if (cm.mode == 1) {
    const int64_t h = cm.h, f = cm.f, H = cm.H, NQ = cm.NQ, NKV = cm.NKV;
    int64_t F, RW;
    double t = 0.0;
    matmul_cost(N, h, (NQ + 2 * NKV) * H, &F, &RW);  // QKV_proj
    t = t + roofline(F, RW, cm);
    matmul_cost(N, NQ * H, h, &F, &RW);  // O_proj
    t = t + roofline(F, RW, cm);
    matmul_cost(N, h, 2 * f, &F, &RW);  // gate + up (SwiGLU, Q27)
    t = t + roofline(F, RW, cm);
    matmul_cost(N, f, h, &F, &RW);  // D_proj
    t = t + roofline(F, RW, cm);
    int64_t Fp = 0, Rp = 0, Fd = 0, Rd = 0, np_ = 0, nd = 0;
    for (const Entry& e : B) {  // mixed batch: per-request sums with B = 1 (Q24)
      attention_cost(e.c, e.m_before, 1, H, NQ, NKV, &F, &RW);
      if (e.phase == PH_PREFILL) {
        Fp += F;
        Rp += RW;
        np_++;
      } else {
        Fd += F;
        Rd += RW;
        nd++;
      }
    }
    if (np_ > 0) t = t + roofline(Fp, Rp, cm);
    if (nd > 0) t = t + roofline(Fd, Rd, cm);
    if (cm.tp > 1) {  // two All_Reduce per layer, bytes linear in c
      double ar = ((double)(2 * (int64_t)cm.e * N * h * (int64_t)(cm.tp - 1)) / (double)cm.tp) / cm.link_bw;
      t = t + ar;
      t = t + ar;
    }
    return (double)cm.layers * t;
  }
  // linear mode over the Table 3 variables
  int64_t np_ = 0, c2 = 0, mc = 0, cp = 0, mp = 0, nd = 0, md = 0;
  for (const Entry& e : B) {
    if (e.phase == PH_PREFILL) {
      np_++;
      c2 += e.c * e.c;
      mc += e.m_before * e.c;
      cp += e.c;
      mp += e.m_before;
    } else {
      nd++;
      md += e.m_before;
    }
  }
  const double* a = cm.lin;
  double t = a[0] + a[1] * (double)N;
  if (np_ > 0) t = t + ((((a[2] + a[3] * (double)c2) + a[4] * (double)mc) + a[5] * (double)cp) + a[6] * (double)mp);
  if (nd > 0) t = t + ((a[7] + a[8] * (double)md) + a[9] * (double)nd);
  return (double)cm.layers * t;
}

struct Trace {
  int64_t* ti;
  int64_t icap, ilen = 0;
  double* td;
  int64_t dcap, dlen = 0;
  bool overflow = false;
  void pi(int64_t v) {
    if (!ti || overflow) return;
    if (ilen >= icap) { overflow = true; return; }
    ti[ilen++] = v;
  }
  void pd(double v) {
    if (!td || overflow) return;
    if (dlen >= dcap) { overflow = true; return; }
    td[dlen++] = v;
  }
};

}  // namespace

extern "C" {

void oracle_attention_cost(int64_t c, int64_t m, int64_t B, int64_t H, int64_t NQ, int64_t NKV, int64_t* flops,
                           int64_t* rw_elems) {
  attention_cost(c, m, B, H, NQ, NKV, flops, rw_elems);
}

void oracle_matmul_cost(int64_t c, int64_t in, int64_t out, int64_t* flops, int64_t* rw_elems) {
  matmul_cost(c, in, out, flops, rw_elems);
}

int64_t oracle_hist_predict(const int32_t* hist, int64_t I) { return hist_predict(hist, I); }

double oracle_batch_time(const oracle_cost_t* cm, int32_t n, const int64_t* c, const int64_t* m,
                         const int32_t* is_prefill) {
  std::vector<Entry> B;
  for (int i = 0; i < n; i++) B.push_back(Entry{i, c[i], m[i], is_prefill[i] ? PH_PREFILL : PH_DECODE});
  return batch_time(*cm, B);
}

int oracle_run(const oracle_config_t* cfg, int32_t n, const int32_t* I, const int32_t* O, const double* T,
               const oracle_cost_t* cms, oracle_summary_t* out, double* t_first, double* t_done, int64_t* n_preempt,
               int64_t* refill_tokens, int64_t* trace_i, int64_t trace_i_cap, double* trace_d, int64_t trace_d_cap,
               int64_t* trace_lens) {
  // ---- call-level validation ----
  if (!cfg || !out || n <= 0 || !I || !O || !T || !cms) return -1;
  if (cfg->order < OR_PREFILL_FIRST || cfg->order > OR_RANK_O) return -2;
  if (cfg->replacement < OR_NRF || cfg->replacement > OR_PF) return -2;
  if (cfg->reserve < OR_RESERVE_SEQ || cfg->reserve > OR_RESERVE_CONTEXT) return -2;
  if ((cfg->replacement == OR_PF) != (cfg->reserve != OR_RESERVE_SEQ)) return -2;  // Q39
  if ((cfg->knobs & ~(OR_KNOB_HOL | OR_KNOB_NRF_ARRIVAL | OR_KNOB_SRF_VISIT_ADMISSION)) || cfg->max_seqs < 0 ||
      cfg->kv_watermark < 0)
    return -2;
  if ((cfg->knobs & OR_KNOB_NRF_ARRIVAL) && cfg->replacement != OR_NRF) return -2;
  if ((cfg->knobs & OR_KNOB_SRF_VISIT_ADMISSION) && cfg->replacement != OR_SRF && cfg->replacement != OR_SRF_HIST)
    return -2;
  if (cfg->kv_block < 0 || (cfg->kv_block > 1 && cfg->replacement == OR_SRF_HIST)) return -2;
  if (cfg->n_cost < 1 || cfg->n_cost > 4) return -3;
  if (cfg->C < 1 || cfg->S < 1 || cfg->max_steps < 1) return -4;
  for (int i = 0; i < n; i++) {
    if (I[i] < 1 || O[i] < 1) return -5;
    if (i > 0 && T[i] < T[i - 1]) return -6;  // sorted by (T, id) (Q1)
    if (cfg->n_cost > 1 && T[i] != 0.0) return -7;  // K cost models share one schedule offline only
  }
  const int K = cfg->n_cost;
  const int repl = cfg->replacement;
  const bool by_arrival = (cfg->knobs & OR_KNOB_NRF_ARRIVAL) != 0;  // Q6 alternative
  const bool finiteM = cfg->M >= 0;
  const int64_t kvb = cfg->kv_block > 1 ? cfg->kv_block : 1;  // Q15 alternative: KV block size
  const int64_t M = finiteM ? cfg->M / kvb : cfg->M, C = cfg->C;   // the KV capacity in blocks

  std::memset(out, 0, sizeof(*out));
  for (int64_t x = 0; x < (int64_t)K * n; x++) {
    t_first[x] = 0.0;
    t_done[x] = 0.0;
  }
  for (int i = 0; i < n; i++) {
    n_preempt[i] = 0;
    refill_tokens[i] = 0;
  }
  Trace tr{trace_i, trace_i_cap, 0, trace_d, trace_d_cap, 0, false};
  if (trace_lens) trace_lens[0] = trace_lens[1] = 0;

  // ---- per-simulation validation (Q35): I+O-1 <= S; must fit M; non-chunked must fit C ----
  for (int i = 0; i < n; i++)
    if ((int64_t)I[i] + O[i] - 1 > cfg->S) {
      out->status = OR_TOO_LONG;
      return 0;
    }
  const int64_t wm = blocks(cfg->kv_watermark, kvb);  // Q16 alternative: free blocks a waiting admission leaves
  for (int i = 0; i < n; i++) {
    int64_t peak = (int64_t)I[i] + O[i] - 1;  // peak KV usage I+O-1
    // a CONTEXT reserve (Orca) of S > M can never be admitted either (Q35); nor, with a watermark, a request
    // whose last refill (s = I + O - 1) could not be admitted into an empty cache
    if ((finiteM && blocks(peak, kvb) + wm > M) || (!cfg->chunked && peak > C) ||
        (finiteM && cfg->reserve == OR_RESERVE_CONTEXT && blocks(cfg->S, kvb) + wm > M)) {
      out->status = OR_NEVER_FITS;
      return 0;
    }
  }

  std::vector<Req> R(n);
  for (int i = 0; i < n; i++) {
    R[i].id = i;
    R[i].I = I[i];
    R[i].O = O[i];
    R[i].T = T[i];
  }
  int32_t hist[18 * 18];
  std::memset(hist, 0, sizeof(hist));

  double clock[4] = {0, 0, 0, 0};
  int next = 0;
  int64_t steps = 0, seq = 0, U = 0, n_done = 0;
  int status = OR_OK;

  // Table 2 "Initial KV reserve": r.I for vLLM/Sarathi (generalised to s = I + g for
  // refills), r.I + r.O - 1 for *^pf, S for Orca
  auto initial_reserve = [&](const Req& r) -> int64_t {
    if (cfg->reserve == OR_RESERVE_PEAK) return r.I + r.O - 1;
    if (cfg->reserve == OR_RESERVE_CONTEXT) return cfg->S;
    return seq_len(r);
  };

  std::vector<int64_t> evs;  // preemption events of the current step: (id, m discarded)
  auto preempt = [&](Req& r) {  // PAPER.md:1644-1646; refill semantics PAPER.md:1570
    U -= held(r, kvb);
    r.refill += r.m;
    r.n_preempt++;
    out->preemptions++;
    evs.push_back(r.id);
    evs.push_back(r.m);
    r.m = 0;
    r.reserved = 0;
    r.filled = false;
    r.st = WAITING;  // "removed from R_r and appended to R_w" (g kept: refill I+g)
    r.preempted_now = true;
  };

  while (true) {
    // (a2) GetNewRequests (Alg. 1 line 3): all arrivals with T <= clock (Q21)
    while (next < n && R[next].T <= clock[0]) {
      R[next].st = WAITING;
      next++;
    }
    if (n_done == n) break;
    if (steps >= cfg->max_steps) {
      status = OR_MAX_STEPS;
      break;
    }

    // (a3) GroupRequests (step 1)
    std::vector<int> Wg, Rr, Rd, Rp;
    for (int i = 0; i < n; i++)
      if (R[i].st == WAITING) Wg.push_back(i);  // by (T, id) = index order (Q1, Q2)
    for (int i = 0; i < n; i++)
      if (R[i].st == RUNNING) Rr.push_back(i);
    std::stable_sort(Rr.begin(), Rr.end(),
                     [&](int a, int b) {  // Q3 (or its alternative: SRF visits in admission order), Q6
                       if (cfg->knobs & OR_KNOB_SRF_VISIT_ADMISSION) return R[a].seq < R[b].seq;
                       return retained_longer(R[a], R[b], repl, by_arrival);
                     });
    for (int i : Rr) (phase_of(R[i]) == PH_DECODE ? Rd : Rp).push_back(i);
    std::vector<std::vector<int>> groups;
    if (cfg->order == OR_PREFILL_FIRST) {  // vLLM {R_w, R_r}
      groups = {Wg, Rr};
    } else if (cfg->order == OR_DECODE_FIRST) {  // Sarathi {R_r^d, R_r^p, R_w}
      groups = {Rd, Rp, Wg};
    } else {  // Rank_org / Rank_I / Rank_O: one group (Q20, Q37)
      std::vector<int> all;
      for (int i = 0; i < n; i++)
        if (R[i].st == WAITING || R[i].st == RUNNING) all.push_back(i);
      std::stable_sort(all.begin(), all.end(), [&](int a, int b) {
        if (cfg->order == OR_RANK_I && R[a].I != R[b].I) return R[a].I < R[b].I;
        if (cfg->order == OR_RANK_O && R[a].O != R[b].O) return R[a].O < R[b].O;
        return a < b;  // (T, id)
      });
      groups = {all};
    }

    // GetNextBatch (steps 2-4)
    for (auto& grp : groups) out->visits += (int64_t)grp.size();
    std::vector<Entry> B;
    int64_t tok = 0;
    int bphase = PH_NONE;
    int64_t trace_hdr = tr.ilen;
    int64_t n_events = 0;
    if (trace_i) {  // header placeholder: step, n_entries, n_events, U_after, tok
      for (int z = 0; z < 5; z++) tr.pi(0);
    }
    evs.clear();
    // one candidate of Algorithm 1's foreach: steps (2)-(4); admits r into B or leaves it
    auto admit_one = [&](Req& r, int id) {
      int ph = phase_of(r);
      // (2) CheckHybridBatching; batch phase = first admitted entry (Q19)
      if (!cfg->hybrid && bphase != PH_NONE && ph != bphase) return;
      // Q16 alternative: at most max_seqs entries per batch (a cap failure never preempts, like Q11)
      if (cfg->max_seqs > 0 && (int64_t)B.size() >= cfg->max_seqs) return;
      // (3a) token limit C, chunked prefill cropping (Q12)
      int64_t c;
      if (ph == PH_DECODE)
        c = 1;
      else
        c = cfg->chunked ? std::min(avail(r), C - tok) : avail(r);
      if (c == 0 || tok + c > C) return;  // token failure never preempts (Q11)
      // SRF+Hist: defer waiting candidates predicted to cause preemption (Q31)
      if (repl == OR_SRF_HIST && r.st == WAITING && finiteM) {
        bool any_running = false;
        int64_t sumrem = 0;
        for (const Req& q : R)
          if (q.st == RUNNING) {
            any_running = true;
            sumrem += std::max(hist_predict(hist, q.I) - q.g, (int64_t)0);
          }
        int64_t rem = std::max(hist_predict(hist, r.I) - r.g, (int64_t)0);
        if (any_running && U + sumrem + seq_len(r) + rem > M) return;
      }
      // (3b) KV limit M: post-batch holdings sum max(reserved, m+c) <= M (Q13, Fig. 3)
      int64_t newheld = blocks(std::max(r.st == WAITING ? initial_reserve(r) : r.reserved, r.m + c), kvb);
      int64_t delta = newheld - held(r, kvb);
      bool fits = true;
      // Q16 alternative: a waiting admission must also leave kv_watermark KVs free (it never preempts, Q5)
      if (finiteM && r.st == WAITING && U + delta + wm > M) return;
      while (finiteM && U + delta > M) {
        if (r.st == WAITING) {  // holds no KVs: skipped, never preempts (Q5)
          fits = false;
          break;
        }
        if (repl == OR_PF) {  // preemption-free: skipped, never preempts (Table 2)
          fits = false;
          break;
        }
        // (4) PreemptLowerPriorityRequest: running, not in B, lower retention (Q4)
        int victim = -1;
        for (int j = 0; j < n; j++) {
          const Req& q = R[j];
          if (j == id || q.st != RUNNING || q.in_batch) continue;
          if (!retained_longer(r, q, repl, by_arrival)) continue;
          if (victim < 0 || retained_longer(R[victim], q, repl, by_arrival)) victim = j;
        }
        if (victim < 0) {  // "If no such request remains, cand is self-preempted" (Q8)
          preempt(r);
          fits = false;
          break;
        }
        preempt(R[victim]);
      }
      if (!fits) return;
      if (r.st == WAITING) {  // (re)admission: reserve the Table 2 "Initial KV reserve"
        r.st = RUNNING;
        r.reserved = initial_reserve(r);
        r.filled = false;
        r.seq = ++seq;
      }
      U += delta;
      tok += c;
      r.in_batch = true;
      B.push_back(Entry{id, c, r.m, ph});
      if (bphase == PH_NONE) bphase = ph;
    };
    const bool hol = cfg->knobs & OR_KNOB_HOL;
    bool wblocked = false;  // Q10 alternative: a waiting candidate was not admitted in this step
    for (auto& grp : groups) {
      for (int id : grp) {
        Req& r = R[id];
        if (r.preempted_now) continue;  // Q9
        const bool was_waiting = r.st == WAITING;
        if (hol && was_waiting && wblocked) continue;  // head-of-line blocking: R_w's visit has ended
        const size_t nb_before = B.size();
        admit_one(r, id);
        if (hol && was_waiting && B.size() == nb_before) wblocked = true;
      }
    }
    n_events = (int64_t)evs.size() / 2;

    if (B.empty()) {
      if (trace_i && !tr.overflow) tr.ilen = trace_hdr;  // drop the header: an idle jump is not a step
      for (Req& q : R) q.preempted_now = false;
      if (n_events != 0) {  // cannot happen: a preemption only occurs for a running candidate that then fits
        status = OR_DEADLOCK;
        break;
      }
      if (next < n) {  // idle: jump to the next arrival, not a step (Q21)
        clock[0] = std::max(clock[0], R[next].T);
        out->idle_jumps++;
        continue;
      }
      status = OR_DEADLOCK;
      break;
    }

    // (a9) Process(B) in simulation: batch time from the cost model
    steps++;
    out->sum_U += U;
    double start = clock[0];
    double d0 = 0.0;
    for (int k = 0; k < K; k++) {
      double d = batch_time(cms[k], B);
      if (k == 0) d0 = d;
      clock[k] = clock[k] + d;  // Q36: one sequential fp64 add per step
    }
    if (trace_i && !tr.overflow) {
      tr.ti[trace_hdr + 0] = steps - 1;
      tr.ti[trace_hdr + 1] = (int64_t)B.size();
      tr.ti[trace_hdr + 2] = n_events;
      tr.ti[trace_hdr + 3] = U;
      tr.ti[trace_hdr + 4] = tok;
      for (const Entry& e : B) {
        tr.pi(e.id);
        tr.pi(e.phase);
        tr.pi(e.c);
        tr.pi(e.m_before);
      }
      for (int64_t v : evs) tr.pi(v);
      tr.pd(start);
      tr.pd(d0);
    }
    // (a10) token generation (Eq. 6); completed requests free KVs at batch end (Q14)
    for (const Entry& e : B) {
      Req& r = R[e.id];
      int64_t s_before = seq_len(r);
      r.m = e.m_before + e.c;
      out->batch_entries++;
      out->processed_tokens += e.c;
      if (e.phase == PH_PREFILL) out->prefill_entries++;
      if (e.c == s_before - e.m_before) {  // all available tokens processed -> g += 1 (Q18)
        r.g++;
        r.filled = true;
        if (!r.has_first) {
          r.has_first = true;
          for (int k = 0; k < K; k++) r.t_first[k] = clock[k];
        }
        if (r.g == r.O) {
          U -= held(r, kvb);
          r.st = DONE;
          for (int k = 0; k < K; k++) r.t_done[k] = clock[k];
          hist[bucket_of(r.I) * 18 + bucket_of(r.O)]++;
          n_done++;
        }
      }
      r.in_batch = false;
    }
    for (Req& q : R) q.preempted_now = false;
    // self-check: U equals the recomputed holdings (c.3 note)
    int64_t Uchk = 0;
    for (const Req& q : R) Uchk += held(q, kvb);
    if (Uchk != U) return -100;
  }

  out->status = status;
  if (trace_lens) {
    trace_lens[0] = tr.overflow ? -1 : tr.ilen;
    trace_lens[1] = tr.overflow ? -1 : tr.dlen;
  }
  if (status != OR_OK) {  // failed simulations: zero-filled rows
    int st = status;
    std::memset(out, 0, sizeof(*out));  // (visits too)
    out->status = st;
    return 0;
  }
  out->steps = steps;
  // (a11) metrics (Q28, Q29): sums in request index order
  for (int k = 0; k < K; k++) {
    double mx = 0.0, s_lat = 0.0, s_ttft = 0.0, s_tpot = 0.0;
    int64_t n_tpot = 0;
    for (int i = 0; i < n; i++) {
      const Req& r = R[i];
      t_first[(int64_t)k * n + i] = r.t_first[k];
      t_done[(int64_t)k * n + i] = r.t_done[k];
      if (i == 0 || r.t_done[k] > mx) mx = r.t_done[k];
      s_lat = s_lat + (r.t_done[k] - r.T);
      s_ttft = s_ttft + (r.t_first[k] - r.T);
      if (r.O > 1) {
        s_tpot = s_tpot + (r.t_done[k] - r.t_first[k]) / (double)(r.O - 1);
        n_tpot++;
      }
    }
    out->makespan[k] = mx - R[0].T;
    out->mean_latency[k] = s_lat / (double)n;
    out->mean_ttft[k] = s_ttft / (double)n;
    out->mean_tpot[k] = n_tpot > 0 ? s_tpot / (double)n_tpot : 0.0;
  }
  for (int i = 0; i < n; i++) {
    n_preempt[i] = R[i].n_preempt;
    refill_tokens[i] = R[i].refill;
  }
  return 0;
}

// ---- exact optimum of the CSP (Sec. "Optimal Scheduling as Constraint Satisfaction Problem") ----
// One request's state after batch j: done, or (g = tokens generated, m = KVs cached, filled).  Batch j chooses for
// every unfinished request either e = 1 (preempt: m := 0, Eq. (4)) or c in [0, s - m] with s = I + g (Eq. (5)); it
// generates a token iff c = s - m (Eq. (6)), s grows by that token, and the batch respects sum c <= C and
// sum m <= M after processing (Eq. (7)).  A request that generated its O-th token is done and holds nothing from
// the next batch on (Q14, Q44).  The objective is sum_j d_j with the batch cost model; an entry is
// a prefill unless the request is filled (its last (re)fill completed, Q17, Q45).  Batches with sum c = 0 are
// excluded (they cost time and change nothing but could be merged, Q43).  Dijkstra from the all-empty state.
struct OptReq {
  int64_t g, m;
  bool filled, done;
};

int oracle_optimum(int32_t n, const int32_t* I, const int32_t* O, int64_t C, int64_t M, int32_t no_preempt,
                   const oracle_cost_t* cm,
                   oracle_opt_t* out) {
  if (n < 1 || !I || !O || !cm || !out || C < 1 || M < 0) return -1;
  for (int i = 0; i < n; i++)
    if (I[i] < 1 || O[i] < 1) return -5;
  using State = std::vector<OptReq>;
  // Requests with the same (I, O) are interchangeable: permuting them maps every schedule to one of the same
  // cost, so a state is identified up to such permutations -- its key lists each request's (g, filled, m) pair
  // with the pairs of every group of identical requests sorted (the canonical representative)
  std::vector<std::vector<int>> groups;
  for (int i = 0; i < n; i++) {
    bool placed = false;
    for (auto& gr : groups)
      if (I[gr[0]] == I[i] && O[gr[0]] == O[i]) {
        gr.push_back(i);
        placed = true;
        break;
      }
    if (!placed) groups.push_back({i});
  }
  auto key = [&](const State& st) {
    std::vector<int64_t> k;
    for (const auto& gr : groups) {
      std::vector<std::pair<int64_t, int64_t>> pr;
      for (int i : gr) {
        const OptReq& r = st[i];
        pr.push_back({r.done ? -1 : 2 * r.g + (r.filled ? 1 : 0), r.done ? 0 : r.m});
      }
      std::sort(pr.begin(), pr.end());
      for (auto& x : pr) k.push_back(x.first), k.push_back(x.second);
    }
    return k;
  };
  std::map<std::vector<int64_t>, double> dist;
  std::map<std::vector<int64_t>, bool> settled;
  using Item = std::pair<double, std::vector<int64_t>>;
  std::priority_queue<Item, std::vector<Item>, std::greater<Item>> pq;
  std::map<std::vector<int64_t>, State> states;
  State start(n);
  for (int i = 0; i < n; i++) start[i] = OptReq{0, 0, false, false};
  dist[key(start)] = 0.0;
  states[key(start)] = start;
  pq.push(Item(0.0, key(start)));
  int64_t n_settled = 0;
  double best = -1.0;
  while (!pq.empty()) {
    const Item top = pq.top();
    pq.pop();
    if (settled[top.second]) continue;
    settled[top.second] = true;
    n_settled++;
    const State u = states[top.second];
    const double du = top.first;
    bool all_done = true;
    for (const OptReq& r : u) all_done = all_done && r.done;
    if (all_done) {
      best = du;
      continue;
    }
    // every batch: each unfinished request picks idle, preempt (m > 0) or a c >= 1; recursion over requests
    State v(n);
    std::vector<Entry> B;
    std::function<void(int, int64_t, int64_t)> rec = [&](int i, int64_t sum_c, int64_t sum_m) {
      if (sum_c > C || sum_m > M) return;  // Eq. (7); both sums only grow with i
      if (i == n) {
        if (sum_c == 0) return;
        const double w = batch_time(*cm, B);
        const double cand = du + w;
        const std::vector<int64_t> kv = key(v);
        auto it = dist.find(kv);
        if (it == dist.end() || cand < it->second) {
          dist[kv] = cand;
          states[kv] = v;
          pq.push(Item(cand, kv));
        }
        return;
      }
      const OptReq& r = u[i];
      if (r.done) {
        v[i] = r;
        rec(i + 1, sum_c, sum_m);
        return;
      }
      const int64_t s = I[i] + r.g;
      v[i] = r;  // idle: c = 0, e = 0
      rec(i + 1, sum_c, sum_m + r.m);
      if (r.m > 0 && !no_preempt) {  // preempt: e = 1, m := 0, c = 0 (Eq. (4)-(5)); off: preemption-free schedules
        v[i] = OptReq{r.g, 0, false, false};
        rec(i + 1, sum_c, sum_m);
      }
      for (int64_t c = 1; c <= s - r.m; c++) {
        const bool token = c == s - r.m;  // Eq. (6)
        const int64_t m2 = r.m + c;
        if (token)
          v[i] = (r.g + 1 == O[i]) ? OptReq{r.g + 1, 0, true, true} : OptReq{r.g + 1, m2, true, false};
        else
          v[i] = OptReq{r.g, m2, false, false};
        B.push_back(Entry{i, c, r.m, r.filled ? PH_DECODE : PH_PREFILL});
        rec(i + 1, sum_c + c, sum_m + m2);  // a request finishing in this batch still holds m2 now (Q44)
        B.pop_back();
      }
    };
    rec(0, 0, 0);
  }
  out->status = best < 0.0 ? 1 : 0;
  out->pad = 0;
  out->states = n_settled;
  out->optimum = best < 0.0 ? 0.0 : best;
  return 0;
}

}  // extern "C"
