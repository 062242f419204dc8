// sim_step.cuh -- the step kernel body (included by simsweep.cu).
//
// One CTA = one simulation of Algorithm 1.  Request state
// lives in shared memory as a ring of CAP slots (slot = request id mod CAP):
// a 16-byte record {I, g, m, reserved} (one LDS.128 per candidate), O,
// admission seq, c of the current batch, and a flag byte.  Per step:
//   (1) a2 arrivals (thread 0 binary search over the sorted T) + slot init
//   (2) a3 GroupRequests: run list (retention order) and Sarathi's
//       decode/prefill split are rebuilt only when the previous step dirtied
//       them; the waiting list (index order) is built lazily, only when a round
//       reaches the waiting group and the group is not skippable
//   (3) a4-a8 GetNextBatch in block-parallel rounds.  The step scalars (tok, U,
//       seq, ...) live in registers, identical in every thread.  A round loads
//       all its candidates first (ILP), classifies them against the current
//       (tok, U), prefix-scans (tokens, KV delta, waiting admissions,
//       admissions, SRF+Hist remainders), and admits the prefix before the first
//       "break" -- a candidate the scan cannot decide: a preemption (running
//       decode short of KV), a cumulative KV / deferral / token failure, a chunk
//       crop, or the first admission when hybrid batching is off.  No break: 2
//       barriers.  A break is resolved literally by thread 0 (+2 barriers).
//       The waiting group is skipped whole when even its smallest request fails
//       a monotone check (hybrid phase, KV, token budget).
//   (4) a9+a10 one pass over the batch list B: Eq. (6) state update + exact
//       integer features; warp REDUX reductions; thread 0 evaluates the cost
//       models, advances the clocks, decides a steady decode run
//   (5) t_first/t_done of this step's events; the steady decode run
//   (6) run-list maintenance only when needed
#pragma once

namespace simsweep {

enum { K_NONE = 0, K_MARK = 1, K_EVENT = 2 };
constexpr int WARP_MAX = 256;  // at most this many candidates left in a group: warp-level admission

// Cold blocks of the step loop, kept out of line so that the hot path stays contiguous in the instruction cache
// (DESIGN.md 6).  Each is called by all threads of the CTA.

// rank orders: drop finished entries of the rank list before their slots are reused
template <int NT, int IPT_>
__device__ __noinline__ int rank_drop_done(int16_t* s_rank, int16_t* s_new, const uint8_t* s_fl, int nrank, Scal& S) {
  nrank = block_compact<NT, IPT_>(
      nrank, [&](int q) { return (s_fl[s_rank[q]] & ST_MASK) != ST_DONE; }, [&](int q) { return s_rank[q]; }, s_new, S);
  for (int q = threadIdx.x; q < nrank; q += NT) s_rank[q] = s_new[q];
  __syncthreads();  // the compacted list is read by other threads before the next barrier otherwise
  return nrank;
}

// rank orders: append the arrivals [nx0, nx1) and sort the one group by (key, T, id) (App. D, Q20, Q37)
template <int NT, int CAP>
__device__ __noinline__ int rank_regroup(int16_t* s_rank, unsigned long long* s_keys, const int4* s_rec,
                                         const int32_t* s_O, int nrank, int nx0, int nx1, int lo, int order) {
  const int tid = threadIdx.x;
  for (int idx = nx0 + tid; idx < nx1; idx += NT) s_rank[nrank + idx - nx0] = (int16_t)(idx & (CAP - 1));
  const int nr = nrank + (nx1 - nx0);
  __syncthreads();
  for (int q = tid; q < nr; q += NT) {
    const int sl = s_rank[q];
    const unsigned idx = (unsigned)(lo + ((sl - lo) & (CAP - 1)));
    const unsigned key = order == SIM_ORDER_RANK_I ? (unsigned)s_rec[sl].x
                         : order == SIM_ORDER_RANK_O ? (unsigned)s_O[sl]
                                                     : 0u;
    s_keys[q] = ((unsigned long long)key << 32) | idx;
  }
  block_bitonic<NT>(s_keys, nr);
  for (int q = tid; q < nr; q += NT) s_rank[q] = (int16_t)(s_keys[q] & (CAP - 1));
  __syncthreads();
  return nr;
}

// |R_w| and the smallest s among the waiting requests at window offsets [w0, L), into S.nW / S.minSW
template <int NT, int CAP>
__device__ __noinline__ void waiting_count(const uint8_t* s_fl, const int4* s_rec, int w0, int L, int lo, Scal& S) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int cnt = 0, mn = 0x7fffffff;
  for (int q = w0 + (int)threadIdx.x; q < L; q += NT) {
    const int sl = (lo + q) & (CAP - 1);
    if ((s_fl[sl] & ST_MASK) == ST_WAIT) {
      const int4 r = s_rec[sl];
      cnt++;
      mn = min(mn, r.x + r.y);
    }
  }
  cnt = (int)__reduce_add_sync(0xffffffffu, (unsigned)cnt);
  mn = (int)__reduce_min_sync(0xffffffffu, (unsigned)mn);
  if (lane == 0) S.wsum[wid][0] = cnt, S.wsum[wid][1] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    int nW = 0, minSW = 0x7fffffff;
#pragma unroll
    for (int w = 0; w < NW; w++) nW += S.wsum[w][0], minSW = min(minSW, S.wsum[w][1]);
    S.nW = nW, S.minSW = minSW;
  }
  __syncthreads();
}

// decode-first general path: stable split of the run list into running decodes, then running prefills
template <int NT, int IPT_>
__device__ __noinline__ void run_split(const int16_t* run, int16_t* s_pl, const uint8_t* s_fl, int nrun, Scal& S) {
  const int nrd = block_partition<NT, IPT_>(
      nrun, [&](int q) { return (s_fl[run[q]] & F_FILLED) != 0; }, [&](int q) { return run[q]; }, s_pl, S);
  if (threadIdx.x == 0) S.nRd = nrd;
  __syncthreads();
}

// SRF+Hist: predictions of the current histogram; sum of the remaining outputs of the running requests
template <int NT>
__device__ __noinline__ long long hist_running_rem(const int16_t* run, const int4* s_rec, int nrun, Scal& S) {
  if (threadIdx.x < 18) S.pred[threadIdx.x] = hist_pred_row(S.hist, threadIdx.x);
  __syncthreads();
  long long r = 0;
  for (int q = threadIdx.x; q < nrun; q += NT) {
    const int4 rc = s_rec[run[q]];
    const int rem = S.pred[bucket_of(rc.x)] - rc.y;
    r += rem > 0 ? rem : 0;
  }
  return block_sum_ll<NT>(r, S);
}

template <int NT, int CAP, int IPT_, bool GM, bool KN>
__global__ void __launch_bounds__(NT, (CAP <= 1024 ? (NT <= 128 ? 3 : 512 / NT) : 1)) sim_kernel(KParams p) {
  using L = Smem<NT, CAP>;
  constexpr int NW = NT / 32;
  constexpr int CH = NT * IPT_;  // candidates per round
  constexpr int SLB = __builtin_ctz(CAP);  // bits of a slot index
  static_assert((CAP & (CAP - 1)) == 0 && CAP <= 32768, "slots are int16 ring indices");
  constexpr unsigned FM = 0xffffffffu;
  // the int32 admission counter (Q6) must not wrap: one step admits at most CAP requests
  constexpr long long SEQ_LIM = 0x7fffffffll - CAP;
  extern __shared__ __align__(16) unsigned char smem[];
  Scal& S = *reinterpret_cast<Scal*>(smem);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ci = p.order ? p.order[blockIdx.x] : (int)blockIdx.x;
  if (kernel_variant(p.cfgs[ci], p.wls[p.cfgs[ci].workload].n, p.lean) != p.variant) return;
  unsigned char* arr = smem + L::scal;
  if constexpr (GM) {  // claim a per-CTA arena of the workspace
    if (tid == 0) S.arena = p.arena_base + (int)atomicAdd(reinterpret_cast<unsigned*>(p.ws + p.ctr_off), 1u);
    __syncthreads();
    arr = p.ws + WS_HEADER + (size_t)S.arena * L::arr_bytes;
  }
  int4* s_rec = reinterpret_cast<int4*>(arr + L::off_rec);  // {I, g, m, res}
  int32_t* s_O = reinterpret_cast<int32_t*>(arr + L::off_int);
  int32_t* s_seq = s_O + CAP;  // admission sequence number (Q6)
  int32_t* s_c = s_seq + CAP;  // c of the current batch
  int16_t* s_rpos = reinterpret_cast<int16_t*>(arr + L::off_rpos);
  uint8_t* s_fl = arr + L::off_fl;
  int16_t* s_runA = reinterpret_cast<int16_t*>(arr + L::off_lists);
  int16_t* s_runB = s_runA + CAP;
  int16_t* s_rank = s_runB + CAP;
  int16_t* s_wl = s_rank + CAP;  // waiting list (index order)
  int16_t* s_pl = s_wl + CAP;    // Sarathi split of the run list (decodes, then prefills)
  int16_t* s_bl = s_pl + CAP;    // the batch B in admission order
  int16_t* s_new = reinterpret_cast<int16_t*>(arr + L::off_union);  // admitted from waiting this step
  int16_t* s_vic = s_new + CAP;                                       // preempted this step
  int32_t* s_ev = reinterpret_cast<int32_t*>(arr + L::off_union + 4 * CAP);  // first-token / completion events
  unsigned long long* s_keys = reinterpret_cast<unsigned long long*>(arr + L::off_union);
  double* s_dbuf = reinterpret_cast<double*>(arr + L::off_union + 4 * CAP);  // CAP/2 doubles (over ev)

#ifdef SIMSWEEP_PROFILE
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
  const sim_config_t cfg = p.cfgs[ci];
  const sim_workload_t wl = p.wls[cfg.workload];
  const int n = wl.n;
  const int K = cfg.n_cost;
  // Q15 alternative (paged KV): every KV quantity below (U, M, holdings, deltas) counts blocks of kvb tokens
  const bool paged = KN && cfg.kv_block > 1;
  const int kvb = paged ? cfg.kv_block : 1;
  auto blk = [&](int x) -> int { return paged ? (x + kvb - 1) / kvb : x; };
  const int M = cfg.M >= 0 ? (int)(cfg.M / kvb) : 0, C = (int)cfg.C;  // host-validated < 2^30
  const bool finiteM = cfg.M >= 0, hybrid = cfg.hybrid != 0, chunked = cfg.chunked != 0;
  const int order = cfg.order;
  const bool srf = cfg.replacement == SIM_SRF || cfg.replacement == SIM_SRF_HIST;
  const bool hist = cfg.replacement == SIM_SRF_HIST && finiteM;
  const bool pf = cfg.replacement == SIM_PF;  // preemption-free: a running KV failure is skipped (Table 2)
  // Table 2 "Initial KV reserve": s = I + g (SEQ), I + O - 1 (PEAK, *^pf), S (CONTEXT, Orca).  Under
  // PEAK / CONTEXT every running request already holds its peak usage, so its KV delta is 0 (kv1 = false:
  // a decode needs no KV); under SEQ a filled request's decode needs exactly one.
  const int rmode = cfg.reserve;
  const bool kv1 = rmode == SIM_RESERVE_SEQ;
  const bool rank = order >= SIM_ORDER_RANK_ORG;
  // alternative readings: head-of-line blocking of R_w (Q10), a cap on |B| and a KV watermark
  // for waiting admissions (Q16); with the defaults (0) every check below is a no-op
  // (KN = false: the kernel instance for configs without knobs, where all of these checks compile away)
  const bool holk = KN && (cfg.knobs & SIM_KNOB_HOL) != 0;
  const bool trc = KN && p.tr.steps != nullptr;  // schedule trace (sim_run_traced; the KN instance)
  const bool arr_ord = KN && (cfg.knobs & SIM_KNOB_NRF_ARRIVAL) != 0;  // NRF run list in arrival order (Q6 alt.)
  // Q3 alternative: SRF visits in admission order (the run list is not re-sorted) and only picks victims by m,
  // so the victim pool is not the run list's tail: the closed form is off and victims are searched literally
  const bool q3alt = KN && (cfg.knobs & SIM_KNOB_SRF_VISIT_ADMISSION) != 0;
  const bool srf_order = srf && !q3alt;
  const int capB = cfg.max_seqs > 0 ? (int)cfg.max_seqs : 0x3fffffff;
  const int Mw = finiteM ? M - blk((int)cfg.kv_watermark) : 0x3fffffff;  // the KV bound of a waiting admission
  const long long row0 = p.row_off[ci], tim0 = p.tim_off[ci];
  double* tf = p.req.t_first + tim0;
  double* td = p.req.t_done + tim0;
  unsigned long long* npre = reinterpret_cast<unsigned long long*>(p.req.n_preempt + row0);
  unsigned long long* refill = reinterpret_cast<unsigned long long*>(p.req.refill_tokens + row0);

  for (int i = tid; i < n; i += NT) {
    npre[i] = 0;
    refill[i] = 0;
  }
  for (int x = tid; x < K * n; x += NT) {
    tf[x] = 0.0;
    td[x] = 0.0;
  }
  // ---- a1: per-simulation validation (Q35) ----
  int bad_long = 0, bad_fit = 0;
  long long ub = 0;  // M infinite: an upper bound of the int32 holdings U (each request holds <= max(peak, reserve))
  for (int i = tid; i < n; i += NT) {
    long long pk = (long long)wl.I[i] + wl.O[i] - 1;  // peak KV usage
    bad_long |= pk > cfg.S;
    bad_fit |= (finiteM && blk((int)pk) + blk((int)cfg.kv_watermark) > M) || (!chunked && pk > cfg.C);
    bad_fit |= finiteM && cfg.reserve == SIM_RESERVE_CONTEXT && blk(cfg.S) + blk((int)cfg.kv_watermark) > M;  // Q35
    if (!finiteM && pk <= cfg.S) ub += blk((int)(cfg.reserve == SIM_RESERVE_CONTEXT ? max(pk, (long long)cfg.S) : pk));
  }
  bad_long = __syncthreads_or(bad_long);
  bad_fit = __syncthreads_or(bad_fit);
  const bool bad_cap = !finiteM && block_sum_ll<NT>(ub, S) > 0x7fffffffll;  // (uniform branch: finiteM)
  if (bad_long || bad_fit || bad_cap) {
    if (tid == 0) {
      sim_result_t r;
      memset(&r, 0, sizeof(r));
      r.status = bad_long ? SIM_S_TOO_LONG : (bad_fit ? SIM_S_NEVER_FITS : SIM_S_CAPACITY);
      p.results[ci] = r;
    }
    return;
  }
  bool anyTheo = false;
  for (int k = 0; k < K; k++) anyTheo |= p.cms[cfg.cost[k]].mode == 1;
  if (tid == 0) {
    for (int k = 0; k < SIM_MAX_COST; k++) S.clock[k] = 0.0;
    S.U = S.seq = 0;
    S.steps = S.preempt = S.entries = S.processed = S.sumU = S.pentries = S.idle = S.visits = S.formed = 0;
    S.next = S.new_next = S.lo = S.n_done = S.n_run = 0;
    S.nrank = S.nW = S.minSW = S.n_ev = S.n_vic = S.nB = 0;
    if (KN) S.tr_ent = S.tr_ev = 0;
    S.r_dirty = S.o_dirty = S.rank_dirty = S.removals = S.wbuilt = 0;
    S.status = 0;
    S.cur = 0;
    S.w_dirty = S.p_dirty = 1;
    S.wstale = 0;
    S.wfirst = 0;
    S.wf_new = -1, S.wf_vic = 0x7fffffff, S.idle_st = 0;
  }
  if (tid < K) S.cm[tid] = p.cms[cfg.cost[tid]];
  for (int i = tid; i < 18 * 18; i += NT) S.hist[i] = 0;
  __syncthreads();
#ifdef SIMSWEEP_PROFILE
  long long prof[24] = {0};
  long long prof_last = clock64();
#endif

  int exit_status = 0;
#ifdef SIMSWEEP_TRACE
  int trn = 0;
#endif
  for (;;) {
    PROF_MARK(10);
    TMARK(1);
    // ---- (1) a2: GetNewRequests (Alg. 1 line 3): all T <= clock, inclusive (Q21) ----
    int nx1;
    if (S.next >= n) {  // everything has arrived (offline after step 1): uniform checks, no barrier
      nx1 = n;
      exit_status = S.n_done == n ? -1 : (S.steps >= cfg.max_steps ? SIM_S_MAX_STEPS : (S.seq > SEQ_LIM ? SIM_S_CAPACITY : 0));
    } else {
      if (tid == 0) {
        int a = S.next, b = n;
        const double clk = S.clock[0];
        while (a < b) {
          int mid = (a + b) >> 1;
          if (wl.T[mid] <= clk)
            a = mid + 1;
          else
            b = mid;
        }
        if (a > S.next) S.wfirst = min(S.wfirst, S.next);  // new arrivals wait
        S.new_next = a;
        int st = 0;
        if (S.n_done == n)
          st = -1;
        else if (a - S.lo > CAP)
          st = SIM_S_CAPACITY;
        else if (S.steps >= cfg.max_steps)
          st = SIM_S_MAX_STEPS;
        else if (S.seq > SEQ_LIM)
          st = SIM_S_CAPACITY;
        S.status = st;
      }
      __syncthreads();
      nx1 = S.new_next;
      exit_status = S.status;
    }
    if (exit_status) break;
    const int nx0 = S.next, lo = S.lo;
    const bool arrived = nx1 > nx0;
    const int nrun = S.n_run;
    int16_t* run = S.cur ? s_runB : s_runA;
    int nrank = S.nrank;
    if (rank && (arrived || S.rank_dirty) && nrank > 0)  // drop finished entries before slot reuse
      nrank = rank_drop_done<NT, IPT_>(s_rank, s_new, s_fl, nrank, S);
    for (int idx = nx0 + tid; idx < nx1; idx += NT) {
      const int sl = idx & (CAP - 1);
      s_rec[sl] = make_int4(wl.I[idx], 0, 0, 0);
      s_O[sl] = wl.O[idx];
      s_seq[sl] = 0;
      s_c[sl] = 0;
      s_fl[sl] = ST_WAIT;
    }
    if (arrived) __syncthreads();
    PROF_MARK(0);
    TMARK(2);
    // ---- (2) a3: GroupRequests (step 1) ----
    if (rank && arrived)  // one group sorted by (key, T, id) (App. D, Q20, Q37)
      nrank = rank_regroup<NT, CAP>(s_rank, s_keys, s_rec, s_O, nrank, nx0, nx1, lo, order);
    int nW = S.nW, minSW = S.minSW, wbuilt = S.wbuilt;
    const int w0 = max(S.wfirst - lo, 0);  // window offsets below w0 hold no waiting request
    if (!rank && (S.w_dirty || arrived)) {  // |R_w| and its smallest s (the skip test); list built lazily
      waiting_count<NT, CAP>(s_fl, s_rec, w0, nx1 - lo, lo, S);
      nW = S.nW, minSW = S.minSW, wbuilt = 0;
    }
    int nRd = 0;
    if (order == SIM_ORDER_DECODE_FIRST && (nrun > CH || q3alt)) {  // general path: stable split of the run list
      if (S.p_dirty) run_split<NT, IPT_>(run, s_pl, s_fl, nrun, S);
      nRd = S.nRd;
    }
    const int16_t* seg0;
    const int16_t* seg1;
    int len0, len1;
    if (order == SIM_ORDER_PREFILL_FIRST) {  // {R_w, R_r}
      seg0 = s_wl, len0 = nW, seg1 = run, len1 = nrun;
    } else if (order == SIM_ORDER_DECODE_FIRST) {
      seg0 = s_pl, len0 = nrun, seg1 = s_wl, len1 = nW;
    } else {
      seg0 = s_rank, len0 = nrank, seg1 = s_rank, len1 = 0;
    }
    const int nP = len0 + len1;
    auto cand = [&](int q) -> int { return q < len0 ? seg0[q] : seg1[q - len0]; };
    // the waiting group's range in P
    const int wbeg = order == SIM_ORDER_PREFILL_FIRST ? 0 : (order == SIM_ORDER_DECODE_FIRST ? len0 : nP);
    const int wend = order == SIM_ORDER_PREFILL_FIRST ? nW : nP;

    long long Rs = 0;
    if (hist)  // SRF+Hist: predictions of the current histogram; sum of remaining outputs of running requests
      Rs = hist_running_rem<NT>(run, s_rec, nrun, S);
    if (tid == 0) {
      S.vt = nrun - 1;
      S.any_pre = 0;
      S.h_pre = 0;
      S.cut = nrun;
      S.n_vic = 0;
      if (nrank != S.nrank) S.nrank = nrank;  // (changed only after the rank helpers' barriers)
      S.visits += nP;
    }
    PROF_MARK(1);
    TMARK(3);

    // ---- (3) a4-a8: GetNextBatch (steps 2-4) ----
    int tok = 0, U = (int)S.U, n_new = 0, n_running = nrun, bph = -1, pos = 0, nB = 0;
    int seq = (int)S.seq;
    int wblk = 0;  // head-of-line knob: a waiting candidate was not admitted in this step

    auto rnew = [&](const int4& rc, int sl) -> int {  // reserve taken at (re)admission
      return rmode == SIM_RESERVE_SEQ ? rc.x + rc.y : (rmode == SIM_RESERVE_PEAK ? rc.x + s_O[sl] - 1 : cfg.S);
    };
    auto preempt = [&](int v) {  // thread 0 only (refill P:1570)
      const int4 rc = s_rec[v];
      U -= blk(max(rc.w, rc.z));
      if (hist) Rs -= max(S.pred[bucket_of(rc.x)] - rc.y, 0);
      const int idx = lo + ((v - lo) & (CAP - 1));
      atomicAdd(&npre[idx], 1ull);
      atomicAdd(&refill[idx], (unsigned long long)rc.z);
      s_rec[v] = make_int4(rc.x, rc.y, 0, 0);
      s_fl[v] = ST_WAIT | F_PRE | (s_fl[v] & F_FIRST);
      if (trc) {
        const long long e = S.tr_ev + S.n_vic;
        if (e < p.tr.cap_events) p.tr.events[e] = sim_trace_event_t{idx, rc.z};
      }
      s_vic[S.n_vic++] = (int16_t)v;
      n_running--;
      S.preempt++;
      S.any_pre = 1;
      S.h_pre = 1;  // a preemption outside the closed form: the run list needs a full compaction
    };
    auto handle_one = [&](int sl) {  // literal sequential resolution of one candidate (thread 0)
      uint8_t fl = s_fl[sl];
      const bool isW = (fl & ST_MASK) == ST_WAIT;
      const int ph = (isW || !(fl & F_FILLED)) ? PH_PRE : PH_DEC;
      if (!hybrid && bph >= 0 && ph != bph) return;  // step 2
      if (KN && nB >= capB) return;                   // max_seqs knob: never preempts (Q16 alternative)
      const int4 rc = s_rec[sl];
      const int s = rc.x + rc.y, avail = s - rc.z;
      const int c = ph == PH_DEC ? 1 : (chunked ? min(avail, C - tok) : avail);
      if (c == 0 || tok + c > C) return;  // token limit never preempts (Q11)
      int rem = 0;
      if (hist && isW) {
        rem = max(S.pred[bucket_of(rc.x)] - rc.y, 0);
        if (n_running > 0 && (long long)U + Rs + s + rem > M) return;  // deferred (Q31)
      }
      const int rw = isW ? rnew(rc, sl) : rc.w;
      const int nh = blk(max(rw, rc.z + c)), held = isW ? 0 : blk(max(rc.w, rc.z)), delta = nh - held;
      if (KN && isW && finiteM && U + delta > Mw) return;  // watermark knob (a waiting candidate never preempts, Q5)
      while (finiteM && U + delta > M) {
        if (isW || pf) return;  // holds no KVs (Q5) / preemption-free: skipped
        if (q3alt) {  // lowest SRF retention among running requests outside B retained less than sl (Q3 alt.)
          const int cm = rc.z, cs = s_seq[sl];
          int best = -1, bm = 0, bs = 0;
          for (int q = 0; q < nrun; q++) {
            const int v = run[q];
            const uint8_t f = s_fl[v];
            if (v == sl || (f & F_INB) || (f & ST_MASK) != ST_RUN) continue;
            const int vm = s_rec[v].z, vs = s_seq[v];
            if (!(cm > vm || (cm == vm && cs < vs))) continue;
            if (best < 0 || vm < bm || (vm == bm && vs > bs)) best = v, bm = vm, bs = vs;
          }
          if (best < 0) {  // self-preemption (Q8)
            preempt(sl);
            return;
          }
          preempt(best);
          continue;
        }
        const int pc = s_rpos[sl];
        int vt = S.vt;
        while (vt > pc) {  // lowest retention = tail of the retention-ordered run list
          const uint8_t f = s_fl[run[vt]];
          if (!(f & F_INB) && (f & ST_MASK) == ST_RUN) break;
          vt--;
        }
        if (vt <= pc) {  // self-preemption (Q8)
          S.vt = vt;
          preempt(sl);
          return;
        }
        preempt(run[vt]);
        S.vt = vt - 1;
      }
      if (isW) {  // (re)admission takes the initial reserve (Table 2, Q13)
        seq++;
        s_seq[sl] = seq;
        s_rec[sl] = make_int4(rc.x, rc.y, rc.z, rw);
        fl = ST_RUN | (fl & F_FIRST);
        s_new[n_new++] = (int16_t)sl;
        n_running++;
        Rs += rem;
      }
      s_fl[sl] = fl | F_INB;
      s_c[sl] = c;
      s_bl[nB++] = (int16_t)sl;
      U += delta;
      tok += c;
      if (bph < 0) bph = ph;
    };
    auto handle = [&](int sl) {
      const uint8_t fl = s_fl[sl];
      if (fl & F_PRE) return;  // Q9: preempted in this step -- not a candidate (and not a failure)
      const bool isW = (fl & ST_MASK) == ST_WAIT;
      if (holk && isW && wblk) return;  // head-of-line knob: R_w's visit has ended
      const int nb0 = nB;
      handle_one(sl);
      if (holk && isW && nB == nb0) wblk = 1;
    };

    // Warp-level admission over [b0, b1) (warp 0 only): positions in P (overWin = false) or offsets in
    // the waiting window (overWin = true: slot (lo + i) mod CAP, waiting and not preempted this step =
    // R_w in index order).  32 candidates per chunk: classify, warp prefix scans, ballot the first break,
    // admit the lanes before it, resolve the break on lane 0 (same handle() as the block path).
    auto warp_run = [&](bool overWin, int b0, int b1) {
      int i0 = b0;
      while (i0 < b1) {
        PROF_CNT(13, 1);
        if (overWin) {  // the rest of R_w fails a monotone check: stop
          const bool wrej = (!hybrid && bph == PH_DEC) || (KN && nB >= capB) || (finiteM && (long long)U + blk(minSW) > (KN ? Mw : M)) ||
                            (chunked ? tok >= C : minSW > C - tok);
          if (wrej) break;
        }
        const int i = i0 + lane;
        int sl = -1;
        if (i < b1) {
          if (overWin) {
            const int s2 = (lo + i) & (CAP - 1);
            if ((s_fl[s2] & (ST_MASK | F_PRE)) == ST_WAIT) sl = s2;
          } else {
            sl = cand(i);
          }
        }
        const int4 rc = s_rec[sl < 0 ? 0 : sl];
        const uint8_t fl = s_fl[sl < 0 ? 0 : sl];
        const bool anyRun0 = n_running > 0;
        const bool isW = (fl & ST_MASK) == ST_WAIT;
        const int ph = (isW || !(fl & F_FILLED)) ? PH_PRE : PH_DEC;
        const int s = rc.x + rc.y, avail = s - rc.z;
        const int rt0 = C - tok;
        const int c = ph == PH_DEC ? 1 : (chunked ? min(avail, rt0) : avail);
        int rem = 0;
        const bool cand0 = sl >= 0 && !(fl & F_PRE) && !(holk && isW && wblk);  // a candidate at all
        bool ok = cand0 && (hybrid || bph < 0 || ph == bph) && c >= 1 && c <= rt0 && (!KN || nB < capB);
        if (hist && isW) {
          rem = max(S.pred[bucket_of(rc.x)] - rc.y, 0);
          ok = ok && !(anyRun0 && (long long)U + Rs + s + rem > M);
        }
        const int rw = isW ? rnew(rc, sl < 0 ? 0 : sl) : rc.w;
        const int delta = blk(max(rw, rc.z + c)) - (isW ? 0 : blk(max(rc.w, rc.z)));
        if (KN && isW && finiteM && U + delta > Mw) ok = false;  // watermark knob
        const bool kvfail = finiteM && U + delta > M;
        const int kind = !ok ? K_NONE : (kvfail ? ((isW || pf) ? K_NONE : K_EVENT) : K_MARK);
        const bool mk = kind == K_MARK;
        const int cc = mk ? (ph == PH_DEC ? 1 : avail) : 0, dd = mk ? delta : 0, ww = mk && isW, kk = mk;
        const int rr = mk ? rem : 0;
        int xc = cc, xd = dd, xw = ww, xk = kk, xr = rr;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int yc = __shfl_up_sync(FM, xc, o), yd = __shfl_up_sync(FM, xd, o);
          const int yw = __shfl_up_sync(FM, xw, o), yk = __shfl_up_sync(FM, xk, o);
          if (lane >= o) xc += yc, xd += yd, xw += yw, xk += yk;
          if (hist) {
            const int yr = __shfl_up_sync(FM, xr, o);
            if (lane >= o) xr += yr;
          }
        }
        const int ec = xc - cc, ed = xd - dd, ew = xw - ww, ek = xk - kk, er = xr - rr;  // exclusive
        bool brk = false;
        if (mk) {
          const int pU = U + ed, rt = C - (tok + ec);
          brk = !hybrid && bph < 0;  // the first admission fixes the batch phase (Q19)
          if (ph == PH_PRE && chunked)
            brk |= rt < avail;
          else
            brk |= cc > rt;
          if (hist && isW) brk |= (anyRun0 || ew > 0) && (long long)pU + Rs + er + s + rem > M;
          if (finiteM) brk |= pU + dd > (KN && isW ? Mw : M);
          if (KN) brk |= nB + ek >= capB;  // max_seqs knob
        } else if (kind == K_EVENT) {
          brk = tok + ec + 1 <= C;  // else a token reject (Q11)
        } else if (holk && isW && cand0) {
          brk = true;  // head-of-line knob: this waiting failure ends R_w's visit (resolved literally)
        }
        const unsigned bm = __ballot_sync(FM, brk);
        const int b = bm ? __ffs(bm) - 1 : 32;
        if (mk && lane < b) {  // admitted: every check passed at its exact position
          s_c[sl] = cc;
          s_bl[nB + ek] = (int16_t)sl;
          if (isW) {
            s_seq[sl] = seq + ew + 1;
            s_rec[sl] = make_int4(rc.x, rc.y, rc.z, rw);
            s_fl[sl] = ST_RUN | F_INB | (fl & F_FIRST);
            s_new[n_new + ew] = (int16_t)sl;
          } else {
            s_fl[sl] = fl | F_INB;
          }
        }
        const bool inner = b < 32;
        const int src = inner ? b : 31;
        const int ac = __shfl_sync(FM, inner ? ec : xc, src), ad = __shfl_sync(FM, inner ? ed : xd, src);
        const int aw = __shfl_sync(FM, inner ? ew : xw, src), ak = __shfl_sync(FM, inner ? ek : xk, src);
        const int ar = __shfl_sync(FM, inner ? er : xr, src);
        tok += ac, U += ad, seq += aw, n_new += aw, n_running += aw, nB += ak, Rs += ar;
        if (inner) {
          PROF_CNT(14, 1);
          const int bsl = __shfl_sync(FM, sl, b);
          __syncwarp();
          if (lane == 0) handle(bsl);
          __syncwarp();
          tok = __shfl_sync(FM, tok, 0), U = __shfl_sync(FM, U, 0), seq = __shfl_sync(FM, seq, 0);
          n_new = __shfl_sync(FM, n_new, 0), n_running = __shfl_sync(FM, n_running, 0);
          nB = __shfl_sync(FM, nB, 0), bph = __shfl_sync(FM, bph, 0), Rs = __shfl_sync(FM, Rs, 0);
          wblk = __shfl_sync(FM, wblk, 0);
          i0 += b + 1;
        } else {
          i0 += 32;
        }
      }
    };

    // Closed form for a group of running decodes visited in retention order (all heads need one KV; the
    // victim pool is the run-list tail, all running and not in B).  Head i (run position p_i) is admitted
    // iff i <= C - tok and F + RS(p_i + 1) >= i, F = M - U, RS(q) = sum of held KVs at run positions >= q
    // (monotone in i).  Admitting a heads evicts the minimal tail suffix [q*, n) with F + RS(q*) >= a;
    // if head a+1 runs out of pool, everything behind it is evicted and it self-preempts (Q8).  This is
    // exactly the sequential head/tail walk of steps (3)-(4), done in O(1) passes.
    // pf: heads = run[0..k) (prefill-first, non-chunked: every running request decodes),
    // else heads = s_pl[0..k) (R_r^d).  Requires nrun <= CH.
    int rp_first = 0;  // after decode_group: first run position of a surviving running prefill (nrun if none)
    auto decode_group = [&](bool tail_sync) {  // heads = decodes (F_FILLED) of the run list, retention order
      const bool fM = finiteM && kv1;  // heads need one KV each (else none: admitted up to the token budget)
      const int F = fM ? M - U : 0x3fffffff;
      const int T = KN ? min(C - tok, capB - nB) : C - tok;  // one token (and one batch slot, max_seqs knob) each
      // warps whose items all lie beyond the run list only meet the barriers and fold the active warps' partials
      const int nact = min(NW, (nrun + 32 * IPT_ - 1) / (32 * IPT_));
      TMARK(10);
      const bool act = wid < nact;
      // (i) reverse scan over run positions of (held, is-head): RS(q) = sum held at >= q, HS(q) = heads at >= q.
      // Paged KV (Q15 alternative): a head needs 0 or 1 new block, so the closed form counts NS(i), the blocks
      // heads 1..i need (= i per token), with NSS(q) = the needs at >= q from a third scan component.
      int hv[IPT_], rsv[IPT_], hsv[IPT_], nv[IPT_], nsv[IPT_], ls = 0, lh = 0, ln = 0;
      bool hh[IPT_];
      int16_t sls[IPT_];
#pragma unroll
      for (int j = 0; j < IPT_; j++) {
        const int q = nrun - 1 - (tid * IPT_ + j);
        hv[j] = 0, hh[j] = false, sls[j] = 0, nv[j] = 0;
        if (q >= 0) {
          const int sl = run[q];
          sls[j] = (int16_t)sl;
          const int4 rc = s_rec[sl];
          hv[j] = blk(max(rc.w, rc.z));
          hh[j] = (s_fl[sl] & F_FILLED) != 0;
          if (paged && hh[j]) nv[j] = blk(max(rc.w, rc.z + 1)) - hv[j];
        }
        ls += hv[j], lh += hh[j], ln += nv[j];
      }
      int xs = ls, xh = lh, xn = ln;
      if (act) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int ys = __shfl_up_sync(FM, xs, o), yh = __shfl_up_sync(FM, xh, o);
          if (lane >= o) xs += ys, xh += yh;
          if (paged) {
            const int yn = __shfl_up_sync(FM, xn, o);
            if (lane >= o) xn += yn;
          }
        }
        if (lane == 31) S.cf_red[wid][0] = xs, S.cf_red[wid][1] = xh, S.cf_red[wid][8] = xn;
      }
      __syncthreads();
      int os = xs - ls, oh = xh - lh, on = xn - ln, k = 0, kn = 0;
      for (int w = 0; w < nact; w++) {
        const int a0 = S.cf_red[w][0], a1 = S.cf_red[w][1], a8 = paged ? S.cf_red[w][8] : 0;
        if (w < wid) os += a0, oh += a1, on += a8;
        k += a1, kn += a8;
      }
#pragma unroll
      for (int j = 0; j < IPT_; j++) os += hv[j], oh += hh[j], on += nv[j], rsv[j] = os, hsv[j] = oh, nsv[j] = on;
      if (!paged) kn = k;
      auto NS = [&](int j) { return paged ? kn - nsv[j] + nv[j] : k - hsv[j] + 1; };  // blocks heads 1..i need
      TMARK(11);
      // (ii) a_kv = #{heads i : F + RS(p_i + 1) >= i}, i = k - HS(p_i) + 1 (monotone in i)
      int akv = k;
      if (fM && F < kn) {  // with F >= kn every head passes (F + RS(p_i + 1) >= F >= kn >= NS(i)): no pass needed
        if (act) {
          int cnt = 0;
#pragma unroll
          for (int j = 0; j < IPT_; j++)
            if (hh[j]) cnt += F + (rsv[j] - hv[j]) >= NS(j);
          cnt = (int)__reduce_add_sync(FM, (unsigned)cnt);
          if (lane == 0) S.cf_red[wid][2] = cnt;
        }
        __syncthreads();
        akv = 0;
        for (int w = 0; w < nact; w++) akv += S.cf_red[w][2];
      }
      TMARK(12);
      const int a = min(min(akv, T), k);
      int NSa = a;  // blocks heads 1..a need (a per token)
      if (paged) {
        if (act) {
          int sn = 0;
#pragma unroll
          for (int j = 0; j < IPT_; j++)
            if (hh[j] && k - hsv[j] + 1 <= a) sn += nv[j];
          sn = (int)__reduce_add_sync(FM, (unsigned)sn);
          if (lane == 0) S.cf_red[wid][9] = sn;
        }
        __syncthreads();
        NSa = 0;
        for (int w = 0; w < nact; w++) NSa += S.cf_red[w][9];
      }
      // (iii) q* = max{q : F + RS(q) >= NS(a)}; the position of head a+1
      const bool needq = fM && F < NSa;
      const bool needp = fM && a == akv && a < min(k, T);
      int qs = nrun, selfp = -1;
      if (needq || needp) {
        if (act) {
          int cq = 0;
#pragma unroll
          for (int j = 0; j < IPT_; j++) {
            const int q = nrun - 1 - (tid * IPT_ + j);
            if (q >= 0) {
              if (needq) cq += F + rsv[j] >= NSa;
              if (hh[j] && k - hsv[j] + 1 == a + 1) S.pa = q;
            }
          }
          cq = (int)__reduce_add_sync(FM, (unsigned)cq);
          if (lane == 0) S.cf_red[wid][3] = cq;
        }
        __syncthreads();
        if (needq) {
          int tot = 0;
          for (int w = 0; w < nact; w++) tot += S.cf_red[w][3];
          qs = tot - 1;
        }
        // head a+1, when the KV (not the token budget) stopped the walk: a victim if it lies in the evicted
        // suffix, else it runs out of pool, evicts everything behind it and self-preempts (Q8)
        if (needp) {
          const int pa = S.pa;
          if (pa < qs) selfp = pa, qs = pa + 1;
        }
      }
      TMARK(13);
      // (iv) apply: evict [qs, nrun) (+ the self-preempted head), admit heads 1..a
      const int nvic0 = S.n_vic;
      const bool evict = qs < nrun || selfp >= 0;
      int tev = 0, teh = 0, ter = 0;
      if (act) {
        int ev = 0, eh = 0, er = 0, pm = nrun;
#pragma unroll
        for (int j = 0; j < IPT_; j++) {
          const int q = nrun - 1 - (tid * IPT_ + j);
          if (q < 0) continue;
          if (q < qs && !hh[j]) pm = min(pm, q);
          const int sl = sls[j];
          if (q >= qs || q == selfp) {
            const int4 rc = s_rec[sl];
            ev++;
            eh += hv[j];
            if (hist) er += max(S.pred[bucket_of(rc.x)] - rc.y, 0);
            const int idx = lo + ((sl - lo) & (CAP - 1));
            atomicAdd(&npre[idx], 1ull);
            atomicAdd(&refill[idx], (unsigned long long)rc.z);
            s_rec[sl] = make_int4(rc.x, rc.y, 0, 0);
            s_fl[sl] = ST_WAIT | F_PRE | (s_fl[sl] & F_FIRST);
            s_vic[nvic0 + (q == selfp ? nrun - qs : q - qs)] = (int16_t)sl;
            if (trc) {  // the oracle's order: the lowest retention (the run list's tail) first, head a+1 last
              const long long e = S.tr_ev + nvic0 + (q == selfp ? nrun - qs : nrun - 1 - q);
              if (e < p.tr.cap_events) p.tr.events[e] = sim_trace_event_t{idx, rc.z};
            }
          } else if (hh[j]) {
            const int i = k - hsv[j] + 1;
            if (i <= a) {
              s_c[sl] = 1;
              s_fl[sl] |= F_INB;
              s_bl[nB + i - 1] = (int16_t)sl;
            }
          }
        }
        if (evict) {  // evictions happened: count them (the common step has none)
          ev = (int)__reduce_add_sync(FM, (unsigned)ev);
          eh = (int)__reduce_add_sync(FM, (unsigned)eh);
          if (hist) er = (int)__reduce_add_sync(FM, (unsigned)er);
        }
        pm = (int)__reduce_min_sync(FM, (unsigned)pm);
        if (lane == 0) S.cf_red[wid][4] = ev, S.cf_red[wid][5] = eh, S.cf_red[wid][6] = er, S.cf_red[wid][7] = pm;
      }
      __syncthreads();
      TMARK(14);
      rp_first = nrun;
      for (int w = 0; w < nact; w++) {
        if (evict) tev += S.cf_red[w][4], teh += S.cf_red[w][5], ter += S.cf_red[w][6];
        rp_first = min(rp_first, S.cf_red[w][7]);
      }
      tok += a;
      U += (kv1 ? NSa : 0) - teh;
      nB += a;
      n_running -= tev;
      Rs -= ter;
      if (a > 0 && bph < 0) bph = PH_DEC;
      if (tid == 0) {
        S.n_vic = nvic0 + tev;
        S.preempt += tev;
        if (tev) S.any_pre = 1;
        S.vt = min(S.vt, (selfp >= 0 ? selfp : qs) - 1);
        S.cut = selfp >= 0 ? selfp : qs;  // run positions >= cut were evicted (a suffix)
      }
      TMARK(15);
      if (tail_sync) __syncthreads();  // evictions and admissions are visible; cf_red may be reused
    };

    // Candidates that never preempt, on warp 0: the waiting group (overWin: window offsets [0, L) = R_w
    // in index order; Q5) or running prefills (P positions [b0, b1) = R_r^p; their KV delta is 0 since
    // reserved >= s >= m + c).  All are in the prefill phase, so a chunk of 32 is resolved in registers:
    // repeat {ballot the lanes that fit alone; prefix-scan them; admit those before the first cumulative
    // failure; drop that failure} -- rejections change no state.  A cropped chunk (chunked prefill)
    // exhausts the token budget and ends the group.
    int wnext = -1;  // after warp_np(1): no window offset below it holds a waiting request (except victims)
    auto warp_np = [&](int src, int b0, int b1) {
      // one call sees one kind: waiting (src 1: KV delta = s = c for a full admission) or running prefills
      // (src 2 / 0: KV delta 0); counts come from ballots, so only the token prefix is scanned
      const bool overWin = src == 1;
      const unsigned lt = (1u << lane) - 1u;
      bool wcont = overWin;  // every waiting request at offsets [b0, i0) was admitted
      if (overWin) wnext = b0;
      for (int i0 = b0; i0 < b1; i0 += 32) {
        TMARK(70);
        if ((!hybrid && bph == PH_DEC) || (chunked && tok >= C) || (KN && nB >= capB)) return;  // all remaining fail
        if (overWin && ((finiteM && (long long)U + blk(minSW) > (KN ? Mw : M)) || (!chunked && minSW > C - tok))) return;
        PROF_CNT(13, 1);
        const int i = i0 + lane;
        int sl = -1;
        if (i < b1) {
          if (overWin) {
            const int s2 = (lo + i) & (CAP - 1);
            if ((s_fl[s2] & (ST_MASK | F_PRE)) == ST_WAIT) sl = s2;
          } else if (src == 2) {  // running prefills (not evicted) in retention order
            const int s2 = run[i];
            if ((s_fl[s2] & (ST_MASK | F_PRE | F_FILLED)) == ST_RUN) sl = s2;
          } else {
            const int s2 = cand(i);
            if (!(s_fl[s2] & F_PRE)) sl = s2;
          }
        }
        if (!__any_sync(FM, sl >= 0)) {  // no candidate in this chunk: nothing to admit or reject
          if (wcont) wnext = min(i0 + 32, b1);
          continue;
        }
        const int4 rc = sl >= 0 ? s_rec[sl] : make_int4(0, 0, 0, 0);  // (no dummy loads: lanes of one warp write)
        const uint8_t fl = sl >= 0 ? s_fl[sl] : (uint8_t)0;
        const int s = rc.x + rc.y, avail = s - rc.z;
        const int rtok = (overWin && sl >= 0) ? rnew(rc, sl) : 0;  // the initial reserve >= s >= c (Q13), tokens
        const int dkv = blk(rtok);                                   // its KV delta (blocks when paged)
        const int rem = (hist && overWin) ? max(S.pred[bucket_of(rc.x)] - rc.y, 0) : 0;
        bool alive = sl >= 0, admitted = false;
        for (;;) {
          const int rt = C - tok;
          const bool anyRun0 = n_running > 0;
          bool fit = alive && rt >= 1 && (chunked || avail <= rt) &&
                     (!finiteM || U + dkv <= (KN && overWin ? Mw : M)) && (!KN || nB < capB);
          if (hist && overWin) fit = fit && !(anyRun0 && (long long)U + Rs + s + rem > M);
          const unsigned fm = __ballot_sync(FM, fit);
          // head-of-line knob: the first waiting lane that fails (alone or cumulatively) ends R_w's visit
          const unsigned failm = (holk && overWin) ? __ballot_sync(FM, alive && !fit) : 0u;
          if (!fm) {
            if (failm) return;
            break;
          }
          const int cc = fit ? avail : 0, rr = fit ? rem : 0, dk = fit ? dkv : 0;
          const bool scand = overWin && (!kv1 || paged);  // KV deltas differ from c under PEAK / CONTEXT or in blocks
          int xc = cc, xr = rr, xd = dk;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int yc = __shfl_up_sync(FM, xc, o);
            if (lane >= o) xc += yc;
            if (hist && overWin) {
              const int yr = __shfl_up_sync(FM, xr, o);
              if (lane >= o) xr += yr;
            }
            if (scand) {
              const int yd = __shfl_up_sync(FM, xd, o);
              if (lane >= o) xd += yd;
            }
          }
          const int ec = xc - cc, er = xr - rr, ek = __popc(fm & lt);
          // full admissions before this lane reserve exactly their c under SEQ (waiting: m = 0, c = s)
          const int ed = overWin ? (scand ? xd - dk : ec) : 0;
          bool brk = false, crop = false;
          if (fit) {
            const int prt = rt - ec;
            if (chunked)
              crop = prt < avail;  // cropped (c = prt >= 1) or exhausted (prt <= 0)
            else
              brk = avail > prt;
            if (finiteM) brk |= U + ed + dkv > (KN && overWin ? Mw : M);
            if (hist && overWin) brk |= (anyRun0 || ek > 0) && (long long)U + ed + Rs + er + s + rem > M;
            if (crop && prt <= 0) brk = true;
            if (KN) brk |= nB + ek >= capB;  // max_seqs knob
          }
          const unsigned bm = __ballot_sync(FM, brk), cm = __ballot_sync(FM, crop && !brk);
          const int b0_ = bm ? __ffs(bm) - 1 : 32, cl = cm ? __ffs(cm) - 1 : 32;
          const int b = failm ? min(b0_, __ffs(failm) - 1) : b0_;                   // first failure
          const int stop = min(b, cl);                                             // lanes < stop: in full
          const bool adm = fit && lane < stop, adc = fit && lane == cl && cl < b;  // + the cropped one
          if (adm || adc) {
            s_c[sl] = adm ? avail : rt - ec;
            s_bl[nB + ek] = (int16_t)sl;
            if (overWin) {
              s_seq[sl] = seq + ek + 1;
              s_rec[sl] = make_int4(rc.x, rc.y, 0, rtok);
              s_fl[sl] = ST_RUN | F_INB | (fl & F_FIRST);
              s_new[n_new + ek] = (int16_t)sl;
            } else {
              s_fl[sl] = fl | F_INB;
            }
            alive = false;
            admitted = true;
          }
          const bool cropped = cl < b && cl < 32;
          const int nadm = __popc(fm & (stop >= 32 ? FM : ((1u << stop) - 1u)));
          const int lastl = stop > 0 ? min(stop, 32) - 1 : 0;
          const int addc = stop > 0 ? __shfl_sync(FM, xc, lastl) : 0;
          const int addr = (hist && overWin && stop > 0) ? __shfl_sync(FM, xr, lastl) : 0;
          const int addd = (scand && stop > 0) ? __shfl_sync(FM, xd, lastl) : addc;
          int cropc = 0, crops = 0, cropr = 0;
          if (cropped) {
            cropc = __shfl_sync(FM, rt - ec, cl);
            crops = __shfl_sync(FM, dkv, cl);
            if (hist && overWin) cropr = __shfl_sync(FM, rem, cl);
          }
          const int nall = nadm + (cropped ? 1 : 0);
          tok += addc + cropc;
          if (overWin) {
            U += addd + crops;
            seq += nall, n_new += nall, n_running += nall;
            Rs += addr + cropr;
          }
          nB += nall;
          if (nall > 0 && bph < 0) bph = PH_PRE;
          if (cropped) break;  // the token budget is exhausted: every later candidate is rejected
          if (holk && overWin && b < 32) return;  // head-of-line knob: a waiting failure ends R_w's visit
          if (b < 32 && lane == b) alive = false;  // rejected (no state change)
          if (b >= 32) break;
        }
        if (wcont) {  // advance the waiting bound past this chunk unless a waiting request is left in it
          const unsigned lf = __ballot_sync(FM, sl >= 0 && !admitted);
          if (lf) {
            wnext = i0 + __ffs(lf) - 1;
            wcont = false;
          } else {
            wnext = min(i0 + 32, b1);
          }
        }
        if (chunked && tok >= C) return;  // cropped: the token budget is exhausted
      }
    };

    bool rfast = false;  // the decode-first running groups were resolved (once per step)
    while (pos < nP) {
      TMARK(20);
      // running decodes in closed form
      if (order == SIM_ORDER_PREFILL_FIRST && pos == nW && nW < nP && !chunked && nrun <= CH && !q3alt) {
        if (hybrid || bph != PH_PRE) decode_group(false);  // else every decode fails step 2 (no running prefills)
        pos = nP;
        PROF_CNT(12, 1);
        continue;
      }
      if (order == SIM_ORDER_DECODE_FIRST && pos == 0 && !rfast && nrun <= CH && !q3alt) {
        rfast = true;
        // {R_r^d, R_r^p, R_w}: decodes in closed form, then running prefills and (if warp-suitable) the
        // waiting group in one pass of warp 0
        if (nrun > 0) decode_group(true);
        PROF_CNT(12, 1);
        if (wid == 0) {
          if (rp_first < nrun) warp_np(2, rp_first, nrun);
          int wdone = nW == 0;
          if (!wdone) {
            const bool wrej = (!hybrid && bph == PH_DEC) || (KN && nB >= capB) || (finiteM && (long long)U + blk(minSW) > (KN ? Mw : M)) ||
                              (chunked ? tok >= C : minSW > C - tok);
            const long long q1 = max(minSW, 1);  // at most 128 admissions possible (no 64-bit division)
            const bool few = (chunked ? (long long)(C - tok) <= 128 : (long long)(C - tok) < 129 * q1) ||
                             (finiteM && (long long)(M - U) < 129 * (long long)blk((int)q1));  // (KV in blocks when paged)
            if (wrej) {
              wdone = 1;
            } else if (few || nx1 - lo <= WARP_MAX) {
              warp_np(1, w0, nx1 - lo);
              wdone = 1;
            }
          }
          if (lane == 0) {
            if (wnext >= 0) S.wf_new = lo + wnext;
            S.r_tok = tok, S.r_U = U, S.r_seq = seq, S.r_Rs = Rs, S.r_nB = nB;
            S.r_new = n_new, S.r_running = n_running, S.r_bph = bph, S.r_wdone = wdone, S.r_wblk = wblk;
          }
        }
        __syncthreads();
        tok = S.r_tok, U = S.r_U, seq = S.r_seq, Rs = S.r_Rs, nB = S.r_nB;
        n_new = S.r_new, n_running = S.r_running, bph = S.r_bph, wblk = S.r_wblk;
        pos = S.r_wdone ? nP : len0;
        __syncthreads();
        continue;
      }
      {  // warp-level mode when few candidates need a decision
        int mode = 0, lim = nP;
        if (pos >= wbeg && pos < wend) {
          const bool wrej = (!hybrid && bph == PH_DEC) || (KN && nB >= capB) || (finiteM && (long long)U + blk(minSW) > (KN ? Mw : M)) ||
                            (chunked ? tok >= C : minSW > C - tok);
          if (wrej) {  // every remaining waiting candidate fails a monotone check: skip the group
            pos = wend;
            continue;
          }
          if (pos == wbeg) {
            // at most 128 admissions possible (floor(x / q) <= 128 <=> x < 129 q): warp-level admission
            const long long q1 = max(minSW, 1);
            const bool few = (chunked ? (long long)(C - tok) <= 128 : (long long)(C - tok) < 129 * q1) ||
                             (finiteM && (long long)(M - U) < 129 * (long long)blk((int)q1));  // (KV in blocks when paged)
            if (few || nx1 - lo <= WARP_MAX) mode = 2, lim = wend;
          }
        } else if (!rank) {
          const int rend = order == SIM_ORDER_DECODE_FIRST ? len0 : nP;  // end of the running group(s)
          if (rend - pos <= WARP_MAX) {
            mode = 1, lim = rend;
            if (order == SIM_ORDER_DECODE_FIRST && pos >= nRd) mode = 3;  // R_r^p: running prefills only
          }
        }
        if (mode) {
          PROF_CNT(11, 1);
          TMARK(60 + mode);
          if (wid == 0) {
            if (mode == 2)
              warp_np(1, w0, nx1 - lo);
            else if (mode == 3)
              warp_np(0, pos, lim);
            else
              warp_run(false, pos, lim);
            if (lane == 0) {
              S.r_tok = tok, S.r_U = U, S.r_seq = seq, S.r_Rs = Rs, S.r_nB = nB;
              S.r_new = n_new, S.r_running = n_running, S.r_bph = bph, S.r_wblk = wblk;
              if (wnext >= 0) S.wf_new = lo + wnext;
            }
          }
          TMARK(65);
          __syncthreads();
          TMARK(66);
          tok = S.r_tok, U = S.r_U, seq = S.r_seq, Rs = S.r_Rs, nB = S.r_nB;
          n_new = S.r_new, n_running = S.r_running, bph = S.r_bph, wblk = S.r_wblk;
          pos = lim;
          __syncthreads();
          TMARK(67);
          continue;
        }
      }
      if (pos >= wbeg && pos < wend) {
        if (!wbuilt) {  // first use this step: build R_w in index order (Q1, Q2), as of the step's
                               // start: requests preempted earlier in this step are not in it (Q9)
          block_compact<NT, IPT_>(
              nx1 - lo, [&](int q) { return (s_fl[(lo + q) & (CAP - 1)] & (ST_MASK | F_PRE)) == ST_WAIT; },
              [&](int q) { return (lo + q) & (CAP - 1); }, s_wl, S);
          wbuilt = 1;
        }
      }
      PROF_CNT(6, 1);
      const bool anyRun0 = n_running > 0;
      int cend = min(pos + CH, nP);
      if (!wbuilt && pos < wbeg && cend > wbeg) cend = wbeg;  // never read an unbuilt waiting list
      if (order == SIM_ORDER_PREFILL_FIRST && pos < wend && cend > wend) cend = wend;  // R_r: closed form
      int slv[IPT_];
      int4 rcv[IPT_];
      uint8_t flv[IPT_];
#pragma unroll
      for (int j = 0; j < IPT_; j++) {
        const int q = pos + tid * IPT_ + j;
        slv[j] = q < cend ? cand(q) : -1;
      }
#pragma unroll
      for (int j = 0; j < IPT_; j++) {
        const int sl = slv[j] < 0 ? 0 : slv[j];
        rcv[j] = s_rec[sl];
        flv[j] = s_fl[sl];
      }
      int kind[IPT_], cc[IPT_], dd[IPT_], rr[IPT_], av[IPT_], ss[IPT_];
      bool ww[IPT_], pre[IPT_], holb[IPT_];
#pragma unroll
      for (int j = 0; j < IPT_; j++) {
        const uint8_t fl = flv[j];
        const int4 rc = rcv[j];
        const bool isW = (fl & ST_MASK) == ST_WAIT;
        const int ph = (isW || !(fl & F_FILLED)) ? PH_PRE : PH_DEC;
        const int s = rc.x + rc.y, avail = s - rc.z;
        const int rt = C - tok;
        const int c = ph == PH_DEC ? 1 : (chunked ? min(avail, rt) : avail);
        int rem = 0;
        const bool cand0 = slv[j] >= 0 && !(fl & F_PRE) && !(holk && isW && wblk);  // a candidate at all
        bool ok = cand0 && (hybrid || bph < 0 || ph == bph) && c >= 1 && c <= rt && (!KN || nB < capB);
        if (hist && isW) {
          rem = max(S.pred[bucket_of(rc.x)] - rc.y, 0);
          ok = ok && !(anyRun0 && (long long)U + Rs + s + rem > M);
        }
        const int rw = isW ? rnew(rc, slv[j] < 0 ? 0 : slv[j]) : rc.w;
        const int delta = blk(max(rw, rc.z + c)) - (isW ? 0 : blk(max(rc.w, rc.z)));
        if (KN && isW && finiteM && U + delta > Mw) ok = false;  // watermark knob
        const bool kvfail = finiteM && U + delta > M;
        kind[j] = !ok ? K_NONE : (kvfail ? ((isW || pf) ? K_NONE : K_EVENT) : K_MARK);
        holb[j] = holk && isW && cand0 && !ok;  // head-of-line knob: this waiting failure ends R_w's visit
        const bool mk = kind[j] == K_MARK;
        cc[j] = mk ? (ph == PH_DEC ? 1 : avail) : 0;
        dd[j] = mk ? delta : 0;
        ww[j] = mk && isW;
        rr[j] = mk ? rem : 0;
        av[j] = avail;
        ss[j] = s;
        pre[j] = ph == PH_PRE;
      }
      int lc = 0, ld = 0, lw = 0, lk = 0, lr = 0;
#pragma unroll
      for (int j = 0; j < IPT_; j++) lc += cc[j], ld += dd[j], lw += ww[j], lk += kind[j] == K_MARK, lr += rr[j];
      int xc = lc, xd = ld, xw = lw, xk = lk, xr = lr;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int yc = __shfl_up_sync(FM, xc, o), yd = __shfl_up_sync(FM, xd, o);
        const int yw = __shfl_up_sync(FM, xw, o), yk = __shfl_up_sync(FM, xk, o);
        if (lane >= o) xc += yc, xd += yd, xw += yw, xk += yk;
        if (hist) {
          const int yr = __shfl_up_sync(FM, xr, o);
          if (lane >= o) xr += yr;
        }
      }
      if (lane == 31)
        S.wsum[wid][0] = xc, S.wsum[wid][1] = xd, S.wsum[wid][2] = xw, S.wsum[wid][3] = xk, S.wsum[wid][4] = xr;
      __syncthreads();
      int oc = xc - lc, od = xd - ld, ow = xw - lw, ok_ = xk - lk, orr = xr - lr;
      int tc = 0, tdk = 0, tw = 0, tk = 0, tr = 0;
#pragma unroll
      for (int w = 0; w < NW; w++) {
        const int a0 = S.wsum[w][0], a1 = S.wsum[w][1], a2 = S.wsum[w][2], a3 = S.wsum[w][3], a4 = S.wsum[w][4];
        if (w < wid) oc += a0, od += a1, ow += a2, ok_ += a3, orr += a4;
        tc += a0, tdk += a1, tw += a2, tk += a3, tr += a4;
      }
      int mybrk = NOBRK;
      {
        int pc = oc, pd = od, pw = ow, pr = orr, pk = ok_;
#pragma unroll
        for (int j = 0; j < IPT_; j++) {
          const int q = pos + tid * IPT_ + j;
          if (kind[j] == K_MARK) {
            const int ptok = tok + pc, pU = U + pd;
            const int rt = C - ptok;
            bool brk = !hybrid && bph < 0;  // the first admission fixes the batch phase (Q19)
            if (pre[j] && chunked)
              brk |= rt < av[j];  // cropped chunk (terminal) or budget exhausted
            else
              brk |= cc[j] > rt;
            if (hist && ww[j]) {
              const bool anyR = anyRun0 || pw > 0;
              brk |= anyR && (long long)pU + Rs + pr + ss[j] + rr[j] > M;
            }
            if (finiteM) brk |= pU + dd[j] > (KN && ww[j] ? Mw : M);
            if (KN) brk |= nB + pk >= capB;  // max_seqs knob
            if (brk) mybrk = min(mybrk, q);
            pc += cc[j], pd += dd[j], pw += ww[j], pr += rr[j], pk++;
          } else if (kind[j] == K_EVENT) {
            if (tok + pc + 1 <= C) mybrk = min(mybrk, q);  // else a token reject (Q11)
          } else if (holb[j]) {
            mybrk = min(mybrk, q);  // resolved literally: it ends R_w's visit
          }
        }
      }
      const int wm = (int)__reduce_min_sync(FM, (unsigned)mybrk);
      if (lane == 0) S.wmin[wid] = wm;
      __syncthreads();
      int b = NOBRK;
#pragma unroll
      for (int w = 0; w < NW; w++) b = min(b, S.wmin[w]);
      {
        int pc = oc, pd = od, pw = ow, pk = ok_, pr = orr;
#pragma unroll
        for (int j = 0; j < IPT_; j++) {
          const int q = pos + tid * IPT_ + j;
          if (q == b) S.pref[0] = pc, S.pref[1] = pd, S.pref[2] = pw, S.pref[3] = pk, S.pref[4] = pr;
          if (kind[j] == K_MARK) {
            if (q < b) {  // admitted: every check passed at its exact position
              const int sl = slv[j];
              s_c[sl] = cc[j];
              s_bl[nB + pk] = (int16_t)sl;
              if (ww[j]) {
                s_seq[sl] = seq + pw + 1;
                const int4 rc = rcv[j];
                s_rec[sl] = make_int4(rc.x, rc.y, rc.z, kv1 ? ss[j] : rnew(rc, sl));
                s_fl[sl] = ST_RUN | F_INB | (flv[j] & F_FIRST);
                s_new[n_new + pw] = (int16_t)sl;
              } else {
                s_fl[sl] = flv[j] | F_INB;
              }
            }
            pc += cc[j], pd += dd[j], pw += ww[j], pk++, pr += rr[j];
          }
        }
      }
      if (b >= cend) {  // no break: every thread advances its copy of the scalars identically
        tok += tc, U += tdk, seq += tw, n_new += tw, n_running += tw, nB += tk, Rs += tr;
        pos = cend;
        continue;
      }
      __syncthreads();  // admissions and the break's prefixes are visible
      if (tid == 0) {
        PROF_CNT(7, 1);
        tok += (int)S.pref[0], U += (int)S.pref[1], seq += (int)S.pref[2], n_new += (int)S.pref[2];
        n_running += (int)S.pref[2], nB += (int)S.pref[3], Rs += S.pref[4];
        handle(cand(b));
        S.r_tok = tok, S.r_U = U, S.r_seq = seq, S.r_Rs = Rs, S.r_nB = nB;
        S.r_new = n_new, S.r_running = n_running, S.r_bph = bph, S.r_wblk = wblk;
      }
      __syncthreads();
      tok = S.r_tok, U = S.r_U, seq = S.r_seq, Rs = S.r_Rs, nB = S.r_nB;
      n_new = S.r_new, n_running = S.r_running, bph = S.r_bph, wblk = S.r_wblk;
      pos = b + 1;
    }
    __syncthreads();  // admissions of the last round are visible
    TMARK(21);
    if (tok == 0) {   // B = {}: idle jump to the next arrival, not a step (Q21)
      if (tid == 0) {
        wfirst_commit(S);
        S.idle_st = 0;
        if (S.any_pre)
          S.idle_st = SIM_S_DEADLOCK;
        else if (nx1 < n) {
          S.clock[0] = fmax(S.clock[0], wl.T[nx1]);
          S.idle++;
          S.next = nx1;
          S.w_dirty = 0;
          S.nW = nW, S.minSW = minSW, S.wbuilt = wbuilt;
          S.rank_dirty = 0;
          S.p_dirty = 0;
        } else
          S.idle_st = SIM_S_DEADLOCK;
      }
      __syncthreads();
      exit_status = S.idle_st;
      if (exit_status) break;
      continue;
    }
    PROF_MARK(2);

    // ---- (4) a9 + a10: Process(B) and the exact integer features in one pass over B ----
    {
      unsigned N = 0, np_ = 0, cp = 0, mp = 0, nd = 0, md = 0, freed = 0, ndone = 0, mdn = 0, nfill = 0;
      int minrem = NOBRK, minfree = NOBRK;  // minfree (paged KV): decodes left before some entry opens a block
      long long c2 = 0, mc = 0, pcm = 0, pce[SIM_MAX_COST] = {0, 0, 0, 0};
      const int nwa = min(NW, (nB + 31) >> 5);  // warps holding batch entries; the others only meet the barrier
      if (wid < nwa) {
      for (int e = tid; e < nB; e += NT) {
        const int sl = s_bl[e];
        uint8_t fl = s_fl[sl];
        const int4 rc = s_rec[sl];
        const int c = s_c[sl], O = s_O[sl];
        const int m0 = rc.z;
        int g = rc.y;
        const int s = rc.x + g, m = m0 + c;
        if (trc) {
          const long long x = S.tr_ent + e;
          if (x < p.tr.cap_entries)
            p.tr.entries[x] = sim_trace_entry_t{lo + ((sl - lo) & (CAP - 1)), (fl & F_FILLED) ? 0 : 1, c, m0};
        }
        N += c;
        if (!(fl & F_FILLED)) {  // prefill entry (incl. refills and chunks)
          np_++;
          cp += c;
          mp += m0;
          c2 += (long long)c * c;
          mc += (long long)m0 * c;
          if (anyTheo) {
            pcm += (long long)c * (c + m0);
#pragma unroll
            for (int k = 0; k < SIM_MAX_COST; k++)
              if (k < K) {
                const int H = S.cm[k].H;
                pce[k] += (long long)((c + H - 1) / H) * (c + m0);
              }
          }
        } else {  // decode entry (c = 1)
          nd++;
          md += m0;
        }
        fl &= ~F_INB;
        bool done = false;
        if (c == s - m0) {  // Eq. (6): all available tokens processed -> one token (Q18)
          g++;
          int evc = 0;
          if (!(fl & F_FILLED)) nfill++;
          fl |= F_FILLED;
          if (!(fl & F_FIRST)) {
            fl |= F_FIRST;
            evc |= 1;
          }
          if (g == O) {
            done = true;
            fl = (fl & ~ST_MASK) | ST_DONE;
            evc |= 2;
            freed += blk(max(rc.w, m));
            ndone++;
            if (hist) atomicAdd(&S.hist[bucket_of(rc.x) * 18 + bucket_of(O)], 1);
          }
          if (evc) s_ev[atomicAdd(&S.n_ev, 1)] = sl | (evc << SLB);
        }
        if (!done) {
          minrem = min(minrem, O - g);
          if (paged) minfree = min(minfree, blk(max(rc.w, m)) * kvb - m);
          mdn += m;
        }
        s_rec[sl] = make_int4(rc.x, g, m, rc.w);
        s_fl[sl] = fl;
      }
      TMARK(30);
      N = __reduce_add_sync(FM, N), np_ = __reduce_add_sync(FM, np_), cp = __reduce_add_sync(FM, cp);
      mp = __reduce_add_sync(FM, mp), nd = __reduce_add_sync(FM, nd), md = __reduce_add_sync(FM, md);
      freed = __reduce_add_sync(FM, freed), ndone = __reduce_add_sync(FM, ndone);
      mdn = __reduce_add_sync(FM, mdn), nfill = __reduce_add_sync(FM, nfill);
      minrem = (int)__reduce_min_sync(FM, (unsigned)minrem);
      if (paged) minfree = (int)__reduce_min_sync(FM, (unsigned)minfree);
      if (np_ > 0) {  // prefill squares: 64-bit, only in warps holding prefill entries
        c2 = warp_sum(c2);
        mc = warp_sum(mc);
        if (anyTheo) {
          pcm = warp_sum(pcm);
#pragma unroll
          for (int k = 0; k < SIM_MAX_COST; k++) pce[k] = warp_sum(pce[k]);
        }
      }
      if (lane == 0) {  // per-warp partials (plain stores; folded by warp 0 after the barrier)
        long long* w = S.wred[wid];
        w[0] = N, w[1] = np_, w[2] = cp, w[3] = mp, w[4] = nd, w[5] = md, w[6] = freed, w[7] = ndone;
        w[8] = mdn, w[9] = nfill, w[10] = minrem, w[11] = c2, w[12] = mc, w[13] = pcm, w[18] = minfree;
#pragma unroll
        for (int k = 0; k < SIM_MAX_COST; k++) w[14 + k] = pce[k];
      }
      }  // wid < nwa
      TMARK(31);
      // clear the preempted-this-step marks (Q9 applies within one step); smallest s among the victims
      // (they join R_w)
      if (wid == 0) {
        const int nv = S.n_vic;
        int vmin = 0x7fffffff, vidx = 0x7fffffff;
        for (int v = lane; v < nv; v += 32) {
          const int sl = s_vic[v];
          s_fl[sl] &= ~F_PRE;
          const int4 rc = s_rec[sl];
          vmin = min(vmin, rc.x + rc.y);
          vidx = min(vidx, lo + ((sl - lo) & (CAP - 1)));
        }
        vmin = (int)__reduce_min_sync(FM, (unsigned)vmin);
        vidx = (int)__reduce_min_sync(FM, (unsigned)vidx);
        if (lane == 0) {
          S.vmin = vmin;
          S.wf_vic = min(S.wf_vic, vidx);  // this step's victims wait from the next step on
        }
      }
      __syncthreads();
      long long tt[19];
      TMARK(33);
      if (wid == 0) {  // lane z folds column z of the per-warp partials; thread 0 gathers them
        long long v = (lane == 10 || lane == 18) ? (long long)NOBRK : 0;
        if (lane < (paged ? 19 : 18)) {
          for (int w = 0; w < nwa; w++) {
            const long long x = S.wred[w][lane];
            v = (lane == 10 || lane == 18) ? min(v, x) : v + x;
          }
        }
#pragma unroll
        for (int z = 0; z < 19; z++) tt[z] = __shfl_sync(FM, v, z);
      }
      TMARK(34);
      double dk[SIM_MAX_COST] = {0.0, 0.0, 0.0, 0.0};  // d_j per cost model (warp 0, lane-parallel Eq. (3) terms)
      if (wid == 0) {
        Feat f;
        f.N = tt[0], f.np = tt[1], f.cp = tt[2], f.mp = tt[3], f.nd = tt[4], f.md = tt[5];
        f.c2 = tt[11], f.mc = tt[12], f.pcm = tt[13];
        f.pceil[0] = tt[14], f.pceil[1] = tt[15], f.pceil[2] = tt[16], f.pceil[3] = tt[17];
        const double d = batch_time_warp(S.cm, K, f, anyTheo);
#pragma unroll
        for (int k = 0; k < SIM_MAX_COST; k++) dk[k] = __shfl_sync(FM, d, k);
      }
      if (tid == 0) {
        const int vmin = S.vmin;
        {
          Feat f;
          f.N = tt[0], f.np = tt[1], f.cp = tt[2], f.mp = tt[3], f.nd = tt[4], f.md = tt[5];
          f.c2 = tt[11], f.mc = tt[12], f.pcm = tt[13];
          f.pceil[0] = tt[14], f.pceil[1] = tt[15], f.pceil[2] = tt[16], f.pceil[3] = tt[17];
          const double start = trc ? S.clock[0] : 0.0;
          for (int k = 0; k < K; k++) S.clock[k] = dadd(S.clock[k], dk[k]);  // Q36
          if (trc) {  // (d_j under cost[0] evaluated again: the same expression, the same bits)
            if (S.steps < p.tr.cap_steps)
              p.tr.steps[S.steps] = sim_trace_step_t{S.steps, nB, S.n_vic, (long long)U, (long long)tok, start,
                                                     batch_time(S.cm[0], f, 0)};
            S.tr_ent += nB;
            S.tr_ev += S.n_vic;
          }
          TMARK(35);
#ifdef SIMSWEEP_PROFILE
          if (ci == 0 && S.steps < DBG_STEPS) {
            int* d = g_dbg[S.steps];
            d[0] = (int)S.steps, d[1] = tok, d[2] = U, d[3] = nB, d[4] = (int)S.preempt, d[5] = S.n_vic;
          }
#endif
          S.steps++;
          S.formed++;
          PROF_CNT(16, 1);
          S.sumU += U;
          S.entries += f.np + f.nd;
          S.processed += f.N;
          S.pentries += f.np;
          const long long fr = tt[6], ndn = tt[7];
          const int Uafter = U - (int)fr;
          S.n_done += (int)ndn;
          // Steady decode run: step j had only decodes, no admission, preemption or completion.  Then step
          // j+1 repeats it exactly (waiting candidates were rejected for reasons that persist: KV and SRF+Hist
          // deferral are monotone in U, token/hybrid rejections are unchanged) until a completion, the KV
          // limit (U + k n_d <= M) or an arrival.  Those steps are charged below without re-forming batches.
          // After an eviction step the same holds when every running request was a decode in B and every
          // waiting candidate (the victims included) fails the KV test at step j+1 already (U only grows).
          bool steady = ndn == 0 && f.np == 0 && f.nd > 0;
          if (steady && S.any_pre) {
            const int nWn = nW - n_new + S.n_vic, minSWn = min(minSW, vmin);
            steady = !rank && f.nd == nrun - S.n_vic &&
                     (nWn == 0 || (finiteM && (long long)Uafter + blk(minSWn) > (KN ? Mw : M)));
          }
          long long Lr = 0;
          if (steady && !trc) {  // (tracing forms every step)
            Lr = tt[10];
            if (paged)  // no entry opens a block during the run: U stays constant
              Lr = min(Lr, tt[18]);
            else if (finiteM && kv1)
              Lr = min(Lr, (long long)(M - Uafter) / f.nd);
            Lr = min(Lr, cfg.max_steps - S.steps);
          }
          S.runL = Lr;
          S.runMD = tt[8];
          S.last_nd = f.nd;
          S.U = Uafter;
          S.seq = seq;
          S.nB = nB;
          const bool changed = n_new > 0 || S.any_pre || ndn > 0;  // run-list membership changed
          S.r_dirty = changed;
          // removals only as the closed form's evicted suffix: the run list is cut, not compacted
          S.removals = S.h_pre || ndn > 0 ? 2 : (S.any_pre ? 1 : 0);
          // R_w gains this step's victims and loses its admissions: |R_w| stays exact; the smallest s becomes a
          // lower bound after admissions (the skip tests only get conservative) and is recounted every 32 of them
          S.nW = nW - n_new + S.n_vic, S.minSW = min(minSW, vmin), S.wbuilt = wbuilt && S.n_vic == 0 && n_new == 0;
          if (n_new > 0) S.wstale++;
          S.w_dirty = arrived || S.wstale >= 32;
          if (S.w_dirty) S.wstale = 0;
          S.rank_dirty = ndn > 0;
          // SRF order can change unless every running request was a decode in B (all +1)
          S.o_dirty = (srf_order && (changed || f.np > 0 || f.nd != nrun)) || (arr_ord && n_new > 0);
          S.p_dirty = changed || tt[9] > 0;
          S.r_new = n_new;
        }
      }
      __syncthreads();
    }
    TMARK(36);
    PROF_MARK(3);

    // ---- (5) event times; steady decode run ----
    {
      const int nev = S.n_ev;
      for (int e = tid; e < nev; e += NT) {
        const int code = s_ev[e], sl = code & (CAP - 1);
        const int idx = lo + ((sl - lo) & (CAP - 1));
        if (code & (1 << SLB))
          for (int k = 0; k < K; k++) tf[(long long)k * n + idx] = S.clock[k];
        if (code & (2 << SLB))
          for (int k = 0; k < K; k++) td[(long long)k * n + idx] = S.clock[k];
      }
      TMARK(40);
      const long long Lr = S.runL;
      if (Lr > 0) {
        constexpr int DB = CAP / 2;
        const int cmax = min(NT, DB / K);
        const long long ndd = S.last_nd, MD = S.runMD, U0 = S.U, du = (kv1 && !paged) ? ndd : 0;  // KV growth/step
        long long E = 0;
        while (E < Lr) {
          const int chunk = (int)min((long long)cmax, Lr - E);
          if (tid < chunk) {  // features of run step E+tid+1 are affine in the step index
            Feat f;
            f.N = ndd, f.np = 0, f.c2 = 0, f.mc = 0, f.cp = 0, f.mp = 0, f.pcm = 0, f.nd = ndd;
            f.md = MD + (E + tid) * ndd;
            for (int k = 0; k < SIM_MAX_COST; k++) f.pceil[k] = 0;
            for (int k = 0; k < K; k++) s_dbuf[k * cmax + tid] = batch_time(S.cm[k], f, k);
          }
          __syncthreads();
          if (tid == 0) {  // the clock chain stays sequential: one fp64 add per step, as in the oracle (Q36)
            int ex = chunk;
            if (nx1 < n) {  // online (K == 1): stop before a step that would start at/after an arrival (Q21)
              const double Tn = wl.T[nx1];
              double clk = S.clock[0];
              for (int t = 0; t < chunk; t++) {
                if (Tn <= clk) {
                  ex = t;
                  break;
                }
                clk = dadd(clk, s_dbuf[t]);
              }
              S.clock[0] = clk;
            } else {
              for (int k = 0; k < K; k++) {
                double clk = S.clock[k];
                const double* db = s_dbuf + k * cmax;
                int t = 0;
                for (; t + 8 <= chunk; t += 8) {  // loads first: the chain is one DADD latency per step
                  double v[8];
#pragma unroll
                  for (int u = 0; u < 8; u++) v[u] = db[t + u];
#pragma unroll
                  for (int u = 0; u < 8; u++) clk = dadd(clk, v[u]);
                }
                for (; t < chunk; t++) clk = dadd(clk, db[t]);
                S.clock[k] = clk;
              }
            }
            S.runEx = ex;
          }
          __syncthreads();
          const int ex = S.runEx;
          E += ex;
          if (ex < chunk) break;
        }
        long long fr2 = 0;
        int nd2 = 0;
        if (E > 0) {
          for (int e = tid; e < nB; e += NT) {  // every B entry is a decode of the steady step
            const int sl = s_bl[e];
            const int4 rc = s_rec[sl];
            const int m = rc.z + (int)E, g = rc.y + (int)E, O = s_O[sl];
            s_rec[sl] = make_int4(rc.x, g, m, rc.w);
            if (g == O) {  // completes at the last run step
              const int idx = lo + ((sl - lo) & (CAP - 1));
              s_fl[sl] = (s_fl[sl] & ~ST_MASK) | ST_DONE;
              for (int k = 0; k < K; k++) td[(long long)k * n + idx] = S.clock[k];
              fr2 += blk(max(rc.w, m));
              nd2++;
              if (hist) atomicAdd(&S.hist[bucket_of(rc.x) * 18 + bucket_of(O)], 1);
            }
          }
        }
        fr2 = block_sum_ll<NT>(fr2, S);
        const long long nd2t = block_sum_ll<NT>((long long)nd2, S);
        if (tid == 0) {
#ifdef SIMSWEEP_PROFILE
          if (ci == 0)
            for (long long k = 1; k <= E && S.steps + k - 1 < DBG_STEPS; k++) {
              int* d = g_dbg[S.steps + k - 1];
              d[0] = (int)(S.steps + k - 1), d[1] = (int)ndd, d[2] = (int)(U0 + k * du), d[3] = (int)ndd;
              d[4] = (int)S.preempt, d[5] = 0;
            }
#endif
          S.steps += E;
          PROF_CNT(17, E);
          S.sumU += E * U0 + du * (E * (E + 1) / 2);
          S.entries += E * ndd;
          S.processed += E * ndd;
          S.visits += E * nP;
          S.U = U0 + E * du - fr2;
          S.n_done += (int)nd2t;
          if (nd2t > 0) S.r_dirty = 1, S.removals = 2, S.rank_dirty = 1, S.p_dirty = 1;
          if (srf_order && E > 0 && ndd != nrun) S.o_dirty = 1;
        }
        __syncthreads();
      }
    }
    TMARK(41);
    PROF_MARK(4);

    // ---- (6) run list (retention order) for the next step ----
    {
      const bool rd = S.r_dirty, od = S.o_dirty;
      int16_t* rl = run;
      int cnt = nrun;
      bool moved = false;
      if (rd) {
        const int nnew = S.r_new;
        if (S.removals == 1) {  // the evicted suffix is cut off, admissions are appended
          const int cut = S.cut;
          for (int q = tid; q < nnew; q += NT) {
            run[cut + q] = s_new[q];
            s_rpos[s_new[q]] = (int16_t)(cut + q);
          }
          cnt = cut + nnew;
          __syncthreads();
        } else if (S.removals) {
          int16_t* nrl = S.cur ? s_runA : s_runB;
          auto src = [&](int q) -> int { return q < nrun ? run[q] : s_new[q - nrun]; };
          cnt = block_compact<NT, IPT_>(
              nrun + nnew, [&](int q) { return (s_fl[src(q)] & ST_MASK) == ST_RUN; }, src, nrl, S);
          rl = nrl;
          if (tid == 0) S.cur ^= 1;
          moved = true;
        } else {  // only admissions: append them (admission order = NRF retention order)
          for (int q = tid; q < nnew; q += NT) {
            run[nrun + q] = s_new[q];
            s_rpos[s_new[q]] = (int16_t)(nrun + q);
          }
          cnt = nrun + nnew;
          __syncthreads();
        }
      }
      TMARK(50);
      if (od) {  // SRF retention order: m descending, then admission order (Q3, Q7); or arrival order (Q6 alt.)
        auto key = [&](int sl) -> unsigned long long {
          if (arr_ord) return (unsigned long long)(unsigned)(lo + ((sl - lo) & (CAP - 1)));  // (T, id) = index
          return ((unsigned long long)(0x3FFFF - s_rec[sl].z) << 46) |
                 ((unsigned long long)(unsigned)s_seq[sl] << SLB) | (unsigned long long)sl;
        };
        int okk = 1;
        for (int q = tid; q + 1 < cnt; q += NT)
          if (key(rl[q]) > key(rl[q + 1])) okk = 0;
        okk = __syncthreads_and(okk);
        if (!okk) {
          PROF_CNT(8, 1);
          for (int q = tid; q < cnt; q += NT) s_keys[q] = key(rl[q]);
          block_bitonic<NT>(s_keys, cnt);
          for (int q = tid; q < cnt; q += NT) rl[q] = (int16_t)(s_keys[q] & (CAP - 1));
          moved = true;
          if (tid == 0) S.p_dirty = 1;
          __syncthreads();
        }
      }
      TMARK(51);
      if (moved)
        for (int q = tid; q < cnt; q += NT) s_rpos[rl[q]] = (int16_t)q;
      __syncwarp();  // (warp 0's lanes read S.n_ev for the event pass without a barrier since)
      if (tid == 0) {
        wfirst_commit(S);
        S.n_run = cnt;
        S.next = nx1;
        S.n_ev = 0;
        int l = lo;
        while (l < nx1 && (s_fl[l & (CAP - 1)] & ST_MASK) == ST_DONE) l++;
        S.lo = l;
      }
      __syncthreads();
      TMARK(52);
      PROF_MARK(5);
    }
  }
#ifdef SIMSWEEP_PROFILE
  if (tid == 0 && ci < PROF_MAX_CFG) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    prof[14] = (long long)t_start, prof[15] = (long long)t_end, prof[9] = smid;
    for (int i = 0; i < 24; i++) g_prof[ci][i] = prof[i];
  }
#endif

#ifdef SIMSWEEP_TRACE
  if (tid == 0 && ci == 0) g_trn = trn;
#endif
  // ---- a11: metrics ----
  const int st = exit_status == -1 ? SIM_S_OK : exit_status;
  __threadfence();
  __syncthreads();
  if (st != SIM_S_OK) {  // failed simulations: zero-filled rows
    for (int i = tid; i < n; i += NT) {
      npre[i] = 0;
      refill[i] = 0;
    }
    for (int x = tid; x < K * n; x += NT) {
      tf[x] = 0.0;
      td[x] = 0.0;
    }
    if (tid == 0) {
      sim_result_t r;
      memset(&r, 0, sizeof(r));
      r.status = st;
      p.results[ci] = r;
    }
    return;
  }
  if (tid < K) {  // sequential sums in request order (identical to the oracle)
    const int k = tid;
    double mx = 0.0, sl = 0.0, st1 = 0.0, stp = 0.0;
    long long ntp = 0;
    for (int i = 0; i < n; i++) {
      const double a = tf[(long long)k * n + i], b = td[(long long)k * n + i], T = wl.T[i];
      if (i == 0 || b > mx) mx = b;
      sl = dadd(sl, b - T);
      st1 = dadd(st1, a - T);
      if (wl.O[i] > 1) {
        stp = dadd(stp, ddiv(b - a, i2d(wl.O[i] - 1)));
        ntp++;
      }
    }
    sim_result_t& r = p.results[ci];
    r.makespan[k] = mx - wl.T[0];
    r.mean_latency[k] = ddiv(sl, i2d(n));
    r.mean_ttft[k] = ddiv(st1, i2d(n));
    r.mean_tpot[k] = ntp > 0 ? ddiv(stp, i2d(ntp)) : 0.0;
  }
  if (tid == 0) {
    sim_result_t& r = p.results[ci];
    r.status = SIM_S_OK;
    r.pad = 0;
    r.steps = S.steps;
    r.preemptions = S.preempt;
    r.batch_entries = S.entries;
    r.processed_tokens = S.processed;
    r.sum_U = S.sumU;
    r.prefill_entries = S.pentries;
    r.idle_jumps = S.idle;
    r.visits = S.visits;
    r.formed_steps = S.formed;
    for (int k = K; k < SIM_MAX_COST; k++) r.makespan[k] = r.mean_latency[k] = r.mean_ttft[k] = r.mean_tpot[k] = 0.0;
  }
}

}  // namespace simsweep
