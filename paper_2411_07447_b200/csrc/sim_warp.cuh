// sim_warp.cuh -- the W <= 1024 step kernel: ONE WARP per simulation (included by simsweep.cu).
//
// Same method, same readings (Q1-Q40) and the same exact mechanisms as the block kernel of
// sim_step.cuh, but every step scalar (clock, U, tok, counters, list lengths) lives in registers and is
// updated identically by all 32 lanes, so a step has no block barrier and no shared-memory broadcast.
// Per-request state is a structure of arrays in shared memory (a ring of CAP slots, slot = id mod CAP).
// Per step (one batch B_j, Algorithm 1):
//   a2  arrivals            ballot over the sorted T (Q21)
//   a3  GroupRequests       run list kept in retention order (NRF: admission order; SRF: m desc, Q3);
//                           R_w is the window in index order (Q1, Q2), counted incrementally; Rank_*
//                           orders keep one list sorted by (key, T, id) (Q20, Q37)
//   a4-a8 GetNextBatch      running decodes: the closed form (decode group, see below); waiting group
//                           and running prefills (never preempt): ballot/prefix-scan admission (Q5);
//                           general groups: 32-candidate rounds, the break resolved literally on lane 0
//   a9  batch latency       exact integer features, warp reductions, fp64 cost models (no FMA, Q36)
//   a10 Process             Eq. (6) token generation, completions, first-token / completion events
//   steady decode runs      charged in closed form (features affine in the step index), clock chain
//                           kept sequential (one fp64 add per step)
#pragma once

namespace simsweep {

struct WHead {  // per-simulation shared header (the rest of the state is in registers)
  sim_cost_model_t cm[SIM_MAX_COST];
  int hist[18 * 18];  // SRF+Hist: log2 histogram of (I, O) at completions (Q31)
  int pred[18];       // SRF+Hist: predicted output length per I bucket
};

template <int CAP>
struct WLayout {
  static constexpr size_t a16(size_t x) { return (x + 15) & ~size_t(15); }
  static constexpr size_t rec = a16(sizeof(WHead));  // int4 {I, g, m, reserved} per slot
  static constexpr size_t O = rec + 16 * CAP;        // int32: output length
  static constexpr size_t seq = O + 4 * CAP;         // int32: admission sequence number (Q6)
  static constexpr size_t c = seq + 4 * CAP;         // int32: c of the current batch
  static constexpr size_t rpos = c + 4 * CAP;        // int16: position in the run list
  static constexpr size_t run = rpos + 2 * CAP;      // int16: run list (retention order)
  static constexpr size_t rank = run + 2 * CAP;      // int16: Rank_* visiting order
  static constexpr size_t bl = rank + 2 * CAP;       // int16: the batch B in admission order
  static constexpr size_t nw = bl + 2 * CAP;         // int16: admitted from R_w this step
  static constexpr size_t vic = nw + 2 * CAP;        // int16: preempted this step
  static constexpr size_t ev = vic + 2 * CAP;        // int16: first-token / completion events (slot | kind << SLB)
  static constexpr size_t fl = ev + 2 * CAP;         // uint8: status and flags
  static constexpr size_t keys = a16(fl + CAP);      // u64: sort keys
  static constexpr size_t bytes = keys + 8 * CAP;
};

// ascending bitonic sort of keys[0, Ln) by one warp (padded with ~0 to a power of two; the buffer holds it)
__device__ __noinline__ void warp_sort_keys(unsigned long long* keys, int Ln) {
  const int lane = threadIdx.x & 31;
  int P2 = 1;
  while (P2 < Ln) P2 <<= 1;
  for (int i = Ln + lane; i < P2; i += 32) keys[i] = ~0ull;
  __syncwarp();
  for (int k = 2; k <= P2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < P2; i += 32) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long a = keys[i], b = keys[ixj];
          if ((a > b) == ((i & k) == 0)) keys[i] = b, keys[ixj] = a;
        }
      }
      __syncwarp();
    }
  }
}

template <int CAP>
__global__ void __launch_bounds__(32) sim_warp_kernel(KParams p) {
  using L = WLayout<CAP>;
  constexpr unsigned FM = 0xffffffffu;
  constexpr int SLB = __builtin_ctz(CAP);  // bits of a slot index
  static_assert((CAP & (CAP - 1)) == 0 && CAP <= 4096, "int16 slots with two event bits");
  extern __shared__ __align__(16) unsigned char smem[];
  WHead& H = *reinterpret_cast<WHead*>(smem);
  const int lane = threadIdx.x;
  const unsigned lt = (1u << lane) - 1u;
  constexpr uint8_t F_MOVE = 64;  // SRF: a prefill entry of this step's batch (its key moved by c)
  constexpr uint8_t F_DEC = 128;  // SRF: a decode entry of this step's batch (its key moved by +1)
  const int ci = p.order ? p.order[blockIdx.x] : (int)blockIdx.x;
  if (variant_of(p.wls[p.cfgs[ci].workload].n) != p.variant) return;
  int4* s_rec = reinterpret_cast<int4*>(smem + L::rec);
  int32_t* s_O = reinterpret_cast<int32_t*>(smem + L::O);
  int32_t* s_seq = reinterpret_cast<int32_t*>(smem + L::seq);
  int32_t* s_c = reinterpret_cast<int32_t*>(smem + L::c);
  int16_t* s_rpos = reinterpret_cast<int16_t*>(smem + L::rpos);
  int16_t* s_run = reinterpret_cast<int16_t*>(smem + L::run);
  int16_t* s_rank = reinterpret_cast<int16_t*>(smem + L::rank);
  int16_t* s_bl = reinterpret_cast<int16_t*>(smem + L::bl);
  int16_t* s_new = reinterpret_cast<int16_t*>(smem + L::nw);
  int16_t* s_vic = reinterpret_cast<int16_t*>(smem + L::vic);
  int16_t* s_ev = reinterpret_cast<int16_t*>(smem + L::ev);
  uint8_t* s_fl = smem + L::fl;
  unsigned long long* s_keys = reinterpret_cast<unsigned long long*>(smem + L::keys);

#ifdef SIMSWEEP_PROFILE
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
  const sim_config_t cfg = p.cfgs[ci];
  const sim_workload_t wl = p.wls[cfg.workload];
  const int n = wl.n;
  const int K = cfg.n_cost;
  const int M = cfg.M >= 0 ? (int)cfg.M : 0, C = (int)cfg.C;  // host-validated < 2^30
  const bool finiteM = cfg.M >= 0, hybrid = cfg.hybrid != 0, chunked = cfg.chunked != 0;
  const int order = cfg.order;
  const bool srf = cfg.replacement == SIM_SRF || cfg.replacement == SIM_SRF_HIST;
  const bool hist = cfg.replacement == SIM_SRF_HIST && finiteM;
  const bool pf = cfg.replacement == SIM_PF;  // preemption-free: a running KV failure is skipped (Table 2)
  const int rmode = cfg.reserve;              // Table 2 "Initial KV reserve": SEQ s, PEAK I+O-1, CONTEXT S
  const bool kv1 = rmode == SIM_RESERVE_SEQ;  // under SEQ a filled request's decode needs exactly one KV
  const bool rank = order >= SIM_ORDER_RANK_ORG;
  const long long row0 = p.row_off[ci], tim0 = p.tim_off[ci];
  double* tf = p.req.t_first + tim0;
  double* td = p.req.t_done + tim0;
  unsigned long long* npre = reinterpret_cast<unsigned long long*>(p.req.n_preempt + row0);
  unsigned long long* refill = reinterpret_cast<unsigned long long*>(p.req.refill_tokens + row0);

  for (int i = lane; i < n; i += 32) npre[i] = 0, refill[i] = 0;
  for (int x = lane; x < K * n; x += 32) tf[x] = 0.0, td[x] = 0.0;
  // ---- a1: per-simulation validation (Q35) ----
  bool bad_long = false, bad_fit = false;
  for (int i = lane; i < n; i += 32) {
    const long long pk = (long long)wl.I[i] + wl.O[i] - 1;  // peak KV usage
    bad_long |= pk > cfg.S;
    bad_fit |= (finiteM && pk > cfg.M) || (!chunked && pk > cfg.C);
    bad_fit |= finiteM && cfg.reserve == SIM_RESERVE_CONTEXT && cfg.S > cfg.M;  // the reserve never fits (Q35)
  }
  bad_long = __any_sync(FM, bad_long);
  bad_fit = __any_sync(FM, bad_fit);
  if (bad_long || bad_fit) {
    if (lane == 0) {
      sim_result_t r;
      memset(&r, 0, sizeof(r));
      r.status = bad_long ? SIM_S_TOO_LONG : SIM_S_NEVER_FITS;
      p.results[ci] = r;
    }
    return;
  }
  bool anyTheo = false;
  for (int k = 0; k < K; k++) anyTheo |= p.cms[cfg.cost[k]].mode == 1;
  if (lane < K) H.cm[lane] = p.cms[cfg.cost[lane]];
  for (int i = lane; i < 18 * 18; i += 32) H.hist[i] = 0;
  __syncwarp();

  // ---- the simulation state held in registers (identical in every lane) ----
  double clk[SIM_MAX_COST] = {0.0, 0.0, 0.0, 0.0};
  long long steps = 0, npreempt = 0, entries = 0, processed = 0, sumU = 0, pentries = 0, idle = 0, visits = 0;
  int U = 0, seq = 0, next = 0, lo = 0, n_done = 0, nrun = 0, nrank = 0;
  int nW = 0, minSW = 0x7fffffff, wstale = 0, wfirst = 0;
  bool w_dirty = true, rank_dirty = false;
  int exit_status = 0;

  auto rnew = [&](const int4& rc, int sl) -> int {  // reserve taken at (re)admission (Table 2, Q39)
    return rmode == SIM_RESERVE_SEQ ? rc.x + rc.y : (rmode == SIM_RESERVE_PEAK ? rc.x + s_O[sl] - 1 : cfg.S);
  };
  auto req_idx = [&](int sl) -> int { return lo + ((sl - lo) & (CAP - 1)); };

  // stable in-place warp compaction of list[0, L) (+ extra[0, Lx) appended) keeping pred(slot); returns the count
  auto compact = [&](int16_t* list, int Lm, const int16_t* extra, int Lx, auto pred) -> int {
    int w = 0;
    for (int b = 0; b < Lm + Lx; b += 32) {
      const int q = b + lane;
      int sl = 0;
      bool keep = false;
      if (q < Lm + Lx) {
        sl = q < Lm ? list[q] : extra[q - Lm];
        keep = pred(sl);
      }
      const unsigned bm = __ballot_sync(FM, keep);
      __syncwarp();  // every lane has read its item before any write (writes never pass reads)
      if (keep) list[w + __popc(bm & lt)] = (int16_t)sl;
      w += __popc(bm);
    }
    __syncwarp();
    return w;
  };
  auto sort_keys = [&](int Ln) { warp_sort_keys(s_keys, Ln); };

  for (;;) {
    // ---- (1) a2: GetNewRequests (Alg. 1 line 3): all T <= clock, inclusive (Q21); T is sorted ----
    int nx1 = next;
    if (next < n) {
      const double c0 = clk[0];
      for (;;) {
        const int i = nx1 + lane;
        const unsigned b = __ballot_sync(FM, i < n && wl.T[i] <= c0);
        if (b == FM) {
          nx1 += 32;
          continue;
        }
        nx1 += __ffs(~b) - 1;
        break;
      }
    }
    exit_status = n_done == n ? -1 : (nx1 - lo > CAP ? SIM_S_CAPACITY : (steps >= cfg.max_steps ? SIM_S_MAX_STEPS : 0));
    if (exit_status) break;
    const bool arrived = nx1 > next;
    for (int idx = next + lane; idx < nx1; idx += 32) {
      const int sl = idx & (CAP - 1);
      s_rec[sl] = make_int4(wl.I[idx], 0, 0, 0);
      s_O[sl] = wl.O[idx];
      s_seq[sl] = 0;
      s_c[sl] = 0;
      s_fl[sl] = ST_WAIT;
    }
    if (arrived) wfirst = min(wfirst, next);  // new arrivals wait
    __syncwarp();
    // ---- (2) a3: GroupRequests (step 1) ----
    if (rank) {  // one group sorted by (key, T, id) (App. D, Q20, Q37)
      if ((arrived || rank_dirty) && nrank > 0)  // drop finished entries before slot reuse
        nrank = compact(s_rank, nrank, s_rank, 0, [&](int sl) { return (s_fl[sl] & ST_MASK) != ST_DONE; });
      if (arrived) {
        const int nr = nrank + (nx1 - next);
        for (int q = lane; q < nr; q += 32) {
          const int sl = q < nrank ? s_rank[q] : ((next + q - nrank) & (CAP - 1));
          const unsigned key = order == SIM_ORDER_RANK_I ? (unsigned)s_rec[sl].x
                               : order == SIM_ORDER_RANK_O ? (unsigned)s_O[sl]
                                                           : 0u;
          s_keys[q] = ((unsigned long long)key << 32) | (unsigned)req_idx(sl);
        }
        __syncwarp();
        sort_keys(nr);
        for (int q = lane; q < nr; q += 32) s_rank[q] = (int16_t)(s_keys[q] & (CAP - 1));
        nrank = nr;
        __syncwarp();
      }
    } else if (w_dirty || arrived) {  // |R_w| and its smallest s (the skip test)
      int cnt = 0, mn = 0x7fffffff;
      for (int q = max(wfirst - lo, 0) + lane; q < nx1 - lo; q += 32) {
        const int sl = (lo + q) & (CAP - 1);
        if ((s_fl[sl] & ST_MASK) == ST_WAIT) {
          const int4 r = s_rec[sl];
          cnt++;
          mn = min(mn, r.x + r.y);
        }
      }
      nW = (int)__reduce_add_sync(FM, (unsigned)cnt);
      minSW = (int)__reduce_min_sync(FM, (unsigned)mn);
    }
    long long Rs = 0;
    if (hist) {  // SRF+Hist: predictions of the current histogram; sum of remaining outputs of running requests
      if (lane < 18) H.pred[lane] = hist_pred_row(H.hist, lane);
      __syncwarp();
      long long r = 0;
      for (int q = lane; q < nrun; q += 32) {
        const int4 rc = s_rec[s_run[q]];
        r += max(H.pred[bucket_of(rc.x)] - rc.y, 0);
      }
      Rs = warp_sum(r);
    }
    const int nP = rank ? nrank : nW + nrun;
    visits += nP;

    // ---- (3) a4-a8: GetNextBatch (steps 2-4) ----
    int tok = 0, n_new = 0, n_running = nrun, bph = -1, nB = 0, n_vic = 0, vt = nrun - 1, cut = nrun;
    bool any_pre = false, h_pre = false;
    auto preempt = [&](int v) {  // lane 0 only (refill P:1570)
      const int4 rc = s_rec[v];
      U -= max(rc.w, rc.z);
      if (hist) Rs -= max(H.pred[bucket_of(rc.x)] - rc.y, 0);
      const int idx = req_idx(v);
      atomicAdd(&npre[idx], 1ull);
      atomicAdd(&refill[idx], (unsigned long long)rc.z);
      s_rec[v] = make_int4(rc.x, rc.y, 0, 0);
      s_fl[v] = ST_WAIT | F_PRE | (s_fl[v] & F_FIRST);
      s_vic[n_vic++] = (int16_t)v;
      n_running--;
      npreempt++;
      any_pre = true;
      h_pre = true;  // a preemption outside the closed form: the run list needs a full compaction
    };
    auto handle = [&](int sl) {  // literal sequential resolution of one candidate (lane 0)
      uint8_t fl = s_fl[sl];
      if (fl & F_PRE) return;  // Q9
      const bool isW = (fl & ST_MASK) == ST_WAIT;
      const int ph = (isW || !(fl & F_FILLED)) ? PH_PRE : PH_DEC;
      if (!hybrid && bph >= 0 && ph != bph) return;  // step 2
      const int4 rc = s_rec[sl];
      const int s = rc.x + rc.y, avail = s - rc.z;
      const int c = ph == PH_DEC ? 1 : (chunked ? min(avail, C - tok) : avail);
      if (c == 0 || tok + c > C) return;  // token limit never preempts (Q11)
      int rem = 0;
      if (hist && isW) {
        rem = max(H.pred[bucket_of(rc.x)] - rc.y, 0);
        if (n_running > 0 && (long long)U + Rs + s + rem > M) return;  // deferred (Q31)
      }
      const int rw = isW ? rnew(rc, sl) : rc.w;
      const int nh = max(rw, rc.z + c), held = isW ? 0 : max(rc.w, rc.z), delta = nh - held;
      while (finiteM && U + delta > M) {
        if (isW || pf) return;  // holds no KVs (Q5) / preemption-free: skipped
        const int pc = s_rpos[sl];
        while (vt > pc) {  // lowest retention = tail of the retention-ordered run list
          const uint8_t f = s_fl[s_run[vt]];
          if (!(f & F_INB) && (f & ST_MASK) == ST_RUN) break;
          vt--;
        }
        if (vt <= pc) {  // self-preemption (Q8)
          preempt(sl);
          return;
        }
        preempt(s_run[vt]);
        vt--;
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
    auto from0 = [&]() {  // lane 0 resolved a break: every lane takes its scalars
      __syncwarp();
      tok = __shfl_sync(FM, tok, 0), U = __shfl_sync(FM, U, 0), seq = __shfl_sync(FM, seq, 0);
      n_new = __shfl_sync(FM, n_new, 0), n_running = __shfl_sync(FM, n_running, 0);
      nB = __shfl_sync(FM, nB, 0), bph = __shfl_sync(FM, bph, 0), Rs = __shfl_sync(FM, Rs, 0);
      vt = __shfl_sync(FM, vt, 0), n_vic = __shfl_sync(FM, n_vic, 0), npreempt = __shfl_sync(FM, npreempt, 0);
      any_pre = __shfl_sync(FM, (int)any_pre, 0), h_pre = __shfl_sync(FM, (int)h_pre, 0);
    };

    // General rounds over list[b0, b1) in visiting order: 32 candidates at a time are classified against
    // the current (tok, U), prefix-scanned (tokens, KV delta, waiting admissions, admissions, SRF+Hist
    // remainders); the lanes before the first "break" (a candidate the scan cannot decide: a preemption,
    // a cumulative token / KV / deferral failure, a chunk crop, the first admission without hybrid
    // batching) are admitted, and lane 0 resolves the break literally (handle).
    auto warp_run = [&](const int16_t* list, int b0, int b1) {
      int i0 = b0;
      while (i0 < b1) {
        const int i = i0 + lane;
        const int sl = i < b1 ? list[i] : -1;
        const int4 rc = s_rec[sl < 0 ? 0 : sl];
        const uint8_t fl = s_fl[sl < 0 ? 0 : sl];
        const bool anyRun0 = n_running > 0;
        const bool isW = (fl & ST_MASK) == ST_WAIT;
        const int ph = (isW || !(fl & F_FILLED)) ? PH_PRE : PH_DEC;
        const int s = rc.x + rc.y, avail = s - rc.z;
        const int rt0 = C - tok;
        const int c = ph == PH_DEC ? 1 : (chunked ? min(avail, rt0) : avail);
        int rem = 0;
        bool ok = sl >= 0 && !(fl & F_PRE) && (hybrid || bph < 0 || ph == bph) && c >= 1 && c <= rt0;
        if (hist && isW) {
          rem = max(H.pred[bucket_of(rc.x)] - rc.y, 0);
          ok = ok && !(anyRun0 && (long long)U + Rs + s + rem > M);
        }
        const int rw = isW ? rnew(rc, sl < 0 ? 0 : sl) : rc.w;
        const int delta = max(rw, rc.z + c) - (isW ? 0 : max(rc.w, rc.z));
        const bool kvfail = finiteM && U + delta > M;
        const int kind = !ok ? K_NONE : (kvfail ? ((isW || pf) ? K_NONE : K_EVENT) : K_MARK);
        const bool mk = kind == K_MARK;
        const int cc = mk ? (ph == PH_DEC ? 1 : avail) : 0, dd = mk ? delta : 0, ww = mk && isW;
        const int rr = mk ? rem : 0;
        int xc = cc, xd = dd, xw = ww, xr = rr;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int yc = __shfl_up_sync(FM, xc, o), yd = __shfl_up_sync(FM, xd, o);
          const int yw = __shfl_up_sync(FM, xw, o);
          if (lane >= o) xc += yc, xd += yd, xw += yw;
          if (hist) {
            const int yr = __shfl_up_sync(FM, xr, o);
            if (lane >= o) xr += yr;
          }
        }
        const unsigned km = __ballot_sync(FM, mk);
        const int ec = xc - cc, ed = xd - dd, ew = xw - ww, ek = __popc(km & lt), er = xr - rr;  // exclusive
        bool brk = false;
        if (mk) {
          const int pU = U + ed, rt = C - (tok + ec);
          brk = !hybrid && bph < 0;  // the first admission fixes the batch phase (Q19)
          if (ph == PH_PRE && chunked)
            brk |= rt < avail;
          else
            brk |= cc > rt;
          if (hist && isW) brk |= (anyRun0 || ew > 0) && (long long)pU + Rs + er + s + rem > M;
          if (finiteM) brk |= pU + dd > M;
        } else if (kind == K_EVENT) {
          brk = tok + ec + 1 <= C;  // else a token reject (Q11)
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
        const int aw = __shfl_sync(FM, inner ? ew : xw, src), ar = __shfl_sync(FM, inner ? er : xr, src);
        const int ak = __popc(km & (inner ? ((1u << b) - 1u) : FM));
        tok += ac, U += ad, seq += aw, n_new += aw, n_running += aw, nB += ak, Rs += ar;
        if (inner) {
          const int bsl = __shfl_sync(FM, sl, b);
          __syncwarp();
          if (lane == 0) handle(bsl);
          from0();
          i0 += b + 1;
        } else {
          i0 += 32;
        }
      }
    };

    // Candidates that never preempt: the waiting group (src 1: window offsets [b0, b1) = R_w in index order,
    // Q5) or running prefills (src 2: run positions [b0, b1) = R_r^p; their KV delta is 0 since
    // reserved >= s >= m + c).  All are in the prefill phase, so a chunk of 32 is resolved in registers:
    // repeat {ballot the lanes that fit alone; prefix-scan them; admit those before the first cumulative
    // failure; drop that failure} -- rejections change no state.  A cropped chunk (chunked prefill)
    // exhausts the token budget and ends the group.
    int wnext = -1;  // after src 1: no window offset below it holds a waiting request (except victims)
    auto warp_np = [&](int src, int b0, int b1) {
      const bool overWin = src == 1;
      bool wcont = overWin;  // every waiting request at offsets [b0, i0) was admitted
      if (overWin) wnext = b0;
      for (int i0 = b0; i0 < b1; i0 += 32) {
        if ((!hybrid && bph == PH_DEC) || (chunked && tok >= C)) return;  // every remaining one fails
        if (overWin && ((finiteM && (long long)U + minSW > M) || (!chunked && minSW > C - tok))) return;
        const int i = i0 + lane;
        int sl = -1;
        if (i < b1) {
          if (overWin) {
            const int s2 = (lo + i) & (CAP - 1);
            if ((s_fl[s2] & (ST_MASK | F_PRE)) == ST_WAIT) sl = s2;
          } else {  // running prefills (not evicted) in retention order
            const int s2 = s_run[i];
            if ((s_fl[s2] & (ST_MASK | F_PRE | F_FILLED)) == ST_RUN) sl = s2;
          }
        }
        const int4 rc = s_rec[sl < 0 ? 0 : sl];
        const uint8_t fl = s_fl[sl < 0 ? 0 : sl];
        const int s = rc.x + rc.y, avail = s - rc.z;
        const int dkv = overWin ? rnew(rc, sl < 0 ? 0 : sl) : 0;  // KV delta: the initial reserve >= s >= c (Q13)
        const int rem = (hist && overWin) ? max(H.pred[bucket_of(rc.x)] - rc.y, 0) : 0;
        bool alive = sl >= 0, admitted = false;
        for (;;) {
          const int rt = C - tok;
          const bool anyRun0 = n_running > 0;
          bool fit = alive && rt >= 1 && (chunked || avail <= rt) && (!finiteM || U + dkv <= M);
          if (hist && overWin) fit = fit && !(anyRun0 && (long long)U + Rs + s + rem > M);
          const unsigned fm = __ballot_sync(FM, fit);
          if (!fm) break;
          const int cc = fit ? avail : 0, rr = fit ? rem : 0, dk = fit ? dkv : 0;
          const bool scand = overWin && !kv1;  // KV deltas differ from c only under a PEAK / CONTEXT reserve
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
            if (finiteM) brk |= U + ed + dkv > M;
            if (hist && overWin) brk |= (anyRun0 || ek > 0) && (long long)U + ed + Rs + er + s + rem > M;
            if (crop && prt <= 0) brk = true;
          }
          const unsigned bm = __ballot_sync(FM, brk), cm = __ballot_sync(FM, crop && !brk);
          const int b = bm ? __ffs(bm) - 1 : 32, cl = cm ? __ffs(cm) - 1 : 32;
          const int stop = min(b, cl);                                             // lanes < stop: in full
          const bool adm = fit && lane < stop, adc = fit && lane == cl && cl < b;  // + the cropped one
          if (adm || adc) {
            s_c[sl] = adm ? avail : rt - ec;
            s_bl[nB + ek] = (int16_t)sl;
            if (overWin) {
              s_seq[sl] = seq + ek + 1;
              s_rec[sl] = make_int4(rc.x, rc.y, 0, dkv);
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
      }
    };

    // Closed form for the running decodes visited in retention order (every head needs one KV under SEQ;
    // the victim pool is the run-list tail, all running and not in B).  Head i (run position p_i) is
    // admitted iff i <= C - tok and F + RS(p_i + 1) >= i, F = M - U, RS(q) = sum of held KVs at run
    // positions >= q (monotone in i).  Admitting a heads evicts the minimal tail suffix [q*, n) with
    // F + RS(q*) >= a; if head a+1 runs out of pool, everything behind it is evicted and it self-preempts
    // (Q8).  This is exactly the sequential head/tail walk of steps (3)-(4).
    // Reverse run index r = s * 256 + j * 32 + lane (q = nrun - 1 - r): superchunks of 8 warp chunks,
    // re-read from shared memory per pass when the run list exceeds one superchunk.
    int rp_first = nrun;  // first run position of a surviving running prefill (nrun if none)
    auto decode_group = [&]() {
      constexpr int DJ = 8;
      const bool fM = finiteM && kv1;  // heads need one KV each (else none: admitted up to the token budget)
      const int F = fM ? M - U : 0x3fffffff;
      const int T = C - tok;
      const int nsc = (nrun + 32 * DJ - 1) / (32 * DJ);
      int hv[DJ], rsv[DJ], hsv[DJ];
      bool hh[DJ];
      int16_t sls[DJ];
      {  // every head fits (F >= k, or no KV needed): admit the first min(k, T) heads -- no scan, no eviction
        int k0 = 0;
        for (int j0 = 0; j0 < nrun; j0 += 32) {
          const int q = nrun - 1 - (j0 + lane);
          k0 += __popc(__ballot_sync(FM, q >= 0 && (s_fl[s_run[q]] & F_FILLED)));
        }
        if (!fM || F >= k0) {
          const int a = min(k0, T);
          int hs = 0, pm = nrun;
          for (int j0 = 0; j0 < nrun; j0 += 32) {
            const int q = nrun - 1 - (j0 + lane);
            int sl = 0;
            bool h = false;
            if (q >= 0) {
              sl = s_run[q];
              h = (s_fl[sl] & F_FILLED) != 0;
            }
            const unsigned hb = __ballot_sync(FM, h);
            const int i = k0 - (hs + __popc(hb & ((2u << lane) - 1u))) + 1;  // head index, front to back
            if (h && i <= a) {
              s_c[sl] = 1;
              s_fl[sl] |= F_INB;
              s_bl[nB + i - 1] = (int16_t)sl;
            }
            if (q >= 0 && !h) pm = min(pm, q);
            hs += __popc(hb);
          }
          rp_first = (int)__reduce_min_sync(FM, (unsigned)pm);
          tok += a;
          U += kv1 ? a : 0;
          nB += a;
          if (a > 0 && bph < 0) bph = PH_DEC;
          vt = min(vt, nrun - 1);
          cut = nrun;
          __syncwarp();
          return;
        }
      }
      int cs = 0, ch = 0;  // carries: held and heads at reverse indices before this superchunk
      auto load = [&](int sc) {
#pragma unroll
        for (int j = 0; j < DJ; j++) {
          const int q = nrun - 1 - (sc * 32 * DJ + j * 32 + lane);
          hv[j] = 0, hh[j] = false, sls[j] = 0;
          if (q >= 0) {
            const int sl = s_run[q];
            sls[j] = (int16_t)sl;
            const int4 rc = s_rec[sl];
            hv[j] = max(rc.w, rc.z);
            hh[j] = (s_fl[sl] & F_FILLED) != 0;
          }
        }
#pragma unroll
        for (int j = 0; j < DJ; j++) {  // inclusive scans: RS(q) and HS(q) (heads at positions >= q)
          if (sc * 32 * DJ + j * 32 >= nrun) break;
          int xs = hv[j];
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int ys = __shfl_up_sync(FM, xs, o);
            if (lane >= o) xs += ys;
          }
          const unsigned hb = __ballot_sync(FM, hh[j]);  // heads are bits: their prefix is a popcount
          rsv[j] = cs + xs, hsv[j] = ch + __popc(hb & ((2u << lane) - 1u));
          cs += __shfl_sync(FM, xs, 31), ch += __popc(hb);
        }
      };
      // pass 1: the scans (kept in registers when one superchunk holds the whole run list); k = #heads
      for (int sc = 0; sc < nsc; sc++) load(sc);
      const int k = ch;
      // pass 2: a_kv = #{heads i : F + RS(p_i + 1) >= i}, i = k - HS(p_i) + 1 (monotone in i)
      int akv = k;
      if (fM) {
        int cnt = 0;
        cs = ch = 0;
        for (int sc = 0; sc < nsc; sc++) {
          if (nsc > 1) load(sc);
#pragma unroll
          for (int j = 0; j < DJ; j++)
            if (hh[j]) cnt += F + (rsv[j] - hv[j]) >= k - hsv[j] + 1;
        }
        akv = (int)__reduce_add_sync(FM, (unsigned)cnt);
      }
      const int a = min(min(akv, T), k);
      // pass 3: q* = max{q : F + RS(q) >= a}; the position of head a+1
      const bool needq = fM && F < a;
      const bool needp = fM && a == akv && a < min(k, T);
      int qs = nrun, selfp = -1;
      if (needq || needp) {
        int cq = 0, pa = -1;
        cs = ch = 0;
        for (int sc = 0; sc < nsc; sc++) {
          if (nsc > 1) load(sc);
#pragma unroll
          for (int j = 0; j < DJ; j++) {
            const int q = nrun - 1 - (sc * 32 * DJ + j * 32 + lane);
            if (q >= 0) {
              if (needq) cq += F + rsv[j] >= a;
              if (hh[j] && k - hsv[j] + 1 == a + 1) pa = q;
            }
          }
        }
        if (needq) qs = (int)__reduce_add_sync(FM, (unsigned)cq) - 1;
        // head a+1, when the KV (not the token budget) stopped the walk: a victim if it lies in the evicted
        // suffix, else it runs out of pool, evicts everything behind it and self-preempts (Q8)
        if (needp) {
          pa = (int)__reduce_max_sync(FM, (unsigned)(pa + 1)) - 1;
          if (pa < qs) selfp = pa, qs = pa + 1;
        }
      }
      // pass 4: apply -- evict [qs, nrun) (+ the self-preempted head), admit heads 1..a
      const bool evict = qs < nrun || selfp >= 0;
      int ev = 0, eh = 0, er = 0, pm = nrun;
      cs = ch = 0;
      for (int sc = 0; sc < nsc; sc++) {
        if (nsc > 1) load(sc);
#pragma unroll
        for (int j = 0; j < DJ; j++) {
          const int q = nrun - 1 - (sc * 32 * DJ + j * 32 + lane);
          if (q < 0) continue;
          const int sl = sls[j];
          if (q < qs && !hh[j]) pm = min(pm, q);
          if (q >= qs || q == selfp) {
            const int4 rc = s_rec[sl];
            ev++;
            eh += hv[j];
            if (hist) er += max(H.pred[bucket_of(rc.x)] - rc.y, 0);
            const int idx = req_idx(sl);
            atomicAdd(&npre[idx], 1ull);
            atomicAdd(&refill[idx], (unsigned long long)rc.z);
            s_rec[sl] = make_int4(rc.x, rc.y, 0, 0);
            s_fl[sl] = ST_WAIT | F_PRE | (s_fl[sl] & F_FIRST);
            s_vic[n_vic + (q == selfp ? nrun - qs : q - qs)] = (int16_t)sl;
          } else if (hh[j]) {
            const int i = k - hsv[j] + 1;
            if (i <= a) {
              s_c[sl] = 1;
              s_fl[sl] |= F_INB;
              s_bl[nB + i - 1] = (int16_t)sl;
            }
          }
        }
      }
      int tev = 0, teh = 0, ter = 0;
      if (evict) {
        tev = (int)__reduce_add_sync(FM, (unsigned)ev);
        teh = (int)__reduce_add_sync(FM, (unsigned)eh);
        if (hist) ter = (int)__reduce_add_sync(FM, (unsigned)er);
      }
      rp_first = (int)__reduce_min_sync(FM, (unsigned)pm);
      tok += a;
      U += (kv1 ? a : 0) - teh;
      nB += a;
      n_running -= tev;
      Rs -= ter;
      if (a > 0 && bph < 0) bph = PH_DEC;
      n_vic += tev;
      npreempt += tev;
      any_pre |= tev > 0;
      vt = min(vt, (selfp >= 0 ? selfp : qs) - 1);
      cut = selfp >= 0 ? selfp : qs;  // run positions >= cut were evicted (a suffix)
      __syncwarp();
    };

    // the groups in the preset's visiting order (Table 2; App. D)
    if (rank) {
      warp_run(s_rank, 0, nrank);
    } else {
      const int w0 = max(wfirst - lo, 0);  // window offsets below w0 hold no waiting request
      for (int g = 0; g < 3; g++) {  // decode-first {R_r^d, R_r^p, R_w}; prefill-first {R_w, R_r}
        const int what = order == SIM_ORDER_DECODE_FIRST ? g : (g == 0 ? 2 : (g == 1 ? 3 : -1));
        if (what == 0 || what == 3) {  // running decodes (closed form) or, with chunking, the whole R_r
          if (nrun == 0) continue;
          if (what == 3 && chunked) {
            warp_run(s_run, 0, nrun);
          } else if (what == 0 || hybrid || bph != PH_PRE) {
            decode_group();
          }
        } else if (what == 1) {  // running prefills
          if (rp_first < nrun) warp_np(2, rp_first, nrun);
        } else if (what == 2 && nW > 0) {  // the waiting group
          warp_np(1, w0, nx1 - lo);
          if (wnext >= 0) wfirst = lo + wnext;
        }
      }
    }
    __syncwarp();

    if (tok == 0) {  // B = {}: idle jump to the next arrival, not a step (Q21)
      if (any_pre || nx1 >= n) {
        exit_status = SIM_S_DEADLOCK;
        break;
      }
      clk[0] = fmax(clk[0], wl.T[nx1]);
      idle++;
      next = nx1;
      w_dirty = false;
      rank_dirty = false;
      continue;
    }
    // ---- (4) a9 + a10: Process(B) and the exact integer features in one pass over B ----
    unsigned N = 0, np_ = 0, cp = 0, mp = 0, nd = 0, md = 0, freed = 0, ndone = 0, mdn = 0, nfill = 0;
    int minrem = NOBRK, n_ev = 0;
    long long c2 = 0, mc = 0, pcm = 0, pce[SIM_MAX_COST] = {0, 0, 0, 0};
    for (int e0 = 0; e0 < nB; e0 += 128) {  // four entries per lane per round, loads first (ILP)
      int slv[4], cv[4], Ov[4];
      int4 rcv[4];
      uint8_t flv[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int e = e0 + u * 32 + lane;
        slv[u] = e < nB ? s_bl[e] : -1;
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int sl = slv[u] < 0 ? 0 : slv[u];
        flv[u] = s_fl[sl], rcv[u] = s_rec[sl], cv[u] = s_c[sl], Ov[u] = s_O[sl];
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        if (e0 + u * 32 >= nB) break;  // uniform
        int evc = 0;
        const int sl = slv[u];
        if (sl >= 0) {
          uint8_t fl = flv[u];
          const int4 rc = rcv[u];
          const int c = cv[u], O = Ov[u];
          const int m0 = rc.z;
          int g = rc.y;
          const int s = rc.x + g, m = m0 + c;
          N += c;
          if (!(fl & F_FILLED)) {  // prefill entry (incl. refills and chunks)
            if (srf) fl |= F_MOVE;  // its SRF key moves by c: re-inserted into the run list order below
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
                  const int Hk = H.cm[k].H;
                  pce[k] += (long long)((c + Hk - 1) / Hk) * (c + m0);
                }
            }
          } else {  // decode entry (c = 1)
            if (srf) fl |= F_DEC;
            nd++;
            md += m0;
          }
          fl &= ~F_INB;
          bool done = false;
          if (c == s - m0) {  // Eq. (6): all available tokens processed -> one token (Q18)
            g++;
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
              freed += max(rc.w, m);
              ndone++;
              if (hist) atomicAdd(&H.hist[bucket_of(rc.x) * 18 + bucket_of(O)], 1);
            }
          }
          if (!done) {
            minrem = min(minrem, O - g);
            mdn += m;
          }
          s_rec[sl] = make_int4(rc.x, g, m, rc.w);
          s_fl[sl] = fl;
        }
        const unsigned em = __ballot_sync(FM, evc != 0);  // first-token / completion events, compacted
        if (evc) s_ev[n_ev + __popc(em & lt)] = (int16_t)(sl | (evc << SLB));
        n_ev += __popc(em);
      }
    }
    N = __reduce_add_sync(FM, N), np_ = __reduce_add_sync(FM, np_), cp = __reduce_add_sync(FM, cp);
    mp = __reduce_add_sync(FM, mp), nd = __reduce_add_sync(FM, nd), md = __reduce_add_sync(FM, md);
    freed = __reduce_add_sync(FM, freed), ndone = __reduce_add_sync(FM, ndone);
    mdn = __reduce_add_sync(FM, mdn), nfill = __reduce_add_sync(FM, nfill);
    minrem = (int)__reduce_min_sync(FM, (unsigned)minrem);
    if (np_ > 0) {  // prefill squares: 64-bit
      c2 = warp_sum(c2);
      mc = warp_sum(mc);
      if (anyTheo) {
        pcm = warp_sum(pcm);
#pragma unroll
        for (int k = 0; k < SIM_MAX_COST; k++) pce[k] = warp_sum(pce[k]);
      }
    }
    // clear the preempted-this-step marks (Q9 applies within one step); the victims join R_w
    int vmin = 0x7fffffff, vidx = 0x7fffffff;
    for (int v = lane; v < n_vic; v += 32) {
      const int sl = s_vic[v];
      s_fl[sl] &= ~F_PRE;
      const int4 rc = s_rec[sl];
      vmin = min(vmin, rc.x + rc.y);
      vidx = min(vidx, req_idx(sl));
    }
    if (n_vic > 0) {
      vmin = (int)__reduce_min_sync(FM, (unsigned)vmin);
      wfirst = min(wfirst, (int)__reduce_min_sync(FM, (unsigned)vidx));  // they wait from the next step on
    }
    {  // a9: batch time of every cost model on the same schedule (all lanes alike; fp64 in the oracle's order)
      Feat f;
      f.N = N, f.np = np_, f.cp = cp, f.mp = mp, f.nd = nd, f.md = md, f.c2 = c2, f.mc = mc, f.pcm = pcm;
#pragma unroll
      for (int k = 0; k < SIM_MAX_COST; k++) f.pceil[k] = pce[k];
      for (int k = 0; k < K; k++) clk[k] = dadd(clk[k], batch_time(H.cm[k], f, k));  // Q36
    }
    steps++;
    sumU += U;
    entries += np_ + nd;
    processed += N;
    pentries += np_;
    const int Uafter = U - (int)freed;
    n_done += (int)ndone;
    // Steady decode run: step j had only decodes, no admission, preemption or completion.  Then step j+1
    // repeats it exactly (waiting candidates were rejected for reasons that persist: KV and SRF+Hist
    // deferral are monotone in U, token/hybrid rejections are unchanged) until a completion, the KV limit
    // (U + k n_d <= M) or an arrival.  Those steps are charged below without re-forming batches.
    long long Lr = 0;
    if (ndone == 0 && np_ == 0 && !any_pre && nd > 0) {
      Lr = minrem;
      if (finiteM && kv1) Lr = min(Lr, (long long)(M - Uafter) / nd);
      Lr = min(Lr, cfg.max_steps - steps);
    }
    U = Uafter;
    bool changed = n_new > 0 || any_pre || ndone > 0;  // run-list membership changed
    // removals only as the closed form's evicted suffix: the run list is cut, not compacted
    int removals = h_pre || ndone > 0 ? 2 : (any_pre ? 1 : 0);
    // R_w gains this step's victims and loses its admissions: |R_w| stays exact; the smallest s becomes a
    // lower bound after admissions (the skip tests only get conservative) and is recounted every 32 of them
    nW = nW - n_new + n_vic, minSW = min(minSW, vmin);
    if (n_new > 0) wstale++;
    w_dirty = arrived || wstale >= 32;
    if (w_dirty) wstale = 0;
    rank_dirty = ndone > 0;
    // SRF order can change unless every running request was a decode in B (all +1)
    bool odirty = srf && (changed || np_ > 0 || (int)nd != nrun);
    __syncwarp();

    // ---- (5) event times; steady decode run ----
    for (int e = lane; e < n_ev; e += 32) {
      const int code = s_ev[e], sl = code & (CAP - 1);
      const int idx = req_idx(sl);
      if (code & (1 << SLB))
        for (int k = 0; k < K; k++) tf[(long long)k * n + idx] = clk[k];
      if (code & (2 << SLB))
        for (int k = 0; k < K; k++) td[(long long)k * n + idx] = clk[k];
    }
    if (Lr > 0) {
      const long long ndd = nd, MD = mdn, U0 = U, du = kv1 ? ndd : 0;  // KV growth per run step
      long long E = 0;
      const double Tn = nx1 < n ? wl.T[nx1] : 0.0;  // online (K == 1): the next arrival
      while (E < Lr) {
        const int chunk = (int)min(32ll, Lr - E);
        double dk[SIM_MAX_COST] = {0.0, 0.0, 0.0, 0.0};
        if (lane < chunk) {  // features of run step E+lane+1 are affine in the step index
          Feat f;
          f.N = ndd, f.np = 0, f.c2 = 0, f.mc = 0, f.cp = 0, f.mp = 0, f.pcm = 0, f.nd = ndd;
          f.md = MD + (E + lane) * ndd;
          for (int k = 0; k < SIM_MAX_COST; k++) f.pceil[k] = 0;
          for (int k = 0; k < K; k++) dk[k] = batch_time(H.cm[k], f, k);
        }
        // the clock chain stays sequential: one fp64 add per step, as in the oracle (Q36)
        int ex = chunk;
        if (nx1 < n) {  // stop before a step that would start at/after an arrival (Q21)
          double c0 = clk[0];
          for (int t = 0; t < chunk; t++) {
            const double d = __shfl_sync(FM, dk[0], t);
            if (Tn <= c0) {
              ex = t;
              break;
            }
            c0 = dadd(c0, d);
          }
          clk[0] = c0;
        } else {
          for (int k = 0; k < K; k++) {
            double c0 = clk[k];
            const double mine = dk[k];
            for (int t = 0; t < chunk; t++) c0 = dadd(c0, __shfl_sync(FM, mine, t));
            clk[k] = c0;
          }
        }
        E += ex;
        if (ex < chunk) break;
      }
      int fr2 = 0, nd2 = 0;
      if (E > 0) {
        for (int e = lane; e < nB; e += 32) {  // every B entry is a decode of the steady step
          const int sl = s_bl[e];
          const int4 rc = s_rec[sl];
          const int m = rc.z + (int)E, g = rc.y + (int)E, O = s_O[sl];
          s_rec[sl] = make_int4(rc.x, g, m, rc.w);
          if (g == O) {  // completes at the last run step
            s_fl[sl] = (s_fl[sl] & ~ST_MASK) | ST_DONE;
            for (int k = 0; k < K; k++) td[(long long)k * n + req_idx(sl)] = clk[k];
            fr2 += max(rc.w, m);
            nd2++;
            if (hist) atomicAdd(&H.hist[bucket_of(rc.x) * 18 + bucket_of(O)], 1);
          }
        }
        fr2 = (int)__reduce_add_sync(FM, (unsigned)fr2);
        nd2 = (int)__reduce_add_sync(FM, (unsigned)nd2);
      }
      steps += E;
      sumU += E * U0 + du * (E * (E + 1) / 2);
      entries += E * ndd;
      processed += E * ndd;
      visits += E * nP;
      U = (int)(U0 + E * du) - fr2;
      n_done += nd2;
      if (nd2 > 0) changed = true, removals = 2, rank_dirty = true;
      if (srf && E > 0 && ndd != nrun) odirty = true;
      __syncwarp();
    }

    // ---- (6) run list (retention order) for the next step ----
    int cnt = nrun;
    bool moved = false;
    if (changed) {
      if (removals == 1) {  // the evicted suffix is cut off, admissions are appended
        for (int q = lane; q < n_new; q += 32) s_run[cut + q] = s_new[q], s_rpos[s_new[q]] = (int16_t)(cut + q);
        cnt = cut + n_new;
      } else if (removals) {
        cnt = compact(s_run, nrun, s_new, n_new, [&](int sl) { return (s_fl[sl] & ST_MASK) == ST_RUN; });
        moved = true;
      } else {  // only admissions: append them (admission order = NRF retention order)
        for (int q = lane; q < n_new; q += 32) s_run[nrun + q] = s_new[q], s_rpos[s_new[q]] = (int16_t)(nrun + q);
        cnt = nrun + n_new;
      }
      __syncwarp();
    }
    if (odirty) {  // SRF retention order: m descending, then admission order (Q3, Q7)
      // Since the last step the decodes of B (D, marked in Process) moved by +1 (+E+1 over a steady run),
      // the other running requests (N) by 0 and the prefill entries of B (movers, marked) by their c.
      // D and N are each still in order, and so is D u N when no D follows an N.  So: drop the movers
      // (stable compaction), check D u N only when some D follows an N, sort the few movers and merge
      // them in by rank; the whole list is sorted only when D u N is out of order.
      auto key = [&](int sl) -> unsigned long long {
        return ((unsigned long long)(0x3FFFF - s_rec[sl].z) << 46) | ((unsigned long long)(unsigned)s_seq[sl] << SLB) |
               (unsigned long long)sl;
      };
      int ns = 0, nm = 0;
      bool inv = false, seenN = false;
      for (int b = 0; b < cnt; b += 32) {
        const int q = b + lane;
        const int sl = q < cnt ? s_run[q] : 0;
        const uint8_t f = q < cnt ? s_fl[sl] : 0;
        const bool mv = q < cnt && (f & F_MOVE), dec = q < cnt && !mv && (f & F_DEC), nn = q < cnt && !mv && !dec;
        const unsigned mb = __ballot_sync(FM, mv), db = __ballot_sync(FM, dec), nb = __ballot_sync(FM, nn);
        if ((seenN && db) || (nb && (db >> (__ffs(nb) - 1)))) inv = true;  // a D after an N
        seenN |= nb != 0;
        __syncwarp();  // every lane has read its item before any write (writes never pass reads)
        if (mv) s_vic[nm + __popc(mb & lt)] = (int16_t)sl;
        if (dec || nn) s_run[ns + __popc((db | nb) & lt)] = (int16_t)sl;
        if (f & (F_MOVE | F_DEC)) s_fl[sl] = f & ~(F_MOVE | F_DEC);
        nm += __popc(mb), ns += __popc(db | nb);
      }
      __syncwarp();
      bool okk = true;
      if (inv) {
        for (int q = lane; okk && q + 1 < ns; q += 32) okk = key(s_run[q]) < key(s_run[q + 1]);
        okk = __all_sync(FM, okk);
      }
      if (!okk) {  // the whole list
        for (int q = lane; q < cnt; q += 32) s_keys[q] = key(q < ns ? s_run[q] : s_vic[q - ns]);
        __syncwarp();
        sort_keys(cnt);
        for (int q = lane; q < cnt; q += 32) s_run[q] = (int16_t)(s_keys[q] & (CAP - 1));
        moved = true;
      } else if (nm > 0) {  // sort the movers, merge them in: mover j lands at ins_j + j, stable i at i + #{ins_j <= i}
        for (int j = lane; j < nm; j += 32) s_keys[j] = key(s_vic[j]);
        __syncwarp();
        sort_keys(nm);
        int16_t* s_ins = s_new;  // free after the membership update
        for (int j = lane; j < nm; j += 32) {
          const unsigned long long x = s_keys[j];
          int lo2 = 0, hi2 = ns;
          while (lo2 < hi2) {  // #{stable keys < x}
            const int mid = (lo2 + hi2) >> 1;
            if (key(s_run[mid]) < x)
              lo2 = mid + 1;
            else
              hi2 = mid;
          }
          s_ins[j] = (int16_t)lo2;
        }
        __syncwarp();
        for (int b = ((ns - 1) >> 5) << 5; b >= 0; b -= 32) {  // back to front: a move never passes a pending read
          const int i = b + lane;
          int sl = 0, sh = 0;
          if (i < ns) {
            sl = s_run[i];
            int lo2 = 0, hi2 = nm;
            while (lo2 < hi2) {  // #{ins_j <= i}
              const int mid = (lo2 + hi2) >> 1;
              if (s_ins[mid] <= i)
                lo2 = mid + 1;
              else
                hi2 = mid;
            }
            sh = lo2;
          }
          __syncwarp();
          if (i < ns && sh) s_run[i + sh] = (int16_t)sl;
        }
        __syncwarp();
        for (int j = lane; j < nm; j += 32) s_run[s_ins[j] + j] = (int16_t)(s_keys[j] & (CAP - 1));
        moved = true;
      } else if (ns < cnt) {
        moved = true;
      }
      __syncwarp();
    } else if (srf) {  // nothing moved: clear the decode marks of B
      for (int e = lane; e < nB; e += 32) s_fl[s_bl[e]] &= ~F_DEC;
      __syncwarp();
    }
    if (moved) {
      for (int q = lane; q < cnt; q += 32) s_rpos[s_run[q]] = (int16_t)q;
    }
    nrun = cnt;
    next = nx1;
    for (;;) {  // lo: the first request not done
      const int i = lo + lane;
      const bool dn = i < nx1 && (s_fl[i & (CAP - 1)] & ST_MASK) == ST_DONE;
      const unsigned b = __ballot_sync(FM, dn);
      if (b == FM) {
        lo += 32;
        continue;
      }
      lo += __ffs(~b) - 1;
      break;
    }
    __syncwarp();
  }

#ifdef SIMSWEEP_PROFILE
  if (lane == 0 && ci < PROF_MAX_CFG) {  // start / end / SM of this simulation (tools/timeline.py)
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_prof[ci][14] = (long long)t_start, g_prof[ci][15] = (long long)t_end, g_prof[ci][9] = smid;
  }
#endif
  // ---- a11: metrics ----
  const int st = exit_status == -1 ? SIM_S_OK : exit_status;
  __syncwarp();
  if (st != SIM_S_OK) {  // failed simulations: zero-filled rows
    __threadfence();
    for (int i = lane; i < n; i += 32) npre[i] = 0, refill[i] = 0;
    for (int x = lane; x < K * n; x += 32) tf[x] = 0.0, td[x] = 0.0;
    if (lane == 0) {
      sim_result_t r;
      memset(&r, 0, sizeof(r));
      r.status = st;
      p.results[ci] = r;
    }
    return;
  }
  __threadfence_block();
  if (lane < K) {  // sequential sums in request order (identical to the oracle)
    const int k = lane;
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
  if (lane == 0) {
    sim_result_t& r = p.results[ci];
    r.status = SIM_S_OK;
    r.pad = 0;
    r.steps = steps;
    r.preemptions = npreempt;
    r.batch_entries = entries;
    r.processed_tokens = processed;
    r.sum_U = sumU;
    r.prefill_entries = pentries;
    r.idle_jumps = idle;
    r.visits = visits;
    for (int k = K; k < SIM_MAX_COST; k++) r.makespan[k] = r.mean_latency[k] = r.mean_ttft[k] = r.mean_tpot[k] = 0.0;
  }
}

}  // namespace simsweep
