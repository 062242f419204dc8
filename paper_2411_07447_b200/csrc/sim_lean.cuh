// sim_lean.cuh -- the lean step kernel: ONE WARP per simulation, decodes advanced lazily (included by simsweep.cu).
//
// The same method and readings as sim_step.cuh (Algorithm 1; Q1-Q40), for the
// configurations that dominate the north-star sweep (lean_ok in simsweep.cu): the vLLM / Sarathi presets
// (prefill-first without chunking, or decode-first), NRF / SRF / PF, no alternative-reading knob, no SRF+Hist,
// no schedule trace, n <= CAP requests.  Everything a step decides (tok, U, seq, list lengths, counters) lives
// in registers, uniform across the warp; lane k < K holds the clock of cost model k; per-request state is a
// structure of arrays in shared memory.
//
// Decode epochs.  Every running decode that is in a batch advances by exactly one token (c = 1, m += 1, g += 1,
// Eq. (6)), and in almost every step either all surviving decodes are in B or none is.  So a running decode
// stores its m and g relative to a decode epoch D (rec = {I, g - D, m - D, reserved}), and a step that admits the
// decodes advances all of them with D += 1.  The decodes a step leaves out (only the token budget can, Q11) are
// compensated (their offsets lowered by one).  The batch features of the decodes come from running sums
// (n_d = the admitted heads, sum m = sum(m - D) + n_d D, Table 3), and the next completion is the smallest
// completion epoch O - (g - D) over the running decodes.  A step therefore costs O(its events) -- the admitted
// prefills, the evicted tail, completions -- not O(|R_r|).
//
// One step (one batch B_j):
//   a2    arrivals: the next arrival time stays in a register; a ballot pass admits every T <= clock (Q21)
//   a3-a8 GetNextBatch:
//         * the running decodes in closed form (decode group): head i (the i-th decode in retention order, at run
//           position p_i) is admitted iff i <= C - tok and F + RS(p_i + 1) >= i (F = M - U, RS = the holdings
//           behind p_i); the predicate is monotone in i, so a walk from the run list's TAIL finds the last
//           admitted head a; the minimal tail suffix [q*, n) with F + RS(q*) >= a is evicted; if the KV stopped
//           the walk, head a+1 evicts everything behind it and self-preempts (Q8)
//         * the waiting group and the running prefills (they never preempt, Q5): 32 candidates per pass,
//           ballot + prefix scan, the first cumulative failure dropped, a cropped chunk ends the group
//   a9    exact integer features (prefill entries explicitly, decodes from the running sums); lane k < K
//         evaluates cost model k (no FMA, Q36)
//   a10   Process: the prefill entries explicitly, the decodes by D += 1; completions at their completion epoch
//   runs  steady decode runs charged in closed form (features affine in the step index) up to the next completion
//         epoch, the KV limit or an arrival; the clock chain stays one sequential fp64 add per step (Q36)
//   a3'   the run list for the next step: the evicted suffix is cut, completions are compacted out, admissions
//         are appended (NRF / PF: admission order) or, for SRF, the entries whose keys moved are merged back by
//         (m desc, seq) (Q3, Q7)
#pragma once

namespace simsweep {

constexpr uint8_t F_INB_L = 8;    // a running prefill admitted into this step's batch
constexpr uint8_t F_MOVE_L = 64;  // SRF: an entry whose retention key moved relative to the others

struct LHead {
  sim_cost_model_t cm[SIM_MAX_COST];
  LTerm term[32];                 // lane 8k + j: Eq. (3) term j of model k (batch_time_lanes)
  double dv[SIM_MAX_COST][8];     // per model: the terms' divisors and reciprocals
  int hist[18 * 18];  // SRF+Hist: log2 histogram of (I, O) at completions (Q31)
  int pred[18];       // SRF+Hist: predicted output length per I bucket (recomputed after completions)
};

// Per-slot arrays (41 B per slot): in shared memory right after LHead, or (GM: workloads of n > 4096 requests, up
// to SIM_MAX_WINDOW) in a per-CTA arena of the caller's workspace, served from L1 / L2; a GM CTA keeps LHead and the
// waiting bitmap (12 B per 32 slots) in shared memory.  Slots are request indices (n <= CAP: no ring).
template <int CAP, bool GM>
struct LLayout {
  static constexpr size_t a16(size_t x) { return (x + 15) & ~size_t(15); }
  static constexpr size_t head = a16(sizeof(LHead));
  static constexpr size_t rec = GM ? 0 : head;       // int4 {I, g | g - D, m | m - D, reserved}
  static constexpr size_t O = rec + 16 * CAP;        // int32
  static constexpr size_t seq = O + 4 * CAP;         // int32 admission sequence number (Q6)
  static constexpr size_t c = seq + 4 * CAP;         // int32 c of this batch's prefill entries  \ u64 sort keys
  static constexpr size_t ev = c + 4 * CAP;          // int32 first-token / completion events   / (SRF merge)
  static constexpr size_t run = ev + 4 * CAP;        // int16 run list (retention order)
  static constexpr size_t run2 = run + 2 * CAP;      // int16 this batch's running prefills; the merge target
  static constexpr size_t nw = run2 + 2 * CAP;       // int16 admitted from R_w this step, in admission order
  static constexpr size_t vic = nw + 2 * CAP;        // int16 preempted this step, then the SRF movers
  static constexpr size_t fl = vic + 2 * CAP;        // uint8 status and flags
  static constexpr size_t arr_bytes = a16(fl + CAP) - rec;  // 41 B per slot
  static constexpr size_t words = CAP / 32;                    // waiting bitmap (GM: in shared memory)
  static constexpr size_t smem = GM ? head + 12 * words : a16(fl + CAP);
};

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// warp sum of non-negative per-lane values below 2^51 in two REDUX: the low 24 bits and the rest apart
__device__ __forceinline__ long long warp_sum_u51(unsigned long long v) {
  const unsigned lo = __reduce_add_sync(0xffffffffu, (unsigned)(v & 0xffffffu));
  const unsigned hi = __reduce_add_sync(0xffffffffu, (unsigned)(v >> 24));
  return ((long long)hi << 24) + (long long)lo;
}

// SRF retention key (ascending = retained longer): m descending, then admission order (Q3, Q7); the slot rides in
// the low bits so that sorting keys sorts slots
template <int SLB>
__device__ __forceinline__ unsigned long long srf_key(int m, int seq, int slot) {
  // bits: 18 of 0x3FFFF - m (m <= S < 2^18) | 31 of seq (< 2^31, SEQ_LIM) | SLB of slot: 49 + SLB <= 64
  return ((unsigned long long)(0x3FFFF - m) << (31 + SLB)) | ((unsigned long long)(unsigned)seq << SLB) | (unsigned)slot;
}

template <int CAP, bool GM>
__global__ void __launch_bounds__(32, 1) sim_lean_kernel(KParams p) {
  using L = LLayout<CAP, GM>;
  constexpr unsigned FM = 0xffffffffu;
  constexpr int SLB = __builtin_ctz(CAP);
  static_assert(SLB <= 15, "int16 slots; slot bits of the SRF key");
  constexpr long long SEQ_LIM = 0x7fffffffll - CAP;  // the int32 admission counter must not wrap
  constexpr int BIG = 0x3fffffff;
  extern __shared__ __align__(16) unsigned char smem[];
  LHead& H = *reinterpret_cast<LHead*>(smem);
  const int lane = threadIdx.x;
  const unsigned lt = (1u << lane) - 1u;
  const int ci = p.order ? p.order[blockIdx.x] : (int)blockIdx.x;
  if (kernel_variant(p.cfgs[ci], p.wls[p.cfgs[ci].workload].n, p.lean) != p.variant) return;
#ifdef SIMSWEEP_PROFILE  // per-simulation start / end / SM (tools/timeline.py); not in the product build
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  struct ProfEnd {
    int ci;
    unsigned long long t0;
    __device__ ~ProfEnd() {
      if (threadIdx.x == 0 && ci < PROF_MAX_CFG) {
        unsigned long long t1;
        unsigned smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_prof[ci][14] = (long long)t0, g_prof[ci][15] = (long long)t1, g_prof[ci][9] = smid;
      }
    }
  } prof_end{ci, t_start};
#endif
  unsigned char* arr = smem;
  if constexpr (GM) {  // claim a per-CTA arena of the workspace (the stride of the block kernel's GM arenas)
    int a0 = 0;
    if (lane == 0) a0 = p.arena_base + (int)atomicAdd(reinterpret_cast<unsigned*>(p.ws + p.ctr_off), 1u);
    a0 = __shfl_sync(FM, a0, 0);
    arr = p.ws + WS_HEADER + (size_t)a0 * Smem<512, SIM_MAX_WINDOW>::arr_bytes;
  }
  int4* s_rec = reinterpret_cast<int4*>(arr + L::rec);
  int32_t* s_O = reinterpret_cast<int32_t*>(arr + L::O);
  int32_t* s_seq = reinterpret_cast<int32_t*>(arr + L::seq);
  int32_t* s_c = reinterpret_cast<int32_t*>(arr + L::c);
  int32_t* s_ev = reinterpret_cast<int32_t*>(arr + L::ev);
  double* s_dbuf = reinterpret_cast<double*>(arr + L::ev);                        // steady run: batch times
  unsigned long long* s_key = reinterpret_cast<unsigned long long*>(arr + L::c);  // SRF merge: CAP keys
  int16_t* s_run = reinterpret_cast<int16_t*>(arr + L::run);
  int16_t* s_run2 = reinterpret_cast<int16_t*>(arr + L::run2);
  int16_t* s_new = reinterpret_cast<int16_t*>(arr + L::nw);
  int16_t* s_vic = reinterpret_cast<int16_t*>(arr + L::vic);
  uint8_t* s_fl = arr + L::fl;
  // GM: the waiting bitmap's words in shared memory: bits, smallest s, smallest PEAK reserve (BIG if empty)
  unsigned* g_wb = reinterpret_cast<unsigned*>(smem + L::head);
  int* g_ws = reinterpret_cast<int*>(g_wb + L::words);
  int* g_wd = g_ws + L::words;

  const sim_config_t cfg = p.cfgs[ci];
  const sim_workload_t wl = p.wls[cfg.workload];
  const int n = wl.n, K = cfg.n_cost;
  const bool finiteM = cfg.M >= 0, hybrid = cfg.hybrid != 0, chunked = cfg.chunked != 0;
  const int M = finiteM ? (int)cfg.M : 0, C = (int)cfg.C;  // host-validated <= 2^30
  const bool pfirst = cfg.order == SIM_ORDER_PREFILL_FIRST;  // {R_w, R_r} (never chunked here), else {R_r^d, R_r^p, R_w}
  const bool srf = cfg.replacement == SIM_SRF || cfg.replacement == SIM_SRF_HIST;  // SRF order (victims, visits)
  const bool hist = cfg.replacement == SIM_SRF_HIST && finiteM;  // SRF+Hist deferral (Q31)
  const int rmode = cfg.reserve, Sctx = cfg.S;
  const long long max_steps = cfg.max_steps;
  const bool kv1 = rmode == SIM_RESERVE_SEQ;  // a decode needs one KV (else its PEAK / CONTEXT reserve covers it, Q39)
  const long long row0 = p.row_off[ci], tim0 = p.tim_off[ci];
  double* tf = p.req.t_first + tim0;
  double* td = p.req.t_done + tim0;
  unsigned long long* npre = reinterpret_cast<unsigned long long*>(p.req.n_preempt + row0);
  unsigned long long* refill = reinterpret_cast<unsigned long long*>(p.req.refill_tokens + row0);
  for (int i = lane; i < n; i += 32) npre[i] = 0, refill[i] = 0;
  for (int x = lane; x < K * n; x += 32) tf[x] = 0.0, td[x] = 0.0;

  // ---- a1: per-simulation validation (Q35) and the int32 holdings bound (M infinite) ----
  {
    int bad_long = 0, bad_fit = 0;
    long long ub = 0;
    for (int i = lane; i < n; i += 32) {
      const long long pk = (long long)wl.I[i] + wl.O[i] - 1;  // peak KV usage
      bad_long |= pk > Sctx;
      bad_fit |= (finiteM && pk > M) || (!chunked && pk > C);
      bad_fit |= finiteM && rmode == SIM_RESERVE_CONTEXT && Sctx > M;
      if (!finiteM && pk <= Sctx) ub += rmode == SIM_RESERVE_CONTEXT ? max(pk, (long long)Sctx) : pk;
    }
    bad_long = __any_sync(FM, bad_long);
    bad_fit = __any_sync(FM, bad_fit);
    const bool bad_cap = !finiteM && warp_sum_ll(ub) > 0x7fffffffll;
    if (bad_long || bad_fit || bad_cap) {
      if (lane == 0) {
        sim_result_t r;
        memset(&r, 0, sizeof(r));
        r.status = bad_long ? SIM_S_TOO_LONG : (bad_fit ? SIM_S_NEVER_FITS : SIM_S_CAPACITY);
        p.results[ci] = r;
      }
      return;
    }
  }
  bool anyTheo = false;
  int Hk[SIM_MAX_COST] = {1, 1, 1, 1};  // attention head dim per model (the ceil(c/H) feature, Eq. (2))
#pragma unroll
  for (int k = 0; k < SIM_MAX_COST; k++)
    if (k < K) {
      const sim_cost_model_t* cm = p.cms + cfg.cost[k];
      anyTheo |= cm->mode == 1;
      Hk[k] = cm->H;
      if (lane == k) H.cm[k] = *cm;
    }
  {  // the per-lane Eq. (3) term table (zeros for lanes of models k >= K or linear; their divisors 1)
    const int k = lane >> 3;
    const sim_cost_model_t one{};  // (mode 0)
    lterm_fill(k < K ? p.cms[cfg.cost[k]] : one, lane & 7, H.term[lane], H.dv[k]);
  }
  __syncwarp();

  for (int i = lane; i < 18 * 18; i += 32) H.hist[i] = 0;
  bool pred_dirty = true;  // SRF+Hist: the histogram changed since the predictions were made
  __syncwarp();
  double clk = 0.0;  // lane k < K: the clock of cost model k
  int U = 0, seq = 0, next = 0, n_done = 0, nrun = 0, nW = 0;
  // the waiting group R_w as a bitmap: word w (32 slots) belongs to lane w % 32, row w / 32; per word the smallest
  // s and (PEAK reserve) the smallest initial reserve of its waiting requests (BIG if none) -- a chunk can hold an
  // admissible candidate only if these pass the step's token and KV limits
  // (GM: the words live in shared memory, g_wb / g_ws / g_wd; lane l keeps a summary of words [32 l, 32 l + 32):
  // gb = which of them hold a waiting request, gs / gd = their smallest s / reserve)
  constexpr int R = GM ? 1 : CAP / 1024;
  unsigned wm[R];
  int wmS[R], wmD[R];
#pragma unroll
  for (int r = 0; r < R; r++) wm[r] = 0u, wmS[r] = BIG, wmD[r] = BIG;
  unsigned gb = 0u;
  int gs = BIG, gd = BIG;
  if constexpr (GM) {
    for (int w = lane; w < (int)L::words; w += 32) g_wb[w] = 0u, g_ws[w] = BIG, g_wd[w] = BIG;
    __syncwarp();
  }
  // R_w gains request slot sl (s, reserve dk): one word's bit and minima (and its summary lane)
  auto wait_add = [&](int sl, int sw, int dk) {
    const int w = sl >> 5;
    if constexpr (GM) {
      if (lane == 0) g_wb[w] |= 1u << (sl & 31), g_ws[w] = min(g_ws[w], sw), g_wd[w] = min(g_wd[w], dk);
      if (lane == (w >> 5)) gb |= 1u << (w & 31), gs = min(gs, sw), gd = min(gd, dk);
    } else {
#pragma unroll
      for (int r = 0; r < R; r++)
        if (r == (w >> 5) && lane == (w & 31)) wm[r] |= 1u << (sl & 31), wmS[r] = min(wmS[r], sw), wmD[r] = min(wmD[r], dk);
    }
  };
  // decode epochs: a running decode holds rec.y = g - D, rec.z = m - D; n_rd of them, SMO = the sum of their m - D,
  // Dmin = a lower bound of their smallest completion epoch O - (g - D) (exact after every completion scan;
  // evictions and left-out decodes only raise the true minimum)
  int D = 0, n_rd = 0, Dmin = BIG;
  long long SMO = 0;
  double Tnext = wl.T[0];  // arrival time of request `next`
  long long steps = 0, preempt = 0, entries = 0, processed = 0, sumU = 0, pentries = 0, idle = 0, visits = 0, formed = 0;
  int exit_status = 0;

  auto is_dec = [&](uint8_t f) { return (f & (ST_MASK | F_FILLED)) == (ST_RUN | F_FILLED); };
  auto m_of = [&](const int4& rc, uint8_t f) { return is_dec(f) ? rc.z + D : rc.z; };  // the current m of a slot

  for (;;) {
    // ---- (1) a2: GetNewRequests (Alg. 1 line 3): all T <= clock, inclusive (Q21) ----
    int nx1 = next;
    if (next < n && Tnext <= __shfl_sync(FM, clk, 0)) {  // (offline: next == n after the first step)
      const double clk0 = __shfl_sync(FM, clk, 0);
      for (;;) {
        const int idx = nx1 + lane;
        const bool arr = idx < n && wl.T[idx] <= clk0;
        const unsigned b = __ballot_sync(FM, arr);  // T is sorted: the arrivals are a prefix
        if (arr) {
          s_rec[idx] = make_int4(wl.I[idx], 0, 0, 0);
          s_O[idx] = wl.O[idx];
          s_seq[idx] = 0;
          s_fl[idx] = ST_WAIT;
        }
        nx1 += __popc(b);
        if (b != FM) break;
      }
      if (nx1 < n) Tnext = wl.T[nx1];
      __syncwarp();
      for (int w = next >> 5; w <= (nx1 - 1) >> 5; w++) {  // the new arrivals join R_w
        const int sl = w * 32 + lane;
        const bool in = sl >= next && sl < nx1;
        const unsigned bits = __ballot_sync(FM, in);
        const int ms = (int)__reduce_min_sync(FM, in ? (unsigned)s_rec[sl].x : (unsigned)BIG);
        const int md_ = rmode == SIM_RESERVE_PEAK
                            ? (int)__reduce_min_sync(FM, in ? (unsigned)(s_rec[sl].x + s_O[sl] - 1) : (unsigned)BIG)
                            : BIG;
        if constexpr (GM) {
          if (lane == 0) g_wb[w] |= bits, g_ws[w] = min(g_ws[w], ms), g_wd[w] = min(g_wd[w], md_);
          if (lane == (w >> 5)) gb |= 1u << (w & 31), gs = min(gs, ms), gd = min(gd, md_);
        } else {
#pragma unroll
          for (int r = 0; r < R; r++)
            if (r == (w >> 5) && lane == (w & 31)) wm[r] |= bits, wmS[r] = min(wmS[r], ms), wmD[r] = min(wmD[r], md_);
        }
      }
      __syncwarp();
      nW += nx1 - next;
    }
    if (n_done == n) {
      exit_status = -1;
      break;
    }
    if (steps >= max_steps) {
      exit_status = SIM_S_MAX_STEPS;
      break;
    }
    if (seq > SEQ_LIM) {
      exit_status = SIM_S_CAPACITY;
      break;
    }
    const int nrun0 = nrun;
    const long long nP = (long long)nW + nrun;
    visits += nP;  // |P| (Alg. 1 line 9)

    // ---- (2) a3-a8: GetNextBatch (steps 2-4) ----
    int tok = 0, n_new = 0, n_pb = 0, bph = -1, n_vic = 0;
    int n_running = nrun;  // running requests (admissions in, victims out), for the SRF+Hist deferral
    long long Rs = 0;      // SRF+Hist: sum of max(O_hat(I) - g, 0) over the running requests (Q31)
    // SRF+Hist: the predictions of the current histogram and Rs over the running requests at run positions < end
    auto hist_sum = [&](int end) {
      if (pred_dirty) {
        if (lane < 18) H.pred[lane] = hist_pred_row(H.hist, lane);
        pred_dirty = false;
        __syncwarp();
      }
      unsigned long long r = 0;
      for (int q = lane; q < end; q += 32) {
        const int sl = s_run[q];
        const int4 rc = s_rec[sl];
        const int g = is_dec(s_fl[sl]) ? rc.y + D : rc.y;
        r += (unsigned)max(H.pred[bucket_of(rc.x)] - g, 0);
      }
      Rs = warp_sum_u51(r);
    };
    int a = 0;          // decodes admitted: the heads at run positions < pa1
    int pf0 = 0;        // run position of the front-most running prefill (set by run_prefills; movers lie at >= pf0)
    int pa1 = 0;        // run position of head a+1 (or the end of the list)
    int cut = nrun;     // run positions >= cut were evicted this step
    auto rnew = [&](const int4& rc, int sl) -> int {  // the reserve taken at (re)admission (Table 2, Q13, Q39)
      return rmode == SIM_RESERVE_SEQ ? rc.x + rc.y : (rmode == SIM_RESERVE_PEAK ? rc.x + s_O[sl] - 1 : Sctx);
    };

    // Candidates that never preempt (Q5), 32 per pass: ballot the lanes that fit alone, prefix-scan their tokens
    // (and KV deltas), admit those before the first cumulative failure, drop that failure, repeat; a cropped chunk
    // (chunked prefill) exhausts the token budget.  One chunk: lanes with `alive` hold a candidate; waiting = R_w
    // (its initial reserve dkv is the KV delta, Q13), else running prefills (KV delta 0: reserved >= s >= m + c).
    // Returns the lanes admitted.
    auto admit_chunk = [&](bool waiting, int sl, const int4& rc, int avail, int dkv, bool alive) -> unsigned {
      const bool scand = waiting && !kv1;  // KV deltas differ from c under PEAK / CONTEXT: scan them too
      const bool hw = hist && waiting;      // SRF+Hist deferral of a waiting candidate (Q31)
      const int rem = hw && alive ? max(H.pred[bucket_of(rc.x)] - rc.y, 0) : 0;
      const int sq = rc.x + rc.y;  // s
      bool admitted = false;
      for (;;) {
        const int rt = C - tok;
        const bool anyRun0 = n_running > 0;
        bool fit = alive && rt >= 1 && (chunked || avail <= rt) && (!finiteM || U + dkv <= M);
        if (hw) fit = fit && !(anyRun0 && (long long)U + Rs + sq + rem > M);  // deferred alone
        const unsigned fm = __ballot_sync(FM, fit);
        if (!fm) break;
        const int L = __ffs(fm) - 1;
        const int av = __shfl_sync(FM, avail, L);
        if ((fm & (fm - 1)) == 0 || av >= rt) {
          // one lane L fits alone (the contended steps), or the first fitting lane takes the whole budget left:
          // nothing can break L (no earlier lane is admitted in this round) -- it is admitted whole, or cropped to
          // the budget (chunked); then no other lane can be admitted (U, tok only grew; or no token is left),
          // which ends the pass exactly as the general round below would
          const int dk1 = __shfl_sync(FM, dkv, L);
          const int c1 = (chunked && av > rt) ? rt : av;
          if (lane == L) {
            s_c[sl] = c1;
            if (waiting) {
              s_seq[sl] = seq + 1;
              s_rec[sl] = make_int4(rc.x, rc.y, 0, dkv);
              s_fl[sl] = ST_RUN | (s_fl[sl] & F_FIRST);
              s_new[n_new] = (int16_t)sl;
            } else {
              s_fl[sl] |= F_INB_L;
              s_run2[n_pb] = (int16_t)sl;
            }
            admitted = true;
          }
          tok += c1;
          if (waiting) {
            U += dk1;  // (SEQ: the reserve is s = c; PEAK / CONTEXT: the initial reserve; cropped: the reserve too)
            seq++, n_new++, n_running++;
            if (hw) Rs += __shfl_sync(FM, rem, L);
          } else {
            n_pb++;
          }
          if (bph < 0) bph = PH_PRE;
          break;
        }
        const int cc = fit ? avail : 0, dk = fit ? dkv : 0, rr = fit ? rem : 0;
        int xc = cc, xd = dk, xr = rr;  // inclusive prefix sums over the lanes that fit alone
        {
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int yc = __shfl_up_sync(FM, xc, o);
            if (lane >= o) xc += yc;
            if (scand) {
              const int yd = __shfl_up_sync(FM, xd, o);
              if (lane >= o) xd += yd;
            }
            if (hw) {
              const int yr = __shfl_up_sync(FM, xr, o);
              if (lane >= o) xr += yr;
            }
          }
        }
        const int ec = xc - cc, ek = __popc(fm & lt), er = xr - rr;
        const int ed = waiting ? (scand ? xd - dk : ec) : 0;  // SEQ: a waiting admission reserves exactly c = s
        bool brk = false, crop = false;
        if (fit) {
          const int prt = rt - ec;
          if (chunked)
            crop = prt < avail;  // cropped (c = prt >= 1) or exhausted (prt <= 0)
          else
            brk = avail > prt;
          if (finiteM) brk |= U + ed + dkv > M;
          if (hw) brk |= (anyRun0 || ek > 0) && (long long)U + ed + Rs + er + sq + rem > M;  // deferred here
          if (crop && prt <= 0) brk = true;
        }
        const unsigned bm = __ballot_sync(FM, brk), cm = __ballot_sync(FM, crop && !brk);
        const int b = bm ? __ffs(bm) - 1 : 32, cl = cm ? __ffs(cm) - 1 : 32;
        const int stop = min(b, cl);
        const bool adm = fit && lane < stop, adc = fit && lane == cl && cl < b;
        if (adm || adc) {
          s_c[sl] = adm ? avail : rt - ec;
          if (waiting) {
            s_seq[sl] = seq + ek + 1;
            s_rec[sl] = make_int4(rc.x, rc.y, 0, dkv);
            s_fl[sl] = ST_RUN | (s_fl[sl] & F_FIRST);
            s_new[n_new + ek] = (int16_t)sl;
          } else {
            s_fl[sl] |= F_INB_L;
            s_run2[n_pb + ek] = (int16_t)sl;
          }
          alive = false;
          admitted = true;
        }
        const bool cropped = cl < b && cl < 32;
        const int nadm = __popc(fm & (stop >= 32 ? FM : ((1u << stop) - 1u)));
        const int lastl = stop > 0 ? min(stop, 32) - 1 : 0;
        const int addc = stop > 0 ? __shfl_sync(FM, xc, lastl) : 0;
        const int addd = (scand && stop > 0) ? __shfl_sync(FM, xd, lastl) : addc;
        const int addr = (hw && stop > 0) ? __shfl_sync(FM, xr, lastl) : 0;
        int cropc = 0, crops = 0, cropr = 0;
        if (cropped) {
          cropc = __shfl_sync(FM, rt - ec, cl);
          crops = __shfl_sync(FM, dkv, cl);
          if (hw) cropr = __shfl_sync(FM, rem, cl);
        }
        const int nall = nadm + (cropped ? 1 : 0);
        tok += addc + cropc;
        if (waiting) {
          U += addd + crops;
          seq += nall, n_new += nall, n_running += nall;
          Rs += addr + cropr;
        } else {
          n_pb += nall;
        }
        if (nall > 0 && bph < 0) bph = PH_PRE;
        if (cropped) break;  // the token budget is exhausted: every later candidate is rejected
        if (b < 32 && lane == b) alive = false;  // rejected (no state change)
        if (b >= 32) break;
      }
      return __ballot_sync(FM, admitted);
    };

    // the running prefills at run positions [0, b1), in retention order (decode-first: R_r^p)
    auto run_prefills = [&](int b1) {
      // [0, b1) holds n_rd decodes and b1 - n_rd running prefills (victims are cut off, completions compacted):
      // find the front-most prefill from the tail (SRF / NRF keep the prefills in progress near the tail)
      int p0 = 0;
      {
        const int need = b1 - n_rd;
        int found = 0;
        for (int top = b1 - 1; top >= 0; top -= 32) {
          const int q = top - lane;
          const bool c = q >= 0 ? (s_fl[s_run[q]] & (ST_MASK | F_PRE | F_FILLED)) == ST_RUN : false;
          const unsigned bb = __ballot_sync(FM, c);
          found += __popc(bb);
          if (found >= need) {
            if (bb) p0 = top - (31 - __clz(bb));
            break;
          }
        }
      }
      pf0 = p0;
      for (int i0 = p0; i0 < b1; i0 += 32) {
        if ((!hybrid && bph == PH_DEC) || (chunked && tok >= C)) return;  // every remaining candidate fails
        const int i = i0 + lane;
        int sl = 0;
        bool cand = false;
        if (i < b1) {
          sl = s_run[i];
          cand = (s_fl[sl] & (ST_MASK | F_PRE | F_FILLED)) == ST_RUN;
        }
        if (!__any_sync(FM, cand)) continue;
        const int4 rc = cand ? s_rec[sl] : make_int4(0, 0, 0, 0);
        admit_chunk(false, sl, rc, rc.x + rc.y - rc.z, 0, cand);
      }
    };

    // R_w in index order (Q1, Q2): only the bitmap words whose smallest s / reserve pass the current token and KV
    // limits can hold an admissible candidate (rejections change no state, so the others are skipped whole)
    auto kv_pass = [&](int ms, int md_, int capM) {  // a word (or group) can hold a candidate passing the KV test
      return rmode == SIM_RESERVE_SEQ ? ms <= capM : (rmode == SIM_RESERVE_PEAK ? md_ <= capM : Sctx <= capM);
    };
    // one bitmap word w (32 slots, `word` = its waiting bits): admit its candidates; returns the bits left waiting
    // and their minima
    auto wait_word = [&](int w, unsigned word, int& ms, int& md_) -> unsigned {
      const int sl = w * 32 + lane;
      const bool isw = (word >> lane) & 1u;
      const int4 rc = isw ? s_rec[sl] : make_int4(0, 0, 0, 0);
      const int sw = rc.x + rc.y, dkv = isw ? rnew(rc, sl) : 0;  // avail = s (m = 0)
      const unsigned admm = admit_chunk(true, sl, rc, sw, dkv, isw);
      const unsigned left = word & ~admm;
      const bool lw = (left >> lane) & 1u;
      ms = (int)__reduce_min_sync(FM, lw ? (unsigned)sw : (unsigned)BIG);
      md_ = rmode == SIM_RESERVE_PEAK ? (int)__reduce_min_sync(FM, lw ? (unsigned)dkv : (unsigned)BIG) : BIG;
      return left;
    };
    auto wait_scan = [&]() {
      if constexpr (GM) {  // two levels: summary lanes, then the 32 words of the first passing lane
        int curL = 0, curW = 0;  // next word to visit: 32 curL + curW
        for (;;) {
          if ((!hybrid && bph == PH_DEC) || (chunked && tok >= C)) return;
          const int capT = chunked ? BIG : C - tok, capM = finiteM ? M - U : BIG;
          const unsigned lb = __ballot_sync(FM, lane >= curL && gb != 0u && gs <= capT && kv_pass(gs, gd, capM));
          if (!lb) return;
          const int Lg = __ffs(lb) - 1;
          const int wj = 32 * Lg + lane;
          const unsigned bj = g_wb[wj];
          const int sj = g_ws[wj], dj = g_wd[wj];
          const unsigned wbm = __ballot_sync(FM, bj != 0u && sj <= capT && kv_pass(sj, dj, capM) && (Lg > curL || lane >= curW));
          if (!wbm) {
            curL = Lg + 1, curW = 0;
            continue;
          }
          const int Wj = __ffs(wbm) - 1, w = 32 * Lg + Wj;
          const unsigned word = __shfl_sync(FM, bj, Wj);
          int ms, md_;
          const unsigned left = wait_word(w, word, ms, md_);
          if (left != word) {  // admissions: the word and its group's summary change
            __syncwarp();  // (every lane has read the words of this group)
            if (lane == 0) g_wb[w] = left, g_ws[w] = ms, g_wd[w] = md_;
            __syncwarp();
            const unsigned b2 = g_wb[wj];
            const int s2 = g_ws[wj], d2 = g_wd[wj];
            const unsigned nb = __ballot_sync(FM, b2 != 0u);
            const int gs2 = (int)__reduce_min_sync(FM, (unsigned)s2), gd2 = (int)__reduce_min_sync(FM, (unsigned)d2);
            if (lane == Lg) gb = nb, gs = gs2, gd = gd2;
          }
          curL = Lg, curW = Wj + 1;
          if (curW == 32) curL++, curW = 0;
          if (chunked && tok >= C) return;
        }
      } else {
#pragma unroll
      for (int r = 0; r < R; r++) {
        int cur = 0;
        for (;;) {
          if ((!hybrid && bph == PH_DEC) || (chunked && tok >= C)) return;  // every remaining candidate fails
          const int capT = chunked ? BIG : C - tok, capM = finiteM ? M - U : BIG;
          const unsigned cb = __ballot_sync(FM, lane >= cur && wm[r] != 0u && wmS[r] <= capT && kv_pass(wmS[r], wmD[r], capM));
          if (!cb) break;
          const int Lc = __ffs(cb) - 1;
          cur = Lc + 1;
          const unsigned word = __shfl_sync(FM, wm[r], Lc);
          int ms, md_;
          const unsigned left = wait_word(r * 32 + Lc, word, ms, md_);
          if (lane == Lc) wm[r] = left, wmS[r] = ms, wmD[r] = md_;
        }
      }
      }
    };

    // the run position of the cnt-th decode (1-based) of the run list, or nrun
    auto nth_head = [&](int cnt) -> int {
      for (int q0 = 0; q0 < nrun; q0 += 32) {
        const int q = q0 + lane;
        const unsigned hb = __ballot_sync(FM, q < nrun && is_dec(s_fl[s_run[q < nrun ? q : 0]]));
        const int h = __popc(hb);
        if (h >= cnt) return q0 + (int)__fns(hb, 0, cnt);
        cnt -= h;
      }
      return nrun;
    };

    // The running decodes in closed form (see the file header); the victim pool is the run list's tail.
    auto decode_group = [&]() {
      const bool fM = finiteM && kv1;  // heads need one KV each (else none: admitted up to the token budget)
      const int F = fM ? M - U : BIG;
      const int T = C - tok;
      const int k = n_rd;
      int qs = nrun;
      if (F >= k && T >= k) {  // every head passes both tests: nothing is evicted
        a = k, pa1 = nrun;
      } else if (F >= k) {  // only the token budget binds (Q11: no preemption): heads 1..T
        a = T;
        pa1 = pfirst ? T : nth_head(T + 1);  // prefill-first: every running request is a decode
      } else {
        // one-victim fast path (the thrash steps): the last two run entries are decodes (heads k-1, k at positions
        // nrun-2, nrun-1) and head k-1 passes (k-1 <= T, F + held(tail) >= k-1): a = k-1, head k fails (F < k, or
        // k > T), and the minimal suffix is the tail alone (or empty if F >= a and the token budget stopped head k)
        // (Sarathi: a running prefill at the tail -- the chunk in progress, smallest m -- and head k before it: if
        // k <= T and F + held(tail) >= k, every head passes, a = k, and the minimal suffix is the tail alone)
        bool fast = false;
        if (nrun >= 2) {
          const int st = s_run[nrun - 1], s2 = s_run[nrun - 2];
          const uint8_t ft = s_fl[st];
          if (is_dec(s_fl[s2])) {
            const int4 rt = s_rec[st];
            if (is_dec(ft)) {
              if (k - 1 <= T && F + max(rt.w, rt.z + D) >= k - 1) {
                a = k - 1;
                pa1 = nrun - 1;
                qs = (k <= T || F < a) ? nrun - 1 : nrun;  // (k <= T: head k stopped by the KV, self-preempts, Q8)
                fast = true;
              }
            } else if (k <= T && F + max(rt.w, rt.z) >= k) {
              a = k;
              pa1 = nrun;
              qs = nrun - 1;  // (F < k = a: the suffix is not empty)
              fast = true;
            }
          }
        }
        if (!fast) {
          // walk from the tail: lane j <-> run position top - j; RSx = the holdings behind the chunk, HSi = its heads
          // behind it; head i (i = k - #heads behind p_i) passes iff i <= T and F + RS(p_i + 1) >= i
          int RSx = 0, HSi = 0, lastfail = nrun;
          bool lastfail_t = false, found = false, kvstop = false;
          a = 0;
          for (int top = nrun - 1; top >= 0; top -= 32) {
            const int q = top - lane;
            int held = 0, head = 0;
            if (q >= 0) {
              const int sl = s_run[q];
              const int4 rc = s_rec[sl];
              head = is_dec(s_fl[sl]) ? 1 : 0;
              held = max(rc.w, head ? rc.z + D : rc.z);
            }
            int xs = held, xh = head;
  #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int ys = __shfl_up_sync(FM, xs, o), yh = __shfl_up_sync(FM, xh, o);
              if (lane >= o) xs += ys, xh += yh;
            }
            const int rsx = RSx + xs - held, i = k - (HSi + xh) + 1;
            const bool tfail = i > T, kfail = F + rsx < i;
            const unsigned hb = __ballot_sync(FM, head);
            const unsigned pb = __ballot_sync(FM, head && !tfail && !kfail);
            if (pb) {  // the tail-most passing head is head a; head a+1 is the nearest failing head behind it
              const int La = __ffs(pb) - 1;
              a = __shfl_sync(FM, i, La);
              const unsigned behind = hb & ((1u << La) - 1u);
              if (behind) {
                const int Lf = 31 - __clz(behind);
                pa1 = top - Lf;
                kvstop = __shfl_sync(FM, (int)tfail, Lf) == 0;
              } else {
                pa1 = lastfail;
                kvstop = lastfail < nrun && !lastfail_t;
              }
              if (top == nrun - 1 && F < a) {  // q* from the same registers: the tail-most q with F + RS(q) >= a
                const unsigned qb = __ballot_sync(FM, q >= 0 && F + RSx + xs >= a);
                if (qb) qs = top - (__ffs(qb) - 1);
              }
              found = true;
              break;
            }
            if (hb) {  // every head of this chunk fails; its front-most one has the lowest rank so far
              const int Lf = 31 - __clz(hb);
              lastfail = top - Lf;
              lastfail_t = __shfl_sync(FM, (int)tfail, Lf) != 0;
            }
            RSx += __shfl_sync(FM, xs, 31);
            HSi += __shfl_sync(FM, xh, 31);
          }
          if (!found) {  // even head 1 fails
            a = 0;
            pa1 = lastfail;
            kvstop = lastfail < nrun && !lastfail_t;
          }
          if (F < a && qs == nrun) {  // q* = the tail-most q with F + RS(q) >= a (walk the tail again)
            int rs = 0;
            for (int top = nrun - 1; top >= 0; top -= 32) {
              const int q = top - lane;
              int held = 0;
              if (q >= 0) {
                const int sl = s_run[q];
                const int4 rc = s_rec[sl];
                held = max(rc.w, is_dec(s_fl[sl]) ? rc.z + D : rc.z);
              }
              int xs = held;
  #pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const int ys = __shfl_up_sync(FM, xs, o);
                if (lane >= o) xs += ys;
              }
              const unsigned qb = __ballot_sync(FM, q >= 0 && F + rs + xs >= a);
              if (qb) {
                qs = top - (__ffs(qb) - 1);
                break;
              }
              rs += __shfl_sync(FM, xs, 31);
            }
          }
          // if the KV stopped the walk at head a+1 and it lies before q*, it evicts everything behind it and
          // self-preempts (Q8): the suffix starts at pa1
          if (kvstop && pa1 < qs) qs = pa1;
        }
      }
      // apply: evict run positions [qs, nrun) (refill semantics P:1570)
      int fr = 0, evd = 0;
      unsigned mev = 0;  // sum of the evicted decodes' m
      for (int q = qs + lane; q < nrun; q += 32) {
        const int sl = s_run[q];
        const int4 rc = s_rec[sl];
        const uint8_t f = s_fl[sl];
        const bool dec = is_dec(f);
        const int m = dec ? rc.z + D : rc.z, g = dec ? rc.y + D : rc.y;
        fr += max(rc.w, m);
        if (dec) {
          evd++;
          mev += m;
        }
        atomicAdd(&npre[sl], 1ull);
        atomicAdd(&refill[sl], (unsigned long long)m);
        s_rec[sl] = make_int4(rc.x, g, 0, 0);
        s_fl[sl] = ST_WAIT | F_PRE | (f & F_FIRST);
        s_vic[q - qs] = (int16_t)sl;
      }
      if (qs < nrun) {
        fr = (int)__reduce_add_sync(FM, (unsigned)fr);
        evd = (int)__reduce_add_sync(FM, (unsigned)evd);
        mev = __reduce_add_sync(FM, mev);
      }
      n_vic = nrun - qs;
      n_rd -= evd;
      SMO -= (long long)mev - (long long)evd * D;
      cut = qs;
      if (pa1 > qs) pa1 = qs;
      tok += a;
      U += (kv1 ? a : 0) - fr;
      if (a > 0 && bph < 0) bph = PH_DEC;
    };

    if (pfirst) {  // vLLM {R_w, R_r}: every running request is a decode (no chunking)
      if (nW > 0) {
        if (hist) hist_sum(nrun);
        wait_scan();
      }
      if (n_rd > 0 && (hybrid || bph != PH_PRE)) decode_group();  // else every decode fails step 2
    } else {  // Sarathi {R_r^d, R_r^p, R_w}
      if (n_rd > 0) decode_group();
      if (cut > n_rd) run_prefills(cut);  // running prefills survive (the run list holds cut entries)
      if (nW > 0) {
        n_running = cut;  // (this step's victims are waiting)
        if (hist) hist_sum(cut);
        wait_scan();
      }
    }
    __syncwarp();

    if (tok == 0) {  // B = {}: idle jump to the next arrival, not a step (Q21)
      if (n_vic == 0 && nx1 < n) {
        if (lane == 0) clk = fmax(clk, wl.T[nx1]);
        idle++;
        next = nx1;
        continue;
      }
      exit_status = SIM_S_DEADLOCK;
      break;
    }

    // ---- (3) a9 + a10: the admitted decodes advance by one epoch; Process the prefill entries explicitly ----
    // the decodes of B: the a heads before pa1, n_d = a, sum m = sum(m - D) + a D over them (Table 3 features)
    long long smo_out = 0;  // sum of m - D over the decodes left out of B (positions [pa1, cut): token budget)
    if (a > 0 && cut > pa1) {  // they do not advance: offsets lowered by one
      unsigned so = 0, cnt = 0;
      for (int q = pa1 + lane; q < cut; q += 32) {
        const int sl = s_run[q];
        if (!is_dec(s_fl[sl])) continue;
        const int4 rc = s_rec[sl];
        so += rc.z + D, cnt++;  // (its m)
        s_rec[sl] = make_int4(rc.x, rc.y - 1, rc.z - 1, rc.w);
      }
      smo_out = (long long)__reduce_add_sync(FM, so) - (long long)__reduce_add_sync(FM, cnt) * D;
    }
    const int nd = a;
    const long long md = a > 0 ? (SMO - smo_out) + (long long)a * D : 0;
    if (a > 0) {
      SMO -= n_rd - a;  // the left-out decodes' offsets were lowered by one
      D++;
    }
    unsigned N = 0, np_ = 0, cp = 0, mp = 0, freed = 0, ndone = 0, nfa = 0;
    int n_ev = 0, dm_new = BIG;
    bool moved = false;  // SRF: some retention key changed relative to the others (movers to merge back)
    long long c2 = 0, mc = 0, pcm = 0, pce[SIM_MAX_COST] = {0, 0, 0, 0};
    unsigned m_new = 0;  // sum of m over the new decodes
    // SRF: a running prefill left out of B but before pa1 is overtaken by the decodes after it (m + 1): it moves
    // too (the block kernel re-sorts whenever nd != |R_r|)
    if (srf && !pfirst && a > 0 && pa1 > a && n_pb < cut - n_rd) {  // (some running prefill is not in B)
      bool mv = false;
      for (int q = pf0 + lane; q < pa1; q += 32) {
        const int sl = s_run[q];
        const uint8_t f = s_fl[sl];
        if ((f & (ST_MASK | F_FILLED | F_INB_L)) == ST_RUN) s_fl[sl] = f | F_MOVE_L, mv = true;
      }
      moved |= __any_sync(FM, mv);
    }
    // the prefill entries: this batch's running prefills (s_run2) then its admissions (s_new), one index space
    {
      const int len = n_pb + n_new;
      for (int e0 = 0; e0 < len; e0 += 32) {
        const int e = e0 + lane;
        const bool sg0 = e < n_pb;  // a running prefill (its retention key moves under SRF)
        unsigned evc = 0;
        int sl = 0;
        if (e < len) {
          sl = sg0 ? s_run2[e] : s_new[e - n_pb];
          uint8_t fl = s_fl[sl];
          const int4 rc = s_rec[sl];
          const int O = s_O[sl];
          const int c = s_c[sl], m0 = rc.z, s = rc.x + rc.y, m = m0 + c;
          int g = rc.y;
          N += c;
          np_++;
          cp += c;
          mp += m0;
          c2 += (long long)c * c;
          mc += (long long)m0 * c;
          if (anyTheo) {
            pcm += (long long)c * (c + m0);
#pragma unroll
            for (int k = 0; k < SIM_MAX_COST; k++)
              if (k < K) pce[k] += (long long)((c + Hk[k] - 1) / Hk[k]) * (c + m0);
          }
          fl &= ~F_INB_L;
          int4 out = make_int4(rc.x, g, m, rc.w);
          if (c == s - m0) {  // Eq. (6): all available tokens processed -> one token (Q18)
            g++;
            fl |= F_FILLED;
            if (!(fl & F_FIRST)) fl |= F_FIRST, evc |= 1;
            if (g == O) {
              fl = (fl & ~ST_MASK) | ST_DONE;
              evc |= 2;
              freed += max(rc.w, m);
              ndone++;
              out = make_int4(rc.x, g, m, rc.w);
              if (hist) atomicAdd(&H.hist[bucket_of(rc.x) * 18 + bucket_of(O)], 1);
            } else {  // the (re)fill completed: a running decode from now on, in epoch form
              nfa++;
              out = make_int4(rc.x, g - D, m - D, rc.w);
              m_new += m;
              dm_new = min(dm_new, O - (g - D));
              if (srf && sg0) fl |= F_MOVE_L, moved = true;
            }
          } else if (srf && sg0) {
            fl |= F_MOVE_L, moved = true;  // a chunk: its key moved (the admissions are merged anyway)
          }
          s_rec[sl] = out;
          s_fl[sl] = fl;
        }
        const unsigned eb = __ballot_sync(FM, evc != 0);
        if (evc) s_ev[n_ev + __popc(eb & lt)] = sl | (int)(evc << 16);
        n_ev += __popc(eb);
      }
    }
    if (n_pb + n_new > 0) {  // (a step of decodes only has nothing to reduce here)
      nfa = __reduce_add_sync(FM, nfa);
      N = __reduce_add_sync(FM, N);
      np_ = __reduce_add_sync(FM, np_), cp = __reduce_add_sync(FM, cp), mp = __reduce_add_sync(FM, mp);
      freed = __reduce_add_sync(FM, freed), ndone = __reduce_add_sync(FM, ndone);
    }
    N += (unsigned)a;
    moved = __any_sync(FM, moved);
    if (np_ > 0) {
      // (c, m < S < 2^18, at most CAP / 32 = 128 entries per lane: every per-lane sum is below 2^44)
      c2 = warp_sum_u51(c2);
      mc = warp_sum_u51(mc);
      if (anyTheo) {
        pcm = warp_sum_u51(pcm);
#pragma unroll
        for (int k = 0; k < SIM_MAX_COST; k++) pce[k] = warp_sum_u51(pce[k]);
      }
    }
    // decode completions: the admitted decodes reaching g = O at this epoch (completion epoch O - (g - D) == D);
    // the new decodes of this step are not in the run list yet and complete later (their epoch > D)
    if (a > 0 && Dmin <= D) {
      int dm = BIG, nd2 = 0, fr2 = 0;
      unsigned so = 0;
      for (int q0 = 0; q0 < cut; q0 += 32) {
        const int q = q0 + lane;
        unsigned evc = 0;
        int sl = 0;
        if (q < cut) {
          sl = s_run[q];
          const uint8_t f = s_fl[sl];
          if (is_dec(f) && !(f & F_INB_L)) {
            const int4 rc = s_rec[sl];
            const int O = s_O[sl], ce = O - rc.y;
            if (ce == D) {
              s_fl[sl] = (f & ~ST_MASK) | ST_DONE;
              s_rec[sl] = make_int4(rc.x, O, rc.z + D, rc.w);
              fr2 += max(rc.w, rc.z + D);
              so += rc.z + D;
              nd2++;
              evc = 2;
              if (hist) atomicAdd(&H.hist[bucket_of(rc.x) * 18 + bucket_of(O)], 1);
            } else {
              dm = min(dm, ce);
            }
          }
        }
        const unsigned eb = __ballot_sync(FM, evc != 0);
        if (evc) s_ev[n_ev + __popc(eb & lt)] = sl | (int)(evc << 16);
        n_ev += __popc(eb);
      }
      const int ndd = (int)__reduce_add_sync(FM, (unsigned)nd2);
      freed += (unsigned)__reduce_add_sync(FM, (unsigned)fr2);
      SMO -= (long long)__reduce_add_sync(FM, so) - (long long)ndd * D;
      Dmin = (int)__reduce_min_sync(FM, (unsigned)dm);  // exact (the run-list prefills turned decodes are in it)
      n_rd -= ndd;
      ndone += ndd;
    }
    // the new decodes join the epoch sums
    if (nfa > 0) {
      SMO += (long long)__reduce_add_sync(FM, m_new) - (long long)nfa * D;
      Dmin = min(Dmin, (int)__reduce_min_sync(FM, (unsigned)dm_new));
      n_rd += (int)nfa;
    }
    // a9: lane k < K charges cost model k; clock += d_j (one fp64 add, Q36)
    {
      Feat f;
      f.N = N, f.np = np_, f.cp = cp, f.mp = mp, f.nd = nd, f.md = md, f.c2 = c2, f.mc = mc, f.pcm = pcm;
#pragma unroll
      for (int k = 0; k < SIM_MAX_COST; k++) f.pceil[k] = pce[k];
      const double d = batch_time_lanes(H.cm, H.term, H.dv, K, f, anyTheo);  // lane-parallel Eq. (3) terms (same bits)
      if (lane < K) clk = dadd(clk, d);
    }
    steps++;
    formed++;
    sumU += U;
    entries += np_ + nd;
    processed += N;
    pentries += np_;
    n_done += (int)ndone;
    preempt += n_vic;
    U -= (int)freed;

    // event times (first token, completion) under every cost model
    if (n_ev > 0) {
      const double c0 = __shfl_sync(FM, clk, 0), c1 = __shfl_sync(FM, clk, 1), c2_ = __shfl_sync(FM, clk, 2),
                   c3 = __shfl_sync(FM, clk, 3);
      __syncwarp();
      for (int e = lane; e < n_ev; e += 32) {
        const int code = s_ev[e], sl = code & 0xffff;
        double* dst[2] = {tf + sl, td + sl};
#pragma unroll
        for (int w = 0; w < 2; w++)
          if (code & ((1 << w) << 16)) {
            dst[w][0] = c0;
            if (K > 1) dst[w][n] = c1;
            if (K > 2) dst[w][2 * (long long)n] = c2_;
            if (K > 3) dst[w][3 * (long long)n] = c3;
          }
      }
    }
    // this step's victims wait from the next step on: clear Q9's mark; R_w gains them (exact count; the smallest
    // s stays a lower bound after admissions, recounted every 32 admission steps)
    for (int v = 0; v < n_vic; v++) {
      const int sl = s_vic[v];
      const int4 rc = s_rec[sl];
      wait_add(sl, rc.x + rc.y, rmode == SIM_RESERVE_PEAK ? rc.x + s_O[sl] - 1 : BIG);
      if (lane == 0) s_fl[sl] &= ~F_PRE;
    }
    nW = nW - n_new + n_vic;
    __syncwarp();

    // ---- (4) steady decode run: step j had only decodes and no admission, preemption or completion; step j+1
    // repeats it exactly (waiting rejections persist: KV is monotone in U, tokens and phases unchanged) until the
    // next completion epoch, the KV limit (U + k nd <= M) or an arrival.  After an eviction step the same holds
    // when every running request was a decode of B and every waiting candidate fails the KV test already.
    {
      bool steady = ndone == 0 && np_ == 0 && nd > 0;
      if (steady && n_vic > 0) {
        int ms = GM ? gs : BIG;
#pragma unroll
        for (int r = 0; r < R; r++) ms = min(ms, wmS[r]);
        ms = (int)__reduce_min_sync(FM, (unsigned)ms);  // the smallest s in R_w
        steady = nd == nrun0 - n_vic && (nW == 0 || (finiteM && (long long)U + ms > M));
      }
      long long Lr = 0;
      if (steady) {
        Lr = (long long)Dmin - D;  // steps until the next completion epoch (at most: Dmin is a lower bound)
        if (finiteM && kv1) Lr = min(Lr, (long long)(M - U) / (long long)nd);
        Lr = min(Lr, max_steps - steps);
      }
      if (Lr > 0) {
        const long long ndl = nd, MD = md + ndl, Ur = U, du = kv1 ? ndl : 0;  // KV growth per run step
        constexpr int DB = 32;
        long long E = 0;
        while (E < Lr) {
          const int chunk = (int)min((long long)DB, Lr - E);
          // lane t: the batch times of run step E + t + 1 under every model (affine features)
          if (lane < chunk) {
            Feat f;
            f.N = ndl, f.np = 0, f.c2 = 0, f.mc = 0, f.cp = 0, f.mp = 0, f.pcm = 0, f.nd = ndl;
            f.md = MD + (E + lane) * ndl;
            for (int k = 0; k < SIM_MAX_COST; k++) f.pceil[k] = 0;
            for (int k = 0; k < K; k++) s_dbuf[k * DB + lane] = batch_time_tab(H.cm[k], H.term + 8 * k, H.dv[k], f, k);
          }
          __syncwarp();
          int ex = chunk;
          if (lane < K) {  // the clock chain stays sequential: one fp64 add per step (Q36)
            const double* db = s_dbuf + lane * DB;
            if (nx1 < n) {  // online (K == 1): stop before a step that would start at/after an arrival (Q21)
              for (int t = 0; t < chunk; t++) {
                if (Tnext <= clk) {
                  ex = t;
                  break;
                }
                clk = dadd(clk, db[t]);
              }
            } else {
              int t = 0;
              for (; t + 8 <= chunk; t += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; u++) v[u] = db[t + u];
#pragma unroll
                for (int u = 0; u < 8; u++) clk = dadd(clk, v[u]);
              }
              for (; t < chunk; t++) clk = dadd(clk, db[t]);
            }
          }
          ex = __shfl_sync(FM, ex, 0);
          __syncwarp();
          E += ex;
          if (ex < chunk) break;
        }
        if (E > 0) {
          const int nout = n_rd - nd;  // decodes left out of B (token budget) do not advance during the run
          if (nout > 0) {
            for (int q = pa1 + lane; q < cut; q += 32) {
              const int sl = s_run[q];
              if (!is_dec(s_fl[sl])) continue;
              const int4 rc = s_rec[sl];
              s_rec[sl] = make_int4(rc.x, rc.y - (int)E, rc.z - (int)E, rc.w);
            }
            SMO -= (long long)nout * E;
          }
          D += (int)E;
          steps += E;
          sumU += E * Ur + du * (E * (E + 1) / 2);
          entries += E * ndl;
          processed += E * ndl;
          visits += E * nP;
          U = (int)(Ur + E * du);
          if (Dmin <= D) {  // completions at the run's last step (their time: the clocks after the run)
            const double c0 = __shfl_sync(FM, clk, 0), c1 = __shfl_sync(FM, clk, 1), c2_ = __shfl_sync(FM, clk, 2),
                         c3 = __shfl_sync(FM, clk, 3);
            int dm = BIG, nd2 = 0, fr2 = 0;
            unsigned so = 0;
            for (int q = lane; q < cut; q += 32) {
              const int sl = s_run[q];
              const uint8_t f = s_fl[sl];
              if (!is_dec(f)) continue;
              const int4 rc = s_rec[sl];
              const int O = s_O[sl], ce = O - rc.y;
              if (ce == D) {
                s_fl[sl] = (f & ~ST_MASK) | ST_DONE;
                s_rec[sl] = make_int4(rc.x, O, rc.z + D, rc.w);
                fr2 += max(rc.w, rc.z + D);
                so += rc.z + D;
                nd2++;
                if (hist) atomicAdd(&H.hist[bucket_of(rc.x) * 18 + bucket_of(O)], 1);
                td[sl] = c0;
                if (K > 1) td[n + sl] = c1;
                if (K > 2) td[2 * (long long)n + sl] = c2_;
                if (K > 3) td[3 * (long long)n + sl] = c3;
              } else {
                dm = min(dm, ce);
              }
            }
            nd2 = (int)__reduce_add_sync(FM, (unsigned)nd2);
            U -= (int)__reduce_add_sync(FM, (unsigned)fr2);
            SMO -= (long long)__reduce_add_sync(FM, so) - (long long)nd2 * D;
            Dmin = (int)__reduce_min_sync(FM, (unsigned)dm);
            n_rd -= nd2;
            n_done += nd2;
            ndone += nd2;
          }
        }
      }
    }

    if (hist && ndone > 0) pred_dirty = true;  // (warp-uniform: the histogram gained this step's completions)
    // ---- (5) the run list for the next step (retention order) ----
    {
      int cnt = cut;  // the evicted suffix is cut off
      int nmov = 0;   // SRF: entries whose keys moved, taken out into s_vic
      auto key_of = [&](int sl) { return srf_key<SLB>(m_of(s_rec[sl], s_fl[sl]), s_seq[sl], sl); };
      if (moved && ndone == 0) {
        // the moved entries often stay in order (a chunk leaves a prefill behind the decodes): if each one is in
        // order with both neighbours, the list is sorted (the others kept their relative order) and stays as is
        bool ok = true;
        for (int q0 = pf0; q0 < cnt; q0 += 32) {  // (every mover is a running prefill: at >= pf0)
          const int q = q0 + lane;
          if (q < cnt) {
            const int sl = s_run[q];
            if (s_fl[sl] & F_MOVE_L) {
              const unsigned long long k = key_of(sl);
              if (q > 0 && key_of(s_run[q - 1]) >= k) ok = false;
              if (q + 1 < cnt && key_of(s_run[q + 1]) <= k) ok = false;
            }
          }
        }
        if (__all_sync(FM, ok)) {
          for (int q = pf0 + lane; q < cnt; q += 32) s_fl[s_run[q]] &= ~F_MOVE_L;
          moved = false;
          __syncwarp();
        }
      }
      if (ndone > 0 || moved) {  // stable in-place compaction: drop completions (and take out the SRF movers)
        __syncwarp();  // (the completion scans read s_run)
        const int c0 = ndone > 0 ? 0 : pf0;  // without completions the entries before the first mover stay
        int w = c0;
        for (int q0 = c0; q0 < cnt; q0 += 32) {
          const int q = q0 + lane;
          int sl = 0;
          uint8_t f = 0;
          if (q < cnt) {
            sl = s_run[q];
            f = s_fl[sl];
          }
          const bool live = q < cnt && (f & ST_MASK) == ST_RUN;
          const bool mov = live && (f & F_MOVE_L);
          const unsigned km = __ballot_sync(FM, live && !mov), mm = __ballot_sync(FM, mov);
          if (live && !mov) s_run[w + __popc(km & lt)] = (int16_t)sl;
          if (mov) {
            s_vic[nmov + __popc(mm & lt)] = (int16_t)sl;
            s_fl[sl] = f & ~F_MOVE_L;
          }
          w += __popc(km);
          nmov += __popc(mm);
        }
        cnt = w;
      }
      // this step's admissions that stay running: appended in admission order (NRF / PF retention = admission
      // order, Q6, Q39), or SRF movers
      for (int e0 = 0; e0 < n_new; e0 += 32) {
        const int e = e0 + lane;
        const int sl = e < n_new ? s_new[e] : 0;
        const bool live = e < n_new && (s_fl[sl] & ST_MASK) == ST_RUN;
        const unsigned km = __ballot_sync(FM, live);
        if (live) {
          if (srf)
            s_vic[nmov + __popc(km & lt)] = (int16_t)sl;
          else
            s_run[cnt + __popc(km & lt)] = (int16_t)sl;
        }
        if (srf)
          nmov += __popc(km);
        else
          cnt += __popc(km);
      }
      __syncwarp();
      if (nmov > 0) {  // SRF: merge the movers back into the (still sorted) kept list by (m desc, seq)
        // The movers are sorted on their own (in lanes when <= 32, else bitonic in s_key), each finds its insertion
        // point ins_t = #{kept j : key_j < key_t} by binary search, and the kept list is shifted in place range by
        // range from its end (range t = [ins_t, ins_t+1) moves by t + 1): O(nmov log nmov + entries moved / 32),
        // never a sort of the whole list.
        const int nk = cnt;
        const bool small = nmov <= 32;
        unsigned long long mk = ~0ull;  // small: lane t holds mover t's key (sorted)
        int ins = nk;                   // small: lane t holds ins_t
        bool append;
        const unsigned long long tail = nk > 0 ? key_of(s_run[nk - 1]) : 0ull;
        if (small) {
          if (lane < nmov) mk = key_of(s_vic[lane]);
          if (nmov > 1) {  // bitonic sort of the first 2^ceil(log2 nmov) lanes' keys (the rest hold ~0)
            const int P2 = 1 << (32 - __clz(nmov - 1));
            for (int k2 = 2; k2 <= P2; k2 <<= 1) {
              for (int j = k2 >> 1; j > 0; j >>= 1) {
                const unsigned long long o = __shfl_xor_sync(FM, mk, j);
                const bool up = (lane & k2) == 0, lower = (lane & j) == 0;
                mk = (lower == up) ? (mk < o ? mk : o) : (mk > o ? mk : o);
              }
            }
          }
          append = nk == 0 || __shfl_sync(FM, mk, 0) > tail;
          if (append) {
            if (lane < nmov) s_run[nk + lane] = (int16_t)(mk & (CAP - 1));
          } else if (lane < nmov) {
            int lo2 = 0, hi2 = nk;
            while (lo2 < hi2) {
              const int mid = (lo2 + hi2) >> 1;
              if (key_of(s_run[mid]) < mk)
                lo2 = mid + 1;
              else
                hi2 = mid;
            }
            ins = lo2;
          }
        } else {
          for (int t = lane; t < nmov; t += 32) s_key[t] = key_of(s_vic[t]);
          int P2 = 1;
          while (P2 < nmov) P2 <<= 1;
          for (int t = nmov + lane; t < P2; t += 32) s_key[t] = ~0ull;
          __syncwarp();
          for (int k2 = 2; k2 <= P2; k2 <<= 1) {
            for (int j = k2 >> 1; j > 0; j >>= 1) {
              for (int i = lane; i < P2; i += 32) {
                const int ixj = i ^ j;
                if (ixj > i) {
                  const unsigned long long x = s_key[i], y = s_key[ixj];
                  if ((x > y) == ((i & k2) == 0)) s_key[i] = y, s_key[ixj] = x;
                }
              }
              __syncwarp();
            }
          }
          append = nk == 0 || s_key[0] > tail;
          for (int t = lane; t < nmov; t += 32) {
            const unsigned long long kt = s_key[t];
            if (append) {
              s_run[nk + t] = (int16_t)(kt & (CAP - 1));
            } else {
              int lo2 = 0, hi2 = nk;
              while (lo2 < hi2) {
                const int mid = (lo2 + hi2) >> 1;
                if (key_of(s_run[mid]) < kt)
                  lo2 = mid + 1;
                else
                  hi2 = mid;
              }
              s_vic[t] = (int16_t)(kt & (CAP - 1));  // mover t in key order
              s_run2[t] = (int16_t)lo2;              // its insertion point
            }
          }
        }
        __syncwarp();
        if (!append) {
          int hi = nk;
          for (int t = nmov - 1; t >= 0; t--) {  // range t = [ins_t, hi) moves up by t + 1 (from its top down)
            const int lo = small ? __shfl_sync(FM, ins, t) : (int)s_run2[t];
            for (int top = hi; top > lo; top -= 32) {
              const int q = top - 1 - lane;
              const bool ok = q >= lo;
              const int16_t v = ok ? s_run[q] : (int16_t)0;
              __syncwarp();
              if (ok) s_run[q + t + 1] = v;
              __syncwarp();
            }
            hi = lo;
          }
          if (small) {
            if (lane < nmov) s_run[ins + lane] = (int16_t)(mk & (CAP - 1));
          } else {
            for (int t = lane; t < nmov; t += 32) s_run[s_run2[t] + t] = s_vic[t];
          }
          __syncwarp();
        }
        cnt = nk + nmov;
      }
      nrun = cnt;
      next = nx1;
      __syncwarp();
    }
  }

  // ---- a11: metrics ----
  const int st = exit_status == -1 ? SIM_S_OK : exit_status;
  __syncwarp();
  if (st != SIM_S_OK) {  // failed simulations: zero-filled rows
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
  if (lane < K) {  // sequential sums in request order (identical to the oracle)
    const int k = lane;
    double mx = 0.0, sl = 0.0, st1 = 0.0, stp = 0.0;
    long long ntp = 0;
    const double* tfk = tf + (long long)k * n;
    const double* tdk = td + (long long)k * n;
    for (int i = 0; i < n; i++) {
      const double a = tfk[i], b = tdk[i], T = wl.T[i];
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
    r.preemptions = preempt;
    r.batch_entries = entries;
    r.processed_tokens = processed;
    r.sum_U = sumU;
    r.prefill_entries = pentries;
    r.idle_jumps = idle;
    r.visits = visits;
    r.formed_steps = formed;
    for (int k = K; k < SIM_MAX_COST; k++) r.makespan[k] = r.mean_latency[k] = r.mean_ttft[k] = r.mean_tpot[k] = 0.0;
  }
}

}  // namespace simsweep
