// simsweep.cu -- libsimsweep.so: CTA-per-simulation step kernel (sm_100a) and
// the C-ABI of include/simsweep.h.  See sim_kernel.cuh for the per-step plan.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "sim_kernel.cuh"
#include "simsweep.h"

namespace simsweep {

enum { K_NONE = 0, K_MARK = 1, K_EVENT = 2 };

#ifdef SIMSWEEP_PROFILE  // phase cycle counters of thread 0 (tools/probe.py); not in the product build
constexpr int PROF_MAX_CFG = 8192;
__device__ long long g_prof[PROF_MAX_CFG][16];
#define PROF_MARK(i)                  \
  if (tid == 0) {                     \
    long long _t = clock64();         \
    prof[i] += _t - prof_last;        \
    prof_last = _t;                   \
  }
#define PROF_CNT(i, v) \
  if (tid == 0) prof[i] += (v);
#else
#define PROF_MARK(i)
#define PROF_CNT(i, v)
#endif

__host__ __device__ inline int variant_of(int n) { return n <= 1024 ? 0 : 1; }

template <int NT>
__device__ __forceinline__ long long block_sum_ll(long long v, Scal& S) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) S.featsum[threadIdx.x >> 5] = v;
  __syncthreads();
  long long t = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; w++) t += S.featsum[w];
  __syncthreads();
  return t;
}

template <int NT, int CAP>
__global__ void __launch_bounds__(NT) sim_kernel(KParams p) {
  using L = Smem<NT, CAP>;
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  Scal& S = *reinterpret_cast<Scal*>(smem);
  int32_t* s_m = reinterpret_cast<int32_t*>(smem + L::off_int);  // r.m: KVs cached
  int32_t* s_g = s_m + CAP;                                        // generated tokens
  int32_t* s_res = s_g + CAP;                                      // reserved KVs
  int32_t* s_seq = s_res + CAP;                                    // admission sequence
  int32_t* s_I = s_seq + CAP;
  int32_t* s_O = s_I + CAP;
  int32_t* s_c = s_O + CAP;  // c of the current batch (0 = not in B)
  int16_t* s_rpos = reinterpret_cast<int16_t*>(smem + L::off_rpos);  // position in the run list
  uint8_t* s_fl = smem + L::off_fl;
  int16_t* s_runA = reinterpret_cast<int16_t*>(smem + L::off_lists);
  int16_t* s_runB = s_runA + CAP;
  int16_t* s_rank = s_runB + CAP;
  int16_t* s_wl = reinterpret_cast<int16_t*>(smem + L::off_union);  // waiting list
  int16_t* s_pl = s_wl + CAP;   // decode-first partition of the run list
  int16_t* s_new = s_pl + CAP;  // admitted-from-waiting this step, in admission order
  int16_t* s_tmp = s_new + CAP;
  unsigned long long* s_keys = reinterpret_cast<unsigned long long*>(smem + L::off_union);

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ci = p.order ? p.order[blockIdx.x] : (int)blockIdx.x;
  const sim_config_t cfg = p.cfgs[ci];
  const sim_workload_t wl = p.wls[cfg.workload];
  const int n = wl.n;
  if (variant_of(n) != p.variant) return;
  const int K = cfg.n_cost;
  const long long M = cfg.M, C = cfg.C;
  const bool finiteM = M >= 0, hybrid = cfg.hybrid != 0, chunked = cfg.chunked != 0;
  const int order = cfg.order;
  const bool srf = cfg.replacement != SIM_NRF;
  const bool hist = cfg.replacement == SIM_SRF_HIST && finiteM;
  const bool rank = order >= SIM_ORDER_RANK_ORG;
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
  for (int i = tid; i < n; i += NT) {
    long long pk = (long long)wl.I[i] + wl.O[i] - 1;  // peak KV usage
    bad_long |= pk > cfg.S;
    bad_fit |= (finiteM && pk > M) || (!chunked && pk > C);
  }
  bad_long = __syncthreads_or(bad_long);
  bad_fit = __syncthreads_or(bad_fit);
  if (bad_long || bad_fit) {
    if (tid == 0) {
      sim_result_t r;
      memset(&r, 0, sizeof(r));
      r.status = bad_long ? SIM_S_TOO_LONG : SIM_S_NEVER_FITS;
      p.results[ci] = r;
    }
    return;
  }
  if (tid == 0) {
    for (int k = 0; k < SIM_MAX_COST; k++) S.clock[k] = 0.0;
    S.U = S.tok = S.Rsum = S.seq = 0;
    S.steps = S.preempt = S.entries = S.processed = S.sumU = S.pentries = S.idle = S.visits = 0;
    S.next = S.new_next = S.lo = S.n_done = S.n_run = S.n_running = 0;
    S.nrank = 0;
    S.status = 0;
    S.cur = 0;
  }
  if (tid < K) S.cm[tid] = p.cms[cfg.cost[tid]];
  for (int i = tid; i < 18 * 18; i += NT) S.hist[i] = 0;
  __syncthreads();
#ifdef SIMSWEEP_PROFILE
  long long prof[16] = {0};
  long long prof_last = clock64();
#endif

  for (;;) {
    PROF_MARK(10);
    // ---- a2: GetNewRequests (Alg. 1 line 3): all T <= clock (inclusive, Q21) ----
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
      S.new_next = a;
      if (S.n_done == n)
        S.status = -1;
      else if (a - S.lo > CAP)
        S.status = SIM_S_CAPACITY;
      else if (S.steps >= cfg.max_steps)
        S.status = SIM_S_MAX_STEPS;
    }
    __syncthreads();
    if (S.status) break;
    const int nx0 = S.next, nx1 = S.new_next, lo = S.lo;
    const int nrun = S.n_run;
    int16_t* run = S.cur ? s_runB : s_runA;
    int nrank = S.nrank;
    if (rank) {  // drop finished entries before slots can be reused by arrivals
      nrank = block_compact<NT>(
          nrank, [&](int q) { return (s_fl[s_rank[q]] & ST_MASK) != ST_DONE; }, [&](int q) { return s_rank[q]; },
          s_tmp, S);
      __syncthreads();
      for (int q = tid; q < nrank; q += NT) s_rank[q] = s_tmp[q];
    }
    for (int idx = nx0 + tid; idx < nx1; idx += NT) {
      const int sl = idx & (CAP - 1);
      s_m[sl] = 0;
      s_g[sl] = 0;
      s_res[sl] = 0;
      s_seq[sl] = 0;
      s_c[sl] = 0;
      s_I[sl] = wl.I[idx];
      s_O[sl] = wl.O[idx];
      s_fl[sl] = ST_WAIT;
    }
    __syncthreads();
    PROF_MARK(0);
    // ---- a3: GroupRequests (step 1) ----
    if (rank) {  // one group sorted by (key, T, id) (App. D, Q20, Q37)
      for (int idx = nx0 + tid; idx < nx1; idx += NT) s_rank[nrank + idx - nx0] = (int16_t)(idx & (CAP - 1));
      const int nr = nrank + (nx1 - nx0);
      if (nx1 > nx0) {
        __syncthreads();
        for (int q = tid; q < nr; q += NT) {
          const int sl = s_rank[q];
          const unsigned idx = (unsigned)(lo + ((sl - lo) & (CAP - 1)));
          const unsigned key = order == SIM_ORDER_RANK_I ? (unsigned)s_I[sl]
                               : order == SIM_ORDER_RANK_O ? (unsigned)s_O[sl]
                                                           : 0u;
          s_keys[q] = ((unsigned long long)key << 32) | idx;
        }
        block_bitonic<NT>(s_keys, nr);
        for (int q = tid; q < nr; q += NT) s_rank[q] = (int16_t)(s_keys[q] & (CAP - 1));
      }
      nrank = nr;
      __syncthreads();
    }
    int nW = 0;
    if (!rank)  // R_w by (T, id) = index order (Q1, Q2)
      nW = block_compact<NT>(
          nx1 - lo, [&](int q) { return (s_fl[(lo + q) & (CAP - 1)] & ST_MASK) == ST_WAIT; },
          [&](int q) { return (lo + q) & (CAP - 1); }, s_wl, S);
    if (order == SIM_ORDER_DECODE_FIRST) {  // {R_r^d, R_r^p, R_w}: stable split of the retention-ordered run list
      const int nd = block_compact<NT>(
          nrun, [&](int q) { return (s_fl[run[q]] & F_FILLED) != 0; }, [&](int q) { return run[q]; }, s_pl, S);
      block_compact<NT>(
          nrun, [&](int q) { return (s_fl[run[q]] & F_FILLED) == 0; }, [&](int q) { return run[q]; }, s_pl + nd, S);
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

    if (hist) {  // SRF+Hist: predictions of the current histogram and sum of remaining outputs
      if (tid < 18) S.pred[tid] = hist_pred_row(S.hist, tid);
      __syncthreads();
      long long r = 0;
      for (int q = tid; q < nrun; q += NT) {
        const int sl = run[q];
        const int rem = S.pred[bucket_of(s_I[sl])] - s_g[sl];
        r += rem > 0 ? rem : 0;
      }
      r = block_sum_ll<NT>(r, S);
      if (tid == 0) S.Rsum = r;
    }
    if (tid == 0) {
      S.tok = 0;
      S.bphase = -1;
      S.vt = nrun - 1;
      S.n_new = 0;
      S.pos = 0;
      S.n_running = nrun;
      S.any_pre = 0;
      S.nrank = nrank;
      S.visits += nP;
    }

    PROF_MARK(1);
    // ---- a4-a8: GetNextBatch (steps 2-4), block-parallel rounds ----
    auto preempt = [&](int v) {  // thread 0 only (refill P:1570)
      const int m = s_m[v];
      S.U -= max(s_res[v], m);
      if (hist) S.Rsum -= max(S.pred[bucket_of(s_I[v])] - s_g[v], 0);
      const int idx = lo + ((v - lo) & (CAP - 1));
      atomicAdd(&npre[idx], 1ull);
      atomicAdd(&refill[idx], (unsigned long long)m);
      s_m[v] = 0;
      s_res[v] = 0;
      s_fl[v] = ST_WAIT | F_PRE | (s_fl[v] & F_FIRST);
      S.n_running--;
      S.preempt++;
      S.any_pre = 1;
    };
    auto handle = [&](int sl) {  // literal sequential resolution of one candidate (thread 0)
      uint8_t fl = s_fl[sl];
      if (fl & F_PRE) return;  // Q9
      const bool isW = (fl & ST_MASK) == ST_WAIT;
      const int ph = (isW || !(fl & F_FILLED)) ? PH_PRE : PH_DEC;
      if (!hybrid && S.bphase >= 0 && ph != S.bphase) return;  // step 2
      const int I = s_I[sl], g = s_g[sl], m = s_m[sl], res = s_res[sl];
      const int s = I + g, avail = s - m;
      const long long c = ph == PH_DEC ? 1 : (chunked ? min((long long)avail, C - S.tok) : (long long)avail);
      if (c == 0 || S.tok + c > C) return;  // token limit never preempts (Q11)
      int rem = 0;
      if (hist && isW) {
        rem = max(S.pred[bucket_of(I)] - g, 0);
        if (S.n_running > 0 && S.U + S.Rsum + s + rem > M) return;  // deferred (Q31)
      }
      const int nh = max(isW ? s : res, m + (int)c), held = isW ? 0 : max(res, m), delta = nh - held;
      while (finiteM && S.U + delta > M) {
        if (isW) return;  // holds no KVs: skipped (Q5)
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
      if (isW) {  // (re)admission reserves s = I + g (Table 2, Q13)
        S.seq++;
        s_seq[sl] = (int)S.seq;
        s_res[sl] = s;
        fl = ST_RUN | (fl & F_FIRST);
        s_new[S.n_new++] = (int16_t)sl;
        S.n_running++;
        S.Rsum += rem;
      }
      s_fl[sl] = fl | F_INB;
      s_c[sl] = (int)c;
      S.U += delta;
      S.tok += c;
      if (S.bphase < 0) S.bphase = ph;
    };

    for (;;) {
      __syncthreads();
      const int pos = S.pos;
      if (pos >= nP) break;
      PROF_CNT(6, 1);
      const long long tok = S.tok, U = S.U, Rs = S.Rsum;
      const int bph = S.bphase;
      const bool anyRun0 = S.n_running > 0;
      const int cend = min(pos + NT * IPT, nP);
      int kind[IPT], cc[IPT], dd[IPT], ww[IPT], rr[IPT], slv[IPT], av[IPT], ss[IPT], phv[IPT];
#pragma unroll
      for (int j = 0; j < IPT; j++) {
        kind[j] = K_NONE;
        cc[j] = dd[j] = ww[j] = rr[j] = av[j] = ss[j] = phv[j] = slv[j] = 0;
        const int q = pos + tid * IPT + j;
        if (q >= cend) continue;
        const int sl = cand(q);
        slv[j] = sl;
        const uint8_t fl = s_fl[sl];
        if (fl & F_PRE) continue;
        const bool isW = (fl & ST_MASK) == ST_WAIT;
        const int ph = (isW || !(fl & F_FILLED)) ? PH_PRE : PH_DEC;
        if (!hybrid && bph >= 0 && ph != bph) continue;
        const int I = s_I[sl], g = s_g[sl], m = s_m[sl], res = s_res[sl];
        const int s = I + g, avail = s - m;
        const long long rt = C - tok;
        const long long c = ph == PH_DEC ? 1 : (chunked ? min((long long)avail, rt) : (long long)avail);
        if (c < 1 || c > rt) continue;
        int rem = 0;
        if (hist && isW) {
          rem = max(S.pred[bucket_of(I)] - g, 0);
          if (anyRun0 && U + Rs + s + rem > M) continue;
        }
        const int held = isW ? 0 : max(res, m);
        const int delta = max(isW ? s : res, m + (int)c) - held;
        if (finiteM && U + delta > M) {
          kind[j] = isW ? K_NONE : K_EVENT;
          continue;
        }
        kind[j] = K_MARK;
        cc[j] = ph == PH_DEC ? 1 : avail;
        dd[j] = delta;
        ww[j] = isW;
        rr[j] = rem;
        av[j] = avail;
        ss[j] = s;
        phv[j] = ph;
      }
      int lc = 0, ld = 0, lw = 0, lr = 0, pc[IPT], pd[IPT], pw[IPT], pr[IPT];
#pragma unroll
      for (int j = 0; j < IPT; j++) {
        pc[j] = lc, pd[j] = ld, pw[j] = lw, pr[j] = lr;
        if (kind[j] == K_MARK) lc += cc[j], ld += dd[j], lw += ww[j], lr += rr[j];
      }
      int xc = lc, xd = ld, xw = lw, xr = lr;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int yc = __shfl_up_sync(0xffffffffu, xc, o), yd = __shfl_up_sync(0xffffffffu, xd, o);
        const int yw = __shfl_up_sync(0xffffffffu, xw, o), yr = __shfl_up_sync(0xffffffffu, xr, o);
        if (lane >= o) xc += yc, xd += yd, xw += yw, xr += yr;
      }
      if (lane == 31) S.wsum[wid][0] = xc, S.wsum[wid][1] = xd, S.wsum[wid][2] = xw, S.wsum[wid][3] = xr;
      __syncthreads();
      int oc = xc - lc, od = xd - ld, ow = xw - lw, orr = xr - lr, tc = 0, tdk = 0, tw = 0, tr = 0;
#pragma unroll
      for (int w = 0; w < NW; w++) {
        const int a0 = S.wsum[w][0], a1 = S.wsum[w][1], a2 = S.wsum[w][2], a3 = S.wsum[w][3];
        if (w < wid) oc += a0, od += a1, ow += a2, orr += a3;
        tc += a0, tdk += a1, tw += a2, tr += a3;
      }
      int mybrk = NOBRK;
#pragma unroll
      for (int j = 0; j < IPT; j++) {
        const int q = pos + tid * IPT + j;
        if (kind[j] == K_MARK) {
          const long long ptok = tok + oc + pc[j], pU = U + od + pd[j];
          const long long rt = C - ptok;
          bool brk = !hybrid && bph < 0;  // the first admission fixes the batch phase (Q19)
          if (phv[j] == PH_PRE && chunked)
            brk |= rt < av[j];  // cropped chunk (terminal) or budget exhausted
          else
            brk |= cc[j] > rt;
          if (hist && ww[j]) {
            const bool anyR = anyRun0 || (ow + pw[j]) > 0;
            brk |= anyR && pU + Rs + orr + pr[j] + ss[j] + rr[j] > M;
          }
          if (finiteM) brk |= pU + dd[j] > M;
          if (brk) mybrk = min(mybrk, q);
        } else if (kind[j] == K_EVENT) {
          if (tok + oc + pc[j] + 1 <= C) mybrk = min(mybrk, q);  // else a token reject (Q11)
        }
      }
      const int wm = (int)__reduce_min_sync(0xffffffffu, (unsigned)mybrk);
      if (lane == 0) S.wmin[wid] = wm;
      __syncthreads();
      int b = NOBRK;
#pragma unroll
      for (int w = 0; w < NW; w++) b = min(b, S.wmin[w]);
#pragma unroll
      for (int j = 0; j < IPT; j++) {
        const int q = pos + tid * IPT + j;
        if (kind[j] == K_MARK && q < b) {  // admitted: every check passed at its exact position
          const int sl = slv[j];
          const uint8_t fl = s_fl[sl];
          s_c[sl] = cc[j];
          if (ww[j]) {
            const int k = ow + pw[j];
            s_seq[sl] = (int)(S.seq + k + 1);
            s_res[sl] = ss[j];
            s_fl[sl] = ST_RUN | F_INB | (fl & F_FIRST);
            s_new[S.n_new + k] = (int16_t)sl;
          } else {
            s_fl[sl] = fl | F_INB;
          }
        }
        if (q == b) S.pref[0] = oc + pc[j], S.pref[1] = od + pd[j], S.pref[2] = ow + pw[j], S.pref[3] = orr + pr[j];
      }
      __syncthreads();
      if (tid == 0) {
        const bool real = b < cend;
        const long long a0 = real ? S.pref[0] : tc, a1 = real ? S.pref[1] : tdk;
        const long long a2 = real ? S.pref[2] : tw, a3 = real ? S.pref[3] : tr;
        S.tok += a0;
        S.U += a1;
        S.seq += a2;
        S.n_new += (int)a2;
        S.n_running += (int)a2;
        S.Rsum += a3;
        if (real) {
          PROF_CNT(7, 1);
          handle(cand(b));
          S.pos = b + 1;
        } else {
          S.pos = cend;
        }
      }
    }
    // (the loop exits right after a barrier: all scalars are current)
    if (S.tok == 0) {  // B = {}: idle jump to the next arrival, not a step (Q21)
      __syncthreads();
      if (tid == 0) {
        if (S.any_pre)
          S.status = SIM_S_DEADLOCK;
        else if (nx1 < n) {
          S.clock[0] = fmax(S.clock[0], wl.T[nx1]);
          S.idle++;
          S.next = nx1;
        } else
          S.status = SIM_S_DEADLOCK;
      }
      __syncthreads();
      if (S.status) break;
      continue;
    }

    PROF_MARK(2);
    // ---- a9: batch latency from exact integer features ----
    {
      long long v[9 + SIM_MAX_COST];
#pragma unroll
      for (int z = 0; z < 9 + SIM_MAX_COST; z++) v[z] = 0;
      for (int q = tid; q < nP; q += NT) {
        const int sl = cand(q);
        const uint8_t fl = s_fl[sl];
        if (!(fl & F_INB)) continue;
        const long long c = s_c[sl], m = s_m[sl];
        v[0] += c;
        if (!(fl & F_FILLED)) {  // prefill entry
          v[1]++;
          v[2] += c * c;
          v[3] += m * c;
          v[4] += c;
          v[5] += m;
          v[6] += c * (c + m);
#pragma unroll
          for (int k = 0; k < SIM_MAX_COST; k++)
            if (k < K) {
              const long long H = S.cm[k].H;
              v[9 + k] += ((c + H - 1) / H) * (c + m);
            }
        } else {  // decode entry (c = 1)
          v[7]++;
          v[8] += m;
        }
      }
#pragma unroll
      for (int z = 0; z < 9 + SIM_MAX_COST; z++) v[z] = warp_sum(v[z]);
      if (lane == 0)
#pragma unroll
        for (int z = 0; z < 9 + SIM_MAX_COST; z++) S.wred[wid][z] = v[z];
      __syncthreads();
      if (tid == 0) {
        Feat f;
        long long t[9 + SIM_MAX_COST];
        for (int z = 0; z < 9 + SIM_MAX_COST; z++) {
          t[z] = 0;
          for (int w = 0; w < NW; w++) t[z] += S.wred[w][z];
        }
        f.N = t[0], f.np = t[1], f.c2 = t[2], f.mc = t[3], f.cp = t[4], f.mp = t[5], f.pcm = t[6];
        f.nd = t[7], f.md = t[8];
        for (int k = 0; k < SIM_MAX_COST; k++) f.pceil[k] = t[9 + k];
        for (int k = 0; k < K; k++) S.clock[k] = dadd(S.clock[k], batch_time(S.cm[k], f, k));  // Q36
        S.steps++;
        S.sumU += S.U;
        S.entries += f.np + f.nd;
        S.processed += f.N;
        S.pentries += f.np;
        S.last_np = f.np;
        S.last_nd = f.nd;
      }
      __syncthreads();
    }

    PROF_MARK(3);
    // ---- a10: Process(B): token generation (Eq. 6), completions free KVs at batch end (Q14) ----
    {
      long long freed = 0, mdn = 0;
      int ndone = 0, minrem = NOBRK;
      for (int q = tid; q < nP; q += NT) {
        const int sl = cand(q);
        uint8_t fl = s_fl[sl];
        if (fl & F_INB) {
          const int c = s_c[sl], m0 = s_m[sl], I = s_I[sl], O = s_O[sl];
          int g = s_g[sl];
          const int s = I + g, m = m0 + c;
          s_m[sl] = m;
          s_c[sl] = 0;
          fl = (fl & ~F_INB) | F_LAST;
          bool done = false;
          if (c == s - m0) {
            g++;
            s_g[sl] = g;
            fl |= F_FILLED;
            const int idx = lo + ((sl - lo) & (CAP - 1));
            if (!(fl & F_FIRST)) {
              fl |= F_FIRST;
              for (int k = 0; k < K; k++) tf[(long long)k * n + idx] = S.clock[k];
            }
            if (g == O) {
              done = true;
              fl = (fl & ~ST_MASK) | ST_DONE;
              for (int k = 0; k < K; k++) td[(long long)k * n + idx] = S.clock[k];
              freed += max(s_res[sl], m);
              ndone++;
              if (hist) atomicAdd(&S.hist[bucket_of(I) * 18 + bucket_of(O)], 1);
            }
          }
          if (!done) {
            minrem = min(minrem, O - g);
            mdn += m;
          }
          s_fl[sl] = fl;
        } else if (fl & (F_PRE | F_LAST)) {
          s_fl[sl] = fl & ~(F_PRE | F_LAST);
        }
      }
      freed = warp_sum(freed);
      mdn = warp_sum(mdn);
      ndone = warp_sum(ndone);
      minrem = (int)__reduce_min_sync(0xffffffffu, (unsigned)minrem);
      if (lane == 0) S.wred[wid][0] = freed, S.wred[wid][1] = mdn, S.wred[wid][2] = ndone, S.wred[wid][3] = minrem;
      __syncthreads();
      if (tid == 0) {
        long long fr = 0, md = 0, nd = 0, mr = NOBRK;
        for (int w = 0; w < NW; w++) fr += S.wred[w][0], md += S.wred[w][1], nd += S.wred[w][2], mr = min(mr, S.wred[w][3]);
        S.U -= fr;
        S.n_done += (int)nd;
        S.n_running -= (int)nd;
        // Steady decode run: step j had only decodes, no admission, preemption or completion.  Then step
        // j+1 repeats it exactly (waiting candidates were rejected for reasons that persist: KV and SRF+Hist
        // deferral are monotone in U, token/hybrid rejections are unchanged) until a completion, the KV
        // limit (U + k n_d <= M) or an arrival.  Those steps are charged below without re-forming batches.
        long long L = 0;
        if (nd == 0 && S.last_np == 0 && !S.any_pre && S.last_nd > 0) {
          L = mr;
          if (finiteM) L = min(L, (M - S.U) / S.last_nd);
          L = min(L, cfg.max_steps - S.steps);
        }
        S.runL = L;
        S.runMD = md;
      }
      __syncthreads();
      const long long L = S.runL;
      if (L > 0) {
        PROF_CNT(9, L);
        // s_new + s_tmp half of the union area is free (no new admissions this step); the P segments
        // (s_wl, s_pl) in the other half are still needed below
        double* dbuf = reinterpret_cast<double*>(s_new);
        constexpr int DB = CAP / 2;  // doubles available
        const int cmax = min(NT, DB / K);
        const long long ndd = S.last_nd, MD = S.runMD, U0 = S.U;
        long long E = 0;
        while (E < L) {
          const int chunk = (int)min((long long)cmax, L - E);
          if (tid < chunk) {  // features of run step E+tid+1 are affine in the step index
            Feat f;
            f.N = ndd, f.np = 0, f.c2 = 0, f.mc = 0, f.cp = 0, f.mp = 0, f.pcm = 0, f.nd = ndd;
            f.md = MD + (E + tid) * ndd;
            for (int k = 0; k < SIM_MAX_COST; k++) f.pceil[k] = 0;
            for (int k = 0; k < K; k++) dbuf[k * cmax + tid] = batch_time(S.cm[k], f, k);
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
                clk = dadd(clk, dbuf[t]);
              }
              S.clock[0] = clk;
            } else {
              for (int k = 0; k < K; k++) {
                double clk = S.clock[k];
                for (int t = 0; t < chunk; t++) clk = dadd(clk, dbuf[k * cmax + t]);
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
        if (tid == 0) {
          S.steps += E;
          S.sumU += E * U0 + ndd * (E * (E + 1) / 2);
          S.entries += E * ndd;
          S.processed += E * ndd;
          S.visits += E * nP;
          S.U = U0 + E * ndd;
        }
        long long fr2 = 0;
        int nd2 = 0;
        if (E > 0) {
          for (int q = tid; q < nP; q += NT) {
            const int sl = cand(q);
            uint8_t fl = s_fl[sl];
            if (!(fl & F_LAST)) continue;
            const int m = s_m[sl] + (int)E, g = s_g[sl] + (int)E, O = s_O[sl];
            s_m[sl] = m;
            s_g[sl] = g;
            if (g == O) {  // completes at the last run step
              const int idx = lo + ((sl - lo) & (CAP - 1));
              s_fl[sl] = (fl & ~ST_MASK) | ST_DONE;
              for (int k = 0; k < K; k++) td[(long long)k * n + idx] = S.clock[k];
              fr2 += max(s_res[sl], m);
              nd2++;
              if (hist) atomicAdd(&S.hist[bucket_of(s_I[sl]) * 18 + bucket_of(O)], 1);
            }
          }
        }
        fr2 = block_sum_ll<NT>(fr2, S);
        const long long nd2t = block_sum_ll<NT>((long long)nd2, S);
        if (tid == 0) {
          S.U -= fr2;
          S.n_done += (int)nd2t;
          S.n_running -= (int)nd2t;
        }
      }
    }

    PROF_MARK(4);
    // ---- run list (retention order) for the next step ----
    {
      int16_t* nrl = S.cur ? s_runA : s_runB;
      const int nnew = S.n_new;
      auto src = [&](int q) -> int { return q < nrun ? run[q] : s_new[q - nrun]; };
      const int cnt = block_compact<NT>(
          nrun + nnew, [&](int q) { return (s_fl[src(q)] & ST_MASK) == ST_RUN; }, src, nrl, S);
      __syncthreads();
      if (srf) {  // SRF retention order: m descending, then admission order (Q3, Q7)
        auto key = [&](int sl) -> unsigned long long {
          return ((unsigned long long)(0x3FFFF - s_m[sl]) << 46) | ((unsigned long long)(unsigned)s_seq[sl] << 12) |
                 (unsigned long long)sl;
        };
        int ok = 1;
        for (int q = tid; q + 1 < cnt; q += NT)
          if (key(nrl[q]) > key(nrl[q + 1])) ok = 0;
        ok = __syncthreads_and(ok);
        if (!ok) {
          PROF_CNT(8, 1);
          for (int q = tid; q < cnt; q += NT) s_keys[q] = key(nrl[q]);
          block_bitonic<NT>(s_keys, cnt);
          for (int q = tid; q < cnt; q += NT) nrl[q] = (int16_t)(s_keys[q] & 0xFFF);
          __syncthreads();
        }
      }
      for (int q = tid; q < cnt; q += NT) s_rpos[nrl[q]] = (int16_t)q;
      if (tid == 0) {
        S.cur ^= 1;
        S.n_run = cnt;
        S.next = nx1;
        int l = lo;
        while (l < nx1 && (s_fl[l & (CAP - 1)] & ST_MASK) == ST_DONE) l++;
        S.lo = l;
      }
      __syncthreads();
      PROF_MARK(5);
    }
  }
#ifdef SIMSWEEP_PROFILE
  if (tid == 0 && ci < PROF_MAX_CFG)
    for (int i = 0; i < 16; i++) g_prof[ci][i] = prof[i];
#endif

  // ---- a11: metrics ----
  const int st = S.status == -1 ? SIM_S_OK : S.status;
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
    for (int k = K; k < SIM_MAX_COST; k++) r.makespan[k] = r.mean_latency[k] = r.mean_ttft[k] = r.mean_tpot[k] = 0.0;
  }
}

// ------------------------------------------------------------------ host side
struct Variant {
  int nt, cap;
  size_t smem;
  void (*fn)(KParams);
};

template <int NT, int CAP>
Variant make_variant() {
  return Variant{NT, CAP, Smem<NT, CAP>::bytes, sim_kernel<NT, CAP>};
}

static Variant g_variants[2] = {make_variant<256, 1024>(), make_variant<512, 4096>()};

static int check_cuda(cudaError_t e) { return e == cudaSuccess ? 0 : SIM_ECUDA; }

}  // namespace simsweep

using namespace simsweep;

extern "C" {

#ifdef SIMSWEEP_PROFILE
int sim_debug_read(int64_t* out, int32_t n_cfgs) {
  return cudaMemcpyFromSymbol(out, g_prof, sizeof(long long) * 16 * (size_t)n_cfgs) == cudaSuccess ? 0 : SIM_ECUDA;
}
#endif

const char* sim_version(void) { return "simsweep 0.1 (sm_100a, CTA-per-simulation)"; }

const char* sim_strerror(int code) {
  switch (code) {
    case 0: return "ok";
    case SIM_EINVAL: return "invalid argument (NULL pointer, n <= 0, bad enum, C < 1, S out of range, n_cost)";
    case SIM_EWORKLOAD: return "invalid workload (I < 1, O < 1, unsorted T, or T != 0 with n_cost > 1)";
    case SIM_ECOST: return "invalid cost model or cost-model index";
    case SIM_ECUDA: return "CUDA runtime error";
    case SIM_ENODEV: return "no sm_100 CUDA device";
    default: return "unknown error";
  }
}

int sim_request_rows(const sim_config_t* cfgs, int32_t n_cfgs, const sim_workload_t* wls, int32_t n_wls,
                     int64_t* rows, int64_t* tim_rows) {
  if (!cfgs || !wls || n_cfgs <= 0 || n_wls <= 0 || !rows || !tim_rows) return SIM_EINVAL;
  int64_t r = 0, t = 0;
  for (int i = 0; i < n_cfgs; i++) {
    if (cfgs[i].workload < 0 || cfgs[i].workload >= n_wls) return SIM_EINVAL;
    if (cfgs[i].n_cost < 1 || cfgs[i].n_cost > SIM_MAX_COST) return SIM_EINVAL;
    r += wls[cfgs[i].workload].n;
    t += (int64_t)cfgs[i].n_cost * wls[cfgs[i].workload].n;
  }
  *rows = r;
  *tim_rows = t;
  return 0;
}

int sim_sweep_device(const sim_config_t* h_cfgs, int32_t n_cfgs, const int32_t* h_wls_n, const sim_config_t* d_cfgs,
                     const sim_workload_t* d_wls, const sim_cost_model_t* d_cms, int32_t n_cms,
                     const int32_t* d_order, const int64_t* d_row_off, const int64_t* d_tim_off,
                     sim_result_t* d_results, sim_request_out_t d_req, void* stream) {
  if (!h_cfgs || !h_wls_n || !d_cfgs || !d_wls || !d_cms || n_cfgs <= 0 || n_cms <= 0 || !d_row_off ||
      !d_tim_off || !d_results || !d_req.t_first || !d_req.t_done || !d_req.n_preempt || !d_req.refill_tokens)
    return SIM_EINVAL;
  bool need[2] = {false, false};
  for (int i = 0; i < n_cfgs; i++) need[variant_of(h_wls_n[h_cfgs[i].workload])] = true;
  KParams kp;
  kp.cfgs = d_cfgs;
  kp.wls = d_wls;
  kp.cms = d_cms;
  kp.order = d_order;
  kp.row_off = d_row_off;
  kp.tim_off = d_tim_off;
  kp.results = d_results;
  kp.req = d_req;
  kp.n_cfgs = n_cfgs;
  int launches = 0;
  // the large-window variant first: its simulations are the longest
  for (int v = 1; v >= 0; v--) {
    if (!need[v]) continue;
    const Variant& V = g_variants[v];
    if (cudaFuncSetAttribute((const void*)V.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)V.smem) !=
        cudaSuccess)
      return SIM_ECUDA;
    kp.variant = v;
    void* args[] = {&kp};
    if (cudaLaunchKernel((const void*)V.fn, dim3(n_cfgs), dim3(V.nt), args, V.smem, (cudaStream_t)stream) !=
        cudaSuccess)
      return SIM_ECUDA;
    launches++;
  }
  return launches;
}

static int validate(const sim_config_t* cfgs, int32_t n_cfgs, const sim_workload_t* wls, int32_t n_wls,
                    const sim_cost_model_t* cms, int32_t n_cms) {
  if (!cfgs || !wls || !cms || n_cfgs <= 0 || n_wls <= 0 || n_cms <= 0) return SIM_EINVAL;
  std::vector<char> multi(n_wls, 0);
  for (int i = 0; i < n_cfgs; i++) {
    const sim_config_t& c = cfgs[i];
    if (c.order < SIM_ORDER_PREFILL_FIRST || c.order > SIM_ORDER_RANK_O) return SIM_EINVAL;
    if (c.replacement < SIM_NRF || c.replacement > SIM_SRF_HIST) return SIM_EINVAL;
    if ((c.hybrid != 0 && c.hybrid != 1) || (c.chunked != 0 && c.chunked != 1)) return SIM_EINVAL;
    if (c.C < 1 || c.S < 1 || c.S > 262143 || c.max_steps < 1) return SIM_EINVAL;
    if (c.n_cost < 1 || c.n_cost > SIM_MAX_COST) return SIM_EINVAL;
    if (c.workload < 0 || c.workload >= n_wls) return SIM_EINVAL;
    for (int k = 0; k < c.n_cost; k++)
      if (c.cost[k] < 0 || c.cost[k] >= n_cms) return SIM_ECOST;
    if (c.n_cost > 1) multi[c.workload] = 1;
  }
  for (int w = 0; w < n_wls; w++) {
    const sim_workload_t& W = wls[w];
    if (W.n <= 0 || !W.I || !W.O || !W.T) return SIM_EINVAL;
    for (int i = 0; i < W.n; i++) {
      if (W.I[i] < 1 || W.O[i] < 1 || W.I[i] > 262143 || W.O[i] > 262143) return SIM_EWORKLOAD;
      if (i > 0 && !(W.T[i] >= W.T[i - 1])) return SIM_EWORKLOAD;
      if (multi[w] && W.T[i] != 0.0) return SIM_EWORKLOAD;
    }
  }
  for (int k = 0; k < n_cms; k++) {
    const sim_cost_model_t& m = cms[k];
    if (m.mode != 0 && m.mode != 1) return SIM_ECOST;
    if (m.layers < 1 || m.e < 1 || m.tp < 1) return SIM_ECOST;
    if (m.mode == 1 && (m.h < 1 || m.f < 1 || m.H < 1 || m.NQ < 1 || m.NKV < 1 || !(m.flops > 0) || !(m.bw > 0) ||
                        (m.tp > 1 && !(m.link_bw > 0))))
      return SIM_ECOST;
  }
  return 0;
}

// longest-processing-time-first estimate of one simulation's step count
static double estimate_steps(const sim_config_t& c, const sim_workload_t& w) {
  double sumIO = 0, sumI = 0, maxO = 0;
  for (int i = 0; i < w.n; i++) {
    sumIO += ((double)w.I[i] + 0.5 * w.O[i]) * w.O[i];
    sumI += w.I[i];
    maxO = std::max(maxO, (double)w.O[i]);
  }
  const double Meff = c.M >= 0 ? (double)std::max<int64_t>(c.M, 1) : 1e18;
  return maxO + sumIO / Meff + sumI / (double)c.C;
}

int sim_sweep(const sim_config_t* cfgs, int32_t n_cfgs, const sim_workload_t* wls, int32_t n_wls,
              const sim_cost_model_t* cms, int32_t n_cms, sim_result_t* results, sim_request_out_t req,
              int32_t device) {
  int rc = validate(cfgs, n_cfgs, wls, n_wls, cms, n_cms);
  if (rc) return rc;
  if (!results) return SIM_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return SIM_ENODEV;
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess) return SIM_ECUDA;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return SIM_ECUDA;
  if (prop.major != 10) return SIM_ENODEV;

  std::vector<int64_t> row_off(n_cfgs), tim_off(n_cfgs);
  int64_t rows = 0, trows = 0;
  for (int i = 0; i < n_cfgs; i++) {
    row_off[i] = rows;
    tim_off[i] = trows;
    rows += wls[cfgs[i].workload].n;
    trows += (int64_t)cfgs[i].n_cost * wls[cfgs[i].workload].n;
  }
  std::vector<double> est(n_cfgs);
  for (int i = 0; i < n_cfgs; i++) est[i] = estimate_steps(cfgs[i], wls[cfgs[i].workload]);
  std::vector<int32_t> order(n_cfgs);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return est[a] > est[b]; });
  std::vector<int32_t> wn(n_wls);
  int64_t wtot = 0;
  for (int w = 0; w < n_wls; w++) wn[w] = wls[w].n, wtot += wls[w].n;

  // one device arena: cfgs | wls | cms | order | row_off | tim_off | results | I O T | outputs
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t off = 0;
  const size_t o_cfg = off;
  off = al(off + sizeof(sim_config_t) * n_cfgs);
  const size_t o_wl = off;
  off = al(off + sizeof(sim_workload_t) * n_wls);
  const size_t o_cm = off;
  off = al(off + sizeof(sim_cost_model_t) * n_cms);
  const size_t o_ord = off;
  off = al(off + 4 * (size_t)n_cfgs);
  const size_t o_ro = off;
  off = al(off + 8 * (size_t)n_cfgs);
  const size_t o_to = off;
  off = al(off + 8 * (size_t)n_cfgs);
  const size_t o_res = off;
  off = al(off + sizeof(sim_result_t) * n_cfgs);
  const size_t o_I = off;
  off = al(off + 4 * (size_t)wtot);
  const size_t o_O = off;
  off = al(off + 4 * (size_t)wtot);
  const size_t o_T = off;
  off = al(off + 8 * (size_t)wtot);
  const size_t o_tf = off;
  off = al(off + 8 * (size_t)trows);
  const size_t o_td = off;
  off = al(off + 8 * (size_t)trows);
  const size_t o_np = off;
  off = al(off + 8 * (size_t)rows);
  const size_t o_rf = off;
  off = al(off + 8 * (size_t)rows);
  char* base = nullptr;
  if (cudaMalloc(&base, off) != cudaSuccess) return SIM_ECUDA;
  cudaStream_t s;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
    cudaFree(base);
    return SIM_ECUDA;
  }
  std::vector<sim_workload_t> dw(n_wls);
  int64_t wo = 0;
  for (int w = 0; w < n_wls; w++) {
    dw[w].n = wls[w].n;
    dw[w].pad = 0;
    dw[w].I = reinterpret_cast<const int32_t*>(base + o_I) + wo;
    dw[w].O = reinterpret_cast<const int32_t*>(base + o_O) + wo;
    dw[w].T = reinterpret_cast<const double*>(base + o_T) + wo;
    wo += wls[w].n;
  }
  rc = 0;
  rc |= check_cuda(cudaMemcpyAsync(base + o_cfg, cfgs, sizeof(sim_config_t) * n_cfgs, cudaMemcpyHostToDevice, s));
  rc |= check_cuda(cudaMemcpyAsync(base + o_wl, dw.data(), sizeof(sim_workload_t) * n_wls, cudaMemcpyHostToDevice, s));
  rc |= check_cuda(cudaMemcpyAsync(base + o_cm, cms, sizeof(sim_cost_model_t) * n_cms, cudaMemcpyHostToDevice, s));
  rc |= check_cuda(cudaMemcpyAsync(base + o_ord, order.data(), 4 * (size_t)n_cfgs, cudaMemcpyHostToDevice, s));
  rc |= check_cuda(cudaMemcpyAsync(base + o_ro, row_off.data(), 8 * (size_t)n_cfgs, cudaMemcpyHostToDevice, s));
  rc |= check_cuda(cudaMemcpyAsync(base + o_to, tim_off.data(), 8 * (size_t)n_cfgs, cudaMemcpyHostToDevice, s));
  wo = 0;
  for (int w = 0; w < n_wls && !rc; w++) {
    rc |= check_cuda(cudaMemcpyAsync(base + o_I + 4 * wo, wls[w].I, 4 * (size_t)wls[w].n, cudaMemcpyHostToDevice, s));
    rc |= check_cuda(cudaMemcpyAsync(base + o_O + 4 * wo, wls[w].O, 4 * (size_t)wls[w].n, cudaMemcpyHostToDevice, s));
    rc |= check_cuda(cudaMemcpyAsync(base + o_T + 8 * wo, wls[w].T, 8 * (size_t)wls[w].n, cudaMemcpyHostToDevice, s));
    wo += wls[w].n;
  }
  sim_request_out_t dreq;
  dreq.t_first = reinterpret_cast<double*>(base + o_tf);
  dreq.t_done = reinterpret_cast<double*>(base + o_td);
  dreq.n_preempt = reinterpret_cast<int64_t*>(base + o_np);
  dreq.refill_tokens = reinterpret_cast<int64_t*>(base + o_rf);
  if (!rc) {
    int l = sim_sweep_device(cfgs, n_cfgs, wn.data(), reinterpret_cast<const sim_config_t*>(base + o_cfg),
                             reinterpret_cast<const sim_workload_t*>(base + o_wl),
                             reinterpret_cast<const sim_cost_model_t*>(base + o_cm), n_cms,
                             reinterpret_cast<const int32_t*>(base + o_ord),
                             reinterpret_cast<const int64_t*>(base + o_ro), reinterpret_cast<const int64_t*>(base + o_to),
                             reinterpret_cast<sim_result_t*>(base + o_res), dreq, s);
    if (l < 0) rc = l;
  }
  if (!rc) {
    rc |= check_cuda(cudaMemcpyAsync(results, base + o_res, sizeof(sim_result_t) * n_cfgs, cudaMemcpyDeviceToHost, s));
    if (req.t_first) rc |= check_cuda(cudaMemcpyAsync(req.t_first, dreq.t_first, 8 * trows, cudaMemcpyDeviceToHost, s));
    if (req.t_done) rc |= check_cuda(cudaMemcpyAsync(req.t_done, dreq.t_done, 8 * trows, cudaMemcpyDeviceToHost, s));
    if (req.n_preempt)
      rc |= check_cuda(cudaMemcpyAsync(req.n_preempt, dreq.n_preempt, 8 * rows, cudaMemcpyDeviceToHost, s));
    if (req.refill_tokens)
      rc |= check_cuda(cudaMemcpyAsync(req.refill_tokens, dreq.refill_tokens, 8 * rows, cudaMemcpyDeviceToHost, s));
    rc |= check_cuda(cudaStreamSynchronize(s));
  }
  cudaStreamDestroy(s);
  cudaFree(base);
  return rc ? SIM_ECUDA : 0;
}

}  // extern "C"
