// sim_kernel.cuh -- the sm_100a step kernel: one CTA per simulation.
//
// Each CTA runs Algorithm 1 for one sim_config_t with the
// request state as a structure of arrays in shared memory (a ring of CAP slots
// indexed by request id mod CAP).  Per step (one batch B_j):
//   a2  arrivals            binary search of the sorted T, slot init
//   a3  GroupRequests       stream compactions build the visiting order P
//   a4-a8 GetNextBatch      block-parallel "rounds": every remaining candidate is
//                           classified against the current (tok, U); a 4-component
//                           block prefix scan (tokens, KV delta, admissions, SRF+Hist
//                           remainders) finds the first candidate whose admission is
//                           not decided by the scan (a break); the prefix before it
//                           is admitted in parallel and thread 0 resolves the break
//                           literally (preemption victims = tail of the retention
//                           list, self-preemption, chunk cropping, deferral)
//   a9  batch latency       block reduction of exact int64 features, fp64 cost model
//                           (__dadd_rn/__dmul_rn/__ddiv_rn: no contraction)
//   a10 Process             parallel m += c, Eq. (6) token generation, completions
//   run-list maintenance    stable compaction (NRF = admission order); SRF order is
//                           re-sorted (bitonic) only when the compacted list is unsorted
// Semantics: DESIGN.md readings Q1-Q40, identical to oracle/oracle.cpp.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "simsweep.h"

namespace simsweep {

constexpr uint8_t ST_WAIT = 1, ST_RUN = 2, ST_DONE = 3, ST_MASK = 3;
constexpr uint8_t F_FILLED = 4, F_INB = 8, F_PRE = 16, F_FIRST = 32, F_LAST = 64;
constexpr int PH_DEC = 0, PH_PRE = 1;
constexpr int NOBRK = 0x7fffffff;

// per-step schedule trace of the launch's only simulation (sim_run_traced), else steps == nullptr
struct TraceDev {
  sim_trace_step_t* steps;
  sim_trace_entry_t* entries;
  sim_trace_event_t* events;
  long long cap_steps, cap_entries, cap_events;
};

struct KParams {
  unsigned char* ws;  // large-window variants: [WS_HEADER (arena counters) | arenas]
  const sim_config_t* cfgs;
  const sim_workload_t* wls;
  const sim_cost_model_t* cms;
  const int32_t* order;
  const int64_t* row_off;
  const int64_t* tim_off;
  sim_result_t* results;
  sim_request_out_t req;
  int32_t n_cfgs;
  int32_t variant;
  int32_t lean;        // route the eligible configs to the lean one-warp kernel (kernel_variant)
  int32_t arena_base;  // GM variants: this launch's first arena (the two GM variants may run concurrently)
  int32_t ctr_off;     // GM variants: byte offset of this launch's arena counter in the workspace header
  TraceDev tr;
};

// exact integer features of one batch (Table 3 variables; Eq. (1)-(2) sums)
struct Feat {
  long long N, np, c2, mc, cp, mp, pcm, nd, md;
  long long pceil[SIM_MAX_COST];
};

struct Scal {
  double clock[SIM_MAX_COST];
  sim_cost_model_t cm[SIM_MAX_COST];
  long long U, seq;
  long long steps, preempt, entries, processed, sumU, pentries, idle, visits, formed;
  long long runL, runMD, last_nd;
  long long tr_ent, tr_ev;  // trace records written before this step
  int runEx;
  long long pref[6];  // exclusive prefixes (c, dKV, admitted-waiting, admitted, SRF+Hist rem) at the break
  long long featsum[16];
  long long wred[16][20];  // per-warp partials of the process pass
  int next, new_next, lo, n_done, n_run, nW, nrank, minSW, n_ev, n_vic, nB, nRd;
  int cf_red[32][10];
  int pa, cut, h_pre, vmin, wstale, wfirst;
  int vt, status, any_pre, cur, wbuilt, arena;
  int idle_st;       // status of an idle jump (not S.status: thread 0 rewrites that at the next loop top)
  int wf_new, wf_vic;  // this step's new first waiting position / smallest victim index, committed at step end
  int w_dirty, p_dirty, r_dirty, o_dirty, rank_dirty, removals;
  long long r_Rs;  // scalars handed back by thread 0 after a break
  int r_tok, r_U, r_seq, r_new, r_running, r_bph, r_nB, r_wdone, r_wblk;
  int wmin[32];
  int wsum[32][6];
  int wcnt[32];
  int hist[18 * 18];
  int pred[18];
};

// thread 0, at the end of a step: the first window position that may hold a waiting request.  Warp 0 finds it
// during GetNextBatch (wf_new) while other warps may still read S.wfirst for this step, so it is staged and
// committed here together with the step's victims (wf_vic), which wait from the next step on.
__device__ __forceinline__ void wfirst_commit(Scal& S) {
  S.wfirst = min(S.wf_new >= 0 ? S.wf_new : S.wfirst, S.wf_vic);
  S.wf_new = -1, S.wf_vic = 0x7fffffff;
}

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double i2d(long long x) { return __ll2double_rn(x); }

// Eq. (3): max(FLOPs / GPU_FLOPS, RW / GPU_bandwidth), RW bytes = e * elements (Q26)
__device__ __forceinline__ double roof(long long F, long long R, const sim_cost_model_t& cm) {
  return fmax(ddiv(i2d(F), cm.flops), ddiv(i2d(R * (long long)cm.e), cm.bw));
}

// batch time d_j of one cost model from the batch features
__device__ double batch_time(const sim_cost_model_t& cm, const Feat& f, int k) {
  if (cm.mode == 1) {
    const long long h = cm.h, ff = cm.f, H = cm.H, NQ = cm.NQ, NKV = cm.NKV, N = f.N;
    const long long qo = (NQ + 2 * NKV) * H, ao = NQ * H;
    double t = 0.0;
    t = dadd(t, roof(2 * N * h * qo, h * qo + N * h + N * qo, cm));                     // QKV_proj
    t = dadd(t, roof(2 * N * ao * h, ao * h + N * ao + N * h, cm));                     // O_proj
    t = dadd(t, roof(2 * N * h * (2 * ff), h * (2 * ff) + N * h + N * (2 * ff), cm));  // gate+up
    t = dadd(t, roof(2 * N * ff * h, ff * h + N * ff + N * h, cm));                     // D_proj
    if (f.np > 0)  // prefill attention, Eq. (1)-(2) summed per request with B = 1 (Q24)
      t = dadd(t, roof(4 * H * NQ * f.pcm, 2 * H * NQ * f.cp + 2 * NQ * f.pcm + 2 * H * NKV * f.pceil[k], cm));
    if (f.nd > 0) {  // decode attention: c = 1, ceil(1/H) = 1
      const long long s1m = f.md + f.nd;
      t = dadd(t, roof(4 * H * NQ * s1m, 2 * H * NQ * f.nd + 2 * NQ * s1m + 2 * H * NKV * s1m, cm));
    }
    if (cm.tp > 1) {  // two All_Reduce per layer
      const double ar = ddiv(ddiv(i2d(2 * (long long)cm.e * N * h * (long long)(cm.tp - 1)), i2d(cm.tp)), cm.link_bw);
      t = dadd(t, ar);
      t = dadd(t, ar);
    }
    return dmul(i2d(cm.layers), t);
  }
  const double* a = cm.lin;
  double t = dadd(a[0], dmul(a[1], i2d(f.N)));
  if (f.np > 0)
    t = dadd(t, dadd(dadd(dadd(dadd(a[2], dmul(a[3], i2d(f.c2))), dmul(a[4], i2d(f.mc))), dmul(a[5], i2d(f.cp))),
                     dmul(a[6], i2d(f.mp))));
  if (f.nd > 0) t = dadd(t, dadd(dadd(a[7], dmul(a[8], i2d(f.md))), dmul(a[9], i2d(f.nd))));
  return dmul(i2d(cm.layers), t);
}

// The same d_j evaluated by a whole warp (lean kernel): lane 8k + j computes term j of model k's Eq. (3) sum (j < 4:
// the matmuls, 4: prefill attention, 5: decode attention, 6: the All_Reduce time), two divisions per lane instead of
// up to fourteen on one lane; lane k < K then adds its model's terms in the order of batch_time above (the same
// dadd sequence, so the same bits) or evaluates its linear model.  Every lane passes the same features; pceil[k] is
// model k's.  Returns d_j of model `lane` in lanes < K (0 elsewhere).  Warp-collective.
__device__ __forceinline__ double batch_time_warp(const sim_cost_model_t* cms, int K, const Feat& f, bool anyTheo) {
  const int lane = threadIdx.x & 31;
  double term = 0.0;
  if (anyTheo) {
    const int k = lane >> 3, j = lane & 7;
    if (k < K && j < 7 && cms[k].mode == 1) {
      const sim_cost_model_t& cm = cms[k];
      const long long h = cm.h, ff = cm.f, H = cm.H, NQ = cm.NQ, NKV = cm.NKV, N = f.N;
      const long long qo = (NQ + 2 * NKV) * H, ao = NQ * H;
      const long long s1m = f.md + f.nd;
      const long long pce = k == 0 ? f.pceil[0] : (k == 1 ? f.pceil[1] : (k == 2 ? f.pceil[2] : f.pceil[3]));
      // branch-free selection of the term's FLOPs F and elements R (exact integers, any association)
      const long long a_in = j == 0 ? h : (j == 1 ? ao : (j == 2 ? h : ff));
      const long long a_out = j == 0 ? qo : (j == 1 ? h : (j == 2 ? 2 * ff : h));
      const long long A = j == 4 ? f.pcm : s1m, B = j == 4 ? f.cp : f.nd, Cc = j == 4 ? pce : s1m;
      const long long F = j < 4 ? 2 * N * a_in * a_out
                                : (j < 6 ? 4 * H * NQ * A : 2 * (long long)cm.e * N * h * (long long)(cm.tp - 1));
      const long long R = j < 4 ? a_in * a_out + N * a_in + N * a_out : 2 * H * NQ * B + 2 * NQ * A + 2 * H * NKV * Cc;
      // roof: fmax(F / flops, e R / bw); All_Reduce: (F / tp) / link_bw.  Only the terms batch_time adds are
      // evaluated: a zero numerator would take the division's slow path (and the term is not summed anyway).
      const bool used = j < 4 || (j == 4 && f.np > 0) || (j == 5 && f.nd > 0) || (j == 6 && cm.tp > 1);
      if (used) {
        const double q1 = ddiv(i2d(F), j == 6 ? i2d(cm.tp) : cm.flops);
        const double q2 = ddiv(j == 6 ? q1 : i2d(R * (long long)cm.e), j == 6 ? cm.link_bw : cm.bw);
        term = j == 6 ? q2 : fmax(q1, q2);
      }
    }
  }
  const int src = 8 * (lane < 4 ? lane : 0);
  double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0, t4 = 0.0, t5 = 0.0, t6 = 0.0;
  if (anyTheo) {
    t0 = __shfl_sync(0xffffffffu, term, src), t1 = __shfl_sync(0xffffffffu, term, src + 1);
    t2 = __shfl_sync(0xffffffffu, term, src + 2), t3 = __shfl_sync(0xffffffffu, term, src + 3);
    t4 = __shfl_sync(0xffffffffu, term, src + 4), t5 = __shfl_sync(0xffffffffu, term, src + 5);
    t6 = __shfl_sync(0xffffffffu, term, src + 6);
  }
  double d = 0.0;
  if (lane < K) {
    const sim_cost_model_t& cm = cms[lane];
    if (cm.mode == 1) {
      double t = 0.0;
      t = dadd(t, t0);
      t = dadd(t, t1);
      t = dadd(t, t2);
      t = dadd(t, t3);
      if (f.np > 0) t = dadd(t, t4);
      if (f.nd > 0) t = dadd(t, t5);
      if (cm.tp > 1) {
        t = dadd(t, t6);
        t = dadd(t, t6);
      }
      d = dmul(i2d(cm.layers), t);
    } else {
      d = batch_time(cm, f, 0);
    }
  }
  return d;
}

// a / b rounded to nearest for a divisor b fixed per simulation, with y = RN(1/b) precomputed (__drcp_rn): q = RN(a y)
// and two residual corrections q <- RN(q + RN(a - b q) y), the residual from one FMA.  After the first correction q is
// within one ulp of a / b; the second is then Markstein's theorem (y within half an ulp of 1/b, q within one ulp of
// a / b => RN(q + (a - b q) y) = RN(a / b)), so the bits are __ddiv_rn's for the operands used here (a = 0 or an
// integer-valued double, b > 0 normal, normal quotient; tools/check_cdiv.c checks 128 M quotients).  Five dependent
// fp64 operations, no reciprocal iteration, no range check, no slow path.
__device__ __forceinline__ double cdiv(double a, double b, double y) {
  double q = __dmul_rn(a, y);
  q = __fma_rn(__fma_rn(-b, q, a), y, q);
  return __fma_rn(__fma_rn(-b, q, a), y, q);
}

// Eq. (3) term j of cost model k as integer coefficients (lean kernel, lane 8k + j; filled once per simulation):
// FLOPs F = cF * xF and e * elements R = c0 x0 + c1 x1 + c2 x2 with the batch variables
//   j < 4 (matmul a_in x a_out):  xF = N, x0 = 1, x1 = N       cF = 2 a_in a_out, c0 = e a_in a_out, c1 = e (a_in + a_out)
//   j = 4 (prefill attention):    xF = sum c(c+m), x0 = sum ceil(c/H)(c+m), x1 = sum c, x2 = sum c(c+m)
//                                 cF = 4 H NQ, c0 = 2 e H NKV, c1 = 2 e H NQ, c2 = 2 e NQ
//   j = 5 (decode attention):     xF = x2 = sum (m+1), x1 = n_d   cF = 4 H NQ, c1 = 2 e H NQ, c2 = e (2 NQ + 2 H NKV)
//   j = 6 (All_Reduce, tp > 1):   xF = N, cF = 2 e h (tp - 1); the time is (F / tp) / link_bw
// -- the integers batch_time forms (exact in int64, so any association gives the same values).  Lanes with j = 7,
// k >= K or a linear model hold zeros (their term is 0 and is not summed).
struct LTerm {
  long long cF, c0, c1, c2;
};
// per model: the two divisors of its terms and their reciprocals {flops, 1/flops, bw, 1/bw, tp, 1/tp, link_bw, 1/link_bw}
// (all 1 for a linear model, whose lanes divide zeros)
__device__ inline void lterm_fill(const sim_cost_model_t& cm, int j, LTerm& t, double* dv) {
  const long long h = cm.h, ff = cm.f, H = cm.H, NQ = cm.NQ, NKV = cm.NKV, e = cm.e;
  const long long qo = (NQ + 2 * NKV) * H, ao = NQ * H;
  t.cF = t.c0 = t.c1 = t.c2 = 0;
  if (cm.mode == 1 && j < 4) {
    const long long a_in = j == 0 ? h : (j == 1 ? ao : (j == 2 ? h : ff));
    const long long a_out = j == 0 ? qo : (j == 1 ? h : (j == 2 ? 2 * ff : h));
    t.cF = 2 * a_in * a_out, t.c0 = e * a_in * a_out, t.c1 = e * (a_in + a_out);
  } else if (cm.mode == 1 && j == 4) {
    t.cF = 4 * H * NQ, t.c0 = 2 * e * H * NKV, t.c1 = 2 * e * H * NQ, t.c2 = 2 * e * NQ;
  } else if (cm.mode == 1 && j == 5) {
    t.cF = 4 * H * NQ, t.c1 = 2 * e * H * NQ, t.c2 = e * (2 * NQ + 2 * H * NKV);
  } else if (cm.mode == 1 && j == 6 && cm.tp > 1) {
    t.cF = 2 * e * h * (long long)(cm.tp - 1);
  }
  if (j == 0 && cm.mode != 1) {
    for (int x = 0; x < 8; x++) dv[x] = 1.0;
  } else if (j == 0) {
    const double tp = i2d(cm.tp);
    dv[0] = cm.flops, dv[1] = __drcp_rn(cm.flops), dv[2] = cm.bw, dv[3] = __drcp_rn(cm.bw);
    dv[4] = tp, dv[5] = __drcp_rn(tp), dv[6] = cm.link_bw, dv[7] = __drcp_rn(cm.link_bw);
  }
}

// batch_time of model k on one lane from the term table (lean kernel's steady runs: one run step per lane): the same
// terms, order and bits as batch_time, the divisions by cdiv
__device__ __forceinline__ double batch_time_tab(const sim_cost_model_t& cm, const LTerm* tk, const double* dv,
                                                 const Feat& f, int k) {
  if (cm.mode != 1) return batch_time(cm, f, k);
  auto term = [&](int j, long long xF, long long x0, long long x1, long long x2) {
    const LTerm& t = tk[j];
    return fmax(cdiv(i2d(t.cF * xF), dv[0], dv[1]), cdiv(i2d(t.c0 * x0 + t.c1 * x1 + t.c2 * x2), dv[2], dv[3]));
  };
  const long long N = f.N, s1m = f.md + f.nd;
  double t = 0.0;
#pragma unroll
  for (int j = 0; j < 4; j++) t = dadd(t, term(j, N, 1, N, 0));
  if (f.np > 0) t = dadd(t, term(4, f.pcm, f.pceil[k], f.cp, f.pcm));
  if (f.nd > 0) t = dadd(t, term(5, s1m, 0, f.nd, s1m));
  if (cm.tp > 1) {
    const double ar = cdiv(cdiv(i2d(tk[6].cF * N), dv[4], dv[5]), dv[6], dv[7]);
    t = dadd(t, ar);
    t = dadd(t, ar);
  }
  return dmul(i2d(cm.layers), t);
}

// batch_time_warp with the per-lane term table (lean kernel): lane 8k + j evaluates term j of model k branch-free
// (cdiv; a zero numerator is exact), lane k < K adds its model's terms in batch_time's order.  Same bits.
__device__ __forceinline__ double batch_time_lanes(const sim_cost_model_t* cms, const LTerm* terms, const double (*dv)[8],
                                                   int K, const Feat& f, bool anyTheo) {
  const int lane = threadIdx.x & 31;
  double term = 0.0;
  if (anyTheo) {
    const int k = lane >> 3, j = lane & 7;
    const LTerm t = terms[lane];
    const long long pce = k == 0 ? f.pceil[0] : (k == 1 ? f.pceil[1] : (k == 2 ? f.pceil[2] : f.pceil[3]));
    const long long s1m = f.md + f.nd;
    const long long xF = j == 4 ? f.pcm : (j == 5 ? s1m : f.N);
    const long long x0 = j == 4 ? pce : 1, x1 = j < 4 ? f.N : (j == 4 ? f.cp : f.nd), x2 = j == 4 ? f.pcm : s1m;
    const long long F = t.cF * xF, Re = t.c0 * x0 + t.c1 * x1 + t.c2 * x2;
    const double* d = dv[k] + (j == 6 ? 4 : 0);
    const double q1 = cdiv(i2d(F), d[0], d[1]);
    const double q2 = cdiv(j == 6 ? q1 : i2d(Re), d[2], d[3]);
    term = j == 6 ? q2 : fmax(q1, q2);
  }
  const int src = 8 * (lane < 4 ? lane : 0);
  double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0, t4 = 0.0, t5 = 0.0, t6 = 0.0;
  if (anyTheo) {
    t0 = __shfl_sync(0xffffffffu, term, src), t1 = __shfl_sync(0xffffffffu, term, src + 1);
    t2 = __shfl_sync(0xffffffffu, term, src + 2), t3 = __shfl_sync(0xffffffffu, term, src + 3);
    t4 = __shfl_sync(0xffffffffu, term, src + 4), t5 = __shfl_sync(0xffffffffu, term, src + 5);
    t6 = __shfl_sync(0xffffffffu, term, src + 6);
  }
  double d = 0.0;
  if (lane < K) {
    const sim_cost_model_t& cm = cms[lane];
    if (cm.mode == 1) {
      double t = 0.0;
      t = dadd(t, t0);
      t = dadd(t, t1);
      t = dadd(t, t2);
      t = dadd(t, t3);
      if (f.np > 0) t = dadd(t, t4);
      if (f.nd > 0) t = dadd(t, t5);
      if (cm.tp > 1) {
        t = dadd(t, t6);
        t = dadd(t, t6);
      }
      d = dmul(i2d(cm.layers), t);
    } else {
      d = batch_time(cm, f, 0);
    }
  }
  return d;
}

__device__ __forceinline__ int bucket_of(int x) {  // floor(log2 x), capped at 17
  int b = 31 - __clz(x);
  return b > 17 ? 17 : b;
}

// SRF+Hist predicted output length per I-bucket (reading Q31): nearest-rank p90 bucket edge
__device__ int hist_pred_row(const int* H, int bi) {
  long long n = 0;
  for (int b = 0; b < 18; b++) n += H[bi * 18 + b];
  if (n >= 8) {
    long long target = (9 * n + 9) / 10, cum = 0;
    for (int b = 0; b < 18; b++) {
      cum += H[bi * 18 + b];
      if (cum >= target) return (1 << (b + 1)) - 1;
    }
  }
  long long col[18];
  n = 0;
  for (int b = 0; b < 18; b++) {
    col[b] = 0;
    for (int a = 0; a < 18; a++) col[b] += H[a * 18 + b];
    n += col[b];
  }
  if (n >= 8) {
    long long target = (9 * n + 9) / 10, cum = 0;
    for (int b = 0; b < 18; b++) {
      cum += col[b];
      if (cum >= target) return (1 << (b + 1)) - 1;
    }
  }
  return 256;
}

// block-wide exclusive scan of one int per thread; returns the prefix, total in *tot.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, Scal& S, int* tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) S.wcnt[wid] = x;
  __syncthreads();
  int off = 0, t = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; w++) {
    int s = S.wcnt[w];
    off += (w < wid) ? s : 0;
    t += s;
  }
  __syncthreads();
  *tot = t;
  return off + x - v;
}

// stable stream compaction of positions [0, L) satisfying pred into out[...]; returns the count.
// Ends with a barrier: the output is visible to the whole block.
template <int NT, int IPT_, typename Pred, typename Val>
__device__ int block_compact(int L, Pred pred, Val val, int16_t* out, Scal& S) {
  int total = 0;
  for (int base = 0; base < L; base += NT * IPT_) {
    int flags = 0, cnt = 0;
#pragma unroll
    for (int j = 0; j < IPT_; j++) {
      int q = base + threadIdx.x * IPT_ + j;
      if (q < L && pred(q)) {
        flags |= 1 << j;
        cnt++;
      }
    }
    int tot;
    int w = total + block_excl_scan<NT>(cnt, S, &tot);
#pragma unroll
    for (int j = 0; j < IPT_; j++)
      if (flags >> j & 1) out[w++] = (int16_t)val(base + threadIdx.x * IPT_ + j);
    total += tot;
  }
  __syncthreads();
  return total;
}

// as block_compact, plus the minimum of key(val(q)) over the selected positions (INT_MAX if none)
template <int NT, int IPT_, typename Pred, typename Val, typename Key>
__device__ int block_compact_min(int L, Pred pred, Val val, Key key, int16_t* out, Scal& S, int* minv) {
  int total = 0, mn = 0x7fffffff;
  for (int base = 0; base < L; base += NT * IPT_) {
    int flags = 0, cnt = 0;
#pragma unroll
    for (int j = 0; j < IPT_; j++) {
      int q = base + threadIdx.x * IPT_ + j;
      if (q < L && pred(q)) {
        flags |= 1 << j;
        cnt++;
        mn = min(mn, key(val(q)));
      }
    }
    int tot;
    int w = total + block_excl_scan<NT>(cnt, S, &tot);
#pragma unroll
    for (int j = 0; j < IPT_; j++)
      if (flags >> j & 1) out[w++] = (int16_t)val(base + threadIdx.x * IPT_ + j);
    total += tot;
  }
  mn = (int)__reduce_min_sync(0xffffffffu, (unsigned)mn);
  if ((threadIdx.x & 31) == 0) S.wmin[threadIdx.x >> 5] = mn;
  __syncthreads();
  int m = 0x7fffffff;
#pragma unroll
  for (int w = 0; w < NT / 32; w++) m = min(m, S.wmin[w]);
  __syncthreads();
  *minv = m;
  return total;
}

// stable partition of positions [0, L): pred-true items (in order), then the others (in order).
// One 2-component scan when L fits one pass.  Ends with a barrier.
template <int NT, int IPT_, typename Pred, typename Val>
__device__ int block_partition(int L, Pred pred, Val val, int16_t* out, Scal& S) {
  if (L > NT * IPT_) {
    const int nt = block_compact<NT, IPT_>(L, pred, val, out, S);
    block_compact<NT, IPT_>(L, [&](int q) { return !pred(q); }, val, out + nt, S);
    return nt;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int flags = 0, ct = 0, cf = 0;
#pragma unroll
  for (int j = 0; j < IPT_; j++) {
    const int q = threadIdx.x * IPT_ + j;
    if (q < L) {
      if (pred(q))
        flags |= 1 << j, ct++;
      else
        cf++;
    }
  }
  int xt = ct, xf = cf;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int yt = __shfl_up_sync(0xffffffffu, xt, o), yf = __shfl_up_sync(0xffffffffu, xf, o);
    if (lane >= o) xt += yt, xf += yf;
  }
  if (lane == 31) S.wsum[wid][0] = xt, S.wsum[wid][1] = xf;
  __syncthreads();
  int ot = xt - ct, of = xf - cf, tt = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; w++) {
    const int a = S.wsum[w][0], b = S.wsum[w][1];
    if (w < wid) ot += a, of += b;
    tt += a;
  }
  of += tt;
#pragma unroll
  for (int j = 0; j < IPT_; j++) {
    const int q = threadIdx.x * IPT_ + j;
    if (q < L) out[(flags >> j & 1) ? ot++ : of++] = (int16_t)val(q);
  }
  __syncthreads();
  return tt;
}

// ascending bitonic sort of keys[0, L) (padded with ~0 to a power of two <= CAP)
template <int NT>
__device__ void block_bitonic(unsigned long long* keys, int L) {
  int P2 = 1;
  while (P2 < L) P2 <<= 1;
  for (int i = L + threadIdx.x; i < P2; i += NT) keys[i] = ~0ull;
  __syncthreads();
  for (int k = 2; k <= P2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P2; i += NT) {
        int ixj = i ^ j;
        if (ixj > i) {
          unsigned long long a = keys[i], b = keys[ixj];
          bool up = (i & k) == 0;
          if ((a > b) == up) {
            keys[i] = b;
            keys[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Per-slot arrays (51 B per slot), relative to the array base: shared memory right after Scal, or (GM
// variant) a per-CTA arena in a caller-provided global workspace, served from L1/L2.
template <int NT, int CAP>
struct Smem {
  static constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
  static constexpr size_t scal = align16(sizeof(Scal));
  static constexpr size_t off_rec = 0;                              // int4 {I, g, m, res} per slot
  static constexpr size_t off_int = off_rec + 16 * CAP;             // O, seq, c (int32)
  static constexpr size_t off_rpos = off_int + 3 * 4 * CAP;         // position in the run list (int16)
  static constexpr size_t off_fl = off_rpos + 2 * CAP;              // flags (uint8)
  static constexpr size_t off_lists = align16(off_fl + CAP);        // runA runB rank wl pl blist (int16)
  // union, 8 B per slot: new (int16) | vic (int16) | ev (int32) -- the steady-run dbuf overlays ev (a steady
  // run has no events) -- or the u64 sort keys
  static constexpr size_t off_union = align16(off_lists + 6 * 2 * CAP);
  static constexpr size_t arr_bytes = (off_union + 8 * CAP + 255) & ~size_t(255);
  static constexpr size_t bytes = scal + arr_bytes;  // all in shared memory
};
constexpr size_t WS_HEADER = 256;  // workspace header: the arena counters (one per GM variant, 64 B apart)

}  // namespace simsweep
