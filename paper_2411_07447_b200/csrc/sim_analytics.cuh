// sim_analytics.cuh -- cost-model analytics (included by simsweep.cu).
//
// The batch-latency model of row a9 (batch_time, sim_kernel.cuh) evaluated on batch SHAPES -- n_p prefill
// entries (c, m_p) and n_d decode entries (m_d) -- instead of simulated batches.  A shape's integer features
// are the sums Process forms over the same entries (Table 3 variables, Eq. (1)-(2) per request), so a shape
// gets bit for bit the d_j a simulated batch with those entries gets.  One thread per (model, item).
#pragma once

namespace simsweep {

// exact integer features of n_p identical prefill entries (c, m_p) and n_d identical decodes (m_d);
// pceil[0] is the per-request ceil(c/H)(c+m) sum for the model the caller evaluates (H of that model)
__device__ __forceinline__ Feat shape_features(long long n_p, long long c, long long m_p, long long n_d, long long m_d,
                                               int H) {
  Feat f;
  if (n_p == 0) c = 0, m_p = 0;
  f.N = n_p * c + n_d;
  f.np = n_p;
  f.cp = n_p * c;
  f.mp = n_p * m_p;
  f.c2 = n_p * (c * c);
  f.mc = n_p * (m_p * c);
  f.pcm = n_p * (c * (c + m_p));
  f.nd = n_d;
  f.md = n_d * m_d;
  f.pceil[0] = n_p * (((c + H - 1) / H) * (c + m_p));
  f.pceil[1] = f.pceil[2] = f.pceil[3] = 0;
  return f;
}

__global__ void batch_times_kernel(const sim_cost_model_t* cms, int n_cms, const sim_batch_shape_t* shapes, int n,
                                   double* out) {
  const long long total = (long long)n * n_cms;
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total; x += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(x / n), i = (int)(x % n);
    const sim_cost_model_t& cm = cms[k];
    const sim_batch_shape_t b = shapes[i];
    out[x] = batch_time(cm, shape_features(b.n_p, b.c, b.m_p, b.n_d, b.m_d, cm.H), 0);
  }
}

// largest m in [0, m_max] with d(n_p prefills (c, m), n_d decodes (m)) <= tau, -1 if none (d is non-decreasing in m)
__global__ void slo_frontier_kernel(const sim_cost_model_t* cms, int n_cms, const sim_slo_query_t* qs, int n,
                                    long long* out) {
  const long long total = (long long)n * n_cms;
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total; x += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(x / n), i = (int)(x % n);
    const sim_cost_model_t& cm = cms[k];
    const sim_slo_query_t q = qs[i];
    auto ok = [&](long long m) { return batch_time(cm, shape_features(q.n_p, q.c, m, q.n_d, m, cm.H), 0) <= q.tau; };
    long long r = -1;
    if (ok(0)) {
      long long lo = 0, hi = q.m_max + 1;  // ok(lo); hi is beyond the range
      while (hi - lo > 1) {
        const long long mid = lo + (hi - lo) / 2;
        if (ok(mid))
          lo = mid;
        else
          hi = mid;
      }
      r = lo;
    }
    out[x] = r;
  }
}

// refill (recompute) time of N KVs, host-link swap time of their K and V, and the break-even interval
__global__ void kv_break_even_kernel(const sim_cost_model_t* cms, int n_cms, const long long* Ns, int n, double xfer_bw,
                                     long long M, double* rec, double* swp, double* itv) {
  const long long total = (long long)n * n_cms;
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total; x += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(x / n), i = (int)(x % n);
    const sim_cost_model_t& cm = cms[k];
    const long long N = Ns[i];
    const double t = batch_time(cm, shape_features(1, N, 0, 0, 0, cm.H), 0);
    const long long kv_bytes = 2ll * cm.layers * cm.NKV * cm.H * cm.e;  // K and V of one token, all layers
    if (rec) rec[x] = t;
    if (swp) swp[x] = ddiv(i2d(N * kv_bytes), xfer_bw);
    if (itv) itv[x] = dmul(ddiv(t, i2d(N)), i2d(M));
  }
}

// Per-operator roofline classification of one layer ("What Makes a Batch Compute-Bound?"):
// the operators of Eq. (3) in batch_time's order, each with its FLOPs, RW elements, Eq. (3) time, intensity
// FLOPs / RW and compute- vs memory-boundness.  Attention is summed per request with B = 1 (Q24).
__device__ __forceinline__ void op_cost(long long F, long long R, const sim_cost_model_t& cm, sim_op_cost_t& o) {
  const double tc = ddiv(i2d(F), cm.flops), tm = ddiv(i2d(R * (long long)cm.e), cm.bw);
  o.flops = F;
  o.rw = R;
  o.time = fmax(tc, tm);  // == roof(F, R, cm)
  o.intensity = R > 0 ? ddiv(i2d(F), i2d(R)) : 0.0;
  o.bound = tc > tm ? 1 : 0;
  o.pad = 0;
}

__global__ void operator_costs_kernel(const sim_cost_model_t* cms, int n_cms, const sim_batch_shape_t* shapes, int n,
                                      sim_op_cost_t* out) {
  const long long total = (long long)n * n_cms;
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total; x += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(x / n), i = (int)(x % n);
    const sim_cost_model_t& cm = cms[k];
    const sim_batch_shape_t b = shapes[i];
    const Feat f = shape_features(b.n_p, b.c, b.m_p, b.n_d, b.m_d, cm.H);
    const long long h = cm.h, ff = cm.f, H = cm.H, NQ = cm.NQ, NKV = cm.NKV, N = f.N;
    const long long qo = (NQ + 2 * NKV) * H, ao = NQ * H;
    sim_op_cost_t* o = out + x * SIM_N_OPS;
    op_cost(2 * N * h * qo, h * qo + N * h + N * qo, cm, o[SIM_OP_QKV]);
    op_cost(2 * N * ao * h, ao * h + N * ao + N * h, cm, o[SIM_OP_O]);
    op_cost(2 * N * h * (2 * ff), h * (2 * ff) + N * h + N * (2 * ff), cm, o[SIM_OP_GATE_UP]);
    op_cost(2 * N * ff * h, ff * h + N * ff + N * h, cm, o[SIM_OP_DOWN]);
    if (f.np > 0) {
      op_cost(4 * H * NQ * f.pcm, 2 * H * NQ * f.cp + 2 * NQ * f.pcm + 2 * H * NKV * f.pceil[0], cm, o[SIM_OP_ATTN_PREFILL]);
    } else {
      o[SIM_OP_ATTN_PREFILL] = sim_op_cost_t{0, 0, 0.0, 0.0, -1, 0};
    }
    if (f.nd > 0) {
      const long long s1m = f.md + f.nd;
      op_cost(4 * H * NQ * s1m, 2 * H * NQ * f.nd + 2 * NQ * s1m + 2 * H * NKV * s1m, cm, o[SIM_OP_ATTN_DECODE]);
    } else {
      o[SIM_OP_ATTN_DECODE] = sim_op_cost_t{0, 0, 0.0, 0.0, -1, 0};
    }
  }
}

}  // namespace simsweep
