// sim_optimum.cuh -- exact optimum of the paper's CSP for tiny workloads (included by
// simsweep.cu).  PAPER.md:317-411, readings Q43-Q45.
//
// Dense state space: request i's local state is 0 = done, else (g, m, filled) at base_i[g] + m (not filled,
// m < I + g) or base_i[g] + I + g (filled, g >= 1); identical requests are stored as the multiset of their local
// states (see OptDev), so the all-done goal is state 0.  Relaxation rounds: every state improved in the last
// round expands every batch it can form (all per-request choices: idle, preempt, any c) and lowers the
// distance of the successor with a 64-bit atomicMin on the bits of the non-negative fp64 path sum.  Rounds
// repeat until nothing improves; the fixed point is the minimum over all schedules of the sequential sums
// (rounding is monotone, so extending a minimal prefix is minimal -- the same value Dijkstra finds).
#pragma once

namespace simsweep {

constexpr int OPT_MAXN = SIM_OPT_MAX_N;
constexpr int OPT_MAXO = 64;
constexpr unsigned long long OPT_INF = 0x7ff0000000000000ull;  // +inf

// Requests are sorted by (I, O); a group is a run of identical requests.  Identical requests are interchangeable
// (permuting them maps every schedule to one of the same cost), so a state is stored once, as the multiset of
// its group's local states: the sorted tuple a_1 <= ... <= a_k is ranked in the combinatorial number system of
// multisets, rank = sum_j binom(a_j + j - 1, j), and the global state is the mixed-radix number of the group
// ranks (radix binom(ns + k - 1, k)).  The all-done goal (every a = 0) is state 0.
struct OptDev {
  int n;
  int I[OPT_MAXN], O[OPT_MAXN];
  long long C, M;
  long long ns[OPT_MAXN];
  int base[OPT_MAXN][OPT_MAXO + 1];
  int nopre;               // SIM_OPT_NO_PREEMPT: preemption-free schedules only
  int ng;                  // groups
  int gs[OPT_MAXN], gk[OPT_MAXN];  // first request and size of each group
  long long gstride[OPT_MAXN];     // mixed-radix stride of each group's rank
};

__host__ __device__ inline long long opt_binom(long long x, int j) {  // binom(x, j), j <= 4, 0 if x < j
  if (x < j) return 0;
  long long r = 1;
  for (int t = 0; t < j; t++) r = r * (x - t) / (t + 1);
  return r;
}

// rank of the sorted tuple a[0..k) (non-decreasing local states) among the multisets of size k
__host__ __device__ inline long long opt_rank(const int* a, int k) {
  long long r = 0;
  for (int j = 0; j < k; j++) r += opt_binom((long long)a[j] + j, j + 1);
  return r;
}

// inverse of opt_rank: the sorted tuple with rank r (local states < ns)
__device__ inline void opt_unrank(long long r, int k, long long ns, int* a) {
  for (int j = k - 1; j >= 0; j--) {  // the largest b = a_j + j with binom(b, j + 1) <= r
    long long lo = j, hi = ns - 1 + j;
    while (lo < hi) {
      const long long mid = (lo + hi + 1) >> 1;
      if (opt_binom(mid, j + 1) <= r)
        lo = mid;
      else
        hi = mid - 1;
    }
    r -= opt_binom(lo, j + 1);
    a[j] = (int)(lo - j);
  }
}

// the global index of per-request local states l[0..n) (canonical: each group's states sorted)
__device__ inline long long opt_index(const OptDev& P, const int* l) {
  long long v = 0;
  for (int q = 0; q < P.ng; q++) {
    int a[OPT_MAXN];
    const int k = P.gk[q];
    for (int t = 0; t < k; t++) a[t] = l[P.gs[q] + t];
    for (int x = 1; x < k; x++)  // insertion sort (k <= 4)
      for (int y = x; y > 0 && a[y - 1] > a[y]; y--) {
        const int tmp = a[y];
        a[y] = a[y - 1], a[y - 1] = tmp;
      }
    v += opt_rank(a, k) * P.gstride[q];
  }
  return v;
}

__global__ void opt_round_kernel(OptDev P, sim_cost_model_t cm, unsigned long long* dist, unsigned char* cur,
                                 unsigned char* nxt, long long nstates, int* changed, long long* reached) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < nstates;
       u += (long long)gridDim.x * blockDim.x) {
    if (!cur[u]) continue;
    cur[u] = 0;
    const double du = __longlong_as_double((long long)dist[u]);
    int g[OPT_MAXN], s[OPT_MAXN], nopt[OPT_MAXN];
    long long m[OPT_MAXN];
    bool fl[OPT_MAXN], dn[OPT_MAXN];
    int loc[OPT_MAXN];
    {
      long long rest = u;
      for (int q = P.ng - 1; q >= 0; q--) {  // decode the group ranks (mixed radix), then each group's tuple
        const long long gr = rest / P.gstride[q];
        rest -= gr * P.gstride[q];
        opt_unrank(gr, P.gk[q], P.ns[P.gs[q]], loc + P.gs[q]);
      }
    }
    for (int i = 0; i < P.n; i++) {  // decode the local states
      const int l = loc[i];
      dn[i] = l == 0, g[i] = 0, m[i] = 0, fl[i] = false;
      if (!dn[i]) {
        int gg = 0;
        while (gg + 1 < P.O[i] && P.base[i][gg + 1] <= l) gg++;
        g[i] = gg;
        const int off = l - P.base[i][gg];
        fl[i] = off == P.I[i] + gg;
        m[i] = fl[i] ? P.I[i] + gg - 1 : off;
      }
      s[i] = P.I[i] + g[i];
      nopt[i] = dn[i] ? 1 : 1 + (m[i] > 0) + (int)(s[i] - m[i]);  // idle, preempt, c = 1 .. s - m
    }
    // every batch this state can form: depth-first over the requests' choices (0 idle, 1 preempt when m > 0,
    // then c = 1 .. s - m), pruned by Eq. (7) -- both sums only grow with depth, and a larger c needs more
    int oi[OPT_MAXN];
    long long scs[OPT_MAXN + 1], sms[OPT_MAXN + 1];
    int lvl = 0;
    oi[0] = -1, scs[0] = 0, sms[0] = 0;
    while (lvl >= 0) {
      const int i = lvl;
      if (++oi[i] >= nopt[i]) {
        lvl--;
        continue;
      }
      const int o = oi[i];
      const bool pre = !dn[i] && m[i] > 0 && o == 1;
      if (pre && P.nopre) continue;  // preemption-free schedules only
      const long long c = (dn[i] || o == 0 || pre) ? 0 : o - (m[i] > 0 ? 1 : 0);
      const long long m2 = dn[i] || pre ? 0 : m[i] + c;
      if (scs[i] + c > P.C || sms[i] + m2 > P.M) {
        if (c > 0) oi[i] = nopt[i];  // every larger chunk fails as well
        continue;
      }
      scs[i + 1] = scs[i] + c, sms[i + 1] = sms[i] + m2;
      if (i + 1 < P.n) {
        lvl++;
        oi[lvl] = -1;
        continue;
      }
      if (scs[P.n] == 0) continue;  // no empty batch (Q43)
      int nl[OPT_MAXN];
      Feat f;
      f.N = f.np = f.cp = f.mp = f.c2 = f.mc = f.pcm = f.nd = f.md = 0;
      f.pceil[0] = f.pceil[1] = f.pceil[2] = f.pceil[3] = 0;
      for (int j = 0; j < P.n; j++) {
        int l = 0;
        const int oj = oi[j];
        if (!dn[j]) {
          if (oj == 0) {  // idle: c = 0, e = 0
            l = fl[j] ? P.base[j][g[j]] + P.I[j] + g[j] : P.base[j][g[j]] + (int)m[j];
          } else if (m[j] > 0 && oj == 1) {  // preempt (Eq. (4))
            l = P.base[j][g[j]];
          } else {  // process cj tokens (Eq. (5)-(6)); a request finishing now still holds m + cj (Q44)
            const long long cj = oj - (m[j] > 0 ? 1 : 0);
            if (cj == s[j] - m[j])  // a token: done, or filled at g + 1
              l = g[j] + 1 == P.O[j] ? 0 : P.base[j][g[j] + 1] + P.I[j] + g[j] + 1;
            else
              l = P.base[j][g[j]] + (int)(m[j] + cj);
            f.N += cj;
            if (fl[j]) {  // decode entry (Q17, Q45)
              f.nd++, f.md += m[j];
            } else {
              f.np++, f.cp += cj, f.mp += m[j], f.c2 += cj * cj, f.mc += m[j] * cj, f.pcm += cj * (cj + m[j]);
              f.pceil[0] += ((cj + cm.H - 1) / cm.H) * (cj + m[j]);
            }
          }
        }
        nl[j] = l;
      }
      const long long v = opt_index(P, nl);
      const double cand = dadd(du, batch_time(cm, f, 0));
      const unsigned long long cb = (unsigned long long)__double_as_longlong(cand);
      const unsigned long long old = atomicMin(&dist[v], cb);
      if (cb < old) {
        nxt[v] = 1;
        *changed = 1;
        if (old == OPT_INF) atomicAdd((unsigned long long*)reached, 1ull);
      }
    }
  }
}

}  // namespace simsweep
