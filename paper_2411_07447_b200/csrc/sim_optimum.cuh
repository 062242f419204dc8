// sim_optimum.cuh -- exact optimum of the paper's CSP for tiny workloads (included by
// simsweep.cu).  PAPER.md:317-411, readings Q43-Q45.
//
// Dense state space: request i's local state is 0 = done, else (g, m, filled) at base_i[g] + m (not filled,
// m < I + g) or base_i[g] + I + g (filled, g >= 1); the global state is the mixed-radix number of the local
// states (stride_i), so the all-done goal is state 0.  Relaxation rounds: every state improved in the last
// round expands every batch it can form (all per-request choices: idle, preempt, any c) and lowers the
// distance of the successor with a 64-bit atomicMin on the bits of the non-negative fp64 path sum.  Rounds
// repeat until nothing improves; the fixed point is the minimum over all schedules of the sequential sums
// (rounding is monotone, so extending a minimal prefix is minimal -- the same value Dijkstra finds).
#pragma once

namespace simsweep {

constexpr int OPT_MAXN = SIM_OPT_MAX_N;
constexpr int OPT_MAXO = 64;
constexpr unsigned long long OPT_INF = 0x7ff0000000000000ull;  // +inf

struct OptDev {
  int n;
  int I[OPT_MAXN], O[OPT_MAXN];
  long long C, M;
  long long ns[OPT_MAXN], stride[OPT_MAXN];
  int base[OPT_MAXN][OPT_MAXO + 1];
};

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
    for (int i = 0; i < P.n; i++) {  // decode the local states
      const int l = (int)((u / P.stride[i]) % P.ns[i]);
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
      long long v = 0;
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
        v += (long long)l * P.stride[j];
      }
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
