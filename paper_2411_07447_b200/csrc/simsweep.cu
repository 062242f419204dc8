// simsweep.cu -- libsimsweep.so: CTA-per-simulation step kernel (sm_100a) and
// the C-ABI of include/simsweep.h.  See sim_kernel.cuh for the per-step plan.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <cmath>
#include <numeric>
#include <vector>

#include "sim_kernel.cuh"
#include "simsweep.h"

namespace simsweep {


#ifdef SIMSWEEP_PROFILE  // phase cycle counters of thread 0 (tools/probe.py); not in the product build
constexpr int PROF_MAX_CFG = 8192;
__device__ long long g_prof[PROF_MAX_CFG][24];
constexpr int DBG_STEPS = 1 << 16;
__device__ int g_dbg[DBG_STEPS][6];  // config 0 only: per full step (steps, tok, U, nB, preemptions, n_vic)
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

#ifdef SIMSWEEP_TRACE  // clock marks of thread 0 of config 0 (tools/tmarks.py); not in the product build
constexpr int TR_MAX = 1 << 22;
__device__ unsigned g_tr[TR_MAX];
__device__ int g_trn;
#define TMARK(i)                                               \
  if (tid == 0 && ci == 0) {                                   \
    unsigned _c;                                               \
    asm volatile("mov.u32 %0, %%clock;" : "=r"(_c)::"memory"); \
    if (trn < TR_MAX / 2) g_tr[2 * trn] = (i), g_tr[2 * trn + 1] = _c; \
    trn++;                                                     \
  }
#else
#define TMARK(i)
#endif

// 0: W <= 1024 and 1: W <= 4096, state in shared memory (the window never exceeds n <= CAP);
// 2: larger workloads, a 32768-slot ring in a per-CTA global-memory arena (SIM_MAX_WINDOW)
__host__ __device__ inline int variant_of(int n) { return n <= 1024 ? 0 : (n <= 4096 ? 1 : 2); }
constexpr int N_SIZES = 3;
// configs with an alternative-reading knob run in a second instance of each size (KN = true), so that the
// default instances carry none of the knob checks
constexpr int32_t SIM_KNOB_TRACE_INTERNAL = 1 << 30;  // set by sim_run_traced only (routes to the KN instance)
__host__ __device__ inline bool has_knobs(const sim_config_t& c) {
  return c.knobs || c.max_seqs || c.kv_watermark || c.kv_block > 1;
}
constexpr int N_GENERAL = 2 * N_SIZES;
// the lean one-warp kernel (sim_lean.cuh) for the configurations that dominate the north-star sweep: the vLLM /
// Sarathi presets (prefill-first without chunking, or decode-first), NRF / SRF / PF, no knob, no SRF+Hist, no trace
constexpr int V_LEAN = N_GENERAL;  // + 0: n <= 1024, + 1: n <= 4096 (state in shared memory), + 2: n <= 32768 (arena)
constexpr int N_VARIANTS = N_GENERAL + 3;
// (n > 4096 with M infinite runs here too: its run list can be as long as the window, but the SRF merge shifts the
// kept list range by range instead of sorting it, and a 512-thread block-kernel CTA holds a whole SM's register file
// for the simulation's duration, 0.5-0.75 s for the 70B AzureConv runs of the north-star sweep)
__host__ __device__ inline bool lean_ok(const sim_config_t& c, int n) {
  return !has_knobs(c) && n <= SIM_MAX_WINDOW &&
         ((c.order == SIM_ORDER_PREFILL_FIRST && !c.chunked) || c.order == SIM_ORDER_DECODE_FIRST);
}
__host__ __device__ inline int kernel_variant(const sim_config_t& c, int n, int lean) {
  if (lean && lean_ok(c, n)) return V_LEAN + (n <= 1024 ? 0 : (n <= 4096 ? 1 : 2));
  return variant_of(n) + (has_knobs(c) ? N_SIZES : 0);
}

#ifndef SIM_NT_SMALL
#define SIM_NT_SMALL 256  // threads per CTA of the W <= 1024 variant
#endif
#ifndef SIM_IPT_SMALL
#define SIM_IPT_SMALL (1024 / SIM_NT_SMALL)  // candidates per thread and round of the W <= 1024 variant
#endif

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

}  // namespace simsweep

#include "sim_step.cuh"
#include "sim_lean.cuh"
#include "sim_analytics.cuh"
#include "sim_optimum.cuh"

namespace simsweep {

// ------------------------------------------------------------------ host side
struct Variant {
  int nt, cap;
  size_t smem;   // dynamic shared memory per CTA
  size_t arena;  // global workspace per CTA (GM variant), else 0
  void (*fn)(KParams);
};

template <int NT, int CAP, int IPT_, bool GM, bool KN>
Variant make_variant() {
  using L = Smem<NT, CAP>;
  return Variant{NT, CAP, GM ? L::scal : L::bytes, GM ? L::arr_bytes : 0, sim_kernel<NT, CAP, IPT_, GM, KN>};
}
template <int CAP, bool GM>
Variant make_lean() {
  return Variant{32, CAP, LLayout<CAP, GM>::smem, GM ? Smem<512, SIM_MAX_WINDOW>::arr_bytes : 0, sim_lean_kernel<CAP, GM>};
}

static Variant g_variants[N_VARIANTS] = {
    make_variant<SIM_NT_SMALL, 1024, SIM_IPT_SMALL, false, false>(), make_variant<512, 4096, 4, false, false>(),
    make_variant<512, SIM_MAX_WINDOW, 4, true, false>(),           make_variant<SIM_NT_SMALL, 1024, SIM_IPT_SMALL, false, true>(),
    make_variant<512, 4096, 4, false, true>(),                     make_variant<512, SIM_MAX_WINDOW, 4, true, true>(),
    make_lean<1024, false>(),                                      make_lean<4096, false>(),
    make_lean<SIM_MAX_WINDOW, true>()};

// SIMSWEEP_LEAN=0 in the environment routes every config to the block kernel (parity tests run both kernels)
static int lean_enabled() {
  const char* e = getenv("SIMSWEEP_LEAN");
  return !(e && e[0] == '0');
}

static int64_t workspace_bytes(const sim_config_t* cfgs, int32_t n_cfgs, const int32_t* wls_n) {
  int64_t big = 0;
  for (int i = 0; i < n_cfgs; i++) big += variant_of(wls_n[cfgs[i].workload]) == 2;
  return big ? (int64_t)WS_HEADER + big * (int64_t)g_variants[2].arena : 0;
}

static int check_cuda(cudaError_t e) { return e == cudaSuccess ? 0 : SIM_ECUDA; }
static unsigned g_attr_set[64];  // kernel attributes already set, per device and variant
struct AuxStreams {              // per device: one stream per variant, a fork event and one join event each
  bool ready = false;
  cudaStream_t s[N_VARIANTS];
  cudaEvent_t done[N_VARIANTS];
  cudaEvent_t fork;
};
static AuxStreams g_aux[64];

}  // namespace simsweep

using namespace simsweep;

extern "C" {

#ifdef SIMSWEEP_TRACE
int sim_trace_read(uint32_t* out, int32_t n, int32_t* count) {
  if (cudaMemcpyFromSymbol(count, g_trn, sizeof(int)) != cudaSuccess) return SIM_ECUDA;
  return cudaMemcpyFromSymbol(out, g_tr, sizeof(unsigned) * 2 * (size_t)n) == cudaSuccess ? 0 : SIM_ECUDA;
}
#endif
#ifdef SIMSWEEP_PROFILE
int sim_debug_read(int64_t* out, int32_t n_cfgs) {
  return cudaMemcpyFromSymbol(out, g_prof, sizeof(long long) * 24 * (size_t)n_cfgs) == cudaSuccess ? 0 : SIM_ECUDA;
}
int sim_debug_steps(int32_t* out, int32_t n) {
  return cudaMemcpyFromSymbol(out, g_dbg, sizeof(int) * 6 * (size_t)n) == cudaSuccess ? 0 : SIM_ECUDA;
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

int64_t sim_workspace_bytes(const sim_config_t* cfgs, int32_t n_cfgs, const int32_t* wls_n) {
  if (!cfgs || !wls_n || n_cfgs <= 0) return SIM_EINVAL;
  return workspace_bytes(cfgs, n_cfgs, wls_n);
}

}  // extern "C"

// Every config field that can be checked without the workload contents (SIM_EINVAL / SIM_ECOST); wls_n[n_wls] is
// the size of each workload.  Shared by sim_validate / sim_sweep (host copies) and sim_sweep_device.
static int validate_configs(const sim_config_t* cfgs, int32_t n_cfgs, const int32_t* wls_n, int32_t n_wls, int32_t n_cms,
                            int32_t internal_knobs = 0) {
  if (!cfgs || !wls_n || n_cfgs <= 0 || n_wls <= 0 || n_cms <= 0) return SIM_EINVAL;
  for (int w = 0; w < n_wls; w++)
    if (wls_n[w] <= 0) return SIM_EINVAL;
  for (int i = 0; i < n_cfgs; i++) {
    const sim_config_t& c = cfgs[i];
    if (c.order < SIM_ORDER_PREFILL_FIRST || c.order > SIM_ORDER_RANK_O) return SIM_EINVAL;
    if (c.replacement < SIM_NRF || c.replacement > SIM_PF) return SIM_EINVAL;
    if (c.reserve < SIM_RESERVE_SEQ || c.reserve > SIM_RESERVE_CONTEXT) return SIM_EINVAL;
    if ((c.replacement == SIM_PF) != (c.reserve != SIM_RESERVE_SEQ)) return SIM_EINVAL;  // Q39
    if ((c.knobs & ~(SIM_KNOB_HOL | SIM_KNOB_NRF_ARRIVAL | SIM_KNOB_SRF_VISIT_ADMISSION | internal_knobs)) || c.max_seqs < 0 ||
        c.kv_watermark < 0 || c.kv_watermark >= (1 << 30) || ((c.knobs & SIM_KNOB_NRF_ARRIVAL) && c.replacement != SIM_NRF) ||
        ((c.knobs & SIM_KNOB_SRF_VISIT_ADMISSION) && c.replacement != SIM_SRF && c.replacement != SIM_SRF_HIST) ||
        c.kv_block < 0 || c.kv_block > (1 << 16) || (c.kv_block > 1 && c.replacement == SIM_SRF_HIST))
      return SIM_EINVAL;  // alternative-reading knobs
    if ((c.hybrid != 0 && c.hybrid != 1) || (c.chunked != 0 && c.chunked != 1)) return SIM_EINVAL;
    if (c.C < 1 || c.C > (1 << 30) || c.M > (1 << 30) || c.S < 1 || c.S > 262143 || c.max_steps < 1) return SIM_EINVAL;
    if (c.n_cost < 1 || c.n_cost > SIM_MAX_COST) return SIM_EINVAL;
    if (c.workload < 0 || c.workload >= n_wls) return SIM_EINVAL;
    for (int k = 0; k < c.n_cost; k++)
      if (c.cost[k] < 0 || c.cost[k] >= n_cms) return SIM_ECOST;
  }
  return 0;
}

// Shared-memory carveout preference of the global-arena variants (percent): small, so that L1 keeps their per-slot
// arrays.  An SM's L1 / shared split cannot change while CTAs are resident, so the SMs that host an arena simulation
// take no shared-memory-resident CTA until it ends.  15 % is the smallest split that holds two lean arena CTAs per
// SM, so all 220 arena simulations of the north-star sweep start at once instead of 148 + a second wave after
// ~160 ms; measured on that sweep (tools/timeline.py --full, profiling build, profiles/r2q6_timelines.md):
// 10 % -> 367.6 ms (148 arena simulations at t = 0), 15 % -> 334.8, 20 % -> 337.5, 30 % -> 334.7, 50 % -> 337.6
// (the sweep equals its longest simulation from 15 % on); round 1: 100 % -> 535 ms (a 28 KB L1).
// SIMSWEEP_GM_CARVEOUT overrides (tools).
static int arena_carveout() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SIMSWEEP_GM_CARVEOUT");
    v = e ? atoi(e) : 15;
    if (v < 0 || v > 100) v = 15;
  }
  return v;
}

// Carveout of the shared-memory-resident block-kernel variants (percent, default 100: the most CTAs per SM).
// SIMSWEEP_SMEM_CARVEOUT overrides (tools: fewer co-resident simulations per SM).
static int smem_carveout() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SIMSWEEP_SMEM_CARVEOUT");
    v = e ? atoi(e) : 100;
    if (v < 0 || v > 100) v = 100;
  }
  return v;
}
// Carveout of the lean n <= 1024 variant: CTAs per SM (sim_set_lean_ctas_per_sm; 0 = auto: two per SM for at most
// 32 simulations per SM, else the maximum).  A CTA takes 45.2 KB + 1 KB; the shared-memory configurations are
// 64 / 100 / 164 / 196 / 228 KB, so k CTAs per SM need 28 / 44 / 72 / 86 / 100 % of the 228 KB.  Measured on the
// grid (tools/gpu_r2q16.sh .. gpu_r2q18.sh, tools/gpu_r2g.sh): 1 per SM 26.09 ms, 2: 23.95-24.13, 3: 24.65,
// 5: 24.89-25.05; full sweep 2 per SM 316-320 ms against 331-350 at 5.  SIMSWEEP_LEAN_CARVEOUT (percent) overrides.
static int g_lean_k = 0;
static int lean_carveout(int n_lean, int nsm) {
  const char* e = getenv("SIMSWEEP_LEAN_CARVEOUT");
  if (e) {
    const int v = atoi(e);
    return v < 0 || v > 100 ? 100 : v;
  }
  static const int pct[6] = {100, 28, 44, 72, 86, 100};
  const int k = g_lean_k ? g_lean_k : (n_lean <= 32 * nsm ? 2 : 5);
  return pct[k];
}

static int launch_sweep(const sim_config_t* h_cfgs, int32_t n_cfgs, const int32_t* h_wls_n, int32_t n_wls,
                        const sim_config_t* d_cfgs, const sim_workload_t* d_wls, const sim_cost_model_t* d_cms,
                        int32_t n_cms, const int32_t* d_order, const int64_t* d_row_off, const int64_t* d_tim_off,
                        sim_result_t* d_results, sim_request_out_t d_req, void* d_workspace, int64_t workspace_bytes_,
                        void* stream, const TraceDev& tr) {
  if (!h_cfgs || !h_wls_n || !d_cfgs || !d_wls || !d_cms || n_cfgs <= 0 || n_cms <= 0 || !d_row_off ||
      !d_tim_off || !d_results || !d_req.t_first || !d_req.t_done || !d_req.n_preempt || !d_req.refill_tokens)
    return SIM_EINVAL;
  // (sim_run_traced's internal routing bit is set after its own validation, never by a caller)
  if (int rc = validate_configs(h_cfgs, n_cfgs, h_wls_n, n_wls, n_cms, tr.steps ? SIM_KNOB_TRACE_INTERNAL : 0)) return rc;
  const int lean = lean_enabled();
  int cnt[N_VARIANTS] = {0};
  for (int i = 0; i < n_cfgs; i++) cnt[kernel_variant(h_cfgs[i], h_wls_n[h_cfgs[i].workload], lean)]++;
  const int64_t wsb = workspace_bytes(h_cfgs, n_cfgs, h_wls_n);
  if (wsb > 0 && (!d_workspace || workspace_bytes_ < wsb)) return SIM_EINVAL;
  KParams kp;
  kp.ws = reinterpret_cast<unsigned char*>(d_workspace);
  kp.cfgs = d_cfgs;
  kp.wls = d_wls;
  kp.cms = d_cms;
  kp.order = d_order;
  kp.row_off = d_row_off;
  kp.tim_off = d_tim_off;
  kp.results = d_results;
  kp.req = d_req;
  kp.n_cfgs = n_cfgs;
  kp.tr = tr;
  kp.lean = lean;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return SIM_ECUDA;
  cudaStream_t main = (cudaStream_t)stream;
  int nneed = 0;
  for (int v = 0; v < N_VARIANTS; v++) nneed += cnt[v] > 0;
  if (wsb > 0 && cudaMemsetAsync(d_workspace, 0, WS_HEADER, main) != cudaSuccess) return SIM_ECUDA;
  // several variants run concurrently on forked streams (joined back into `stream` with events), so a sweep that
  // mixes kernels is as long as its longest variant, not their sum
  AuxStreams& ax = g_aux[dev];
  if (nneed > 1) {
    if (!ax.ready) {
      for (int v = 0; v < N_VARIANTS; v++)
        if (cudaStreamCreateWithFlags(&ax.s[v], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ax.done[v], cudaEventDisableTiming) != cudaSuccess)
          return SIM_ECUDA;
      if (cudaEventCreateWithFlags(&ax.fork, cudaEventDisableTiming) != cudaSuccess) return SIM_ECUDA;
      ax.ready = true;
    }
    if (cudaEventRecord(ax.fork, main) != cudaSuccess) return SIM_ECUDA;
  }
  int launches = 0;
  // the large-window variants first: their simulations are the longest
  static const int launch_order[N_VARIANTS] = {2, 2 + N_SIZES, V_LEAN + 2, V_LEAN + 1, 1, 1 + N_SIZES, V_LEAN, 0, N_SIZES};
  for (int vi = 0; vi < N_VARIANTS; vi++) {
    const int v = launch_order[vi];
    if (!cnt[v]) continue;
    const Variant& V = g_variants[v];
    if (!(g_attr_set[dev] >> v & 1)) {
      if (cudaFuncSetAttribute((const void*)V.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)V.smem) !=
          cudaSuccess)
        return SIM_ECUDA;
      // shared-memory resident state: the largest carveout, so that more CTAs fit per SM; the global-arena
      // variant keeps the carveout small and leaves the rest of the 256 KB to L1
      if (v != V_LEAN)
        cudaFuncSetAttribute((const void*)V.fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                             V.arena ? arena_carveout() : smem_carveout());
      g_attr_set[dev] |= 1u << v;
    }
    if (v == V_LEAN) {  // its occupancy depends on the launch (sim_set_lean_ctas_per_sm): set when it changes
      static int last[64];
      int nsm = 148;
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      const int cv = lean_carveout(cnt[v], nsm);
      if (last[dev] != cv + 1) {
        if (cudaFuncSetAttribute((const void*)V.fn, cudaFuncAttributePreferredSharedMemoryCarveout, cv) != cudaSuccess)
          return SIM_ECUDA;
        last[dev] = cv + 1;
      }
    }
    kp.variant = v;
    // the three GM variants share the workspace: disjoint arenas, one counter each
    kp.arena_base = v == 2 + N_SIZES ? cnt[2] : (v == V_LEAN + 2 ? cnt[2] + cnt[2 + N_SIZES] : 0);
    kp.ctr_off = v == 2 + N_SIZES ? 64 : (v == V_LEAN + 2 ? 128 : 0);
    cudaStream_t s = nneed > 1 ? ax.s[v] : main;
    if (nneed > 1 && cudaStreamWaitEvent(s, ax.fork, 0) != cudaSuccess) return SIM_ECUDA;
    void* args[] = {&kp};
    if (cudaLaunchKernel((const void*)V.fn, dim3(n_cfgs), dim3(V.nt), args, V.smem, s) != cudaSuccess)
      return SIM_ECUDA;
    if (nneed > 1 && (cudaEventRecord(ax.done[v], s) != cudaSuccess || cudaStreamWaitEvent(main, ax.done[v], 0) != cudaSuccess))
      return SIM_ECUDA;
    launches++;
  }
  return launches;
}

extern "C" {

int sim_set_lean_ctas_per_sm(int32_t k) {
  if (k < 0 || k > 5) return SIM_EINVAL;
  g_lean_k = k;
  return 0;
}

int sim_sweep_device(const sim_config_t* h_cfgs, int32_t n_cfgs, const int32_t* h_wls_n, int32_t n_wls,
                     const sim_config_t* d_cfgs, const sim_workload_t* d_wls, const sim_cost_model_t* d_cms,
                     int32_t n_cms, const int32_t* d_order, const int64_t* d_row_off, const int64_t* d_tim_off,
                     sim_result_t* d_results, sim_request_out_t d_req, void* d_workspace, int64_t workspace_bytes_,
                     void* stream) {
  const TraceDev none{nullptr, nullptr, nullptr, 0, 0, 0};
  return launch_sweep(h_cfgs, n_cfgs, h_wls_n, n_wls, d_cfgs, d_wls, d_cms, n_cms, d_order, d_row_off, d_tim_off,
                      d_results, d_req, d_workspace, workspace_bytes_, stream, none);
}

static int validate_cms(const sim_cost_model_t* cms, int32_t n_cms) {
  if (!cms || n_cms <= 0) return SIM_EINVAL;
  for (int k = 0; k < n_cms; k++) {
    const sim_cost_model_t& m = cms[k];
    if (m.mode != 0 && m.mode != 1) return SIM_ECOST;
    if (m.layers < 1 || m.e < 1 || m.tp < 1 || m.H < 1) return SIM_ECOST;
    if (m.mode == 1 && (m.h < 1 || m.f < 1 || m.NQ < 1 || m.NKV < 1 || !(m.flops > 0) || !(m.bw > 0) ||
                        (m.tp > 1 && !(m.link_bw > 0))))
      return SIM_ECOST;
  }
  return 0;
}

static int validate(const sim_config_t* cfgs, int32_t n_cfgs, const sim_workload_t* wls, int32_t n_wls,
                    const sim_cost_model_t* cms, int32_t n_cms) {
  if (!cfgs || !wls || !cms || n_cfgs <= 0 || n_wls <= 0 || n_cms <= 0) return SIM_EINVAL;
  std::vector<int32_t> wn(n_wls);
  for (int w = 0; w < n_wls; w++) wn[w] = wls[w].n;
  if (int rc = validate_configs(cfgs, n_cfgs, wn.data(), n_wls, n_cms)) return rc;
  std::vector<char> multi(n_wls, 0);
  for (int i = 0; i < n_cfgs; i++)
    if (cfgs[i].n_cost > 1) multi[cfgs[i].workload] = 1;
  for (int w = 0; w < n_wls; w++) {
    const sim_workload_t& W = wls[w];
    if (W.n <= 0 || !W.I || !W.O || !W.T) return SIM_EINVAL;
    for (int i = 0; i < W.n; i++) {
      if (W.I[i] < 1 || W.O[i] < 1 || W.I[i] > 262143 || W.O[i] > 262143) return SIM_EWORKLOAD;
      if (i > 0 && !(W.T[i] >= W.T[i - 1])) return SIM_EWORKLOAD;
      if (multi[w] && W.T[i] != 0.0) return SIM_EWORKLOAD;
    }
  }
  return validate_cms(cms, n_cms);
}

// longest-processing-time-first estimate of one simulation's step count from per-workload statistics
struct WlStats {
  double sumIO, sumPO, sumO, sumI, maxO;
};

static WlStats workload_stats(const sim_workload_t& w) {
  WlStats st{0, 0, 0, 0, 0};
  for (int i = 0; i < w.n; i++) {
    st.sumIO += ((double)w.I[i] + 0.5 * w.O[i]) * w.O[i];
    st.sumPO += ((double)w.I[i] + w.O[i] - 1) * w.O[i];
    st.sumO += w.O[i];
    st.sumI += w.I[i];
    st.maxO = std::max(st.maxO, (double)w.O[i]);
  }
  return st;
}

// KV-time area / M: the average usage is ~(I + O/2) per running request under SEQ, the whole reserve
// (I + O - 1 or S) under the preemption-free reserves
static double estimate_steps(const sim_config_t& c, const WlStats& st) {
  const double Meff = c.M >= 0 ? (double)std::max<int64_t>(c.M, 1) : 1e18;
  const double area = c.reserve == SIM_RESERVE_PEAK      ? st.sumPO
                      : c.reserve == SIM_RESERVE_CONTEXT ? (double)c.S * st.sumO
                                                         : st.sumIO;
  return st.maxO + area / Meff + st.sumI / (double)c.C;
}

// Per-device cache of the host entry point: one device arena, one pinned staging buffer and one stream,
// grown on demand and reused across calls (guarded by a mutex; released at process exit).
struct DevCache {
  std::mutex mu;
  char* dbuf = nullptr;
  size_t dcap = 0;
  char* hbuf = nullptr;
  size_t hcap = 0;
  cudaStream_t stream = nullptr;
  int checked = 0;  // 1 = sm_100 device, -1 = unsupported
};
static DevCache g_cache[64];

static int cache_reserve(DevCache& c, size_t dbytes, size_t hbytes) {
  if (!c.stream && cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking) != cudaSuccess) return SIM_ECUDA;
  if (dbytes > c.dcap) {
    if (c.dbuf) cudaFree(c.dbuf);
    c.dcap = 0;
    const size_t want = dbytes + dbytes / 4;
    if (cudaMalloc(&c.dbuf, want) != cudaSuccess) return SIM_ECUDA;
    c.dcap = want;
  }
  if (hbytes > c.hcap) {
    if (c.hbuf) cudaFreeHost(c.hbuf);
    c.hcap = 0;
    const size_t want = hbytes + hbytes / 4;
    if (cudaMallocHost(&c.hbuf, want) != cudaSuccess) return SIM_ECUDA;
    c.hcap = want;
  }
  return 0;
}

}  // extern "C"

// the host entry points: validate, stage inputs (one H2D), launch, copy outputs (and the trace) back
static int host_run(const sim_config_t* cfgs_in, int32_t n_cfgs, const sim_workload_t* wls, int32_t n_wls,
                    const sim_cost_model_t* cms, int32_t n_cms, sim_result_t* results, sim_request_out_t req,
                    int32_t device, sim_trace_t* trace) {
  int rc = validate(cfgs_in, n_cfgs, wls, n_wls, cms, n_cms);
  if (rc) return rc;
  if (!results) return SIM_EINVAL;
  if (trace && (n_cfgs != 1 || trace->cap_steps < 0 || trace->cap_entries < 0 || trace->cap_events < 0 ||
                (trace->cap_steps && !trace->steps) || (trace->cap_entries && !trace->entries) ||
                (trace->cap_events && !trace->events)))
    return SIM_EINVAL;
  sim_config_t tcfg;
  const sim_config_t* cfgs = cfgs_in;
  if (trace) {  // a traced simulation runs in the knob instance (KN), which carries the trace writes
    tcfg = cfgs_in[0];
    tcfg.knobs |= SIM_KNOB_TRACE_INTERNAL;
    cfgs = &tcfg;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return SIM_ENODEV;
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess) return SIM_ECUDA;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return SIM_ECUDA;
  DevCache& cache = g_cache[dev];
  std::lock_guard<std::mutex> lock(cache.mu);
  if (cache.checked == 0) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return SIM_ECUDA;
    cache.checked = prop.major == 10 ? 1 : -1;
  }
  if (cache.checked < 0) return SIM_ENODEV;

  std::vector<int64_t> row_off(n_cfgs), tim_off(n_cfgs);
  int64_t rows = 0, trows = 0;
  for (int i = 0; i < n_cfgs; i++) {
    row_off[i] = rows;
    tim_off[i] = trows;
    rows += wls[cfgs[i].workload].n;
    trows += (int64_t)cfgs[i].n_cost * wls[cfgs[i].workload].n;
  }
  std::vector<WlStats> stats(n_wls);
  for (int w = 0; w < n_wls; w++) stats[w] = workload_stats(wls[w]);
  std::vector<double> est(n_cfgs);
  for (int i = 0; i < n_cfgs; i++) est[i] = estimate_steps(cfgs[i], stats[cfgs[i].workload]);
  std::vector<int32_t> order(n_cfgs);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return est[a] > est[b]; });
  std::vector<int32_t> wn(n_wls);
  int64_t wtot = 0;
  for (int w = 0; w < n_wls; w++) wn[w] = wls[w].n, wtot += wls[w].n;

  // arena layout: inputs (staged in pinned memory, one H2D) | outputs
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
  const size_t o_I = off;
  off = al(off + 4 * (size_t)wtot);
  const size_t o_O = off;
  off = al(off + 4 * (size_t)wtot);
  const size_t o_T = off;
  off = al(off + 8 * (size_t)wtot);
  const size_t in_bytes = off;
  const size_t o_res = off;
  off = al(off + sizeof(sim_result_t) * n_cfgs);
  const size_t o_tf = off;
  off = al(off + 8 * (size_t)trows);
  const size_t o_td = off;
  off = al(off + 8 * (size_t)trows);
  const size_t o_np = off;
  off = al(off + 8 * (size_t)rows);
  const size_t o_rf = off;
  off = al(off + 8 * (size_t)rows);
  const int64_t wsb = workspace_bytes(cfgs, n_cfgs, wn.data());
  const size_t o_ws = off;
  off = al(off + (size_t)wsb);
  const size_t o_ts = off;
  off = al(off + (trace ? sizeof(sim_trace_step_t) * (size_t)trace->cap_steps : 0));
  const size_t o_te = off;
  off = al(off + (trace ? sizeof(sim_trace_entry_t) * (size_t)trace->cap_entries : 0));
  const size_t o_tv = off;
  off = al(off + (trace ? sizeof(sim_trace_event_t) * (size_t)trace->cap_events : 0));
  if ((rc = cache_reserve(cache, off, in_bytes))) return rc;
  char* base = cache.dbuf;
  char* h = cache.hbuf;
  cudaStream_t s = cache.stream;
  // the previous call's stream work has completed (it synchronized before returning)
  std::memcpy(h + o_cfg, cfgs, sizeof(sim_config_t) * n_cfgs);
  sim_workload_t* dw = reinterpret_cast<sim_workload_t*>(h + o_wl);
  int64_t wo = 0;
  for (int w = 0; w < n_wls; w++) {
    dw[w].n = wls[w].n;
    dw[w].pad = 0;
    dw[w].I = reinterpret_cast<const int32_t*>(base + o_I) + wo;
    dw[w].O = reinterpret_cast<const int32_t*>(base + o_O) + wo;
    dw[w].T = reinterpret_cast<const double*>(base + o_T) + wo;
    std::memcpy(h + o_I + 4 * wo, wls[w].I, 4 * (size_t)wls[w].n);
    std::memcpy(h + o_O + 4 * wo, wls[w].O, 4 * (size_t)wls[w].n);
    std::memcpy(h + o_T + 8 * wo, wls[w].T, 8 * (size_t)wls[w].n);
    wo += wls[w].n;
  }
  std::memcpy(h + o_cm, cms, sizeof(sim_cost_model_t) * n_cms);
  std::memcpy(h + o_ord, order.data(), 4 * (size_t)n_cfgs);
  std::memcpy(h + o_ro, row_off.data(), 8 * (size_t)n_cfgs);
  std::memcpy(h + o_to, tim_off.data(), 8 * (size_t)n_cfgs);
  rc = check_cuda(cudaMemcpyAsync(base, h, in_bytes, cudaMemcpyHostToDevice, s));
  sim_request_out_t dreq;
  dreq.t_first = reinterpret_cast<double*>(base + o_tf);
  dreq.t_done = reinterpret_cast<double*>(base + o_td);
  dreq.n_preempt = reinterpret_cast<int64_t*>(base + o_np);
  dreq.refill_tokens = reinterpret_cast<int64_t*>(base + o_rf);
  TraceDev tr{nullptr, nullptr, nullptr, 0, 0, 0};
  if (trace) {
    tr.steps = reinterpret_cast<sim_trace_step_t*>(base + o_ts);
    tr.entries = reinterpret_cast<sim_trace_entry_t*>(base + o_te);
    tr.events = reinterpret_cast<sim_trace_event_t*>(base + o_tv);
    tr.cap_steps = trace->cap_steps, tr.cap_entries = trace->cap_entries, tr.cap_events = trace->cap_events;
  }
  if (!rc) {
    int l = launch_sweep(cfgs, n_cfgs, wn.data(), n_wls, reinterpret_cast<const sim_config_t*>(base + o_cfg),
                             reinterpret_cast<const sim_workload_t*>(base + o_wl),
                             reinterpret_cast<const sim_cost_model_t*>(base + o_cm), n_cms,
                             reinterpret_cast<const int32_t*>(base + o_ord),
                             reinterpret_cast<const int64_t*>(base + o_ro), reinterpret_cast<const int64_t*>(base + o_to),
                             reinterpret_cast<sim_result_t*>(base + o_res), dreq, wsb ? base + o_ws : nullptr, wsb,
                             s, tr);
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
  }
  rc |= check_cuda(cudaStreamSynchronize(s));
  if (!rc && trace) {  // totals from the result (every step, entry and preemption is counted there)
    trace->n_steps = results[0].steps;
    trace->n_entries = results[0].batch_entries;
    trace->n_events = results[0].preemptions;
    const int64_t ns = std::min(trace->n_steps, trace->cap_steps), ne = std::min(trace->n_entries, trace->cap_entries),
                  nv = std::min(trace->n_events, trace->cap_events);
    if (ns > 0) rc |= check_cuda(cudaMemcpy(trace->steps, tr.steps, sizeof(sim_trace_step_t) * ns, cudaMemcpyDeviceToHost));
    if (ne > 0)
      rc |= check_cuda(cudaMemcpy(trace->entries, tr.entries, sizeof(sim_trace_entry_t) * ne, cudaMemcpyDeviceToHost));
    if (nv > 0)
      rc |= check_cuda(cudaMemcpy(trace->events, tr.events, sizeof(sim_trace_event_t) * nv, cudaMemcpyDeviceToHost));
  }
  return rc ? (rc < 0 ? rc : SIM_ECUDA) : 0;
}

extern "C" {

int sim_validate(const sim_config_t* cfgs, int32_t n_cfgs, const sim_workload_t* wls, int32_t n_wls,
                 const sim_cost_model_t* cms, int32_t n_cms) {
  return validate(cfgs, n_cfgs, wls, n_wls, cms, n_cms);
}

int sim_sweep(const sim_config_t* cfgs, int32_t n_cfgs, const sim_workload_t* wls, int32_t n_wls,
              const sim_cost_model_t* cms, int32_t n_cms, sim_result_t* results, sim_request_out_t req,
              int32_t device) {
  return host_run(cfgs, n_cfgs, wls, n_wls, cms, n_cms, results, req, device, nullptr);
}

int sim_run_traced(const sim_config_t* cfg, const sim_workload_t* wls, int32_t n_wls, const sim_cost_model_t* cms,
                   int32_t n_cms, sim_result_t* result, sim_request_out_t req, sim_trace_t* trace, int32_t device) {
  if (!trace) return SIM_EINVAL;
  return host_run(cfg, 1, wls, n_wls, cms, n_cms, result, req, device, trace);
}

}  // extern "C"

// ---- cost-model analytics: host buffers in and out, one kernel each ----
static bool shape_ok(int64_t n_p, int64_t c, int64_t m_p, int64_t n_d, int64_t m_d) {
  if (n_p < 0 || n_d < 0 || n_p + n_d < 1 || m_p < 0 || m_d < 0 || (n_p > 0 && c < 1)) return false;
  const double lim = 4.0e18;  // every feature sum below 2^62 (checked in floating point, no overflow)
  const double P = (double)n_p, Cc = (double)c, Mp = (double)m_p;
  return P * Cc * (Cc + Mp) < lim && P * Cc + (double)n_d < lim && (double)n_d * (double)m_d < lim && P * Mp < lim;
}

template <typename In, typename Out, typename Launch>
static int run_analytics(const sim_cost_model_t* cms, int32_t n_cms, const In* in, int32_t n, Out** outs, int n_outs,
                         int32_t device, Launch launch) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return SIM_ENODEV;
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess) return SIM_ECUDA;
  const size_t total = (size_t)n * n_cms;
  sim_cost_model_t* d_cms = nullptr;
  In* d_in = nullptr;
  Out* d_out = nullptr;
  int rc = 0;
  rc |= check_cuda(cudaMalloc(&d_cms, sizeof(sim_cost_model_t) * n_cms));
  rc |= check_cuda(cudaMalloc(&d_in, sizeof(In) * n));
  rc |= check_cuda(cudaMalloc(&d_out, sizeof(Out) * total * n_outs));
  if (!rc) rc |= check_cuda(cudaMemcpy(d_cms, cms, sizeof(sim_cost_model_t) * n_cms, cudaMemcpyHostToDevice));
  if (!rc) rc |= check_cuda(cudaMemcpy(d_in, in, sizeof(In) * n, cudaMemcpyHostToDevice));
  if (!rc) {
    const int threads = 128, blocks = (int)std::min<size_t>((total + threads - 1) / threads, 148 * 16);
    launch(blocks, threads, d_cms, d_in, d_out, total);
    rc |= check_cuda(cudaGetLastError());
  }
  for (int o = 0; o < n_outs && !rc; o++)
    if (outs[o]) rc |= check_cuda(cudaMemcpy(outs[o], d_out + o * total, sizeof(Out) * total, cudaMemcpyDeviceToHost));
  cudaFree(d_cms);
  cudaFree(d_in);
  cudaFree(d_out);
  return rc ? SIM_ECUDA : 0;
}

extern "C" {

int sim_batch_times(const sim_cost_model_t* cms, int32_t n_cms, const sim_batch_shape_t* shapes, int32_t n,
                    double* out, int32_t device) {
  if (!shapes || !out || n <= 0) return SIM_EINVAL;
  if (int rc = validate_cms(cms, n_cms)) return rc;
  for (int i = 0; i < n; i++)
    if (!shape_ok(shapes[i].n_p, shapes[i].c, shapes[i].m_p, shapes[i].n_d, shapes[i].m_d)) return SIM_EINVAL;
  double* outs[1] = {out};
  return run_analytics(cms, n_cms, shapes, n, outs, 1, device,
                       [&](int b, int t, const sim_cost_model_t* dc, const sim_batch_shape_t* di, double* dout, size_t) {
                         batch_times_kernel<<<b, t>>>(dc, n_cms, di, n, dout);
                       });
}

int sim_slo_frontier(const sim_cost_model_t* cms, int32_t n_cms, const sim_slo_query_t* q, int32_t n, int64_t* out,
                     int32_t device) {
  if (!q || !out || n <= 0) return SIM_EINVAL;
  if (int rc = validate_cms(cms, n_cms)) return rc;
  for (int i = 0; i < n; i++)
    if (q[i].m_max < 0 || !(q[i].tau > 0) || !shape_ok(q[i].n_p, q[i].c, q[i].m_max, q[i].n_d, q[i].m_max))
      return SIM_EINVAL;
  int64_t* outs[1] = {out};
  return run_analytics(cms, n_cms, q, n, outs, 1, device,
                       [&](int b, int t, const sim_cost_model_t* dc, const sim_slo_query_t* di, int64_t* dout, size_t) {
                         slo_frontier_kernel<<<b, t>>>(dc, n_cms, di, n, reinterpret_cast<long long*>(dout));
                       });
}

int sim_operator_costs(const sim_cost_model_t* cms, int32_t n_cms, const sim_batch_shape_t* shapes, int32_t n,
                       sim_op_cost_t* out, int32_t device) {
  if (!shapes || !out || n <= 0) return SIM_EINVAL;
  if (int rc = validate_cms(cms, n_cms)) return rc;
  for (int k = 0; k < n_cms; k++)
    if (!(cms[k].flops > 0) || !(cms[k].bw > 0) || cms[k].h < 1 || cms[k].f < 1 || cms[k].NQ < 1 || cms[k].NKV < 1)
      return SIM_ECOST;
  for (int i = 0; i < n; i++)
    if (!shape_ok(shapes[i].n_p, shapes[i].c, shapes[i].m_p, shapes[i].n_d, shapes[i].m_d)) return SIM_EINVAL;
  // run_analytics sizes its output as n * n_cms records: one record per (model, shape) holding SIM_N_OPS operators
  struct Rec {
    sim_op_cost_t op[SIM_N_OPS];
  };
  Rec* recs[1] = {reinterpret_cast<Rec*>(out)};
  return run_analytics(cms, n_cms, shapes, n, recs, 1, device,
                       [&](int b, int t, const sim_cost_model_t* dc, const sim_batch_shape_t* di, Rec* dout, size_t) {
                         operator_costs_kernel<<<b, t>>>(dc, n_cms, di, n, reinterpret_cast<sim_op_cost_t*>(dout));
                       });
}

int sim_kv_break_even(const sim_cost_model_t* cms, int32_t n_cms, const int64_t* N, int32_t n, double xfer_bw, int64_t M,
                      double* recompute, double* swap, double* interval, int32_t device) {
  if (!N || n <= 0 || !(xfer_bw > 0) || M <= 0) return SIM_EINVAL;
  if (int rc = validate_cms(cms, n_cms)) return rc;
  for (int i = 0; i < n; i++)
    if (N[i] < 1 || !shape_ok(1, N[i], 0, 0, 0)) return SIM_EINVAL;
  double* outs[3] = {recompute, swap, interval};
  return run_analytics(cms, n_cms, N, n, outs, 3, device,
                       [&](int b, int t, const sim_cost_model_t* dc, const int64_t* di, double* dout, size_t total) {
                         kv_break_even_kernel<<<b, t>>>(dc, n_cms, reinterpret_cast<const long long*>(di), n, xfer_bw,
                                                        (long long)M, dout, dout + total, dout + 2 * total);
                       });
}

}  // extern "C"

namespace simsweep {
__global__ void opt_fill_kernel(unsigned long long* dist, unsigned char* cur, unsigned char* nxt, long long n) {
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n; x += (long long)gridDim.x * blockDim.x)
    dist[x] = OPT_INF, cur[x] = 0, nxt[x] = 0;
}
}  // namespace simsweep

extern "C" {

int sim_optimum(const sim_opt_problem_t* probs, int32_t n_probs, const sim_cost_model_t* cm, sim_opt_result_t* out,
                int32_t device) {
  if (!probs || !out || n_probs <= 0) return SIM_EINVAL;
  if (int rc = validate_cms(cm, 1)) return rc;
  constexpr long long MAX_STATES = 1ll << 28;  // canonical states: 8 B of distance + 2 flags each (2.5 GB)
  std::vector<OptDev> P(n_probs);
  std::vector<long long> nst(n_probs), start_of(n_probs);
  long long cap = 0;
  for (int q = 0; q < n_probs; q++) {
    const sim_opt_problem_t& pr = probs[q];
    if (pr.n < 1 || pr.n > OPT_MAXN || pr.C < 1 || pr.M < 0) return SIM_EINVAL;
    OptDev& d = P[q];
    memset(&d, 0, sizeof(d));
    if (pr.flags & ~SIM_OPT_NO_PREEMPT) return SIM_EINVAL;
    d.n = pr.n, d.C = pr.C, d.M = pr.M, d.nopre = (pr.flags & SIM_OPT_NO_PREEMPT) ? 1 : 0;
    // requests sorted by (I, O) so that identical ones are adjacent (a group); the optimum does not depend on the
    // order of the requests
    std::vector<std::pair<int, int>> req;
    for (int i = 0; i < pr.n; i++) {
      if (pr.I[i] < 1 || pr.O[i] < 1 || pr.O[i] > OPT_MAXO || pr.I[i] > (1 << 20)) return SIM_EINVAL;
      req.push_back({pr.I[i], pr.O[i]});
    }
    std::sort(req.begin(), req.end());
    for (int i = 0; i < pr.n; i++) {
      d.I[i] = req[i].first, d.O[i] = req[i].second;
      long long b = 1;  // local id 0 = done; block g holds the I+g unfilled states (+ the filled one for g >= 1)
      for (int g = 0; g < d.O[i]; g++) {
        d.base[i][g] = (int)std::min<long long>(b, MAX_STATES + 1);
        b += d.I[i] + g + (g >= 1 ? 1 : 0);
        if (b > MAX_STATES) break;
      }
      d.base[i][d.O[i]] = (int)std::min<long long>(b, MAX_STATES + 1);
      d.ns[i] = b;
    }
    long long total = 1, start = 0;
    for (int i = 0; i < pr.n;) {
      int j = i;
      while (j < pr.n && d.I[j] == d.I[i] && d.O[j] == d.O[i]) j++;
      const int k = j - i, g = d.ng++;
      d.gs[g] = i, d.gk[g] = k;
      d.gstride[g] = total;
      // radix: multisets of size k from ns local states, binom(ns + k - 1, k) (overflow-safe test first)
      const long long ns = d.ns[i];
      long long radix = ns > MAX_STATES ? MAX_STATES + 1 : 1;
      for (int t = 0; t < k && radix <= MAX_STATES; t++) radix = radix * (ns + t) / (t + 1);
      int ones[OPT_MAXN];
      for (int t = 0; t < k; t++) ones[t] = 1;  // every request at (g = 0, m = 0): local id 1
      if (total <= MAX_STATES && radix <= MAX_STATES) start += opt_rank(ones, k) * total;
      total = (total > MAX_STATES || radix > MAX_STATES || total * radix > MAX_STATES) ? MAX_STATES + 1 : total * radix;
      i = j;
    }
    nst[q] = total;
    start_of[q] = start;
    if (total <= MAX_STATES) cap = std::max(cap, total);
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return SIM_ENODEV;
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess) return SIM_ECUDA;
  unsigned long long* dist = nullptr;
  unsigned char *cur = nullptr, *nxt = nullptr;
  int* changed = nullptr;
  long long* reached = nullptr;
  int rc = 0;
  if (cap > 0) {
    rc |= check_cuda(cudaMalloc(&dist, 8 * (size_t)cap));
    rc |= check_cuda(cudaMalloc(&cur, (size_t)cap));
    rc |= check_cuda(cudaMalloc(&nxt, (size_t)cap));
  }
  rc |= check_cuda(cudaMalloc(&changed, sizeof(int)));
  rc |= check_cuda(cudaMalloc(&reached, sizeof(long long)));
  for (int q = 0; q < n_probs && !rc; q++) {
    sim_opt_result_t& r = out[q];
    memset(&r, 0, sizeof(r));
    const OptDev& d = P[q];
    long long peak = 0;
    for (int i = 0; i < d.n; i++) peak = std::max<long long>(peak, (long long)d.I[i] + d.O[i] - 1);
    if (nst[q] > MAX_STATES) {
      r.status = 2;
      continue;
    }
    if (peak > d.M) {  // that request can never hold its last KVs (Eq. (7))
      r.status = 1;
      continue;
    }
    const long long ns = nst[q];
    const int threads = 256, blocks = (int)std::min<long long>((ns + threads - 1) / threads, 148 * 16);
    opt_fill_kernel<<<blocks, threads>>>(dist, cur, nxt, ns);
    const long long start = start_of[q];
    const unsigned long long zero = 0ull;
    const unsigned char one = 1;
    const long long one_ll = 1;
    rc |= check_cuda(cudaMemcpy(dist + start, &zero, 8, cudaMemcpyHostToDevice));
    rc |= check_cuda(cudaMemcpy(cur + start, &one, 1, cudaMemcpyHostToDevice));
    rc |= check_cuda(cudaMemcpy(reached, &one_ll, 8, cudaMemcpyHostToDevice));
    int rounds = 0;
    unsigned char *a = cur, *b = nxt;
    while (!rc) {
      rc |= check_cuda(cudaMemset(changed, 0, sizeof(int)));
      opt_round_kernel<<<blocks, threads>>>(d, *cm, dist, a, b, ns, changed, reached);
      rc |= check_cuda(cudaGetLastError());
      int h = 0;
      rc |= check_cuda(cudaMemcpy(&h, changed, sizeof(int), cudaMemcpyDeviceToHost));
      rounds++;
      if (!h) break;
      std::swap(a, b);  // the processed flags were all cleared: the old frontier array is the next one
    }
    unsigned long long goal = OPT_INF;
    long long nreach = 0;
    rc |= check_cuda(cudaMemcpy(&goal, dist, 8, cudaMemcpyDeviceToHost));  // state 0 = every request done
    rc |= check_cuda(cudaMemcpy(&nreach, reached, 8, cudaMemcpyDeviceToHost));
    r.rounds = rounds;
    r.states = nreach;
    if (goal == OPT_INF) {
      r.status = 1;
    } else {
      double v;
      memcpy(&v, &goal, 8);
      r.optimum = v;
    }
  }
  cudaFree(dist);
  cudaFree(cur);
  cudaFree(nxt);
  cudaFree(changed);
  cudaFree(reached);
  return rc ? SIM_ECUDA : 0;
}

}  // extern "C"
