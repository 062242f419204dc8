/* ORACLE -- test infrastructure only.
 *
 * Plain, slow, literal CPU implementation of the InferMax step-level
 * simulator (arXiv 2411.07447, Algorithm 1) used to prove
 * the CUDA path correct.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no code,
 * header, table or constant with paper_2411_07447_b200/ (the product).
 *
 * Semantics: DESIGN.md "Readings" Q1-Q40 (frozen from SURVEY.md 8(c), plus Q39-Q40 for the preemption-free reserves).
 */
#ifndef INFERMAX_ORACLE_H
#define INFERMAX_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* GroupRequests orders (Table 2; App. D) */
enum { OR_PREFILL_FIRST = 0, OR_DECODE_FIRST = 1, OR_RANK_ORG = 2, OR_RANK_I = 3, OR_RANK_O = 4 };
/* replacement policies (Table 2; Sec. SRF) */
enum { OR_NRF = 0, OR_SRF = 1, OR_SRF_HIST = 2, OR_PF = 3 /* preemption-free, Table 2 PAPER.md:1603,1606 */ };
/* initial KV reserve at (re)admission (Table 2 column "Initial KV reserve") */
enum { OR_RESERVE_SEQ = 0 /* s = I + g (r.I) */, OR_RESERVE_PEAK = 1 /* I + O - 1 (*^pf) */,
       OR_RESERVE_CONTEXT = 2 /* S (Orca) */ };
/* per-simulation status */
enum { OR_OK = 0, OR_TOO_LONG = 1, OR_NEVER_FITS = 2, OR_MAX_STEPS = 3, OR_DEADLOCK = 4 };

typedef struct {
  int32_t order, hybrid, chunked, replacement;
  int32_t S, n_cost;
  int64_t C;         /* token limit per batch */
  int64_t M;         /* KV capacity in tokens, < 0 = infinite (what-if) */
  int64_t max_steps;
  int32_t reserve;   /* OR_RESERVE_*; != SEQ iff replacement == OR_PF (reading Q39) */
  int32_t knobs;     /* OR_KNOB_* alternative readings */
  int32_t max_seqs;  /* Q16 alternative: |B| <= max_seqs (0 = no cap) */
  int32_t kv_block;  /* Q15 alternative: KVs allocated in blocks of this many tokens (0 / 1 = per token) */
  int64_t kv_watermark; /* Q16 alternative: KVs a waiting admission must leave free (0 = none) */
} oracle_config_t;
enum { OR_KNOB_HOL = 1 /* Q10 alternative: the first waiting candidate not admitted ends R_w's visit */,
       OR_KNOB_NRF_ARRIVAL = 2 /* Q6 alternative: NRF visits and retains running requests in arrival order */,
       OR_KNOB_SRF_VISIT_ADMISSION = 4 /* Q3 alternative: SRF visits in admission order, SRF only for victims */ };

typedef struct {
  int32_t mode; /* 0 = linear, 1 = theoretical (Eq. 3) */
  int32_t layers, h, f, H, NQ, NKV, e, tp, pad;
  double lin[10]; /* a0 a1 | b0 b1 b2 b3 b4 | d0 d1 d2 (per layer, seconds) */
  double flops, bw, link_bw;
} oracle_cost_t;

typedef struct {
  int32_t status, pad;
  int64_t steps, preemptions, batch_entries, processed_tokens, sum_U, prefill_entries, idle_jumps, visits;
  double makespan[4], mean_latency[4], mean_ttft[4], mean_tpot[4];
} oracle_summary_t;

/* Runs one simulation.  Returns 0, or < 0 on a call error (bad enum, n <= 0,
 * unsorted T, I < 1, O < 1, n_cost not in 1..4, n_cost > 1 with non-zero T).
 * Per-request outputs are k-major: t_first[k*n + i].  Trace buffers may be
 * NULL; trace_lens[0..1] receive the int64 / double lengths written (or -1 on
 * overflow). */
int oracle_run(const oracle_config_t* cfg, int32_t n, const int32_t* I, const int32_t* O, const double* T,
               const oracle_cost_t* cms, oracle_summary_t* out, double* t_first, double* t_done,
               int64_t* n_preempt, int64_t* refill_tokens, int64_t* trace_i, int64_t trace_i_cap,
               double* trace_d, int64_t trace_d_cap, int64_t* trace_lens);

/* Batch time of one batch given its entries (c, m_before, is_prefill). */
double oracle_batch_time(const oracle_cost_t* cm, int32_t n, const int64_t* c, const int64_t* m,
                         const int32_t* is_prefill);

/* Eq. (1)-(2) for B requests sharing (c, m): FLOPs and RW in elements. */
void oracle_attention_cost(int64_t c, int64_t m, int64_t B, int64_t H, int64_t NQ, int64_t NKV,
                           int64_t* flops, int64_t* rw_elems);
/* (c x in) @ (in x out) matmul: 2*c*in*out FLOPs; RW elements in*out + c*in + c*out. */
void oracle_matmul_cost(int64_t c, int64_t in, int64_t out, int64_t* flops, int64_t* rw_elems);
/* SRF+Hist output-length prediction from an 18x18 histogram (reading Q31). */
int64_t oracle_hist_predict(const int32_t* hist, int64_t I);

/* Exact optimum of the paper's CSP for a tiny offline workload, by Dijkstra over every
 * reachable schedule state (readings Q43-Q45).  status 0 = optimum found, 1 = the
 * all-done state is unreachable (some I+O-1 > M).  states = number of reachable states (all are settled). */
typedef struct {
  int32_t status;
  int32_t pad;
  int64_t states;
  double optimum; /* min over schedules of sum_j d_j (seconds) */
} oracle_opt_t;
int oracle_optimum(int32_t n, const int32_t* I, const int32_t* O, int64_t C, int64_t M, int32_t no_preempt,
                   const oracle_cost_t* cm,
                   oracle_opt_t* out);

#ifdef __cplusplus
}
#endif
#endif
