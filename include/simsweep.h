/* simsweep.h -- C-ABI of libsimsweep.so, the B200 (sm_100a) step-level
 * simulator of multi-batch LLM-serving schedulers (arXiv 2411.07447).
 *
 * One SIMULATION = Algorithm 1 "Scheduler(M, C)" run on
 * one workload until every request has generated its O tokens, under one
 * scheduler preset (Table 2; Table "Schedulers used",
 * PAPER.md:39-57), one replacement policy (NRF, Table 2; SRF / SRF+Hist,
 * PAPER.md:647-653) and 1..4 batch-latency models.
 * The semantics of every step are the readings Q1-Q40 of DESIGN.md.
 *
 * Conventions (all entry points):
 *  - plain pointers and sizes only; the CALLER owns every buffer.  sim_sweep()
 *    keeps one device arena, one pinned staging buffer and one stream per device
 *    for reuse across calls (grow-only, mutex-guarded: calls are thread-safe and
 *    serialized per device); sim_sweep_device() allocates nothing.
 *  - return value: 0 on success, < 0 on a call-level error (SIM_EINVAL ...;
 *    sim_strerror() names it).  Problems of one simulation are reported in its
 *    sim_result_t.status (SIM_S_*), never in the return value.
 *  - results of failed simulations (status != SIM_S_OK) are zero-filled.
 */
#ifndef SIMSWEEP_H
#define SIMSWEEP_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* GroupRequests order (step 1; Table 2; App. D) */
enum {
  SIM_ORDER_PREFILL_FIRST = 0, /* vLLM {R_w, R_r} */
  SIM_ORDER_DECODE_FIRST = 1,  /* Sarathi {R_r^d, R_r^p, R_w} */
  SIM_ORDER_RANK_ORG = 2,      /* one group by (T, id) */
  SIM_ORDER_RANK_I = 3,        /* one group by (I, T, id) */
  SIM_ORDER_RANK_O = 4         /* one group by (O, T, id) -- hypothetical, reads O */
};
/* cache replacement policy on preemption */
enum {
  SIM_NRF = 0,      /* newest (most recently admitted) request first, Table 2 */
  SIM_SRF = 1,      /* shortest (smallest m) request first */
  SIM_SRF_HIST = 2, /* SRF + online output-length histogram deferral */
  SIM_PF = 3        /* preemption-free (Table 2): never preempts; requires a
                       PEAK or CONTEXT reserve; running order = admission order (reading Q39) */
};
/* initial KV reserve at (re)admission (Table 2 "Initial KV reserve") */
enum {
  SIM_RESERVE_SEQ = 0,    /* s = I + g: r.I for vLLM / Sarathi, generalised to refills (reading Q13) */
  SIM_RESERVE_PEAK = 1,   /* I + O - 1: the *^pf schedulers */
  SIM_RESERVE_CONTEXT = 2 /* S: Orca */
};
/* alternative readings (sim_config_t.knobs bits) */
enum {
  SIM_KNOB_HOL = 1, /* Q10 alternative: the first waiting candidate that is not admitted ends the visit of R_w for
                       this step (vLLM's head-of-line blocking; a rank order skips the later waiting candidates) */
  SIM_KNOB_NRF_ARRIVAL = 2 /* Q6 alternative (NRF only): running requests are visited and retained in arrival
                              order (T, id) -- vLLM's FCFS running queue -- instead of admission order, so a refilled
                              request keeps its place and the newest ARRIVAL is preempted first */,
  SIM_KNOB_SRF_VISIT_ADMISSION = 4 /* Q3 alternative (SRF / SRF+Hist only): running requests are visited in admission
                                      order; SRF only chooses the victims (smallest m, later admission first) */
};
/* per-simulation status */
enum {
  SIM_S_OK = 0,
  SIM_S_TOO_LONG = 1,   /* some request has I+O-1 > S */
  SIM_S_NEVER_FITS = 2, /* I+O-1 (+ kv_watermark) > M, or > C without chunked prefill (reading Q35) */
  SIM_S_MAX_STEPS = 3,  /* more than max_steps batches */
  SIM_S_DEADLOCK = 4,   /* B empty, nothing arriving, requests unfinished (defensive) */
  SIM_S_CAPACITY = 5    /* a limit of this implementation: more than SIM_MAX_WINDOW arrived-but-unfinished requests
                           (only if n > SIM_MAX_WINDOW); or, with M infinite, KV holdings that could exceed 2^31 - 1
                           (sum over requests of max(I+O-1, the initial reserve) >= 2^31; the holdings are int32);
                           or more than 2^31 - 1 - n (re)admissions (the admission sequence number, reading Q6) */
};
/* call-level errors */
enum {
  SIM_EINVAL = -1,    /* NULL pointer, n <= 0, bad enum, C not in [1, 2^30], M > 2^30, S not in [1, 2^18), n_cost not 1..4,
                         replacement == SIM_PF without a PEAK / CONTEXT reserve or vice versa, unknown knob bits,
                         SIM_KNOB_NRF_ARRIVAL without SIM_NRF, SIM_KNOB_SRF_VISIT_ADMISSION without SRF,
                         max_seqs < 0, kv_watermark not in [0, 2^30), kv_block not in [0, 2^16] or > 1 with SRF+Hist */
  SIM_EWORKLOAD = -2, /* I < 1, O < 1, T not sorted, or T != 0 with n_cost > 1 */
  SIM_ECOST = -3,     /* cost-model index out of range or bad cost-model fields */
  SIM_ECUDA = -4,     /* a CUDA runtime error (device, allocation, launch) */
  SIM_ENODEV = -5     /* no sm_100 device */
};

#define SIM_MAX_COST 4
/* largest simultaneously tracked request window (arrived and not finished,
 * counted from the oldest unfinished request); larger -> SIM_S_CAPACITY.
 * Workloads of n <= 4096 requests never exceed it (state in shared memory);
 * larger ones use a per-simulation arena of the caller's workspace. */
#define SIM_MAX_WINDOW 32768

/* One simulation.  96 bytes, naturally aligned. */
typedef struct {
  int32_t order;       /* SIM_ORDER_* */
  int32_t hybrid;      /* 0/1: hybrid prefill+decode batches (step 2) */
  int32_t chunked;     /* 0/1: chunked prefill */
  int32_t replacement; /* SIM_NRF / SIM_SRF / SIM_SRF_HIST / SIM_PF */
  int32_t S;           /* model context size; requests need I+O-1 <= S */
  int32_t workload;    /* index into the workload table */
  int64_t C;           /* token limit per batch, 1 .. 2^30 */
  int64_t M;           /* KV-cache capacity in tokens, <= 2^30; < 0 = infinite (what-if) */
  int64_t max_steps;   /* livelock guard (>= 1) */
  int32_t n_cost;      /* 1..4 cost models charged on the same schedule; > 1 only for offline (all T = 0) */
  int32_t cost[SIM_MAX_COST]; /* indices into the cost-model table; the clock of cost[0] drives arrivals */
  int32_t reserve;     /* SIM_RESERVE_*; != SEQ iff replacement == SIM_PF */
  int32_t knobs;       /* SIM_KNOB_* bits: alternative readings (0 = the frozen semantics) */
  int32_t max_seqs;    /* Q16 alternative: at most this many entries per batch, like vLLM's max_num_seqs (0 = no cap) */
  int64_t kv_watermark;/* Q16 alternative: KVs a waiting admission must leave free, like vLLM's watermark (0 = none) */
  int32_t kv_block;    /* Q15 alternative: KVs are allocated in blocks of this many tokens, like vLLM's paged cache;
                          M and kv_watermark stay in tokens (capacity floor(M / kv_block) blocks); 0 or 1 = per token */
  int32_t pad;
} sim_config_t;

/* One workload: n requests sorted by (T, id).  The pointers are HOST memory
 * for sim_sweep() and DEVICE memory for sim_sweep_device(). */
typedef struct {
  int32_t n;      /* >= 1 */
  int32_t pad;
  const int32_t* I; /* [n] input tokens, >= 1 */
  const int32_t* O; /* [n] output tokens, >= 1 */
  const double* T;  /* [n] arrival times in seconds, non-decreasing */
} sim_workload_t;

/* One batch-latency model (Sec. "Cost Models for Batch Times").  mode 0 =
 * linear over the Table 3 variables, per layer
 *   t = a0 + a1 N + [n_p>0](b0 + b1 sum c^2 + b2 sum mc + b3 sum c + b4 sum m)
 *                 + [n_d>0](d0 + d1 sum m + d2 n_d),
 * mode 1 = Eq. (3) roofline per operator with Eq. (1)-(2) for
 * attention; batch time = layers * t.  flops / bw are aggregate over tp GPUs;
 * link_bw is the per-GPU All_Reduce bandwidth.  Evaluation order: DESIGN.md 2. */
typedef struct {
  int32_t mode;
  int32_t layers, h, f, H, NQ, NKV, e, tp;
  int32_t pad;
  double lin[10]; /* a0 a1 | b0 b1 b2 b3 b4 | d0 d1 d2, seconds per layer */
  double flops, bw, link_bw;
} sim_cost_model_t;

/* Per-simulation result (one per config). */
typedef struct {
  int32_t status; /* SIM_S_* */
  int32_t pad;
  int64_t steps;            /* number of batches B_j */
  int64_t preemptions;      /* including self-preemptions */
  int64_t batch_entries;    /* sum_j |B_j| */
  int64_t processed_tokens; /* sum_j sum_{B_j} c */
  int64_t sum_U;            /* sum_j KV holdings right after admission (kv usage = sum_U / (steps M)) */
  int64_t prefill_entries;  /* entries in the prefill phase */
  int64_t idle_jumps;       /* clock jumps to the next arrival (not steps) */
  int64_t visits;           /* sum over GetNextBatch calls of |P| (candidates visited, Alg. 1 line 9) */
  double makespan[SIM_MAX_COST];     /* max t_done - min T, per cost model */
  double mean_latency[SIM_MAX_COST]; /* mean t_done - T */
  double mean_ttft[SIM_MAX_COST];    /* mean t_first - T */
  double mean_tpot[SIM_MAX_COST];    /* mean (t_done - t_first)/(O-1) over O > 1 */
  int64_t formed_steps;     /* implementation counter, not a method output: the steps whose batch the kernel formed
                               explicitly; the rest (steps - formed_steps) were charged as steady decode runs */
} sim_result_t;

/* Per-request outputs.  Config i owns rows [row_off[i], row_off[i] + n_i) of
 * n_preempt / refill_tokens and rows [tim_off[i], tim_off[i] + n_cost_i * n_i)
 * of t_first / t_done, k-major (t_first[tim_off[i] + k*n_i + r]).  Offsets are
 * the exclusive prefix sums of n_i and n_cost_i * n_i in config order. */
typedef struct {
  double* t_first;        /* time the first token was generated */
  double* t_done;         /* time the O-th token was generated */
  int64_t* n_preempt;     /* times the request was preempted */
  int64_t* refill_tokens; /* sum of m discarded at its preemptions */
} sim_request_out_t;

/* Simulate n_cfgs configurations.  HOST buffers: cfgs[n_cfgs], wls[n_wls]
 * (with host arrays), cms[n_cms], results[n_cfgs] and req (sized by the
 * offsets above; any member may be NULL to skip it).  Uses CUDA device
 * `device` (or the current device if < 0).  Inputs are staged into a cached
 * pinned buffer and copied with one H2D; outputs are copied straight into the
 * caller's buffers (pinned buffers are fastest).  Returns 0 / SIM_E*.  Blocking. */
int sim_sweep(const sim_config_t* cfgs, int32_t n_cfgs, const sim_workload_t* wls, int32_t n_wls,
              const sim_cost_model_t* cms, int32_t n_cms, sim_result_t* results, sim_request_out_t req,
              int32_t device);

/* Same computation with everything already resident on the device.
 * d_cfgs[n_cfgs], d_wls[n_wls] (struct array in device memory whose I/O/T
 * point to device memory), d_cms[n_cms], d_results[n_cfgs], d_row_off[n_cfgs],
 * d_tim_off[n_cfgs] and the members of d_req are DEVICE pointers.  The host
 * arrays h_cfgs / h_wls_n (n of each workload) describe the same configs and
 * (n_wls entries) are used to validate every config field that does not need
 * the workload contents (the checks of sim_validate() below except I, O and T:
 * enums, knobs, C, M, S, n_cost, workload and cost indices; SIM_EINVAL /
 * SIM_ECOST), to choose kernel variants and the launch order; d_order[n_cfgs]
 * (device, may be NULL) is a permutation giving the launch order (e.g.
 * longest-first).  Launches asynchronously on `stream` (cudaStream_t, NULL =
 * legacy default stream) and does not synchronize; validation of workload
 * contents is the caller's responsibility (sim_validate() on the host copies,
 * which sim_sweep and the Python DeviceSweep do).  d_workspace
 * (device, caller-owned, may be NULL when sim_workspace_bytes() is 0) holds
 * the state of simulations whose workload has n > 4096 requests; its first 4
 * bytes are reset on `stream` before use, so one workspace serves successive
 * calls on one stream.  Returns the number of kernel launches issued (>= 1) or
 * SIM_E* (SIM_EINVAL if the workspace is missing or smaller than needed). */
int sim_sweep_device(const sim_config_t* h_cfgs, int32_t n_cfgs, const int32_t* h_wls_n, int32_t n_wls,
                     const sim_config_t* d_cfgs, const sim_workload_t* d_wls, const sim_cost_model_t* d_cms,
                     int32_t n_cms, const int32_t* d_order, const int64_t* d_row_off, const int64_t* d_tim_off,
                     sim_result_t* d_results, sim_request_out_t d_req, void* d_workspace,
                     int64_t workspace_bytes, void* stream);

/* Host-only validation of a sweep, exactly the checks sim_sweep() makes before it touches the device: every
 * config field (SIM_EINVAL / SIM_ECOST), every cost model (SIM_ECOST) and every workload's contents (I, O >= 1,
 * T sorted, T = 0 when n_cost > 1: SIM_EWORKLOAD).  HOST buffers.  Returns 0 or the first error found. */
int sim_validate(const sim_config_t* cfgs, int32_t n_cfgs, const sim_workload_t* wls, int32_t n_wls,
                 const sim_cost_model_t* cms, int32_t n_cms);

/* ---- per-step schedule trace of one simulation (the schedule log of PAPER.md:714-719) ----
 * One record per step j (a batch B_j; an idle arrival jump is not a step), in step order; the entries of B_j in
 * admission order (Algorithm 1's B); the preemptions of step j in the order they happened
 * (PAPER.md:1644-1646). */
typedef struct {
  int64_t step;      /* j, 0-based */
  int32_t n_entries; /* |B_j| (its entries follow the previous steps' in `entries`) */
  int32_t n_events;  /* preemptions during step j */
  int64_t U;         /* KV holdings after B_j was formed (before its completions free theirs) */
  int64_t tok;       /* sum of c over B_j */
  double start;      /* clock (cost model cost[0]) when the batch starts */
  double d;          /* its batch time d_j under cost[0] */
} sim_trace_step_t; /* 48 bytes */

typedef struct {
  int32_t id;       /* request index in the workload */
  int32_t phase;    /* 1 = prefill (incl. refills and chunks), 0 = decode */
  int32_t c;        /* tokens processed in this step */
  int32_t m_before; /* m of the request before the step */
} sim_trace_entry_t; /* 16 bytes */

typedef struct {
  int32_t id; /* the preempted request */
  int32_t m;  /* its m when it was preempted (the KVs discarded) */
} sim_trace_event_t; /* 8 bytes */

typedef struct {            /* HOST buffers, caller-owned */
  sim_trace_step_t* steps;  /* [cap_steps] */
  int64_t cap_steps;
  sim_trace_entry_t* entries; /* [cap_entries] */
  int64_t cap_entries;
  sim_trace_event_t* events; /* [cap_events] */
  int64_t cap_events;
  int64_t n_steps, n_entries, n_events; /* out: the totals; records beyond a cap are not written (call again
                                           with caps >= the totals for the whole log) */
} sim_trace_t;

/* Simulate ONE configuration (cfg->workload indexes wls) and record its schedule.  Same semantics, inputs and
 * outputs as sim_sweep() with n_cfgs = 1 (result[1], req sized for it), plus `trace`.  Steady decode runs are
 * not compressed while tracing (every step is formed), which changes no result.  Returns 0 / SIM_E*
 * (SIM_EINVAL for a NULL trace or negative caps).  Blocking. */
int sim_run_traced(const sim_config_t* cfg, const sim_workload_t* wls, int32_t n_wls, const sim_cost_model_t* cms,
                   int32_t n_cms, sim_result_t* result, sim_request_out_t req, sim_trace_t* trace, int32_t device);

/* Device workspace bytes sim_sweep_device() needs for these configs (host
 * arrays; wls_n = n of each workload): ~1.7 MB per simulation whose workload
 * has n > 4096 requests, 0 if there is none.  Returns >= 0 or SIM_EINVAL. */
int64_t sim_workspace_bytes(const sim_config_t* cfgs, int32_t n_cfgs, const int32_t* wls_n);

/* Scratch-free helper: total rows of the per-request outputs for n_cfgs configs
 * (rows = sum n_i, tim_rows = sum n_cost_i * n_i).  Returns 0 / SIM_EINVAL. */
int sim_request_rows(const sim_config_t* cfgs, int32_t n_cfgs, const sim_workload_t* wls, int32_t n_wls,
                     int64_t* rows, int64_t* tim_rows);

/* ---- Cost-model analytics: the batch-latency model of
 * row a9 evaluated on batch shapes instead of simulated batches.  All three
 * calls take HOST buffers, evaluate on CUDA device `device` (current if < 0),
 * are blocking, return 0 / SIM_E*, and use the expression order of DESIGN.md 2
 * (fp64, no contraction), so a shape gets the exact d_j a simulated batch with
 * the same entries gets. */

/* One batch shape: n_p prefill entries, each processing c tokens on top of m_p
 * cached KVs, plus n_d decode entries, each on top of m_d cached KVs
 * (Eq. (1)-(2) per request).  n_p, n_d >= 0, n_p + n_d >= 1,
 * c >= 1 when n_p > 0; every feature sum must stay below 2^62. */
typedef struct {
  int64_t n_p, c, m_p, n_d, m_d;
} sim_batch_shape_t;

/* Batch time (seconds) of every shape under every cost model:
 * out[k * n + i] = d(shapes[i]) under cms[k] (k-major).  SIM_EINVAL on a bad
 * shape or n <= 0, SIM_ECOST on a bad model. */
int sim_batch_times(const sim_cost_model_t* cms, int32_t n_cms, const sim_batch_shape_t* shapes, int32_t n,
                    double* out, int32_t device);

/* SLO frontier (Fig. SLO, "TPOT threshold of 1s" :574): a hybrid batch of n_p prefills
 * (c, m) and n_d decodes (m) sharing one m.  For every query and model, the
 * largest m in [0, m_max] whose batch time is <= tau (binary search; the time
 * is non-decreasing in m for non-negative linear coefficients and for Eq. (3)),
 * or -1 when even m = 0 exceeds tau.  out[k * n + i]. */
typedef struct {
  int64_t n_p, c, n_d, m_max;
  double tau; /* seconds (the paper's TPOT threshold: 1 s) */
} sim_slo_query_t;
int sim_slo_frontier(const sim_cost_model_t* cms, int32_t n_cms, const sim_slo_query_t* q, int32_t n, int64_t* out,
                     int32_t device);

/* Recompute vs swap and the 5-minute rule for KVs (Eq. (8)-(9),
 * PAPER.md:257-274).  For N[i] >= 1 KVs of one request and every model k:
 *   recompute[k*n+i] = d(one prefill entry, c = N, m = 0)          (refill cost)
 *   swap[k*n+i]      = N * 2 * layers * NKV * H * e / xfer_bw       (K and V over the host link)
 *   interval[k*n+i]  = recompute / N * M    (break-even interval t^N_recom M / N)
 * xfer_bw in bytes/s (> 0), M > 0.  Any output pointer may be NULL. */
int sim_kv_break_even(const sim_cost_model_t* cms, int32_t n_cms, const int64_t* N, int32_t n, double xfer_bw, int64_t M,
                      double* recompute, double* swap, double* interval, int32_t device);

/* Per-operator roofline classification ("What Makes a Batch Compute-Bound?"; Eq. (1)-(3),
 * PAPER.md:1703-1729).  For one layer of the batch shape shapes[i] under model cms[k], each operator o of
 * Eq. (3) (SIM_OP_*): its FLOPs and RW (elements; bytes = e * RW, reading Q26), its Eq. (3) time
 * max(FLOPs / flops, e * RW / bw), its intensity FLOPs / RW (FLOPs per element, the unit of PAPER.md:538:
 * attention -> 128 for large-c prefills and 2 / (1/128 + 1) ~ 1.98 for decodes on Llama-2-7B) and whether it is
 * compute-bound (FLOPs / flops > e * RW / bw).  Attention is summed per request with B = 1 (reading Q24).  The
 * operator times, summed in SIM_OP order (absent attentions skipped) and multiplied by `layers`, are the
 * theoretical batch time of sim_batch_times() when tp = 1 (tp > 1 adds two All_Reduce terms, not operators of
 * Eq. (3)).  The linear-mode coefficients are not used (every model carries its dims and GPU constants).
 * out[(k * n + i) * SIM_N_OPS + o].  HOST buffers, blocking; SIM_EINVAL on a bad shape or n <= 0, SIM_ECOST on
 * a bad model (flops and bw must be > 0). */
enum {
  SIM_OP_QKV = 0,          /* (N x h)(h x (N_Q + 2 N_KV) H) */
  SIM_OP_O = 1,            /* (N x N_Q H)(N_Q H x h) */
  SIM_OP_GATE_UP = 2,      /* (N x h)(h x 2f), SwiGLU (reading Q27) */
  SIM_OP_DOWN = 3,         /* (N x f)(f x h) */
  SIM_OP_ATTN_PREFILL = 4, /* Eq. (1)-(2) over the n_p prefill entries */
  SIM_OP_ATTN_DECODE = 5,  /* Eq. (1)-(2) over the n_d decode entries (c = 1) */
  SIM_N_OPS = 6
};
typedef struct {
  int64_t flops;    /* FLOPs of the operator (one layer) */
  int64_t rw;       /* elements read or written */
  double time;      /* Eq. (3) seconds, one layer */
  double intensity; /* flops / rw (FLOPs per element); 0 when the operator is absent */
  int32_t bound;    /* 1 compute-bound, 0 memory-bound, -1 absent (no prefill / decode entry) */
  int32_t pad;
} sim_op_cost_t; /* 40 bytes */
int sim_operator_costs(const sim_cost_model_t* cms, int32_t n_cms, const sim_batch_shape_t* shapes, int32_t n,
                       sim_op_cost_t* out, int32_t device);

/* ---- Exact optimum of the paper's CSP ----
 * A tiny offline workload of n <= SIM_OPT_MAX_N requests.  Every batch j chooses for each unfinished request
 * either preemption (e = 1: m := 0, Eq. (4)) or c in [0, s - m] (Eq. (5)); a token is generated iff
 * c = s - m (Eq. (6)); sum c <= C and sum m <= M after processing (Eq. (7)); a finished request holds its KVs
 * until the end of the batch that finished it.  The objective is sum_j d_j under the cost model (entries are
 * prefills unless the request's last (re)fill completed).  Batches with sum c = 0 are not considered (a
 * preemption can always ride with the next batch; readings Q43-Q45).  Solved exactly on the GPU by parallel
 * relaxation rounds over the dense state space (every reachable state, fp64 path sums), so the result is the
 * minimum over ALL schedules: a lower bound for every simulated preset.  Identical requests (same I and O) are
 * interchangeable, so a state is stored once per multiset of their local states (`states` counts those). */
#define SIM_OPT_MAX_N 4
#define SIM_OPT_NO_PREEMPT 1
typedef struct {
  int32_t n;                   /* requests, 1..SIM_OPT_MAX_N */
  int32_t I[SIM_OPT_MAX_N];    /* >= 1 */
  int32_t O[SIM_OPT_MAX_N];    /* >= 1 */
  int32_t flags;               /* bit 0 (SIM_OPT_NO_PREEMPT): e = 0 always -- the optimum over preemption-free schedules */
  int64_t C;                   /* token limit per batch, >= 1 */
  int64_t M;                   /* KV limit per batch, >= 0 (finite) */
} sim_opt_problem_t;
typedef struct {
  int32_t status;  /* 0 ok, 1 unreachable (some I + O - 1 > M), 2 state space too large (> 2^28 states) */
  int32_t rounds;  /* relaxation rounds until no state improved */
  int64_t states;  /* reachable states */
  double optimum;  /* min over schedules of sum_j d_j (seconds); 0 unless status 0 */
} sim_opt_result_t;
/* Solves n_probs problems in turn under cost model cm on CUDA device `device` (current if < 0).  HOST buffers;
 * blocking; returns 0 / SIM_E* (SIM_EINVAL on a bad problem, SIM_ECOST on a bad model). */
int sim_optimum(const sim_opt_problem_t* probs, int32_t n_probs, const sim_cost_model_t* cm, sim_opt_result_t* out,
                int32_t device);

/* Occupancy of the lean shared-memory kernel (configurations with n <= 1024 requests): how many of its
 * one-warp simulations share an SM.  Every simulation is one dependent chain, so a sweep whose length is set by a
 * few long simulations runs fastest with few per SM (the long ones lose less to their neighbours' issue slots and
 * instruction-cache footprint than the sweep gains from concurrency: BASELINE configs[1] 24.89 ms at 5 per SM,
 * 23.95-24.13 at 2, 26.09 at 1); a sweep of many equally long simulations needs the concurrency.  k = 1 .. 5 fixes
 * it (5 = the shared-memory maximum); k = 0 (the default) picks 2 when the launch has at most 32 such simulations
 * per SM, else 5.  Process-wide, host-only; applies to later sim_sweep / sim_sweep_device calls.  Returns 0, or
 * SIM_EINVAL for k outside 0 .. 5. */
int sim_set_lean_ctas_per_sm(int32_t k);

const char* sim_strerror(int code);
const char* sim_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SIMSWEEP_H */
