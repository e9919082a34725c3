/*
 * padsim.h — C ABI of the B200-native what-if evaluator for power-aware
 * prefill/decode disaggregation ("Power Aware Dynamic Reallocation For
 * Inference", arXiv 2601.12241; /root/reference/PAPER.md cited "P:<line>",
 * SPEC.md cited "S:<line>", readings "A<n>"/"c.N" = SURVEY.md §8(c) and
 * DESIGN.md §3).
 *
 * What it computes (BASELINE.json north_star; SURVEY.md §8(a) rows a1–a8):
 * for every candidate allocation — an xPyD split of the node's GPUs into
 * prefill and decode roles with per-GPU power caps under a node budget
 * (P:129), optionally with the paper's dynamic reallocation policy
 * (Algorithm 1) — replay every trace at every QPS point through
 * the prefill/decode latency-and-power model, score
 * every request against the TTFT/TPOT SLOs, reduce to SLO
 * attainment and goodput per (candidate, QPS), and take the argmax per QPS.
 *
 * Conventions
 *  - Every function is extern "C", returns int status (PADSIM_OK = 0, <0 =
 *    error), never throws, never aborts.  padsim_last_error() gives a static
 *    message for the last failure on that context.
 *  - Input pointers are caller-owned HOST memory unless the parameter name
 *    starts with "d_" (device memory); they are read during the call only.
 *  - Output buffers are caller-allocated with the documented sizes.
 *  - A padsim_ctx owns its device buffers (cudaMalloc) and is bound to one
 *    CUDA device; it is not thread-safe (one ctx per host thread/stream).
 *  - "stream" parameters are cudaStream_t passed as void* (NULL = default).
 *  - All times are FP64 seconds, all powers int32 watts.  Results are
 *    deterministic: bit-identical for identical inputs.
 *  - There is no CPU fallback: without a usable CUDA device every compute
 *    call fails with PADSIM_ECUDA.
 */
#ifndef PADSIM_H
#define PADSIM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PADSIM_MAX_GPUS 64      /* simulated GPUs per node (cfg 5: 64)          */
#define PADSIM_MAX_ANCHORS 8    /* anchors per power->speedup curve             */
#define PADSIM_MAX_SLOTS 32     /* KV request buffer bound (32)          */
#define PADSIM_MAX_DECODE_BATCH 256
#define PADSIM_MAX_PREFILL_BATCH 256

enum {
    PADSIM_OK = 0,
    PADSIM_EINVAL = -1,   /* null pointer, bad size, bad policy field              */
    PADSIM_ERANGE = -2,   /* a cap outside [min_w, max_w]            */
    PADSIM_EBUDGET = -3,  /* Σ caps > budget; bad_index = first offender   */
    PADSIM_EROLE = -4,    /* prefill or decode role count outside [1, N−1] */
    PADSIM_EMODEL = -5,   /* anchors unsorted / non-monotone / not spanning
                             [min_w,max_w] / first speedup != 1 / params <= 0
                                                           */
    PADSIM_EDOMAIN = -6,  /* token count < 1 or unsorted arrivals    */
    PADSIM_ECUDA = -7,    /* CUDA runtime/kernel error or no device                */
    PADSIM_ENOMEM = -8    /* host or device allocation failure                     */
};

typedef struct padsim_ctx padsim_ctx;

/* a2 — one synthetic trace, sorted by arrival.  s_unit[i] are cumulative
 * arrival times of a unit-rate process (first gap > 0 or 0); the arrival at
 * QPS-per-GPU q on N GPUs is s_unit[i] * (1.0/(q*(double)N)) (A16).
 * phase[i] ∈ {0,1} selects the per-phase TPOT SLO.  in_tok ≥ 1,
 * out_tok ≥ 1 (the first output token comes from prefill).          */
typedef struct {
    int32_t n_req;
    const double* s_unit;
    const int32_t* in_tok;
    const int32_t* out_tok;
    const uint8_t* phase;    /* nullable: all phase 0 */
} padsim_trace;

/* A1 — piecewise-linear power->speedup curve (D1 S:92, D3 S:94):
 * anchors strictly increasing in w, w[0] = min_w, w[n-1] = max_w,
 * s non-decreasing, s[0] = 1.0.                                             */
typedef struct { int32_t n; int32_t w[PADSIM_MAX_ANCHORS]; double s[PADSIM_MAX_ANCHORS]; } padsim_curve;

/* a3 — latency/power model (c.1, defaults D2 S:93):
 *   prefill_lat(T,b,w) = ((double)T / (rate*(1+eff*(b-1)))) / s_pre(w)
 *   decode_lat(n,C,w)  = (fixed + per_seq*n [+ per_ctx*C]) / s_dec(w)
 *   kv_lat(T)          = overhead + (T*kv_bytes)/fabric_bw                  */
typedef struct {
    int32_t min_w, max_w;              /* cap range (400–750 W), max_w − min_w ≤ 511 */
    padsim_curve prefill, decode;
    double prefill_base_rate;          /* tokens/s at min_w, batch 1  (> 0)     */
    double prefill_batch_eff;          /* per extra batch member      (>= 0)    */
    double decode_fixed_s;             /* per step at min_w           (> 0)     */
    double decode_per_seq_s;           /* per active sequence         (>= 0)    */
    double decode_per_ctx_tok_s;       /* per active context token (>= 0; 0 = SPEC form, A15) */
    double kv_bytes_per_token;         /* (> 0) Llama-3.1-8B: 131072     */
    double fabric_bw_Bps;              /* (> 0)                                  */
    double transfer_overhead_s;        /* (> 0)                                  */
    int32_t max_prefill_batch;         /* [1, 256]  (A9: 16)                     */
    int32_t prefill_token_budget;      /* >= 1      (16384)               */
    int32_t max_decode_batch;          /* [1, 256]  (64)                  */
    int32_t transfer_slots;            /* [1, 32]   (32)                  */
    int32_t prefill_chunk_tokens;      /* >= 1, coalesced mode only (512) */
    int32_t decode_ctx_growth;         /* 0/1. 1: the decode context of a step counts the
                                          tokens generated so far, C = Σ (in_i + s − join_i)
                                          (A40); boundaries of a segment are then the
                                          arithmetic-series sums t0 + (k·L1 + k(k−1)/2·d) */
} padsim_model;

/* Algorithm 1 constants for one candidate.  kind: 0 static,
 * 1 dyn-power, 2 dyn-gpu, 3 dyn-both, 4 coalesced — the
 * paper's non-disaggregated baseline with chunked prefill (SPEC
 * S:262–269; readings A33–A37): every GPU serves both phases at its cap,
 * role[] is ignored, no KV transfer (transfer_end = prefill_end), one engine
 * step = ≤ prefill_chunk_tokens of the head prompt fused with the active
 * decode batch.  For kind 1–3:
 * tick_s > 0 (MIN_TIME), settle_s > 0, reassign_s > 0
 * (P:294), cooldown_s >= settle_s, window_s >= 0, power_step_w > 0,
 * decode_ceiling_w ∈ [min_w, max_w], queue_threshold >= 0,
 * window_stamp ∈ {0, 1}.                                                      */
typedef struct {
    int32_t kind;
    int32_t queue_threshold, power_step_w, decode_ceiling_w;
    int32_t window_stamp;   /* controller TTFT samples stamped at 0: the first token
                               (prefill end, reading A22 — the default) or 1: request
                               completion; TPOT samples are always
                               stamped at completion                                  */
    double cooldown_s, tick_s, window_s, settle_s, reassign_s;
} padsim_policy;

/* D7 — candidate set: n_cand rows of n_gpus entries.  role 0 = prefill,
 * 1 = decode; cap_w = initial per-GPU cap.  policy[n_cand].               */
typedef struct {
    int32_t n_gpus, n_cand;
    const uint8_t* role;
    const int32_t* cap_w;
    const padsim_policy* policy;
} padsim_candidates;

/* SLOs: inclusive ≤ (A6). All > 0.           */
typedef struct { double ttft_s; double tpot_s[2]; } padsim_slo;
/* Node GPU power budget (4800 W).  cand_budget_w (nullable) gives a
 * budget per candidate [n_cand] instead — e.g. Fig. 5a's 4P4D-750W reference
 * at 6000 W next to 4800 W candidates; it bounds Σ caps (validation)
 * and DistributeUniformPower / the N·min_w check of a dynamic candidate.      */
typedef struct { int32_t budget_w; const int32_t* cand_budget_w; } padsim_budget;

/* a7/a8 results.  met[c*n_qps+q] = Σ over traces of requests meeting both
 * SLOs (int, exact); goodput = Σ over traces (ascending) of met/duration;
 * near_boundary = requests within 1e-9 relative of an SLO; argmax[q] =
 * candidate maximising (Σmet ↓, Σcaps ↑, index ↑) (A25).  Any pointer may
 * be NULL.  bad_index: first offending candidate on EBUDGET/ERANGE/EROLE,
 * else -1.                                                                  */
typedef struct {
    int64_t* met;
    double* goodput;
    int64_t* near_boundary;
    int32_t* argmax;
    int32_t bad_index;
} padsim_result;

/* ---- context ------------------------------------------------------------ */
/* padsim_create: bind a context to CUDA device `cuda_device`; `cuda_stream`
 * (cudaStream_t as void*, NULL = the legacy default stream) is the stream the
 * one-shot padsim_evaluate_allocations runs on.  ECUDA without a device.     */
int padsim_create(int32_t cuda_device, void* cuda_stream, padsim_ctx** out);
void padsim_destroy(padsim_ctx* ctx);
const char* padsim_last_error(const padsim_ctx* ctx);
const char* padsim_version(void);

/* ---- evaluate_allocations (north_star) ------------------------------------
 * One-shot host API: validate, upload, run every replay (n_cand × n_qps ×
 * n_traces), reduce, argmax, download.  Synchronous.  qps_per_gpu[n_qps] > 0.
 */
int padsim_evaluate_allocations(padsim_ctx* ctx, const padsim_trace* traces, int32_t n_traces,
                                const double* qps_per_gpu, int32_t n_qps,
                                const padsim_model* model, const padsim_candidates* cands,
                                const padsim_slo* slo, const padsim_budget* budget,
                                padsim_result* out);

/* ---- split API (inputs resident in HBM between calls) ---------------------
 * padsim_plan: validate + upload inputs + precompute model tables (a3) on the
 * device; synchronous; replaces any previous plan.  flags: PADSIM_RECORDS
 * keeps per-request records (memory n_cand*n_qps*Σn_req*40 B).
 * padsim_run: launch the replay, seed-reduction and argmax kernels on
 * `stream`; asynchronous; results stay in ctx-owned device buffers.
 * padsim_fetch: copy the last run's results to host (synchronises stream).
 */
#define PADSIM_RECORDS 1u
#define PADSIM_JOINT 2u     /* N <= 8: replay static candidates in the joint kernel instead
                               of the factorized stage A / stage C path (cross-check, ablation) */
int padsim_plan(padsim_ctx* ctx, const padsim_trace* traces, int32_t n_traces,
                const double* qps_per_gpu, int32_t n_qps, const padsim_model* model,
                const padsim_candidates* cands, const padsim_slo* slo,
                const padsim_budget* budget, uint32_t flags, int32_t* bad_index);
int padsim_run(padsim_ctx* ctx, void* stream);
int padsim_fetch(padsim_ctx* ctx, void* stream, padsim_result* out);

/* Device views of the last run's outputs (valid until the next plan/destroy):
 * d_met i64[C*Q], d_goodput f64[C*Q], d_near i64[C*Q], d_argmax i32[Q],
 * per replay r = (c*Q + q)*S + s: d_rep_met i32, d_rep_near i32,
 * d_rep_duration f64, d_rep_goodput f64, d_rep_events i64 [C*Q*S].          */
typedef struct {
    int64_t* d_met; double* d_goodput; int64_t* d_near; int32_t* d_argmax;
    int32_t* d_rep_met; int32_t* d_rep_near; double* d_rep_duration; double* d_rep_goodput;
    int64_t* d_rep_events;
    int32_t n_cand, n_qps, n_traces;
    int64_t* d_aux_events;   /* DES instants of shared prefill stages (factorized static
                                path: one per prefill group x QPS x trace), n_aux_events */
    int32_t n_aux_events;
} padsim_device_results;
int padsim_get_device_results(padsim_ctx* ctx, padsim_device_results* out);

/* Device time of the replay kernel(s) of the last padsim_run in ms, measured
 * with CUDA events recorded on the run's stream around the replay launches
 * (synchronises on the end event).                                          */
int padsim_replay_kernel_ms(padsim_ctx* ctx, float* ms);

/* Per-kernel device times of the last padsim_run in ms (CUDA events on the
 * run's stream): [0] stage A (static prefill), [1] stage C (static decode),
 * [2] joint + coalesced replays (dynamic candidates, static when N > 8,
 * policy kind 4), which start after [0] on a side stream concurrently with
 * [1]; 0 if not run.                                                       */
int padsim_kernel_times_ms(padsim_ctx* ctx, float* ms3);

/* ---- SLO scaling, QPS/W, max QPS at 80 % ---------------
 * Static trajectories do not depend on the SLOs, so extra SLO sets are scored
 * on the same replays for the cost of a compare (Fig. 5b TPOT 25 ms, Fig. 8
 * SLO scaling 0.5x–2x).  padsim_set_slo_sweep (after padsim_plan,
 * before padsim_run): up to PADSIM_MAX_SLO_SWEEP extra SLO sets (all > 0).
 * padsim_fetch_extras (synchronises), any pointer may be NULL:
 *   met_sweep[(c*Q + q)*8 + k]  Σ over traces of requests meeting SLO set k
 *   qps_per_watt[c*Q + q]       Σ over traces (ascending) of goodput / avg
 *                               provisioned GPU W
 *   avg_watts[c*Q + q]          Σ over traces of the time-weighted mean of the
 *                               Σ of effective caps over [a_0, last completion]
 *                               (static: Σ caps); divide by n_traces for a mean
 *   max_qps80[c*9 + k]          k = 0: main SLO, k = 1..8: sweep set k−1 — the
 *                               QPS index with the largest QPS among those with
 *                               5·Σmet ≥ 4·Σ n_req (≥ 80 % attainment),
 *                               −1 if none.                                      */
#define PADSIM_MAX_SLO_SWEEP 8
int padsim_set_slo_sweep(padsim_ctx* ctx, const padsim_slo* slos, int32_t n_slo);
int padsim_fetch_extras(padsim_ctx* ctx, void* stream, int64_t* met_sweep, double* qps_per_watt,
                        double* avg_watts, int32_t* max_qps80);

/* Per-replay host copies (synchronises): arrays of C*Q*S, any may be NULL. */
int padsim_fetch_replays(padsim_ctx* ctx, void* stream, int32_t* met, int32_t* near_boundary,
                         double* duration, double* goodput, int64_t* events);

/* Per-request records of the last run (plan flag PADSIM_RECORDS): for replay
 * r = (c*Q + q)*S + s, request i at [r*R_max + i] where R_max = max n_req;
 * arrays of C*Q*S*R_max, any may be NULL.                                   */
int padsim_fetch_records(padsim_ctx* ctx, void* stream, double* ttft, double* tpot,
                         double* prefill_end, double* completion, double* transfer_end,
                         int32_t* r_max);

/* One candidate x one trace x one QPS point, per-request records (SURVEY §8(b)
 * parity/debug helper; the same kernels as padsim_evaluate_allocations): plans
 * `ctx` with PADSIM_RECORDS for cands->n_cand == 1, runs it on the ctx's stream
 * and copies the records of the replay to the caller's buffers, each
 * [trace->n_req] doubles (any may be NULL):  ttft = prefill_end − arrival,
 * tpot = (completion − prefill_end)/(out−1), 0 for out = 1 (A7), prefill_end,
 * completion.  Errors as padsim_plan (EINVAL if n_cand != 1).  Re-plans ctx. */
int padsim_replay_records(padsim_ctx* ctx, const padsim_trace* trace, double qps_per_gpu,
                          const padsim_model* model, const padsim_candidates* one,
                          const padsim_slo* slo, const padsim_budget* budget, double* ttft,
                          double* tpot, double* prefill_end, double* completion);

/* ---- Fig. 6 TTFT decomposition, percentiles ----------
 * padsim_fetch_decomposition (synchronises; any pointer may be NULL):
 *   rep_queue[r], rep_exec[r]   r = (c*Q + q)*S + s: Σ over the replay's
 *       requests of (prefill batch start − arrival) and (prefill end − batch
 *       start) — the queueing-delay / prefill-execution split of TTFT that
 *       Fig. 6 reports (TTFT = queue + exec + KV transfer)
 *   sum_queue[c*Q + q], sum_exec[c*Q + q]   Σ over traces (ascending) of the
 *       per-replay sums; divide by Σ_s n_req for per-request means.
 * Summation order inside a replay is batch-completion order (the oracle sums
 * in request-id order): FP64 agreement is to rounding (≤ 1e-9 relative).
 * padsim_fetch_percentiles (plan flag PADSIM_RECORDS, after padsim_run;
 * synchronises): nearest-rank percentiles (S:426–432, 1-based rank
 * ⌈p·n/100⌉) of each replay's TTFT and TPOT records, pcts[k] ∈ [1, 100],
 * 1 ≤ n_pct ≤ PADSIM_MAX_PCT, out[(r*2 + m)*n_pct + k] (m = 0 TTFT, 1 TPOT),
 * NaN for an empty trace. Exact (a sort; no arithmetic). EINVAL otherwise.  */
#define PADSIM_MAX_PCT 16
int padsim_fetch_decomposition(padsim_ctx* ctx, void* stream, double* rep_queue, double* rep_exec,
                               double* sum_queue, double* sum_exec);
int padsim_fetch_percentiles(padsim_ctx* ctx, void* stream, const int32_t* pcts, int32_t n_pct,
                             double* out);

/* a8 across ranks: argmax per QPS over a device met array
 * d_met[n_cand * n_qps] (e.g. the all-gathered scores of every rank's shard)
 * with the key (Σmet ↓, Σcaps ↑, index ↑) (A25).  d_capsum[n_cand] (device,
 * nullable) gives each candidate's Σ initial caps; NULL uses the planned
 * candidates' (then n_cand must equal the plan's).  Asynchronous on stream.  */
int padsim_argmax_device(padsim_ctx* ctx, void* stream, const int64_t* d_met, const int32_t* d_capsum,
                         int32_t n_cand, int32_t n_qps, int32_t* d_argmax);

/* ---- step_controller (north_star; Algorithm 1) -----------------
 * A PURE HOST FUNCTION (no context, no device, no allocation; thread-safe:
 * it touches only *inout and *out).  One controller invocation at time now_s
 * on the full controller state of one node:
 *   1. time-driven transitions due by now_s, in the A10 kind order:
 *      settle: every GPU with settle_deadline_s[g] <= now_s takes
 *      eff = cmd when cmd < eff and, if pending_raise_w[g] > 0, cmd = eff =
 *      pending_raise_w[g] (sinks are raised at the donors' settle instant,
 *      source-before-sink); the deadline is cleared (< 0).
 *      role flip: a draining GPU whose drain completed
 *      (stats->drained_empty_s[g] >= 0) flips roles at drained_empty_s[g] +
 *      reassign_s; if that time is <= now_s the flip is applied (role ^= 1,
 *      draining = 0), otherwise flip_deadline_s[g] holds it.
 *   2. the Alg. 1 decision on the window statistics (guards strict as printed,
 *      P:229–240, A20; cooldown strict; |Q_P| > THRESHOLD; PowerLimitsReached
 *      checked before moving, A18): MovePower (donors −min(step,
 *      cap−floor), recipients +min(⌊F/|rec|⌋, ceiling−cap)), else MoveGPU of
 *      the least-loaded donor (load[g], lowest id) + DistributeUniformPower
 *      (clamp(B/N, min_w, max_w)) when the policy allows, the donor
 *      role keeps >= 1 GPU and no role change is pending, else saturated.
 *      Draining GPUs belong to neither pool (A26).  Policy masking S:323.
 *   3. a move commands decreases at once (cmd), holds raises in
 *      pending_raise_w, sets every GPU's settle_deadline_s = now_s + settle_s,
 *      marks the MoveGPU donor draining, and sets last_move_s = now_s.
 * Errors: EINVAL (null / n_gpus outside [2, 64] / role not 0/1 / bad policy),
 * EMODEL (model), ERANGE (a cap outside [min_w, max_w]).                     */
typedef struct {
    uint8_t role[PADSIM_MAX_GPUS];         /* 0 prefill, 1 decode                      */
    uint8_t draining[PADSIM_MAX_GPUS];     /* drain in progress: in neither pool (A26) */
    int32_t cmd_cap_w[PADSIM_MAX_GPUS];    /* commanded caps                           */
    int32_t eff_cap_w[PADSIM_MAX_GPUS];    /* effective caps (what the budget charges)  */
    int32_t pending_raise_w[PADSIM_MAX_GPUS];  /* raise applied at the settle, 0 = none */
    double settle_deadline_s[PADSIM_MAX_GPUS]; /* < 0: none                             */
    double flip_deadline_s[PADSIM_MAX_GPUS];   /* < 0: none (set once the drain is done) */
    int32_t n_gpus;
    double last_move_s;                    /* Alg. 1 last_move_time, 0 initially */
} padsim_ctrl_state;
typedef struct {
    double ttft_stat_s, tpot_stat_s;       /* window p90 statistics (A22), 0 = empty   */
    double ttft_slo_s, tpot_slo_s;         /* SLOs in effect                   */
    double rate_p, rate_d;                 /* Alg. 1 inputs, unused by the guards (A21) */
    int32_t q_prefill, q_decode;           /* |Q_P| queued prompts; |Q_D| (A21) */
    int32_t load[PADSIM_MAX_GPUS];         /* P: outstanding tokens, D: active+pending  */
    double drained_empty_s[PADSIM_MAX_GPUS];   /* draining GPU: when it became empty, else < 0 */
} padsim_window_stats;
typedef struct {
    int32_t kind;                          /* 0 none, 1 move-power, 2 move-gpu, 3 saturated */
    int32_t direction;                     /* 0 D->P, 1 P->D, -1 none                 */
    int32_t gpu;                           /* drained GPU (move-gpu) else -1           */
    int32_t new_cap_w[PADSIM_MAX_GPUS];    /* targets once the move settles            */
} padsim_action;
int padsim_step_controller(const padsim_policy* policy, const padsim_budget* budget,
                           const padsim_model* model, padsim_ctrl_state* inout,
                           const padsim_window_stats* stats, double now_s, padsim_action* out);

/* The same Alg. 1 decision (step 2 only; no transitions, no state change) run
 * on the device by the __device__ code the dynamic replay kernel uses
 * (controller.cuh ctl_step): for parity tests of the kernel's controller
 * against the host step.  Reads role, draining, cmd_cap_w, pending_raise_w,
 * last_move_s of *state.  Synchronous on the context's stream.              */
int padsim_controller_decide_device(padsim_ctx* ctx, const padsim_policy* policy,
                                    const padsim_budget* budget, const padsim_model* model,
                                    const padsim_ctrl_state* state, const padsim_window_stats* stats,
                                    double now_s, padsim_action* out);

/* ---- launch tuning (tests, ablations) ----------------------------------------
 * padsim_set_tuning (before padsim_plan; kept until changed): overrides of the
 * launch configuration the planner otherwise picks from the workload size.
 * Results never depend on it (every variant is parity-tested); 0 / -1 = auto.
 *   stage_a_threads      32, 128 or 256 threads per stage-A CTA
 *   stage_c_classes      3 or 5 decode-pool classes
 *   stage_c_batch_lists  bit k: class k uses sorted batch lists (-1 auto)
 *   joint_threads        32 or 128 threads per joint-replay CTA
 *   joint_reg_cap        1: the 168-register one-warp joint variant, 0: not (-1 auto)
 *   joint_lanes_per_warp replays per warp item of the joint kernel (1..32)
 *   joint_after_stage_a  1: joint replays wait for stage A (-1 auto)
 *   serialize            1: padsim_run launches every kernel on its stream, one
 *                        after another (per-kernel times in isolation, for the
 *                        roofline), 0: concurrent streams (read at run time)
 *   joint_groups         N ≤ 8 joint replays: 1 lane groups (one lane per simulated
 *                        GPU, 4 replays per warp; group_path.cuh), 0 one thread per
 *                        replay (dynamic_path.cuh), -1 auto (one thread per replay:
 *                        measured faster)
 *   wide_path            8 < N ≤ 64 static candidates: 1/-1 the factorized
 *                        warp-per-replay stages (wide_path.cuh), 0 the joint kernel
 *   wide_chunk           traces per stage A → C chunk of the wide path (0 auto:
 *                        as many as half the free device memory holds)        */
typedef struct {
    int32_t stage_a_threads, stage_c_classes, stage_c_batch_lists;
    int32_t joint_threads, joint_reg_cap, joint_lanes_per_warp, joint_after_stage_a;
    int32_t serialize;
    int32_t joint_groups, wide_path, wide_chunk;
} padsim_tuning;
int padsim_set_tuning(padsim_ctx* ctx, const padsim_tuning* tuning);

/* Kernel launches issued by the last padsim_run (for the bench's launch count). */
int padsim_launch_count(padsim_ctx* ctx, int32_t* n);

/* Which path the planner chose for the static candidates of the current plan
 * (*path): 0 none, 1 thread-per-replay factorized stages (stageA_kernel /
 * stageC_kernel, N ≤ 8), 2 warp-per-replay factorized stages (stageA_wide_kernel /
 * stageC_wide_kernel: 8 < N ≤ 64, or N ≤ 8 with ≤ 8 static replays per SM),
 * 3 the joint kernel.  PADSIM_EINVAL without a plan.                         */
int padsim_static_path(padsim_ctx* ctx, int32_t* path);

/* ---- a1 candidate enumeration (host) ----------------------------------------
 * All pool-uniform (x, p, d): x ∈ [1, N−1] prefill GPUs at p W, N−x decode
 * GPUs at d W, p,d ∈ {min_w + k·step_w} ∩ [min_w, max_w], x·p + (N−x)·d ≤ B
 * (== B if exact).  Lexicographic (x, p, d) order.
 * out_xpd may be NULL to count; *n_out = total count (may exceed cap).       */
int padsim_enumerate_pool_uniform(int32_t n_gpus, int32_t budget_w, int32_t min_w, int32_t max_w,
                                  int32_t step_w, int32_t exact, int32_t* out_xpd, int32_t cap,
                                  int32_t* n_out);

#ifdef __cplusplus
}
#endif
#endif
