/*
 * padsim_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded-per-replay CPU discrete-event simulator of
 * the what-if evaluation defined by "Power Aware Dynamic Reallocation For
 * Inference" (arXiv 2601.12241, /root/reference/PAPER.md, cited "P:<line>")
 * under the readings of SURVEY.md §8(c) / DESIGN.md §3 (cited "c.N", "A<n>").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant with the product (paper_2601_12241_b200/, include/):
 * it has its own structs, its own model evaluation, its own event loop (a
 * binary heap, one event per decode step), its own controller.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread.
 */
#ifndef PADSIM_ORACLE_H
#define PADSIM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_MAX_ANCHORS 8
#define OR_MAX_GPUS 64

typedef struct { int32_t n; int32_t w[OR_MAX_ANCHORS]; double s[OR_MAX_ANCHORS]; } or_curve;

typedef struct {
    int32_t min_w, max_w;
    or_curve prefill, decode;
    double rate;          /* prefill tokens/s at the lowest anchor, batch 1 */
    double eff;           /* prefill batch efficiency per extra request      */
    double dec_fixed;     /* decode step fixed cost (s) at lowest anchor     */
    double dec_per_seq;   /* decode step cost per active sequence (s)        */
    double dec_per_ctx;   /* decode step cost per active context token (s)   */
    double kvb;           /* KV bytes per prompt token                       */
    double bw;            /* fabric bytes/s                                  */
    double ovh;           /* transfer fixed overhead (s)                     */
    int32_t max_pb;       /* max prefill batch (requests)                    */
    int32_t pb_tokens;    /* prefill batch token budget                      */
    int32_t max_db;       /* max decode batch                                */
    int32_t slots;        /* KV transfer request buffer (32)          */
    int32_t chunk;        /* coalesced mode: prefill chunk tokens (512) */
    int32_t ctx_growth;   /* 1: decode context counts generated tokens (A40)  */
} or_model;

typedef struct {
    int32_t kind;         /* 0 static, 1 dyn-power, 2 dyn-gpu, 3 dyn-both,
                             4 coalesced (non-disaggregated, chunked prefill) */
    int32_t threshold;    /* Alg.1 THRESHOLD on |Q_P|                        */
    int32_t step_w;       /* MovePower step (W)                              */
    int32_t dec_ceiling_w;/* decode dynamic ceiling (600 W)           */
    int32_t window_stamp; /* TTFT window samples stamped at 0: first token
                             (A22), 1: completion        */
    double cooldown_s, tick_s, window_s, settle_s, reassign_s;
} or_policy;

typedef struct { double ttft; double tpot[2]; } or_slo;

typedef struct {
    int32_t met, near_boundary, n_req, pad;
    double duration, goodput;
    int64_t events;       /* heap events processed (diagnostic)             */
    int32_t n_moves_power, n_moves_gpu, n_saturated, n_flips;
    double avg_watts;     /* time-weighted mean of Σ effective caps over [a_0, last completion] */
    double qps_per_watt;  /* goodput / avg_watts                                  */
    double sum_queue;     /* Σ_i (prefill start − arrival), request-id order (Fig. 6)    */
    double sum_exec;      /* Σ_i (prefill end − prefill start), request-id order               */
} or_summary;

/* log records for invariant tests (budget, cooldown, role bounds, masking) */
enum { OR_LOG_MOVE_POWER = 1, OR_LOG_MOVE_GPU = 2, OR_LOG_SATURATED = 3,
       OR_LOG_SETTLE = 4, OR_LOG_FLIP = 5, OR_LOG_BUDGET = 6, OR_LOG_ROLES = 7,
       OR_LOG_CAPS = 8 };
typedef struct { double t; int32_t type, gpu, a, b; } or_log_rec;
/* one controller tick: what Alg. 1 saw (window statistics, |Q_P|, per-GPU
 * load, drain-completion times), what it decided, and the node state after
 * the tick (for the host step_controller parity test)                       */
typedef struct {
    double t, ttft_stat, tpot_stat, ttft_slo, tpot_slo;
    int32_t q_prefill, kind, direction, gpu;
    int32_t load[OR_MAX_GPUS];
    double drained_empty[OR_MAX_GPUS];     /* draining GPU emptied at, else -1 */
    uint8_t role[OR_MAX_GPUS], draining[OR_MAX_GPUS];
    int32_t cmd[OR_MAX_GPUS], eff[OR_MAX_GPUS], raise_to[OR_MAX_GPUS];
    double last_move;
} or_tick_rec;
typedef struct { int32_t cap; int32_t n; or_log_rec* recs; int32_t tcap; int32_t tn; or_tick_rec* ticks; } or_log;

/* model functions (c.1) */
double or_speedup(const or_curve* c, int32_t w);
double or_prefill_lat(const or_model* m, int64_t tokens, int32_t b, int32_t w);
double or_decode_lat(const or_model* m, int32_t n, int64_t ctx, int32_t w);
double or_kv_lat(const or_model* m, int32_t tokens);
double or_p90(const double* v, int32_t n); /* nearest rank, copies + sorts  */
double or_percentile(const double* v, int32_t n, int32_t p);   /* nearest rank, p in 1..100 */

/* One replay: one candidate (role[N], cap[N], policy) x one trace x one QPS.
 * Outputs per request (nullable arrays of n_req).  Returns 0 or <0 on bad
 * input / allocation failure.                                               */
int or_replay(const or_model* m, int32_t n_gpus, const uint8_t* role, const int32_t* cap,
              const or_policy* pol, int32_t budget_w, const or_slo* slo,
              int32_t n_req, const double* s_unit, const int32_t* in_tok,
              const int32_t* out_tok, const uint8_t* phase, double qps_per_gpu,
              double* ttft, double* tpot, double* prefill_end, double* completion,
              double* transfer_end, double* prefill_start, or_summary* sum, or_log* log);

/* Whole evaluation: n_cand x n_qps x n_traces replays over n_threads host
 * threads; Σ over traces in ascending trace order; argmax per QPS with key
 * (Σmet desc, Σcaps asc, index asc) (c.4).  Optional per-replay outputs
 * indexed [(c*n_qps + q)*n_traces + s].                                      */
int or_evaluate(const or_model* m, int32_t n_gpus, int32_t n_cand, const uint8_t* role,
                const int32_t* cap, const or_policy* pol, int32_t budget_w,
                const int32_t* cand_budget_w /* nullable: per-candidate budgets [n_cand] */,
                const or_slo* slo, int32_t n_traces, const int32_t* n_req, const double* const* s_unit,
                const int32_t* const* in_tok, const int32_t* const* out_tok,
                const uint8_t* const* phase, int32_t n_qps, const double* qps,
                int32_t n_threads, int64_t* met, double* goodput, int64_t* near_boundary,
                int32_t* argmax, int32_t* rep_met, double* rep_goodput, double* rep_duration);

/* met count of one replay's per-request records against K SLO sets (the
 * inclusive rule of S:407, per-phase TPOT SLO): out_met[k].           */
int or_met_for_slos(int32_t n_req, const double* ttft, const double* tpot, const uint8_t* phase,
                    int32_t n_slo, const or_slo* slos, int32_t* out_met);

/* Pool-uniform candidate enumeration by brute force over (x, p, d) (a1). */
int or_enumerate(int32_t n_gpus, int32_t budget_w, int32_t min_w, int32_t max_w, int32_t step_w,
                 int32_t exact, int32_t* out_xpd, int32_t cap, int32_t* n_out);

/* Alg. 1 decision (pure), for controller parity with the product. */
typedef struct {
    uint8_t role[OR_MAX_GPUS];      /* 0 P, 1 D                               */
    uint8_t draining[OR_MAX_GPUS];
    int32_t cmd[OR_MAX_GPUS];       /* commanded caps                         */
    int32_t n_gpus;
    int32_t drain_pending;          /* a role change is in progress           */
    double last_move;
} or_ctl_state;
typedef struct {
    double ttft_stat, tpot_stat, ttft_slo, tpot_slo;
    int32_t q_prefill;
    int32_t load[OR_MAX_GPUS];      /* P: outstanding tokens; D: active+pending */
} or_ctl_obs;
typedef struct {
    int32_t kind;                   /* 0 none, 1 move-power, 2 move-gpu, 3 saturated */
    int32_t direction;              /* 0 D->P, 1 P->D                          */
    int32_t gpu;                    /* drained GPU for move-gpu                */
    int32_t new_cap[OR_MAX_GPUS];   /* caps after the move settles             */
} or_ctl_action;
int or_step_controller(const or_policy* pol, const or_model* m, int32_t budget_w,
                       or_ctl_state* st, const or_ctl_obs* obs, double now, or_ctl_action* act);

#ifdef __cplusplus
}
#endif
#endif
