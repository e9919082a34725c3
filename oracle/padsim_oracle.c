/*
 * padsim_oracle.c — TEST INFRASTRUCTURE ONLY (see padsim_oracle.h).
 *
 * Plain heap-based discrete-event simulator of the paper's disaggregated,
 * power-capped node.  Every rule below names the passage it follows:
 *   P:<line>  /root/reference/PAPER.md (the authority on what is computed)
 *   S:<line>  /root/reference/SPEC.md  (surrogate constants, worked examples)
 *   c.N / A<n> the readings of SURVEY.md §8(c), restated in DESIGN.md §3.
 * It deliberately does nothing clever: one heap event per decode step, FIFO
 * ring buffers, p90 by sorting the window, linear scans for routing.
 *
 * Parity status: model (c.1), static replay (c.2), controller (Alg. 1, c.3)
 * and dynamic replay (c.3) are pinned by tests/test_oracle_*.py (Appendix A
 * values, Lindley recursion, M/D/1, hand-worked one/two-request examples,
 * SPEC controller examples, invariants, brute force).  Absolute attainment
 * levels versus the paper's figures: parity unpinned (figures absent).
 */
#include "padsim_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* c.1 model evaluation — SPEC perf-model S:40–74, defaults D1/D2 S:92–93.   */
/* Pinned operation order, no FMA (built with -ffp-contract=off).           */
/* ------------------------------------------------------------------------ */

/* Piecewise-linear interpolation over the anchors (SPEC D3 S:94), exact at
 * anchors; the power→speedup relation of Fig. 4a/b.          */
double or_speedup(const or_curve* c, int32_t w) {
    int n = c->n;
    if (w == c->w[n - 1]) return c->s[n - 1];
    int j = 0;
    for (int k = 0; k < n - 1; k++)
        if (c->w[k] <= w) j = k;
    double diff = c->s[j + 1] - c->s[j];
    double frac = (double)(w - c->w[j]) / (double)(c->w[j + 1] - c->w[j]);
    return c->s[j] + diff * frac;
}

/* prefill_latency: whole-batch latency for T tokens, b requests. */
double or_prefill_lat(const or_model* m, int64_t tokens, int32_t b, int32_t w) {
    double be = 1.0 + m->eff * (double)(b - 1);
    double den = m->rate * be;
    return ((double)tokens / den) / or_speedup(&m->prefill, w);
}

/* decode_step_latency; optional context term (A15), 0 = SPEC.    */
double or_decode_lat(const or_model* m, int32_t n, int64_t ctx, int32_t w) {
    double t = m->dec_fixed + m->dec_per_seq * (double)n;
    if (m->dec_per_ctx != 0.0) t = t + m->dec_per_ctx * (double)ctx;
    return t / or_speedup(&m->decode, w);
}

/* A40 context-growing decode: the decode context of the step that ends at
 * boundary s is C(s) = Σ_active (in_i + s − join_i) (prompt plus the tokens
 * generated before the step), so within a constant-composition segment the
 * step latency grows by d = per_ctx·n / s_dec(w) per step and boundary k of
 * the segment is the arithmetic-series sum
 *     t_seg + ((double)k·L1 + (double)(k(k−1)/2)·d),
 * L1 = decode_lat(n, C(step0+1), w).  With ctx_growth = 0 the context is
 * Σ in_i (A15) and the boundary is A14's t_seg + (double)k·L.              */
static long seg_ctx(const or_model* m, long ctx_in, int n, int step_next, long sum_join) {
    if (!m->ctx_growth) return ctx_in;
    return ctx_in + (long)n * step_next - sum_join;
}
static double seg_growth(const or_model* m, int n, int32_t w) {
    if (!m->ctx_growth || m->dec_per_ctx == 0.0) return 0.0;
    return (m->dec_per_ctx * (double)n) / or_speedup(&m->decode, w);
}
static double seg_boundary(const or_model* m, double t_seg, double L1, double d, int k) {
    if (!m->ctx_growth) return t_seg + (double)k * L1;
    long tri = (long)k * (long)(k - 1) / 2;
    return t_seg + ((double)k * L1 + (double)tri * d);
}

/* kv_transfer_latency: bulk KV pull, lands in TPOT.      */
double or_kv_lat(const or_model* m, int32_t tokens) {
    return m->ovh + ((double)tokens * m->kvb) / m->bw;
}

static int cmp_double(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* nearest-rank percentile: value at 1-based rank ceil(p/100 · n)
 * = (p·n + 99)/100 of the sorted samples, p integer in [1, 100]; n ≥ 1.        */
double or_percentile(const double* v, int32_t n, int32_t p) {
    if (n <= 0 || p < 1 || p > 100) return NAN;
    double* tmp = (double*)malloc(sizeof(double) * (size_t)n);
    if (!tmp) return NAN;
    memcpy(tmp, v, sizeof(double) * (size_t)n);
    qsort(tmp, (size_t)n, sizeof(double), cmp_double);
    int k = (p * n + 99) / 100;
    double r = tmp[k - 1];
    free(tmp);
    return r;
}

/* p90 nearest rank: 1-based rank ceil(0.9 n) = (90n+99)/100,
 * empty → 0 which counts as "SLO met".                       */
double or_p90(const double* v, int32_t n) {
    if (n <= 0) return 0.0;
    double* tmp = (double*)malloc(sizeof(double) * (size_t)n);
    if (!tmp) return NAN;
    memcpy(tmp, v, sizeof(double) * (size_t)n);
    qsort(tmp, (size_t)n, sizeof(double), cmp_double);
    int k = (90 * n + 99) / 100;
    double r = tmp[k - 1];
    free(tmp);
    return r;
}

/* ------------------------------------------------------------------------ */
/* a1: candidate enumeration — pool-uniform caps, Σ ≤ B,      */
/* grid 400 + k·step within [min,max].  Brute force.          */
/* ------------------------------------------------------------------------ */
int or_enumerate(int32_t n_gpus, int32_t budget_w, int32_t min_w, int32_t max_w, int32_t step_w,
                 int32_t exact, int32_t* out_xpd, int32_t cap, int32_t* n_out) {
    if (n_gpus < 2 || step_w <= 0 || min_w > max_w || !n_out) return -1;
    int cnt = 0;
    for (int x = 1; x <= n_gpus - 1; x++) {
        int y = n_gpus - x;
        for (int p = min_w; p <= max_w; p += step_w) {
            for (int d = min_w; d <= max_w; d += step_w) {
                long total = (long)x * p + (long)y * d;
                int ok = exact ? (total == budget_w) : (total <= budget_w);
                if (!ok) continue;
                if (out_xpd && cnt < cap) {
                    out_xpd[3 * cnt + 0] = x;
                    out_xpd[3 * cnt + 1] = p;
                    out_xpd[3 * cnt + 2] = d;
                }
                cnt++;
            }
        }
    }
    *n_out = cnt;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 1 "Dynamic Resources Scheduling" as a pure step,   */
/* with the readings A18–A21, A24, A26.                      */
/* ------------------------------------------------------------------------ */
int or_step_controller(const or_policy* pol, const or_model* m, int32_t budget_w,
                       or_ctl_state* st, const or_ctl_obs* obs, double now, or_ctl_action* act) {
    int n = st->n_gpus;
    act->kind = 0;
    act->direction = -1;
    act->gpu = -1;
    for (int g = 0; g < n; g++) act->new_cap[g] = st->cmd[g];
    if (pol->kind == 0) return 0;                       /* static never acts */
    if (!((now - st->last_move) > pol->cooldown_s)) return 0;  /* P:231, P:240 strict */

    int ttft_gt = obs->ttft_stat > obs->ttft_slo;
    int ttft_lt = obs->ttft_stat < obs->ttft_slo;
    int tpot_gt = obs->tpot_stat > obs->tpot_slo;
    int tpot_lt = obs->tpot_stat < obs->tpot_slo;
    int dir;
    if (ttft_gt && obs->q_prefill > pol->threshold && tpot_lt) dir = 0;
    else if (tpot_gt && ttft_lt) dir = 1;
    else return 0;
    act->direction = dir;

    int from = dir == 0 ? 1 : 0;          /* role donating (1 = decode) */
    int to = dir == 0 ? 0 : 1;
    int ceil_to = to == 0 ? m->max_w : pol->dec_ceiling_w;   /* P:449 decode peak 600 W */
    int floor_from = m->min_w;
    int n_don = 0, n_rec = 0, all_rec_ceil = 1, all_don_floor = 1;
    for (int g = 0; g < n; g++) {
        if (st->draining[g]) continue;     /* A26: a draining GPU is in neither pool */
        if (st->role[g] == from) { n_don++; if (st->cmd[g] > floor_from) all_don_floor = 0; }
        if (st->role[g] == to)   { n_rec++; if (st->cmd[g] < ceil_to) all_rec_ceil = 0; }
    }
    int limits = all_rec_ceil || all_don_floor;   /* PowerLimitsReached */
    int power_ok = pol->kind == 1 || pol->kind == 3;
    int gpu_ok = pol->kind == 2 || pol->kind == 3;

    if (power_ok && !limits) {
        /* MovePower: every donor −min(step, cap−floor);
         * F = Σ; every recipient +min(⌊F/|rec|⌋, ceiling−cap); rest unallocated. */
        long F = 0;
        for (int g = 0; g < n; g++) {
            if (st->draining[g] || st->role[g] != from) continue;
            int r = st->cmd[g] - floor_from;
            if (r > pol->step_w) r = pol->step_w;
            if (r < 0) r = 0;
            act->new_cap[g] = st->cmd[g] - r;
            F += r;
        }
        long share = n_rec > 0 ? F / n_rec : 0;
        for (int g = 0; g < n; g++) {
            if (st->draining[g] || st->role[g] != to) continue;
            long room = (long)ceil_to - st->cmd[g];
            long r = share < room ? share : room;
            if (r < 0) r = 0;
            act->new_cap[g] = st->cmd[g] + (int)r;
        }
        act->kind = 1;
    } else if (gpu_ok && n_don >= 2 && !st->drain_pending) {
        /* MoveGPU: donor with the least outstanding work
         * (S:349), tie lowest id; then DistributeUniformPower.      */
        int best = -1;
        for (int g = 0; g < n; g++) {
            if (st->draining[g] || st->role[g] != from) continue;
            if (best < 0 || obs->load[g] < obs->load[best]) best = g;
        }
        int u = budget_w / n;
        if (u < m->min_w) u = m->min_w;
        if (u > m->max_w) u = m->max_w;
        for (int g = 0; g < n; g++) act->new_cap[g] = u;
        act->kind = 2;
        act->gpu = best;
        st->draining[best] = 1;
        st->drain_pending = 1;
    } else {
        act->kind = 3;       /* saturated: no action, last_move unchanged */
        return 0;
    }
    for (int g = 0; g < n; g++) st->cmd[g] = act->new_cap[g];
    st->last_move = now;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Event heap.  Total order: (time, kind, key) — A10 kind order             */
/* settle < role-flip < prefill-end < decode-step < transfer-end < arrival  */
/* < tick; key = worker id or request id.                                   */
/* ------------------------------------------------------------------------ */
enum { K_SETTLE = 0, K_FLIP = 1, K_PEND = 2, K_DSTEP = 3, K_TEND = 4, K_ARR = 5, K_TICK = 6 };
typedef struct { double t; int kind; int key; } ev_t;
typedef struct { ev_t* a; int n, cap; } heap_t;

static int ev_less(const ev_t* x, const ev_t* y) {
    if (x->t != y->t) return x->t < y->t;
    if (x->kind != y->kind) return x->kind < y->kind;
    return x->key < y->key;
}
static int heap_push(heap_t* h, double t, int kind, int key) {
    if (h->n == h->cap) {
        int nc = h->cap ? 2 * h->cap : 64;
        ev_t* na = (ev_t*)realloc(h->a, sizeof(ev_t) * (size_t)nc);
        if (!na) return -1;
        h->a = na;
        h->cap = nc;
    }
    int i = h->n++;
    h->a[i].t = t; h->a[i].kind = kind; h->a[i].key = key;
    while (i > 0) {
        int p = (i - 1) / 2;
        if (!ev_less(&h->a[i], &h->a[p])) break;
        ev_t tmp = h->a[i]; h->a[i] = h->a[p]; h->a[p] = tmp;
        i = p;
    }
    return 0;
}
static ev_t heap_pop(heap_t* h) {
    ev_t top = h->a[0];
    h->a[0] = h->a[--h->n];
    int i = 0;
    for (;;) {
        int l = 2 * i + 1, r = l + 1, s = i;
        if (l < h->n && ev_less(&h->a[l], &h->a[s])) s = l;
        if (r < h->n && ev_less(&h->a[r], &h->a[s])) s = r;
        if (s == i) break;
        ev_t tmp = h->a[i]; h->a[i] = h->a[s]; h->a[s] = tmp;
        i = s;
    }
    return top;
}

/* FIFO ring of request ids, capacity = number of requests. */
typedef struct { int* buf; int cap, head, len; } ring_t;
static void ring_push(ring_t* r, int v) { r->buf[(r->head + r->len) % r->cap] = v; r->len++; }
static int ring_pop(ring_t* r) { int v = r->buf[r->head]; r->head = (r->head + 1) % r->cap; r->len--; return v; }
static int ring_at(const ring_t* r, int k) { return r->buf[(r->head + k) % r->cap]; }

typedef struct {
    int role, draining, flip_sched, flip_to;
    int cmd, eff, raise_to;
    /* prefill worker (P:281 local scheduler) */
    ring_t q; long outstanding; int busy; int* batch; int bn;
    /* decode worker (continuous batching) */
    int* act_id; int* act_fin; int n_act; long ctx; long sum_join;
    ring_t pend; int step, step0; double t_seg, L, dL;
    int in_step, at_boundary, comp_changed, dirty;
    double empty_at;      /* draining: the instant it became empty (flip at +reassign) */
} wk_t;

typedef struct { double* stamp; double* val; int n, lo; } samples_t;

static void log_put(or_log* lg, double t, int type, int gpu, int a, int b) {
    if (!lg || lg->n >= lg->cap) { if (lg) lg->n++; return; }
    or_log_rec* r = &lg->recs[lg->n++];
    r->t = t; r->type = type; r->gpu = gpu; r->a = a; r->b = b;
}

static int valid_curve(const or_curve* c, int min_w, int max_w) {
    if (c->n < 2 || c->n > OR_MAX_ANCHORS) return 0;
    if (c->w[0] != min_w || c->w[c->n - 1] != max_w) return 0;
    if (c->s[0] != 1.0) return 0;
    for (int k = 1; k < c->n; k++) {
        if (!(c->w[k] > c->w[k - 1])) return 0;
        if (!(c->s[k] >= c->s[k - 1])) return 0;
    }
    return 1;
}

static int valid_model(const or_model* m) {
    if (!(m->min_w > 0 && m->min_w < m->max_w)) return 0;
    if (!valid_curve(&m->prefill, m->min_w, m->max_w)) return 0;
    if (!valid_curve(&m->decode, m->min_w, m->max_w)) return 0;
    if (!(m->rate > 0 && m->eff >= 0 && m->dec_fixed > 0 && m->dec_per_seq >= 0 &&
          m->dec_per_ctx >= 0 && m->kvb > 0 && m->bw > 0 && m->ovh > 0)) return 0;
    if (m->max_pb < 1 || m->pb_tokens < 1 || m->max_db < 1 || m->slots < 1 || m->slots > 32) return 0;
    if (m->chunk < 1) return 0;
    if (m->ctx_growth != 0 && m->ctx_growth != 1) return 0;
    return 1;
}

/* ------------------------------------------------------------------------ */
/* Coalesced (non-disaggregated) replay — the paper's baseline: "vLLM in    */
/* coalesced mode ... generated using chunked prefill", SPEC         */
/* coalesced_step, readings A33–A37:             */
/*  A33 every GPU serves both phases at its cap; roles are ignored; no KV    */
/*      transfer (transfer_end = prefill_end).                               */
/*  A34 arrivals go to the GPU with the least outstanding prompt tokens      */
/*      (remaining, queued + in service), lowest id (as A8).                 */
/*  A35 one engine step = at most one chunk of ≤ chunk tokens of the head    */
/*      prompt (FIFO, no packing across prompts) fused with every active     */
/*      decode sequence: lat = prefill_lat(c,1,w) + decode_lat(n,C,w) when   */
/*      both are present, else the one present.  A chunk step ends   */
/*      at t + lat.                                                          */
/*  A36 the last chunk's step end is the first token (prefill_end, TTFT);    */
/*      the request then joins this GPU's decode batch at that boundary      */
/*      (pending FIFO when max_db is full) and needs out−1 more steps;       */
/*      out = 1 completes at prefill_end with TPOT 0 (A7).                   */
/*  A37 runs of decode-only steps are constant-composition segments,         */
/*      boundary k at t_seg + (double)k·L (A14); a chunk step, a join or a   */
/*      leave ends the segment.                                              */
/* One heap event per engine step; kind order as A10 (step end < arrival).  */
/* ------------------------------------------------------------------------ */
typedef struct {
    ring_t q; int done_tok; long outstanding;          /* prompt FIFO, head progress */
    int* act_id; int* act_fin; int n_act; long ctx;     /* decode batch               */
    long sum_join;                                       /* Σ join steps (A40)         */
    ring_t pend; int step, step0; double t_seg, L, dL;
    int in_step, at_boundary, comp_changed, seg_valid;
    int c_id, c_tok;                                     /* chunk of the step in flight */
} cw_t;

static int replay_coalesced(const or_model* m, int32_t N, const int32_t* cap, int32_t B,
                            const or_slo* slo, int32_t R, const double* s_unit,
                            const int32_t* in_tok, const int32_t* out_tok, const uint8_t* phase,
                            double qps, double* o_ttft, double* o_tpot, double* o_pe, double* o_comp,
                            double* o_te, double* o_ps, or_summary* sum) {
    long capsum = 0;
    for (int g = 0; g < N; g++) {
        if (cap[g] < m->min_w || cap[g] > m->max_w) return -2;
        capsum += cap[g];
    }
    if (capsum > B) return -3;
    for (int i = 0; i < R; i++) {
        if (in_tok[i] < 1 || out_tok[i] < 1) return -6;
        if (!(s_unit[i] >= 0) || !isfinite(s_unit[i])) return -1;
        if (i > 0 && !(s_unit[i] >= s_unit[i - 1])) return -1;
        if (phase[i] > 1) return -1;
    }
    memset(sum, 0, sizeof(*sum));
    sum->n_req = R;
    sum->avg_watts = (double)capsum;
    if (R == 0) return 0;

    int rc = -8;
    double* a = (double*)malloc(sizeof(double) * (size_t)R);
    double* pe = (double*)malloc(sizeof(double) * (size_t)R);
    double* ps = (double*)malloc(sizeof(double) * (size_t)R);
    double* comp = (double*)malloc(sizeof(double) * (size_t)R);
    double* tpot = (double*)malloc(sizeof(double) * (size_t)R);
    cw_t* W = (cw_t*)calloc((size_t)N, sizeof(cw_t));
    heap_t h = {0};
    if (!a || !pe || !ps || !comp || !tpot || !W) goto out;
    for (int g = 0; g < N; g++) {
        cw_t* w = &W[g];
        w->q.buf = (int*)malloc(sizeof(int) * (size_t)R); w->q.cap = R;
        w->pend.buf = (int*)malloc(sizeof(int) * (size_t)R); w->pend.cap = R;
        w->act_id = (int*)malloc(sizeof(int) * (size_t)m->max_db);
        w->act_fin = (int*)malloc(sizeof(int) * (size_t)m->max_db);
        w->c_id = -1;
        if (!w->q.buf || !w->pend.buf || !w->act_id || !w->act_fin) goto out;
    }
    double inv_lam = 1.0 / (qps * (double)N);          /* a2 */
    for (int i = 0; i < R; i++) a[i] = s_unit[i] * inv_lam;
    for (int i = 0; i < R; i++)
        if (heap_push(&h, a[i], K_ARR, i)) goto out;

    int completed = 0;
    int64_t events = 0;
    while (completed < R) {
        if (h.n == 0) { rc = -9; goto out; }
        double t = h.a[0].t;
        while (h.n > 0 && h.a[0].t == t) {
            ev_t e = heap_pop(&h);
            events++;
            if (e.kind == K_DSTEP) {
                cw_t* w = &W[e.key];
                w->step++;
                w->in_step = 0;
                w->at_boundary = 1;
                int k = 0;
                while (k < w->n_act) {             /* sequences emitting their last token */
                    if (w->act_fin[k] == w->step) {
                        int i = w->act_id[k];
                        comp[i] = t;
                        tpot[i] = (t - pe[i]) / (double)(out_tok[i] - 1);
                        completed++;
                        w->ctx -= in_tok[i];
                        w->sum_join -= w->act_fin[k] - (out_tok[i] - 1);
                        w->act_id[k] = w->act_id[w->n_act - 1];
                        w->act_fin[k] = w->act_fin[w->n_act - 1];
                        w->n_act--;
                        w->comp_changed = 1;
                    } else {
                        k++;
                    }
                }
                if (w->c_id >= 0) {                /* the step's prefill chunk (A35/A36) */
                    int i = w->c_id;
                    w->done_tok += w->c_tok;
                    w->outstanding -= w->c_tok;
                    if (w->done_tok == in_tok[i]) {
                        ring_pop(&w->q);
                        w->done_tok = 0;
                        pe[i] = t;
                        if (out_tok[i] == 1) {
                            comp[i] = t;
                            tpot[i] = 0.0;
                            completed++;
                        } else {
                            ring_push(&w->pend, i);
                        }
                    }
                    w->c_id = -1;
                }
            } else {                               /* K_ARR (A34) */
                int i = e.key;
                int best = 0;
                for (int g = 1; g < N; g++)
                    if (W[g].outstanding < W[best].outstanding) best = g;
                ring_push(&W[best].q, i);
                W[best].outstanding += in_tok[i];
            }
        }
        /* dispatch after the instant, worker-id order (A10) */
        for (int g = 0; g < N; g++) {
            cw_t* w = &W[g];
            if (w->in_step) { w->at_boundary = 0; continue; }
            int was_idle = !w->at_boundary;
            int joined = 0;
            while (w->n_act < m->max_db && w->pend.len > 0) {
                int i = ring_pop(&w->pend);
                w->act_id[w->n_act] = i;
                w->act_fin[w->n_act] = w->step + (out_tok[i] - 1);
                w->n_act++;
                w->ctx += in_tok[i];
                w->sum_join += w->step;
                joined = 1;
            }
            if (w->q.len > 0) {
                int i = ring_at(&w->q, 0);
                int c = in_tok[i] - w->done_tok;
                if (c > m->chunk) c = m->chunk;
                if (w->done_tok == 0) ps[i] = t;
                double lat = or_prefill_lat(m, c, 1, cap[g]);
                if (w->n_act > 0)
                    lat = lat + or_decode_lat(m, w->n_act,
                                              seg_ctx(m, w->ctx, w->n_act, w->step + 1, w->sum_join), cap[g]);
                if (heap_push(&h, t + lat, K_DSTEP, g)) goto out;
                w->c_id = i;
                w->c_tok = c;
                w->in_step = 1;
                w->seg_valid = 0;
            } else if (w->n_act > 0) {
                if (was_idle || joined || w->comp_changed || !w->seg_valid) {
                    w->t_seg = t;
                    w->step0 = w->step;
                    w->L = or_decode_lat(m, w->n_act, seg_ctx(m, w->ctx, w->n_act, w->step + 1, w->sum_join),
                                         cap[g]);
                    w->dL = seg_growth(m, w->n_act, cap[g]);
                    w->seg_valid = 1;
                }
                double nb = seg_boundary(m, w->t_seg, w->L, w->dL, w->step + 1 - w->step0);
                if (heap_push(&h, nb, K_DSTEP, g)) goto out;
                w->in_step = 1;
            }
            w->at_boundary = 0;
            w->comp_changed = 0;
        }
    }
    {
        int met = 0, near = 0;
        double last = 0.0, sq = 0.0, se = 0.0;
        for (int i = 0; i < R; i++) {
            sq = sq + (ps[i] - a[i]);
            se = se + (pe[i] - ps[i]);
            double tt = pe[i] - a[i];
            double ts = slo->tpot[phase[i]];
            if (tt <= slo->ttft && tpot[i] <= ts) met++;
            if (fabs(tt - slo->ttft) <= 1e-9 * slo->ttft || fabs(tpot[i] - ts) <= 1e-9 * ts) near++;
            if (i == 0 || comp[i] > last) last = comp[i];
            if (o_ttft) o_ttft[i] = tt;
            if (o_tpot) o_tpot[i] = tpot[i];
            if (o_pe) o_pe[i] = pe[i];
            if (o_comp) o_comp[i] = comp[i];
            if (o_te) o_te[i] = pe[i];
            if (o_ps) o_ps[i] = ps[i];
        }
        sum->met = met;
        sum->near_boundary = near;
        sum->duration = last - a[0];
        sum->goodput = sum->duration > 0 ? (double)met / sum->duration : 0.0;
        sum->events = events;
        sum->avg_watts = (double)capsum;
        sum->qps_per_watt = sum->goodput / sum->avg_watts;
        sum->sum_queue = sq;
        sum->sum_exec = se;
    }
    rc = 0;
out:
    if (W) {
        for (int g = 0; g < N; g++) {
            free(W[g].q.buf); free(W[g].pend.buf); free(W[g].act_id); free(W[g].act_fin);
        }
    }
    free(W); free(a); free(pe); free(ps); free(comp); free(tpot);
    free(h.a);
    return rc;
}

/* The replay: c.2 (static) + c.3 (dynamic).                                 */
int or_replay(const or_model* m, int32_t N, const uint8_t* role, const int32_t* cap,
              const or_policy* pol, int32_t B, const or_slo* slo,
              int32_t R, const double* s_unit, const int32_t* in_tok,
              const int32_t* out_tok, const uint8_t* phase, double qps,
              double* o_ttft, double* o_tpot, double* o_pe, double* o_comp, double* o_te,
              double* o_ps, or_summary* sum, or_log* lg) {
    if (!m || !role || !cap || !pol || !slo || !sum || N < 2 || N > OR_MAX_GPUS || R < 0) return -1;
    if (!valid_model(m)) return -5;
    if (!(qps > 0) || !(slo->ttft > 0 && slo->tpot[0] > 0 && slo->tpot[1] > 0)) return -1;
    if (pol->kind == 4)
        return replay_coalesced(m, N, cap, B, slo, R, s_unit, in_tok, out_tok, phase, qps, o_ttft,
                                o_tpot, o_pe, o_comp, o_te, o_ps, sum);
    int np = 0;
    long capsum = 0;
    for (int g = 0; g < N; g++) {
        if (role[g] > 1) return -4;
        np += role[g] == 0;
        if (cap[g] < m->min_w || cap[g] > m->max_w) return -2;
        capsum += cap[g];
    }
    if (np < 1 || np > N - 1) return -4;
    if (capsum > B) return -3;
    int dynamic = pol->kind != 0;
    if (pol->kind < 0 || pol->kind > 3) return -1;
    if (dynamic) {
        if (!(pol->tick_s > 0 && pol->settle_s > 0 && pol->reassign_s > 0 &&
              pol->cooldown_s >= pol->settle_s && pol->window_s >= 0 && pol->step_w > 0 &&
              pol->threshold >= 0 && pol->dec_ceiling_w >= m->min_w &&
              (pol->window_stamp == 0 || pol->window_stamp == 1) &&
              pol->dec_ceiling_w <= m->max_w && (long)N * m->min_w <= B)) return -1;
    }
    for (int i = 0; i < R; i++) {
        if (in_tok[i] < 1 || out_tok[i] < 1) return -6;
        if (!(s_unit[i] >= 0) || !isfinite(s_unit[i])) return -1;
        if (i > 0 && !(s_unit[i] >= s_unit[i - 1])) return -1;
        if (phase[i] > 1) return -1;
    }
    memset(sum, 0, sizeof(*sum));
    sum->n_req = R;
    sum->avg_watts = (double)capsum;     /* nothing happens: the initial provisioning */
    if (R == 0) return 0;

    int rc = -8;
    double* a = (double*)malloc(sizeof(double) * (size_t)R);
    double* pe = (double*)malloc(sizeof(double) * (size_t)R);
    double* comp = (double*)malloc(sizeof(double) * (size_t)R);
    double* tpot = (double*)malloc(sizeof(double) * (size_t)R);
    double* te = (double*)malloc(sizeof(double) * (size_t)R);
    double* ps = (double*)malloc(sizeof(double) * (size_t)R);   /* prefill (batch) start */
    int* done = (int*)calloc((size_t)R, sizeof(int));
    wk_t* W = (wk_t*)calloc((size_t)N, sizeof(wk_t));
    ring_t twait = {0};
    samples_t s_ttft = {0}, s_tpot = {0};
    heap_t h = {0};
    if (!a || !pe || !comp || !tpot || !te || !ps || !done || !W) goto out;
    twait.buf = (int*)malloc(sizeof(int) * (size_t)R); twait.cap = R;
    s_ttft.stamp = (double*)malloc(sizeof(double) * (size_t)R);
    s_ttft.val = (double*)malloc(sizeof(double) * (size_t)R);
    s_tpot.stamp = (double*)malloc(sizeof(double) * (size_t)R);
    s_tpot.val = (double*)malloc(sizeof(double) * (size_t)R);
    if (!twait.buf || !s_ttft.stamp || !s_ttft.val || !s_tpot.stamp || !s_tpot.val) goto out;
    for (int g = 0; g < N; g++) {
        wk_t* w = &W[g];
        w->role = role[g];
        w->cmd = w->eff = cap[g];
        w->q.buf = (int*)malloc(sizeof(int) * (size_t)R); w->q.cap = R;
        w->pend.buf = (int*)malloc(sizeof(int) * (size_t)R); w->pend.cap = R;
        w->batch = (int*)malloc(sizeof(int) * (size_t)m->max_pb);
        w->act_id = (int*)malloc(sizeof(int) * (size_t)m->max_db);
        w->act_fin = (int*)malloc(sizeof(int) * (size_t)m->max_db);
        if (!w->q.buf || !w->pend.buf || !w->batch || !w->act_id || !w->act_fin) goto out;
    }

    /* a2: arrivals at QPS q: a_i = s_unit_i · (1/(q·N)) (Poisson). */
    double inv_lam = 1.0 / (qps * (double)N);
    for (int i = 0; i < R; i++) a[i] = s_unit[i] * inv_lam;
    for (int i = 0; i < R; i++)
        if (heap_push(&h, a[i], K_ARR, i)) goto out;
    long tick_k = 1;
    if (dynamic && heap_push(&h, (double)tick_k * pol->tick_s, K_TICK, 0)) goto out;

    int completed = 0, tbusy = 0, phase2_seen = 0, drain_pending = 0;
    /* provisioned power ("average provisioned GPU power"): Σ eff caps is
     * piecewise constant, changing only at settle instants; integrated over [a_0, last] */
    long w_sum = 0;
    for (int g = 0; g < N; g++) w_sum += W[g].eff;
    double w_acc = 0.0, w_prev = a[0];
    double last_move = 0.0;    /* Alg. 1 "last_move_time ← 0", A24 */
    int64_t events = 0;
    if (lg) {
        long c0 = 0; for (int g = 0; g < N; g++) c0 += W[g].eff;
        log_put(lg, 0.0, OR_LOG_BUDGET, -1, (int)c0, 0);
        int p0 = 0; for (int g = 0; g < N; g++) p0 += W[g].role == 0;
        log_put(lg, 0.0, OR_LOG_ROLES, -1, p0, N - p0);
    }

#define COMPLETE(ID, T, TP) do { int id_ = (ID); comp[id_] = (T); tpot[id_] = (TP); done[id_] = 1; \
        completed++; s_tpot.stamp[s_tpot.n] = (T); s_tpot.val[s_tpot.n] = (TP); s_tpot.n++; \
        if (pol->window_stamp) {   /* TTFT sampled at completion */ \
            s_ttft.stamp[s_ttft.n] = (T); s_ttft.val[s_ttft.n] = pe[id_] - a[id_]; s_ttft.n++; } } while (0)

    while (completed < R) {
        if (h.n == 0) { rc = -9; goto out; }     /* cannot happen: progress guaranteed */
        double t = h.a[0].t;
        /* ---- process every event of this instant in (kind, key) order (A10) ---- */
        while (h.n > 0 && h.a[0].t == t) {
            ev_t e = heap_pop(&h);
            events++;
            switch (e.kind) {
            case K_SETTLE: {
                /* source-before-sink: decreases take effect
                 * at settle; raises are applied at the same instant.           */
                for (int g = 0; g < N; g++) {
                    wk_t* w = &W[g];
                    int changed = 0;
                    if (w->cmd < w->eff) { w->eff = w->cmd; changed = 1; }
                    if (w->raise_to > 0) { w->cmd = w->eff = w->raise_to; w->raise_to = 0; changed = 1; }
                    if (changed && w->role == 1) w->dirty = 1;
                }
                if (t > a[0]) {
                    w_acc = w_acc + (double)w_sum * (t - w_prev);
                    w_prev = t;
                }
                w_sum = 0;
                for (int g = 0; g < N; g++) w_sum += W[g].eff;
                if (lg) {
                    long c = 0; for (int g = 0; g < N; g++) c += W[g].eff;
                    log_put(lg, t, OR_LOG_SETTLE, -1, 0, 0);
                    log_put(lg, t, OR_LOG_BUDGET, -1, (int)c, 0);
                    for (int g = 0; g < N; g++) log_put(lg, t, OR_LOG_CAPS, g, W[g].eff, W[g].role);
                }
                break;
            }
            case K_FLIP: {
                /* role change after drain + reassignment latency */
                wk_t* w = &W[e.key];
                w->role = w->flip_to;
                w->draining = 0;
                w->flip_sched = 0;
                w->busy = 0; w->bn = 0; w->outstanding = 0;
                w->n_act = 0; w->ctx = 0; w->sum_join = 0; w->in_step = 0; w->dirty = 0; w->step0 = w->step;
                drain_pending = 0;
                sum->n_flips++;
                if (lg) {
                    int p = 0; for (int g = 0; g < N; g++) p += W[g].role == 0 && !W[g].draining;
                    int d = 0; for (int g = 0; g < N; g++) d += W[g].role == 1 && !W[g].draining;
                    log_put(lg, t, OR_LOG_FLIP, e.key, w->role, 0);
                    log_put(lg, t, OR_LOG_ROLES, -1, p, d);
                }
                break;
            }
            case K_PEND: {
                /* prefill batch end: first token (TTFT); each member goes to
                 * the 32-slot KV request buffer in member order (A12).    */
                wk_t* w = &W[e.key];
                for (int k = 0; k < w->bn; k++) {
                    int i = w->batch[k];
                    pe[i] = t;
                    w->outstanding -= in_tok[i];
                    if (!pol->window_stamp) {      /* A22: TTFT known at the first token */
                        s_ttft.stamp[s_ttft.n] = t; s_ttft.val[s_ttft.n] = t - a[i]; s_ttft.n++;
                    }
                    if (tbusy < m->slots) {
                        tbusy++;
                        te[i] = t + or_kv_lat(m, in_tok[i]);
                        if (heap_push(&h, te[i], K_TEND, i)) goto out;
                    } else {
                        ring_push(&twait, i);
                    }
                }
                w->busy = 0;
                w->bn = 0;
                break;
            }
            case K_DSTEP: {
                /* one decode step: every active sequence emits one token; those
                 * reaching their last token complete (TPOT P:339).      */
                wk_t* w = &W[e.key];
                w->step++;
                w->in_step = 0;
                w->at_boundary = 1;
                int k = 0;
                while (k < w->n_act) {
                    if (w->act_fin[k] == w->step) {
                        int i = w->act_id[k];
                        double tp = (t - pe[i]) / (double)(out_tok[i] - 1);
                        COMPLETE(i, t, tp);
                        w->ctx -= in_tok[i];
                        w->sum_join -= w->act_fin[k] - (out_tok[i] - 1);
                        w->act_id[k] = w->act_id[w->n_act - 1];
                        w->act_fin[k] = w->act_fin[w->n_act - 1];
                        w->n_act--;
                        w->comp_changed = 1;
                    } else {
                        k++;
                    }
                }
                break;
            }
            case K_TEND: {
                int i = e.key;
                tbusy--;
                if (twait.len > 0) {
                    int j = ring_pop(&twait);
                    tbusy++;
                    te[j] = t + or_kv_lat(m, in_tok[j]);
                    if (heap_push(&h, te[j], K_TEND, j)) goto out;
                }
                if (out_tok[i] == 1) {
                    COMPLETE(i, t, 0.0);          /* S:280 D4: TPOT 0, completes now */
                } else {
                    /* A13: decode worker with the fewest active+pending, lowest id */
                    int best = -1; long bl = 0;
                    for (int g = 0; g < N; g++) {
                        if (W[g].role != 1 || W[g].draining) continue;
                        long l = W[g].n_act + W[g].pend.len;
                        if (best < 0 || l < bl) { best = g; bl = l; }
                    }
                    ring_push(&W[best].pend, i);
                }
                break;
            }
            case K_ARR: {
                int i = e.key;
                if (phase[i] == 1) phase2_seen = 1;   /* SLO schedule switch */
                /* A8: prefill worker with the least outstanding tokens, lowest id */
                int best = -1; long bl = 0;
                for (int g = 0; g < N; g++) {
                    if (W[g].role != 0 || W[g].draining) continue;
                    if (best < 0 || W[g].outstanding < bl) { best = g; bl = W[g].outstanding; }
                }
                ring_push(&W[best].q, i);
                W[best].outstanding += in_tok[i];
                break;
            }
            case K_TICK: {
                /* Alg. 1 loop body every MIN_TIME. Window [t−W, t]. */
                double lo_t = t - pol->window_s;
                double* buf = (double*)malloc(sizeof(double) * (size_t)(R > 0 ? R : 1));
                if (!buf) goto out;
                int nb = 0;
                while (s_ttft.lo < s_ttft.n && s_ttft.stamp[s_ttft.lo] < lo_t) s_ttft.lo++;
                for (int k = s_ttft.lo; k < s_ttft.n; k++)
                    if (s_ttft.stamp[k] >= lo_t && s_ttft.stamp[k] <= t) buf[nb++] = s_ttft.val[k];
                double ttft_stat = or_p90(buf, nb);
                nb = 0;
                while (s_tpot.lo < s_tpot.n && s_tpot.stamp[s_tpot.lo] < lo_t) s_tpot.lo++;
                for (int k = s_tpot.lo; k < s_tpot.n; k++)
                    if (s_tpot.stamp[k] >= lo_t && s_tpot.stamp[k] <= t) buf[nb++] = s_tpot.val[k];
                double tpot_stat = or_p90(buf, nb);
                free(buf);

                or_ctl_state st;
                or_ctl_obs ob;
                or_ctl_action act;
                memset(&st, 0, sizeof st);
                memset(&ob, 0, sizeof ob);
                st.n_gpus = N;
                st.drain_pending = drain_pending;
                st.last_move = last_move;
                ob.q_prefill = 0;
                for (int g = 0; g < N; g++) {
                    st.role[g] = (uint8_t)W[g].role;
                    st.draining[g] = (uint8_t)W[g].draining;
                    st.cmd[g] = W[g].raise_to > 0 ? W[g].raise_to : W[g].cmd;
                    if (W[g].role == 0) { ob.q_prefill += W[g].q.len; ob.load[g] = (int)W[g].outstanding; }
                    else ob.load[g] = W[g].n_act + W[g].pend.len;
                }
                ob.ttft_stat = ttft_stat;
                ob.tpot_stat = tpot_stat;
                ob.ttft_slo = slo->ttft;
                ob.tpot_slo = phase2_seen ? slo->tpot[1] : slo->tpot[0];
                or_step_controller(pol, m, B, &st, &ob, t, &act);
                or_tick_rec* tr_ = (lg && lg->ticks && lg->tn < lg->tcap) ? &lg->ticks[lg->tn] : NULL;
                if (lg && lg->ticks) lg->tn++;
                if (tr_) {
                    memset(tr_, 0, sizeof(*tr_));
                    tr_->t = t; tr_->ttft_stat = ttft_stat; tr_->tpot_stat = tpot_stat;
                    tr_->ttft_slo = ob.ttft_slo; tr_->tpot_slo = ob.tpot_slo; tr_->q_prefill = ob.q_prefill;
                    tr_->kind = act.kind; tr_->direction = act.direction; tr_->gpu = act.gpu;
                    for (int g = 0; g < N; g++) {
                        tr_->load[g] = ob.load[g];
                        tr_->drained_empty[g] = (W[g].draining && W[g].flip_sched) ? W[g].empty_at : -1.0;
                    }
                }
                if (act.kind == 1 || act.kind == 2) {
                    last_move = st.last_move;
                    if (act.kind == 2) {
                        int g = act.gpu;
                        wk_t* w = &W[g];
                        w->draining = 1;
                        w->flip_to = 1 - w->role;
                        drain_pending = 1;
                        if (w->role == 0) {
                            /* re-route queued prompts in queue order */
                            while (w->q.len > 0) {
                                int i = ring_pop(&w->q);
                                w->outstanding -= in_tok[i];
                                int best = -1; long bl = 0;
                                for (int g2 = 0; g2 < N; g2++) {
                                    if (W[g2].role != 0 || W[g2].draining) continue;
                                    if (best < 0 || W[g2].outstanding < bl) { best = g2; bl = W[g2].outstanding; }
                                }
                                ring_push(&W[best].q, i);
                                W[best].outstanding += in_tok[i];
                            }
                        } else {
                            while (w->pend.len > 0) {
                                int i = ring_pop(&w->pend);
                                int best = -1; long bl = 0;
                                for (int g2 = 0; g2 < N; g2++) {
                                    if (W[g2].role != 1 || W[g2].draining) continue;
                                    long l = W[g2].n_act + W[g2].pend.len;
                                    if (best < 0 || l < bl) { best = g2; bl = l; }
                                }
                                ring_push(&W[best].pend, i);
                            }
                        }
                        sum->n_moves_gpu++;
                        log_put(lg, t, OR_LOG_MOVE_GPU, g, act.direction, 0);
                    } else {
                        sum->n_moves_power++;
                        log_put(lg, t, OR_LOG_MOVE_POWER, -1, act.direction, 0);
                    }
                    /* source-before-sink: decreases commanded now (charged at the
                     * old cap until settle), raises at the settle instant.       */
                    for (int g = 0; g < N; g++) {
                        int tgt = act.new_cap[g];
                        if (tgt < W[g].cmd) W[g].cmd = tgt;
                        else if (tgt > W[g].cmd) W[g].raise_to = tgt;
                    }
                    if (heap_push(&h, t + pol->settle_s, K_SETTLE, 0)) goto out;
                    if (lg) {
                        long c = 0; for (int g = 0; g < N; g++) c += W[g].eff;
                        log_put(lg, t, OR_LOG_BUDGET, -1, (int)c, 0);
                    }
                } else if (act.kind == 3) {
                    sum->n_saturated++;
                    log_put(lg, t, OR_LOG_SATURATED, -1, act.direction, 0);
                }
                if (tr_) {
                    for (int g = 0; g < N; g++) {
                        tr_->role[g] = (uint8_t)W[g].role; tr_->draining[g] = (uint8_t)W[g].draining;
                        tr_->cmd[g] = W[g].cmd; tr_->eff[g] = W[g].eff; tr_->raise_to[g] = W[g].raise_to;
                    }
                    tr_->last_move = last_move;
                }
                tick_k++;
                if (heap_push(&h, (double)tick_k * pol->tick_s, K_TICK, 0)) goto out;
                break;
            }
            }
        }

        /* ---- dispatch after the whole instant, in worker-id order (A10) ---- */
        for (int g = 0; g < N; g++) {
            wk_t* w = &W[g];
            if (w->role != 0 || w->busy || w->q.len == 0) continue;
            /* A9: FIFO prefix, ≤ max_pb requests, Σin ≤ pb_tokens, head always */
            long tok = in_tok[ring_at(&w->q, 0)];
            int b = 1;
            while (b < m->max_pb && b < w->q.len) {
                int nx = ring_at(&w->q, b);
                if (tok + in_tok[nx] > m->pb_tokens) break;
                tok += in_tok[nx];
                b++;
            }
            for (int k = 0; k < b; k++) {
                w->batch[k] = ring_pop(&w->q);
                ps[w->batch[k]] = t;
            }
            w->bn = b;
            w->busy = 1;
            double end = t + or_prefill_lat(m, tok, b, w->eff);
            if (heap_push(&h, end, K_PEND, g)) goto out;
        }
        for (int g = 0; g < N; g++) {
            wk_t* w = &W[g];
            if (w->role != 1 || w->in_step) { w->at_boundary = 0; continue; }
            /* idle, or at a step boundary at t: admit pending joins  */
            int was_idle = !w->at_boundary;
            int joined = 0;
            while (w->n_act < m->max_db && w->pend.len > 0) {
                int i = ring_pop(&w->pend);
                w->act_id[w->n_act] = i;
                w->act_fin[w->n_act] = w->step + (out_tok[i] - 1);
                w->n_act++;
                w->ctx += in_tok[i];
                w->sum_join += w->step;
                joined = 1;
            }
            if (w->n_act > 0) {
                if (was_idle || joined || w->comp_changed || w->dirty) {
                    /* new constant-composition segment, reads the effective cap */
                    w->t_seg = t;
                    w->step0 = w->step;
                    w->L = or_decode_lat(m, w->n_act, seg_ctx(m, w->ctx, w->n_act, w->step + 1, w->sum_join),
                                         w->eff);
                    w->dL = seg_growth(m, w->n_act, w->eff);
                    w->dirty = 0;
                }
                /* A14: step k of a segment ends at t_seg + (double)k * L (A40 with growth) */
                double nb = seg_boundary(m, w->t_seg, w->L, w->dL, w->step + 1 - w->step0);
                if (heap_push(&h, nb, K_DSTEP, g)) goto out;
                w->in_step = 1;
            }
            w->at_boundary = 0;
            w->comp_changed = 0;
        }
        /* drained worker: flip after reassign_s once empty */
        for (int g = 0; g < N; g++) {
            wk_t* w = &W[g];
            if (!w->draining || w->flip_sched) continue;
            int empty = w->role == 0 ? (!w->busy && w->q.len == 0)
                                     : (w->n_act == 0 && w->pend.len == 0 && !w->in_step);
            if (empty) {
                w->flip_sched = 1;
                w->empty_at = t;
                if (heap_push(&h, t + pol->reassign_s, K_FLIP, g)) goto out;
            }
        }
    }
#undef COMPLETE

    /* c.2 step 5–6, metrics (D11 inclusive ≤). */
    {
        int met = 0, near = 0;
        double last = 0.0, sq = 0.0, se = 0.0;
        for (int i = 0; i < R; i++) {
            /* Fig. 6 decomposition: TTFT = queueing + prefill exec */
            sq = sq + (ps[i] - a[i]);
            se = se + (pe[i] - ps[i]);
            if (o_ps) o_ps[i] = ps[i];
            double tt = pe[i] - a[i];
            double ts = slo->tpot[phase[i]];
            if (tt <= slo->ttft && tpot[i] <= ts) met++;
            if (fabs(tt - slo->ttft) <= 1e-9 * slo->ttft || fabs(tpot[i] - ts) <= 1e-9 * ts) near++;
            if (i == 0 || comp[i] > last) last = comp[i];
            if (o_ttft) o_ttft[i] = tt;
            if (o_tpot) o_tpot[i] = tpot[i];
            if (o_pe) o_pe[i] = pe[i];
            if (o_comp) o_comp[i] = comp[i];
            if (o_te) o_te[i] = te[i];
        }
        sum->met = met;
        sum->near_boundary = near;
        sum->duration = last - a[0];
        sum->goodput = sum->duration > 0 ? (double)met / sum->duration : 0.0;
        sum->events = events;
        w_acc = w_acc + (double)w_sum * (last - w_prev);
        sum->avg_watts = sum->duration > 0 ? w_acc / sum->duration : (double)w_sum;
        sum->sum_queue = sq;
        sum->sum_exec = se;
        sum->qps_per_watt = sum->avg_watts > 0 ? sum->goodput / sum->avg_watts : 0.0;
    }
    rc = 0;
out:
    if (W) {
        for (int g = 0; g < N; g++) {
            free(W[g].q.buf); free(W[g].pend.buf); free(W[g].batch);
            free(W[g].act_id); free(W[g].act_fin);
        }
    }
    free(W); free(a); free(pe); free(comp); free(tpot); free(te); free(ps); free(done);
    free(twait.buf); free(s_ttft.stamp); free(s_ttft.val); free(s_tpot.stamp); free(s_tpot.val);
    free(h.a);
    return rc;
}

int or_met_for_slos(int32_t R, const double* ttft, const double* tpot, const uint8_t* phase,
                    int32_t K, const or_slo* slos, int32_t* out_met) {
    if (R < 0 || K < 0 || (R > 0 && (!ttft || !tpot || !phase)) || (K > 0 && (!slos || !out_met)))
        return -1;
    for (int k = 0; k < K; k++) {
        int m = 0;
        for (int i = 0; i < R; i++)
            if (ttft[i] <= slos[k].ttft && tpot[i] <= slos[k].tpot[phase[i]]) m++;
        out_met[k] = m;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Whole evaluation over host threads + seed aggregation + argmax (c.4).     */
/* ------------------------------------------------------------------------ */
typedef struct {
    const or_model* m; int32_t N, C, S, Q; const uint8_t* role; const int32_t* cap;
    const or_policy* pol; int32_t B; const int32_t* cand_B; const or_slo* slo; const int32_t* n_req;
    const double* const* s_unit; const int32_t* const* in_tok; const int32_t* const* out_tok;
    const uint8_t* const* phase; const double* qps;
    int32_t* r_met; int32_t* r_near; double* r_good; double* r_dur;
    long next; pthread_mutex_t mu; int err;
} job_t;

static void* worker_main(void* arg) {
    job_t* J = (job_t*)arg;
    long total = (long)J->C * J->Q * J->S;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        long r = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (r >= total) break;
        int s = (int)(r % J->S);
        int q = (int)((r / J->S) % J->Q);
        int c = (int)(r / ((long)J->S * J->Q));
        or_summary sm;
        int rc = or_replay(J->m, J->N, J->role + (size_t)c * J->N, J->cap + (size_t)c * J->N,
                           &J->pol[c], J->cand_B ? J->cand_B[c] : J->B, J->slo, J->n_req[s], J->s_unit[s], J->in_tok[s],
                           J->out_tok[s], J->phase[s], J->qps[q], NULL, NULL, NULL, NULL, NULL,
                           NULL, &sm, NULL);
        if (rc) { J->err = rc; continue; }
        J->r_met[r] = sm.met;
        J->r_near[r] = sm.near_boundary;
        J->r_good[r] = sm.goodput;
        J->r_dur[r] = sm.duration;
    }
    return NULL;
}

int or_evaluate(const or_model* m, int32_t N, int32_t C, const uint8_t* role,
                const int32_t* cap, const or_policy* pol, int32_t B, const int32_t* cand_B,
                const or_slo* slo, int32_t S, const int32_t* n_req, const double* const* s_unit,
                const int32_t* const* in_tok, const int32_t* const* out_tok,
                const uint8_t* const* phase, int32_t Q, const double* qps,
                int32_t n_threads, int64_t* met, double* goodput, int64_t* near_boundary,
                int32_t* argmax, int32_t* rep_met, double* rep_goodput, double* rep_duration) {
    if (C < 1 || S < 1 || Q < 1 || n_threads < 1) return -1;
    long total = (long)C * Q * S;
    job_t J;
    memset(&J, 0, sizeof J);
    J.m = m; J.N = N; J.C = C; J.S = S; J.Q = Q; J.role = role; J.cap = cap; J.pol = pol;
    J.B = B; J.cand_B = cand_B; J.slo = slo; J.n_req = n_req; J.s_unit = s_unit; J.in_tok = in_tok;
    J.out_tok = out_tok; J.phase = phase; J.qps = qps;
    J.r_met = (int32_t*)malloc(sizeof(int32_t) * (size_t)total);
    J.r_near = (int32_t*)malloc(sizeof(int32_t) * (size_t)total);
    J.r_good = (double*)malloc(sizeof(double) * (size_t)total);
    J.r_dur = (double*)malloc(sizeof(double) * (size_t)total);
    if (!J.r_met || !J.r_near || !J.r_good || !J.r_dur) {
        free(J.r_met); free(J.r_near); free(J.r_good); free(J.r_dur);
        return -8;
    }
    pthread_mutex_init(&J.mu, NULL);
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
    int started = 0;
    for (int k = 0; k < n_threads; k++)
        if (pthread_create(&th[k], NULL, worker_main, &J) == 0) started++;
    if (started == 0) worker_main(&J);
    for (int k = 0; k < started; k++) pthread_join(th[k], NULL);
    free(th);
    pthread_mutex_destroy(&J.mu);
    int rc = J.err;
    if (rc == 0) {
        for (int c = 0; c < C; c++) {
            for (int q = 0; q < Q; q++) {
                int64_t sm = 0, sn = 0;
                double sg = 0.0;
                for (int s = 0; s < S; s++) {      /* ascending trace order */
                    long r = ((long)c * Q + q) * S + s;
                    sm += J.r_met[r];
                    sn += J.r_near[r];
                    sg += J.r_good[r];
                    if (rep_met) rep_met[r] = J.r_met[r];
                    if (rep_goodput) rep_goodput[r] = J.r_good[r];
                    if (rep_duration) rep_duration[r] = J.r_dur[r];
                }
                if (met) met[(long)c * Q + q] = sm;
                if (goodput) goodput[(long)c * Q + q] = sg;
                if (near_boundary) near_boundary[(long)c * Q + q] = sn;
            }
        }
        if (argmax) {
            /* A25: (Σmet ↓, Σcaps ↑ [QPS/W spirit, P:339], index ↑) */
            for (int q = 0; q < Q; q++) {
                int best = 0;
                int64_t bm = -1; long bc = 0;
                for (int c = 0; c < C; c++) {
                    int64_t mc = 0;
                    for (int s = 0; s < S; s++) mc += J.r_met[((long)c * Q + q) * S + s];
                    long cs = 0;
                    for (int g = 0; g < N; g++) cs += cap[(size_t)c * N + g];
                    if (mc > bm || (mc == bm && cs < bc)) { best = c; bm = mc; bc = cs; }
                }
                argmax[q] = best;
            }
        }
    }
    free(J.r_met); free(J.r_near); free(J.r_good); free(J.r_dur);
    return rc;
}
