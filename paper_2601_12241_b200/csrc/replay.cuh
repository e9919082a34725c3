// replay.cuh — the per-replay event-driven queueing simulation (rows a4–a7),
// one CUDA thread per (candidate, QPS point, trace) replay.
//
// Semantics: DESIGN.md §3.  Design:
//  * the loop advances instant by instant: t = min over every GPU's next
//    event, the next arrival, the earliest in-flight KV transfer and (dynamic)
//    the next settle / role flip / controller tick; all events of the instant
//    are handled in the kind order of A10, then one dispatch pass;
//  * decode steps are *skipped ahead*: a decode GPU only materialises the
//    boundaries where something happens (a member leaves, pending requests
//    join, or its cap changed).  Boundary k of a segment is at
//    t_seg + (double)k * L exactly as A14 pins it, so skipping is bit-exact;
//    the CPU oracle steps every boundary — parity tests prove equivalence;
//  * queues (prefill FIFO, KV-wait FIFO, decode pending FIFO) are singly
//    linked through one per-request `link` array; per-request prefill end
//    times live in `pe`; decode batches in `mem` — all in a lane-interleaved
//    per-warp scratch region so lanes touching the same request index
//    coalesce;
//  * the trace (s_unit, kv, in, out, phase) of the CTA is staged once in
//    shared memory with cp.async.bulk (TMA bulk copy) and read by all 128
//    replays of the CTA;
//  * the controller (dynamic) is ctl_step() from controller.cuh; window p90
//    comparisons are exact integer counts (p90 > S ⇔ #{v ≤ S} < k with
//    k = ⌈0.9 n⌉), maintained incrementally as samples enter/leave.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "controller.cuh"

namespace padsim {

#define PAD_INF __longlong_as_double(0x7ff0000000000000ULL)

enum : unsigned char { F_DRAIN = 1, F_DIRTY = 2, F_BND = 4, F_CHG = 8 };

template <int NMAX>
struct Gpus {
    double tnext[NMAX];      // next event time of this GPU (INF = none)
    double tseg[NMAX];       // D: segment start
    double L[NMAX];          // D: segment step latency
    long long a0[NMAX];      // P: outstanding tokens   | D: active count
    int qh[NMAX], qt[NMAX], ql[NMAX];   // P: prompt queue | D: pending-join FIFO
    int b0[NMAX];            // P: batch head           | D: last materialised step
    int b1[NMAX];            // P: batch size           | D: next boundary to materialise
    int step0[NMAX];         // D: step index at segment start
    int minfin[NMAX];        // D: smallest finish step among active
    long long ctx[NMAX];     // D: Σ prompt tokens of active (A15 term)
    int eff[NMAX], cmd[NMAX], rse[NMAX];  // effective / commanded cap, pending raise
    unsigned char role[NMAX], fl[NMAX];
};

struct TraceView {
    const double* s_unit;
    const double* kv;
    const int* in_tok;
    const int* out_tok;
    const unsigned char* phase;
    int R;
};

// lane-interleaved scratch accessors
struct Scratch {
    int* link;             // [i*32]
    double* pe;            // [i*32]
    int2* mem;             // [(g*max_db + k)*32]  {fin, id}
    int* ordt;             // [k*32] TTFT window: request ids in prefill-end order
    double* tst;           // [k*32] TPOT window: completion stamps
    unsigned char* tfl;    // [k*32] TPOT window: flags (le0, lt0, le1, lt1)
};

template <int NMAX>
struct CtlView {
    const Gpus<NMAX>* G;
    __device__ int role(int g) const { return G->role[g]; }
    __device__ bool draining(int g) const { return (G->fl[g] & F_DRAIN) != 0; }
    __device__ int target(int g) const { return G->rse[g] > 0 ? G->rse[g] : G->cmd[g]; }
    __device__ long long load(int g) const {
        return G->role[g] == 0 ? G->a0[g] : G->a0[g] + (long long)G->ql[g];
    }
};

struct ReplayResult {
    int met, near;
    double duration, goodput;
    long long events;
    double watts;                  // time-weighted mean of Σ effective caps
};

template <int NMAX, bool DYN>
struct Replay {
    const Plan& P;
    const TraceView& T;
    const Scratch& X;
    Gpus<NMAX> G;
    int N, R, max_db;
    double inv_lam;
    // KV transfer stage (≤ 32 in flight) + waiting FIFO
    double tr_te[PADSIM_MAX_SLOTS];
    int tr_id[PADSIM_MAX_SLOTS];
    int tbusy, tmin, twh, twt, twl;
    // metrics
    int completed, met, near;
    double maxcomp;
    // per-request records (nullable)
    long long rec_base;
    // dynamic state
    padsim_policy pol;
    double tick_t, settle_t, flip_t, last_move;
    long long tick_k;
    int flip_g, drain_pending, phase2;
    int w_th, w_tlo, w_tle, w_tlt;                       // TTFT window
    int w_ph, w_plo, w_ple0, w_plt0, w_ple1, w_plt1;     // TPOT window
    int* metk;            // this replay's sweep counters (global, kMaxSloSweep)
    int nk;
    long long w_sum;
    double w_acc, w_prev, a0t;

    __device__ Replay(const Plan& p, const TraceView& t, const Scratch& x) : P(p), T(t), X(x) {}

    __device__ __forceinline__ int& LNK(int i) { return X.link[(size_t)i * 32]; }
    __device__ __forceinline__ double& PE(int i) { return X.pe[(size_t)i * 32]; }
    __device__ __forceinline__ int2& MEM(int g, int k) { return X.mem[((size_t)g * max_db + k) * 32]; }
    __device__ __forceinline__ double arr(int i) const { return T.s_unit[i] * inv_lam; }
    __device__ __forceinline__ double bnd(int g, int s) const {
        return G.tseg[g] + (double)(s - G.step0[g]) * G.L[g];
    }

    // smallest boundary index s > last materialised with time >= tau
    __device__ int first_bnd_ge(int g, double tau) const {
        const int stepm = G.b0[g];
        float xf = __fdividef((float)(tau - G.tseg[g]), (float)G.L[g]);
        int s = G.step0[g] + (int)ceilf(xf);
        if (s <= stepm) s = stepm + 1;
        while (bnd(g, s) < tau) s++;
        while (s - 1 > stepm && bnd(g, s - 1) >= tau) s--;
        return s;
    }

    __device__ __forceinline__ void tmin_rescan() {
        int k = 0;
        for (int j = 1; j < tbusy; j++)
            if (tr_te[j] < tr_te[k] || (tr_te[j] == tr_te[k] && tr_id[j] < tr_id[k])) k = j;
        tmin = k;
    }

    __device__ __forceinline__ void transfer_start(int i, double t) {
        const int k = tbusy++;
        tr_te[k] = t + T.kv[i];
        tr_id[k] = i;
        if (k == 0 || tr_te[k] < tr_te[tmin] || (tr_te[k] == tr_te[tmin] && i < tr_id[tmin])) tmin = k;
    }

    __device__ void complete(int i, double t, double tpot) {
        completed++;
        const double pe = PE(i);
        const double ttft = pe - arr(i);
        const double ts = T.phase[i] ? P.tpot_slo1 : P.tpot_slo0;
        met += (ttft <= P.ttft_slo && tpot <= ts) ? 1 : 0;
        near += (fabs(ttft - P.ttft_slo) <= 1e-9 * P.ttft_slo || fabs(tpot - ts) <= 1e-9 * ts) ? 1 : 0;
        maxcomp = fmax(maxcomp, t);
        for (int z = 0; z < nk; z++) {
            const double tz = T.phase[i] ? P.sw.tpot1[z] : P.sw.tpot0[z];
            if (ttft <= P.sw.ttft[z] && tpot <= tz) metk[z]++;
        }
        if (DYN) {
            unsigned char f = (tpot <= P.tpot_slo0 ? 1 : 0) | (tpot < P.tpot_slo0 ? 2 : 0) |
                              (tpot <= P.tpot_slo1 ? 4 : 0) | (tpot < P.tpot_slo1 ? 8 : 0);
            X.tst[(size_t)w_ph * 32] = t;
            X.tfl[(size_t)w_ph * 32] = f;
            w_ph++;
            w_ple0 += f & 1; w_plt0 += (f >> 1) & 1; w_ple1 += (f >> 2) & 1; w_plt1 += (f >> 3) & 1;
        }
        if (rec_base >= 0) {
            P.rec_ttft[rec_base + i] = ttft;
            P.rec_tpot[rec_base + i] = tpot;
            P.rec_pe[rec_base + i] = pe;
            P.rec_comp[rec_base + i] = t;
        }
    }

    // A8: prefill GPU with the least outstanding tokens (queued + in service), lowest id
    __device__ void route_prompt(int i) {
        int best = -1;
        long long bl = 0;
#pragma unroll
        for (int g = 0; g < NMAX; g++) {
            if (g >= N) break;
            if (G.role[g] != 0 || (G.fl[g] & F_DRAIN)) continue;
            if (best < 0 || G.a0[g] < bl) { best = g; bl = G.a0[g]; }
        }
        LNK(i) = kNoIdx;
        if (G.ql[best] == 0) G.qh[best] = i; else LNK(G.qt[best]) = i;
        G.qt[best] = i;
        G.ql[best]++;
        G.a0[best] += T.in_tok[i];
    }

    // A13: decode GPU with the fewest active + pending, lowest id; joins at the
    // first step boundary at or after t (A14)
    __device__ void route_decode(int i, double t) {
        int best = -1;
        long long bl = 0;
#pragma unroll
        for (int g = 0; g < NMAX; g++) {
            if (g >= N) break;
            if (G.role[g] != 1 || (G.fl[g] & F_DRAIN)) continue;
            const long long l = G.a0[g] + G.ql[g];
            if (best < 0 || l < bl) { best = g; bl = l; }
        }
        const int v = best;
        LNK(i) = kNoIdx;
        if (G.ql[v] == 0) G.qh[v] = i; else LNK(G.qt[v]) = i;
        G.qt[v] = i;
        G.ql[v]++;
        if (G.a0[v] > 0 && !(G.fl[v] & F_BND) && G.a0[v] < max_db && G.ql[v] == 1) {
            const int s = first_bnd_ge(v, t);
            if (s < G.b1[v]) { G.b1[v] = s; G.tnext[v] = bnd(v, s); }
        }
    }

    // kind 2: prefill batch end → first token (TTFT), members enter the KV buffer
    __device__ void batch_end(int g, double t) {
        int i = G.b0[g];
        const int n = G.b1[g];
        for (int k = 0; k < n; k++) {
            const int nx = LNK(i);
            PE(i) = t;
            G.a0[g] -= T.in_tok[i];
            if (DYN) {
                const double ttft = t - arr(i);
                X.ordt[(size_t)w_th * 32] = i;
                w_th++;
                w_tle += ttft <= P.ttft_slo ? 1 : 0;
                w_tlt += ttft < P.ttft_slo ? 1 : 0;
            }
            if (tbusy < P.m.slots) {
                transfer_start(i, t);
            } else {
                LNK(i) = kNoIdx;
                if (twl == 0) twh = i; else LNK(twt) = i;
                twt = i;
                twl++;
            }
            i = nx;
        }
        G.tnext[g] = PAD_INF;
        G.b1[g] = 0;
    }

    // kind 3: a materialised decode step boundary
    __device__ void boundary(int g, double t) {
        const int s = G.b1[g];
        G.b0[g] = s;
        G.fl[g] |= F_BND;
        G.tnext[g] = PAD_INF;
        if (s == G.minfin[g]) {
            int n = (int)G.a0[g];
            int mf = 0x7fffffff;
            int k = 0;
            while (k < n) {
                const int2 e = MEM(g, k);
                if (e.x == s) {
                    const int id = e.y;
                    complete(id, t, (t - PE(id)) / (double)(T.out_tok[id] - 1));
                    G.ctx[g] -= T.in_tok[id];
                    n--;
                    MEM(g, k) = MEM(g, n);
                } else {
                    mf = e.x < mf ? e.x : mf;
                    k++;
                }
            }
            G.a0[g] = n;
            G.minfin[g] = mf;
            G.fl[g] |= F_CHG;
        }
    }

    // kind 4: KV transfer end (earliest (te, id) first)
    __device__ void transfer_end(double t) {
        const int k = tmin;
        const int i = tr_id[k];
        tbusy--;
        tr_te[k] = tr_te[tbusy];
        tr_id[k] = tr_id[tbusy];
        if (twl > 0) {
            const int j = twh;
            twh = LNK(j);
            twl--;
            tr_te[tbusy] = t + T.kv[j];
            tr_id[tbusy] = j;
            tbusy++;
        }
        if (tbusy > 0) tmin_rescan();
        if (rec_base >= 0) P.rec_te[rec_base + i] = t;
        if (T.out_tok[i] == 1) complete(i, t, 0.0);       // S:280 D4
        else route_decode(i, t);
    }

    __device__ void dispatch(double t) {
        for (int g = 0; g < N; g++) {
            if (G.role[g] == 0) {
                if (G.tnext[g] != PAD_INF || G.ql[g] == 0) continue;
                // A9: FIFO prefix, ≤ max_pb, Σin ≤ budget, head always admitted
                const int h = G.qh[g];
                long long tok = T.in_tok[h];
                int b = 1, j = h;
                const int ql = G.ql[g];
                while (b < P.m.max_pb && b < ql) {
                    const int nx = LNK(j);
                    const long long tt = tok + T.in_tok[nx];
                    if (tt > P.m.pb_tokens) break;
                    tok = tt;
                    j = nx;
                    b++;
                }
                G.b0[g] = h;
                G.b1[g] = b;
                G.ql[g] = ql - b;
                if (ql > b) G.qh[g] = LNK(j);
                const double lat = ((double)tok / P.m.den[b]) / P.m.spre[G.eff[g] - P.m.min_w];
                G.tnext[g] = t + lat;
            } else {
                bool at_bnd = (G.fl[g] & F_BND) != 0;
                if (G.a0[g] > 0 && !at_bnd) {
                    if (G.tnext[g] != t) continue;       // mid-step
                    G.b0[g] = G.b1[g];                   // join boundary exactly at t
                    at_bnd = true;
                }
                if (!at_bnd && G.ql[g] == 0) continue;  // idle, nothing pending
                const bool was_idle = !at_bnd;
                bool joined = false;
                int n = (int)G.a0[g];
                const int step = G.b0[g];
                while (n < max_db && G.ql[g] > 0) {
                    const int i = G.qh[g];
                    G.ql[g]--;
                    if (G.ql[g] > 0) G.qh[g] = LNK(i);
                    const int fin = step + (T.out_tok[i] - 1);
                    MEM(g, n) = make_int2(fin, i);
                    n++;
                    G.ctx[g] += T.in_tok[i];
                    G.minfin[g] = fin < G.minfin[g] ? fin : G.minfin[g];
                    joined = true;
                }
                G.a0[g] = n;
                if (n > 0) {
                    if (was_idle || joined || (G.fl[g] & (F_CHG | F_DIRTY))) {
                        G.tseg[g] = t;
                        G.step0[g] = step;
                        const int ci = G.eff[g] - P.m.min_w;
                        if (P.m.dec_per_ctx == 0.0) {
                            G.L[g] = P.m.ltab[(size_t)ci * max_db + (n - 1)];
                        } else {
                            double x = P.m.dec_fixed + P.m.dec_per_seq * (double)n;
                            x = x + P.m.dec_per_ctx * (double)G.ctx[g];
                            G.L[g] = x / P.m.sdec[ci];
                        }
                        G.fl[g] &= (unsigned char)~F_DIRTY;
                    }
                    G.b1[g] = G.minfin[g];
                    G.tnext[g] = bnd(g, G.minfin[g]);
                } else {
                    G.tnext[g] = PAD_INF;
                    G.minfin[g] = 0x7fffffff;
                }
                G.fl[g] &= (unsigned char)~(F_BND | F_CHG);
            }
        }
    }

    // ---- dynamic-only pieces ------------------------------------------------
    __device__ void settle(double t) {
        for (int g = 0; g < N; g++) {
            bool changed = false;
            if (G.cmd[g] < G.eff[g]) { G.eff[g] = G.cmd[g]; changed = true; }
            if (G.rse[g] > 0) { G.eff[g] = G.cmd[g] = G.rse[g]; G.rse[g] = 0; changed = true; }
            if (changed && G.role[g] == 1) {
                G.fl[g] |= F_DIRTY;
                if (G.a0[g] > 0) {
                    const int s = first_bnd_ge(g, t);
                    if (s < G.b1[g]) { G.b1[g] = s; G.tnext[g] = bnd(g, s); }
                }
            }
        }
        settle_t = PAD_INF;
        if (t > a0t) {
            w_acc = w_acc + (double)w_sum * (t - w_prev);
            w_prev = t;
        }
        long long ws = 0;
        for (int g = 0; g < N; g++) ws += G.eff[g];
        w_sum = ws;
    }

    __device__ void flip(double) {
        const int g = flip_g;
        G.role[g] = (unsigned char)(1 - G.role[g]);
        G.fl[g] = 0;
        G.tnext[g] = PAD_INF;
        G.a0[g] = 0;
        G.ql[g] = 0;
        G.b0[g] = 0;
        G.b1[g] = 0;
        G.step0[g] = 0;
        G.minfin[g] = 0x7fffffff;
        G.ctx[g] = 0;
        drain_pending = 0;
        flip_g = -1;
        flip_t = PAD_INF;
    }

    __device__ void tick(double t) {
        if ((t - last_move) > pol.cooldown_s) {
            const double lo = t - pol.window_s;
            while (w_tlo < w_th) {
                const int id = X.ordt[(size_t)w_tlo * 32];
                const double pe = PE(id);
                if (!(pe < lo)) break;
                const double ttft = pe - arr(id);
                w_tle -= ttft <= P.ttft_slo ? 1 : 0;
                w_tlt -= ttft < P.ttft_slo ? 1 : 0;
                w_tlo++;
            }
            while (w_plo < w_ph && X.tst[(size_t)w_plo * 32] < lo) {
                const unsigned char f = X.tfl[(size_t)w_plo * 32];
                w_ple0 -= f & 1; w_plt0 -= (f >> 1) & 1; w_ple1 -= (f >> 2) & 1; w_plt1 -= (f >> 3) & 1;
                w_plo++;
            }
            const int nt = w_th - w_tlo, np = w_ph - w_plo;
            const int kt = (90 * nt + 99) / 100, kp = (90 * np + 99) / 100;
            CtlSignals sg;
            sg.ttft_gt = w_tle < kt;
            sg.ttft_lt = w_tlt >= kt;
            sg.tpot_gt = (phase2 ? w_ple1 : w_ple0) < kp;
            sg.tpot_lt = (phase2 ? w_plt1 : w_plt0) >= kp;
            int qp = 0;
            for (int g = 0; g < N; g++) if (G.role[g] == 0) qp += G.ql[g];
            sg.q_prefill = qp;
            int newcap[NMAX];
            int gsel, dir;
            CtlView<NMAX> view{&G};
            const int act = ctl_step(pol, P.m.min_w, P.m.max_w, P.B, N, view, drain_pending != 0,
                                     last_move, t, sg, newcap, &gsel, &dir);
            if (act == ACT_MOVE_POWER || act == ACT_MOVE_GPU) {
                last_move = t;
                if (act == ACT_MOVE_GPU) {
                    const int g = gsel;
                    G.fl[g] |= F_DRAIN;
                    drain_pending = 1;
                    flip_g = g;
                    int i = G.qh[g];
                    const int n = G.ql[g];
                    G.ql[g] = 0;
                    if (G.role[g] == 0) {
                        for (int k = 0; k < n; k++) {
                            const int nx = LNK(i);
                            G.a0[g] -= T.in_tok[i];
                            route_prompt(i);
                            i = nx;
                        }
                    } else {
                        for (int k = 0; k < n; k++) {
                            const int nx = LNK(i);
                            route_decode(i, t);
                            i = nx;
                        }
                    }
                }
                for (int g = 0; g < N; g++) {
                    const int tg = newcap[g];
                    if (tg < G.cmd[g]) G.cmd[g] = tg;
                    else if (tg > G.cmd[g]) G.rse[g] = tg;
                }
                settle_t = t + pol.settle_s;
            }
        }
        tick_k++;
        tick_t = (double)tick_k * pol.tick_s;
    }

    __device__ void drain_check(double t) {
        if (flip_g < 0 || flip_t != PAD_INF) return;
        const int g = flip_g;
        const bool empty = G.role[g] == 0 ? (G.tnext[g] == PAD_INF && G.ql[g] == 0)
                                          : (G.a0[g] == 0 && G.ql[g] == 0);
        if (empty) flip_t = t + pol.reassign_s;
    }

    __device__ ReplayResult run(int c, int q, long long rec) {
        N = P.N;
        R = T.R;
        max_db = P.m.max_db;
        inv_lam = 1.0 / (P.qps[q] * (double)N);
        rec_base = rec;
        const unsigned char* crole = P.role + (size_t)c * N;
        const int* ccap = P.cap + (size_t)c * N;
#pragma unroll
        for (int g = 0; g < NMAX; g++) {
            const bool on = g < N;
            G.role[g] = on ? crole[g] : 2;
            G.eff[g] = G.cmd[g] = on ? ccap[g] : P.m.min_w;
            G.rse[g] = 0;
            G.tnext[g] = PAD_INF;
            G.tseg[g] = 0.0;
            G.L[g] = 1.0;
            G.a0[g] = 0;
            G.qh[g] = G.qt[g] = kNoIdx;
            G.ql[g] = 0;
            G.b0[g] = G.b1[g] = 0;
            G.step0[g] = 0;
            G.minfin[g] = 0x7fffffff;
            G.ctx[g] = 0;
            G.fl[g] = 0;
        }
        tbusy = 0; tmin = 0; twh = twt = kNoIdx; twl = 0;
        completed = 0; met = 0; near = 0;
        maxcomp = -PAD_INF;
        if (DYN) {
            pol = P.pol[c];
            tick_k = 1;
            tick_t = (double)tick_k * pol.tick_s;
            settle_t = flip_t = PAD_INF;
            last_move = 0.0;
            flip_g = -1; drain_pending = 0; phase2 = 0;
            w_th = w_tlo = w_tle = w_tlt = 0;
            w_ph = w_plo = w_ple0 = w_plt0 = w_ple1 = w_plt1 = 0;
        }
        nk = P.sw.n;
        for (int z = 0; z < nk; z++) metk[z] = 0;
        w_sum = P.sw.capsum[c];
        a0t = R > 0 ? arr(0) : 0.0;
        w_acc = 0.0;
        w_prev = a0t;
        long long events = 0;
        int na = 0;
        double ta = R > 0 ? arr(0) : PAD_INF;
        while (completed < R) {
            double t = ta;
#pragma unroll
            for (int g = 0; g < NMAX; g++)
                if (g < N) t = fmin(t, G.tnext[g]);
            if (tbusy > 0) t = fmin(t, tr_te[tmin]);
            if (DYN) t = fmin(t, fmin(tick_t, fmin(settle_t, flip_t)));
            events++;
            if (DYN) {
                if (settle_t == t) settle(t);
                if (flip_t == t) flip(t);
            }
            for (int g = 0; g < N; g++)
                if (G.role[g] == 0 && G.tnext[g] == t) batch_end(g, t);
            for (int g = 0; g < N; g++)
                if (G.role[g] == 1 && G.tnext[g] == t) boundary(g, t);
            while (tbusy > 0 && tr_te[tmin] == t) transfer_end(t);
            while (ta == t) {
                if (DYN && T.phase[na] == 1) phase2 = 1;     // S:375 SLO switch
                route_prompt(na);
                na++;
                ta = na < R ? arr(na) : PAD_INF;
            }
            if (DYN && tick_t == t) tick(t);
            dispatch(t);
            if (DYN) drain_check(t);
        }
        ReplayResult res;
        res.met = met;
        res.near = near;
        res.duration = R > 0 ? maxcomp - arr(0) : 0.0;
        res.goodput = res.duration > 0 ? (double)met / res.duration : 0.0;
        res.events = events;
        if (R > 0) w_acc = w_acc + (double)w_sum * (maxcomp - w_prev);
        res.watts = res.duration > 0 ? w_acc / res.duration : (double)w_sum;
        return res;
    }
};

// ---------------------------------------------------------------------------
// TMA (cp.async.bulk) trace staging helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    }
}

template <int NMAX, bool DYN>
__global__ void __launch_bounds__(kThreads) replay_kernel(const __grid_constant__ Plan P) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ unsigned long long bar;
    __shared__ int s_item;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    char* cta_scratch = P.scratch + (size_t)blockIdx.x * P.scratch_per_cta;
    char* wbase = cta_scratch + (size_t)warp * P.warp_bytes;
    Scratch X;
    X.link = (int*)(wbase + P.off_link) + lane;
    X.pe = (double*)(wbase + P.off_pe) + lane;
    X.mem = (int2*)(wbase + P.off_mem) + lane;
    X.ordt = DYN ? (int*)(wbase + P.off_ordt) + lane : nullptr;
    X.tst = DYN ? (double*)(wbase + P.off_tst) + lane : nullptr;
    X.tfl = DYN ? (unsigned char*)(wbase + P.off_tfl) + lane : nullptr;
    if (tid == 0) mbar_init(&bar, 1);
    __syncthreads();
    unsigned phase = 0;
    int cur_s = -1;
    const int per_trace = P.items_per_trace;
    const int QC = P.Q * P.n_clist;
    for (;;) {
        if (tid == 0) s_item = (int)atomicAdd(P.work, 1u);
        __syncthreads();
        const int item = s_item;
        if (item >= P.n_items) break;
        const int s = item / per_trace;
        const int u = (item - s * per_trace) * kThreads + tid;
        const long long off = P.toff[s];
        const int R = P.nreq[s];
        TraceView T;
        T.R = R;
        if (P.smem_trace) {
            const int Rp = (R + 15) & ~15;
            double* sd = (double*)smem;
            double* kvd = sd + Rp;
            int* inp = (int*)(kvd + Rp);
            int* outp = inp + Rp;
            unsigned char* php = (unsigned char*)(outp + Rp);
            if (s != cur_s) {
                if (tid == 0 && Rp > 0) {
                    // order the CTA's earlier generic-proxy reads before the async-proxy writes
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    const unsigned b8 = (unsigned)Rp * 8u, b4 = (unsigned)Rp * 4u, b1 = (unsigned)Rp;
                    mbar_expect_tx(&bar, 2 * b8 + 2 * b4 + b1);
                    bulk_g2s(sd, P.s_unit + off, b8, &bar);
                    bulk_g2s(kvd, P.kv + off, b8, &bar);
                    bulk_g2s(inp, P.in_tok + off, b4, &bar);
                    bulk_g2s(outp, P.out_tok + off, b4, &bar);
                    bulk_g2s(php, P.phase + off, b1, &bar);
                }
                if (Rp > 0) {
                    mbar_wait(&bar, phase);
                    phase ^= 1;
                }
                cur_s = s;
            }
            T.s_unit = sd; T.kv = kvd; T.in_tok = inp; T.out_tok = outp; T.phase = php;
        } else {
            T.s_unit = P.s_unit + off; T.kv = P.kv + off; T.in_tok = P.in_tok + off;
            T.out_tok = P.out_tok + off; T.phase = P.phase + off;
        }
        if (u < QC) {
            const int q = u / P.n_clist;
            const int c = P.clist[u - q * P.n_clist];
            const long long r = ((long long)c * P.Q + q) * P.S + s;
            Replay<NMAX, DYN> rp(P, T, X);
            rp.metk = P.sw.rep_met + r * kMaxSloSweep;
            const ReplayResult res = rp.run(c, q, P.rec_ttft ? r * P.Rmax : -1);
            P.rep_met[r] = res.met;
            P.rep_near[r] = res.near;
            P.rep_dur[r] = res.duration;
            P.rep_good[r] = res.goodput;
            P.rep_events[r] = res.events;
            P.sw.rep_watts[r] = res.watts;
        }
        __syncthreads();   // every replay of the item done before the trace is replaced
    }
}

}  // namespace padsim
