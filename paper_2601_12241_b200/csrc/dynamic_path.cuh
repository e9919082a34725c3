// dynamic_path.cuh — joint replay (rows a4–a7, and a6 for dynamic candidates):
// prefill, KV buffer, decode and the Algorithm 1 controller in one event loop
// per replay (one thread per replay).  NG = 8 (nodes of up to 8 simulated
// GPUs, per-GPU next-event/routing keys in registers, per-GPU state in shared
// memory) or NG = 64 (cfg 5: keys in shared memory with per-group-of-8 minima
// in registers, refreshed lazily; per-GPU state in lane-interleaved global
// scratch).
//
// Same semantics as replay.cuh (DESIGN.md §3 c.2/c.3), different storage:
//  * per-GPU next event time and the two routing keys (prefill: outstanding
//    tokens; decode: active + pending; INT_MAX when the GPU is not eligible —
//    other role or draining) are register arrays, role masks are bitmasks;
//  * the remaining per-GPU state is a [field][gpu][thread] shared-memory SoA,
//    so every handler body is shared across GPUs (run-time GPU index) and
//    bank-conflict free;
//  * handlers run only for the GPUs that have an event at the instant, and
//    the dispatch pass visits only GPUs touched at the instant;
//  * CTAs are bound to one trace; warps pull 32-replay items from that
//    trace's counter (no CTA barrier per item);
//  * window p90 comparisons are exact integer counts (controller.cuh).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "controller.cuh"
#include "replay.cuh"

// Decode batches of the joint replay: PADSIM_JBL = 1 sorted per-GPU batch lists
// in a per-lane ring of u64 (fin << 32 | id) entries (as stageC_kernel<BL>), 0 =
// the timing wheel (bucket heads + occupancy bitmap in global scratch).
#ifndef PADSIM_JBL
#define PADSIM_JBL 1
#endif

namespace padsim {

constexpr int kJG = 8;     // GPU slots of the small-node variant (N ≤ 8)
constexpr int kIntMax = 0x7fffffff;

template <int NG> struct MaskT { using type = unsigned; };
template <> struct MaskT<64> { using type = unsigned long long; };
__device__ __forceinline__ int mffs(unsigned m) { return __ffs(m) - 1; }
__device__ __forceinline__ int mffs(unsigned long long m) { return __ffsll((long long)m) - 1; }

// Per-GPU next event time + routing keys (kp: prefill outstanding tokens, kd:
// decode active+pending; INT_MAX = not eligible).
template <int NG> struct WTab;

template <> struct WTab<8> {                // register arrays, predicated selects
    double tn[8];
    int kp[8], kd[8];
    __device__ __forceinline__ void init(int g, int role) {
#pragma unroll
        for (int v = 0; v < 8; v++) if (v == g) { tn[v] = PAD_INF; kp[v] = role == 0 ? 0 : kIntMax; kd[v] = role == 1 ? 0 : kIntMax; }
    }
    __device__ __forceinline__ double tmin(double cur) {
#pragma unroll
        for (int g = 0; g < 8; g++) cur = tn[g] < cur ? tn[g] : cur;
        return cur;
    }
    __device__ __forceinline__ unsigned eq(double t) {
        unsigned m = 0;
#pragma unroll
        for (int g = 0; g < 8; g++) if (tn[g] == t) m |= 1u << g;
        return m;
    }
    __device__ __forceinline__ void set_t(int gd, double v) {
#pragma unroll
        for (int g = 0; g < 8; g++) tn[g] = (g == gd) ? v : tn[g];
    }
    __device__ __forceinline__ double get_t(int gd) const {
        double v = tn[0];
#pragma unroll
        for (int g = 1; g < 8; g++) v = (g == gd) ? tn[g] : v;
        return v;
    }
    __device__ __forceinline__ int arg_p() {
        int best = 0, bl = kp[0];
#pragma unroll
        for (int g = 1; g < 8; g++) if (kp[g] < bl) { bl = kp[g]; best = g; }
        return best;
    }
    __device__ __forceinline__ int arg_d() {
        int best = 0, bl = kd[0];
#pragma unroll
        for (int g = 1; g < 8; g++) if (kd[g] < bl) { bl = kd[g]; best = g; }
        return best;
    }
    __device__ __forceinline__ void add_p(int gd, int d) {
#pragma unroll
        for (int g = 0; g < 8; g++) kp[g] += (g == gd) ? d : 0;
    }
    __device__ __forceinline__ void add_d(int gd, int d) {
#pragma unroll
        for (int g = 0; g < 8; g++) kd[g] += (g == gd) ? d : 0;
    }
    __device__ __forceinline__ void set_p(int gd, int v) {
#pragma unroll
        for (int g = 0; g < 8; g++) kp[g] = (g == gd) ? v : kp[g];
    }
    __device__ __forceinline__ void set_d(int gd, int v) {
#pragma unroll
        for (int g = 0; g < 8; g++) kd[g] = (g == gd) ? v : kd[g];
    }
};

template <> struct WTab<64> {               // memory arrays + lazily refreshed group minima
    double* tn; int* kp; int* kd; int st;   // [g*st]
    double gt[8];
    int gpv[8], gpi[8], gdv[8], gdi[8];
    unsigned dt, dp, dd;                    // dirty groups
    __device__ __forceinline__ void init(int g, int role) {
        tn[g * st] = PAD_INF;
        kp[g * st] = role == 0 ? 0 : kIntMax;
        kd[g * st] = role == 1 ? 0 : kIntMax;
        dt = dp = dd = 0xffu;
    }
    __device__ __forceinline__ void refresh_t() {
        for (unsigned m = dt; m; m &= m - 1) {
            const int gi = __ffs(m) - 1;
            double v = PAD_INF;
            for (int j = 0; j < 8; j++) { const double x = tn[(gi * 8 + j) * st]; v = x < v ? x : v; }
#pragma unroll
            for (int z = 0; z < 8; z++) gt[z] = (z == gi) ? v : gt[z];
        }
        dt = 0;
    }
    __device__ __forceinline__ double tmin(double cur) {
        refresh_t();
#pragma unroll
        for (int z = 0; z < 8; z++) cur = gt[z] < cur ? gt[z] : cur;
        return cur;
    }
    __device__ __forceinline__ unsigned long long eq(double t) {
        unsigned long long m = 0;
#pragma unroll
        for (int z = 0; z < 8; z++) {
            if (gt[z] == t) {
                for (int j = 0; j < 8; j++)
                    if (tn[(z * 8 + j) * st] == t) m |= 1ull << (z * 8 + j);
            }
        }
        return m;
    }
    __device__ __forceinline__ void set_t(int g, double v) { tn[g * st] = v; dt |= 1u << (g >> 3); }
    __device__ __forceinline__ double get_t(int g) const { return tn[g * st]; }
    __device__ __forceinline__ void refresh_k(int* k, unsigned& dirty, int (&gv)[8], int (&gi)[8]) {
        for (unsigned m = dirty; m; m &= m - 1) {
            const int z = __ffs(m) - 1;
            int bv = k[(z * 8) * st], bi = z * 8;
            for (int j = 1; j < 8; j++) { const int x = k[(z * 8 + j) * st]; if (x < bv) { bv = x; bi = z * 8 + j; } }
#pragma unroll
            for (int y = 0; y < 8; y++) { gv[y] = (y == z) ? bv : gv[y]; gi[y] = (y == z) ? bi : gi[y]; }
        }
        dirty = 0;
    }
    __device__ __forceinline__ int arg_p() {
        refresh_k(kp, dp, gpv, gpi);
        int best = gpi[0], bl = gpv[0];
#pragma unroll
        for (int z = 1; z < 8; z++) if (gpv[z] < bl) { bl = gpv[z]; best = gpi[z]; }
        return best;
    }
    __device__ __forceinline__ int arg_d() {
        refresh_k(kd, dd, gdv, gdi);
        int best = gdi[0], bl = gdv[0];
#pragma unroll
        for (int z = 1; z < 8; z++) if (gdv[z] < bl) { bl = gdv[z]; best = gdi[z]; }
        return best;
    }
    __device__ __forceinline__ void add_p(int g, int d) { kp[g * st] += d; dp |= 1u << (g >> 3); }
    __device__ __forceinline__ void add_d(int g, int d) { kd[g * st] += d; dd |= 1u << (g >> 3); }
    __device__ __forceinline__ void set_p(int g, int v) { kp[g * st] = v; dp |= 1u << (g >> 3); }
    __device__ __forceinline__ void set_d(int g, int v) { kd[g * st] = v; dd |= 1u << (g >> 3); }
};

// per-GPU SoA: shared memory with stride TB (NG = 8) or lane-interleaved
// global scratch with stride 32 (NG = 64); field[g * ws]
struct JWork {
    double* tseg; double* L;
    long long* sj;   // D: Σ join steps of the active members (A40)
    double* dL;      // D: per-step latency growth of the segment (A40)
    int* a0;    // P: outstanding tokens | D: active count
    int* qh; int* qt; int* ql;        // P: prompt FIFO | D: pending joins
    int* b0;    // P: batch head | D: last materialised step
    int* b1;    // P: batch size | D: next boundary to materialise
    int* st0; int* mfin; int* eff; int* cmd; int* rse; int* ctx;
    int* bf;    // D: ring index of the batch list's front (PADSIM_JBL)
    unsigned char* fl;
};
// per-GPU SoA bytes: with the context term (CX) 4 doubles (tseg, L, sj, dL) + 13 ints +
// flags; without it 2 doubles + 12 ints + flags (no sj, dL, ctx: 65 instead of 89 B per
// GPU, so a one-warp CTA needs 16.6 instead of 22.8 KB and 13 instead of 9 fit an SM)
template <int TB, bool CX>
__host__ __device__ constexpr size_t j_work_bytes() {
    return (size_t)kJG * TB * (CX ? 4 * sizeof(double) + 13 * sizeof(int) + 1 : 2 * sizeof(double) + 12 * sizeof(int) + 1);
}

enum : unsigned char { JF_DRAIN = 1, JF_DIRTY = 2 };


// dynamic shared memory of the joint kernel (same base as the kernel's smem[])
extern __shared__ __align__(128) unsigned char joint_dyn_smem[];

template <int NG, int TB, bool CX>
__host__ __device__ constexpr size_t joint_smem_base() {
    return NG == 8 ? j_work_bytes<TB, CX>() : (size_t)NG * TB * (sizeof(double) + 2 * sizeof(int));
}
// + the per-thread Fig. 6 decomposition accumulators (2 doubles)
template <int NG, int TB, bool CX>
__host__ __device__ constexpr size_t joint_smem_bytes() {
    return ((joint_smem_base<NG, TB, CX>() + 15) & ~(size_t)15) + 2 * TB * sizeof(double);
}


template <typename Mask>
struct JCtlView {
    const JWork* W;
    Mask pmask;
    int ws;
    __device__ int role(int g) const { return ((pmask >> g) & 1u) ? 0 : 1; }
    __device__ bool draining(int g) const { return (W->fl[g * ws] & JF_DRAIN) != 0; }
    __device__ int target(int g) const {
        const int r = W->rse[g * ws];
        return r > 0 ? r : W->cmd[g * ws];
    }
    __device__ long long load(int g) const {
        const int o = g * ws;
        return ((pmask >> g) & 1u) ? (long long)W->a0[o] : (long long)W->a0[o] + W->ql[o];
    }
};

// CX: the decode step has a context term (decode_per_ctx_tok_s != 0, A15/A40);
// without it the per-GPU context sums are not kept (no in_tok loads at joins and
// leaves) and the growth code is compiled out
template <bool DYN, int TB, int NG, bool CX>
struct JReplay {
    using Mask = typename MaskT<NG>::type;
    const Plan& P;
    const TraceView& T;
    const Scratch& X;
    const JWork& W;
    int ws;              // stride of the per-GPU SoA
    int N, R, max_db;
    double inv_lam;
    WTab<NG> tab;
    Mask pmask, dmask;
    // KV buffer: slots in lane-interleaved scratch
    double* tte;
    int* tti;
    int* heads;          // [(g*wheel + b)*32]
    unsigned* bits;      // [(g*wheel/32 + k)*32]
    unsigned long long* ring;   // PADSIM_JBL: per-lane [g][RB] batch lists
    size_t accoff;              // byte offset of the Fig. 6 accumulators in shared memory
    int RB, RBm;
    double* wts;         // TTFT window stamps [k], per-lane contiguous (FIFO walk)
    unsigned char* wtf;  // TTFT window flags (≤ SLO, < SLO) [k]
    int Wh, Wm, nwords;
    int tbusy, mk, mid, twh, twt, twl;
    double mte;
    int completed, met, near;
    double maxcomp;
    long long rec_base;
    // dynamic
    padsim_policy pol;
    int Bc;              // this candidate's node budget (DistributeUniformPower)
    double tick_t, settle_t, flip_t, last_move;
    long long tick_k;
    int flip_g, drain_pending, phase2;
    int w_th, w_tlo, w_tle, w_tlt, w_ph, w_plo, w_ple0, w_plt0, w_ple1, w_plt1;
    double wh_t, wh_p;   // oldest TTFT / TPOT window stamps, as of the last window walk
    Mask touched;
    // SLO sweep + provisioned power (time-weighted Σ effective caps)
    int* metk;            // this replay's sweep counters (global, kMaxSloSweep)
    int nk;
    long long w_sum;
    double w_acc, w_prev, a0t;
    bool gr;             // A40 context growth (ctx_growth with a context cost)

    __device__ JReplay(const Plan& p, const TraceView& t, const Scratch& x, const JWork& w)
        : P(p), T(t), X(x), W(w) {}

    __device__ __forceinline__ int& LNK(int i) { return X.link[(size_t)i * 32]; }
    __device__ __forceinline__ double& PE(int i) { return X.pe[(size_t)i * 32]; }
    __device__ __forceinline__ double arr(int i) const { return T.s_unit[i] * inv_lam; }
    __device__ __forceinline__ void set_tnext(int g, double v) { tab.set_t(g, v); }
    __device__ __forceinline__ double get_tnext(int g) const { return tab.get_t(g); }
    __device__ __forceinline__ void add_kp(int g, int d) { tab.add_p(g, d); }
    __device__ __forceinline__ void add_kd(int g, int d) { tab.add_d(g, d); }
    __device__ __forceinline__ double bnd(int o, int s) const {
        return seg_bnd(W.tseg[o], W.L[o], (CX && gr) ? W.dL[o] : 0.0, s - W.st0[o], gr);
    }
    __device__ int first_bnd_ge(int o, double tau) const {
        return seg_first_ge(W.tseg[o], W.L[o], (CX && gr) ? W.dL[o] : 0.0, W.st0[o], W.b0[o], tau, gr);
    }

    __device__ void complete(int i, double t, double tpot) {
        completed++;
        const double pe = PE(i);
        const double ttft = pe - arr(i);
        const double ts = T.phase[i] ? P.tpot_slo1 : P.tpot_slo0;
        met += (ttft <= P.ttft_slo && tpot <= ts) ? 1 : 0;
        near += (fabs(ttft - P.ttft_slo) <= 1e-9 * P.ttft_slo || fabs(tpot - ts) <= 1e-9 * ts) ? 1 : 0;
        maxcomp = fmax(maxcomp, t);
#pragma unroll 1
        for (int z = 0; z < nk; z++) {
            const double tz = T.phase[i] ? P.sw.tpot1[z] : P.sw.tpot0[z];
            if (ttft <= P.sw.ttft[z] && tpot <= tz) metk[z]++;
        }
        if (DYN && pol.window_stamp) {       // TTFT sampled at completion
            const unsigned char f = (ttft <= P.ttft_slo ? 1 : 0) | (ttft < P.ttft_slo ? 2 : 0);
            wts[w_th] = t;
            wtf[w_th] = f;
            w_th++;
            w_tle += f & 1;
            w_tlt += f >> 1;
        }
        if (DYN) {
            const unsigned char f = (tpot <= P.tpot_slo0 ? 1 : 0) | (tpot < P.tpot_slo0 ? 2 : 0) |
                                    (tpot <= P.tpot_slo1 ? 4 : 0) | (tpot < P.tpot_slo1 ? 8 : 0);
            X.tst[w_ph] = t;
            X.tfl[w_ph] = f;
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

    // A8: least outstanding non-draining prefill GPU, lowest id
    __device__ void route_prompt(int i) {
        const int best = tab.arg_p();
        const int tin = T.in_tok[i];
        add_kp(best, tin);
        const int o = best * ws;
        W.a0[o] += tin;
        LNK(i) = kNoIdx;
        const int qn = W.ql[o];
        if (qn == 0) W.qh[o] = i; else LNK(W.qt[o]) = i;
        W.qt[o] = i;
        W.ql[o] = qn + 1;
        touched |= ((Mask)1) << best;
    }

    // A13/A14: fewest active+pending non-draining decode GPU, lowest id; joins
    // at the first step boundary at or after t
    __device__ void route_decode(int i, double t, Mask bm_now) {
        const int best = tab.arg_d();
        add_kd(best, 1);
        const int o = best * ws;
        LNK(i) = kNoIdx;
        const int qn = W.ql[o];
        if (qn == 0) W.qh[o] = i; else LNK(W.qt[o]) = i;
        W.qt[o] = i;
        W.ql[o] = qn + 1;
        touched |= ((Mask)1) << best;
        const int na = W.a0[o];
        if (na > 0 && !((bm_now >> best) & 1u) && na < max_db && qn == 0) {
            const int s = first_bnd_ge(o, t);
            if (s < W.b1[o]) { W.b1[o] = s; set_tnext(best, bnd(o, s)); }
        }
    }

    __device__ void batch_end(int g, double t) {
        const int o = g * ws;
        int i = W.b0[o];
        const int n = W.b1[o];
        const double bstart = W.tseg[o];      // prefill workers keep the batch start here
        double bq = 0.0, be = 0.0;            // Fig. 6 decomposition, this batch
        int dec = 0;
        for (int z = 0; z < n; z++) {
            const int nx = LNK(i);
            PE(i) = t;
            dec += T.in_tok[i];
            bq = bq + (bstart - arr(i));
            be = be + (t - bstart);
            if (DYN && !pol.window_stamp) {   // A22: TTFT known at the first token
                const double ttft = t - arr(i);
                const unsigned char f = (ttft <= P.ttft_slo ? 1 : 0) | (ttft < P.ttft_slo ? 2 : 0);
                wts[w_th] = t;
                wtf[w_th] = f;
                w_th++;
                w_tle += f & 1;
                w_tlt += f >> 1;
            }
            if (tbusy < P.m.slots) {
                const double te = t + T.kv[i];
                tte[tbusy * 32] = te;
                tti[tbusy * 32] = i;
                if (tbusy == 0 || te < mte || (te == mte && i < mid)) { mte = te; mid = i; mk = tbusy; }
                tbusy++;
            } else {
                LNK(i) = kNoIdx;
                if (twl == 0) twh = i; else LNK(twt) = i;
                twt = i;
                twl++;
            }
            i = nx;
        }
        {   // per-thread accumulators in shared memory (no extra registers)
            double* acc = (double*)(joint_dyn_smem + accoff) +
                          threadIdx.x;
            acc[0] = acc[0] + bq;
            acc[TB] = acc[TB] + be;
        }
        W.a0[o] -= dec;
        if (!(W.fl[o] & JF_DRAIN)) add_kp(g, -dec);
        W.b1[o] = 0;
        set_tnext(g, PAD_INF);
    }

    // returns true when the composition changed (leaves).  Decode batches are
    // a timing wheel: bucket (finish step mod Wh) chains its members through
    // link[]; an occupancy bitmap gives the next finish step.
    __device__ bool boundary(int g, double t) {
        const int o = g * ws;
        const int s = W.b1[o];
        W.b0[o] = s;
        set_tnext(g, PAD_INF);
        if (s != W.mfin[o]) return false;
        int left = 0;
        auto leave = [&](int id) {
            complete(id, t, (t - PE(id)) / (double)(T.out_tok[id] - 1));
            if (CX) W.ctx[o] -= T.in_tok[id];
            if (CX && gr) W.sj[o] -= s - (T.out_tok[id] - 1);      // its join step (A40)
            left++;
        };
        int mf = kIntMax;
        if (PADSIM_JBL) {
            // pop the front entries with fin == s; the first one left is the new front
            const int n0 = W.a0[o];
            const unsigned long long* rg = ring + (size_t)g * RB;
            int f = W.bf[o];
            unsigned long long e = rg[f];
            for (;;) {
                leave((int)(unsigned)e);
                f = (f + 1) & RBm;
                if (left == n0) break;
                e = rg[f];
                if ((int)(e >> 32) != s) break;
            }
            W.bf[o] = f;
            W.a0[o] = n0 - left;
            if (left < n0) mf = (int)(e >> 32);
        } else {
            const int b = s & Wm;
            int id = heads[((size_t)g * Wh + b) * 32];
            while (id != kNoIdx) {
                const int nx = LNK(id);
                leave(id);
                id = nx;
            }
            unsigned* bw = bits + (size_t)g * nwords * 32;
            bw[(size_t)(b >> 5) * 32] &= ~(1u << (b & 31));
            const int n = W.a0[o] - left;
            W.a0[o] = n;
            if (n > 0) {
                const int st = (b + 1) & Wm;
                int wi = st >> 5;
                unsigned mword = bw[(size_t)wi * 32] & (0xffffffffu << (st & 31));
                while (mword == 0u) {
                    wi = (wi + 1) & (nwords - 1);
                    mword = bw[(size_t)wi * 32];
                }
                mf = s + ((((wi << 5) + __ffs(mword) - 1) - b) & Wm);
            }
        }
        W.mfin[o] = mf;
        if (!(W.fl[o] & JF_DRAIN)) add_kd(g, -left);
        return true;
    }

    __device__ void transfer_end(double t, Mask bm_now) {
        const int i = mid;
        tbusy--;
        if (mk != tbusy) { tte[mk * 32] = tte[tbusy * 32]; tti[mk * 32] = tti[tbusy * 32]; }
        if (twl > 0) {
            const int j = twh;
            twh = LNK(j);
            twl--;
            tte[tbusy * 32] = t + T.kv[j];
            tti[tbusy * 32] = j;
            tbusy++;
        }
        // earliest (te, id) in flight: slots read four at a time (independent loads)
        mte = PAD_INF;
        for (int z0 = 0; z0 < tbusy; z0 += 4) {
            double ev[4];
            int dv[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const bool ok = z0 + j < tbusy;
                ev[j] = ok ? tte[(z0 + j) * 32] : PAD_INF;
                dv[j] = ok ? tti[(z0 + j) * 32] : 0x7fffffff;
            }
#pragma unroll
            for (int j = 0; j < 4; j++)
                if (ev[j] < mte || (ev[j] == mte && dv[j] < mid)) { mte = ev[j]; mid = dv[j]; mk = z0 + j; }
        }
        if (rec_base >= 0) P.rec_te[rec_base + i] = t;
        if (T.out_tok[i] == 1) complete(i, t, 0.0);
        else route_decode(i, t, bm_now);
    }

    __device__ void dispatch_prefill(int g, double t) {
        const int o = g * ws;
        const int qn = W.ql[o];
        if (get_tnext(g) != PAD_INF || qn == 0) return;
        const int h = W.qh[o];
        long long tok = T.in_tok[h];
        int b = 1, j = h;
        while (b < P.m.max_pb && b < qn) {
            const int nx = LNK(j);
            const long long tt = tok + T.in_tok[nx];
            if (tt > P.m.pb_tokens) break;
            tok = tt;
            j = nx;
            b++;
        }
        W.b0[o] = h;
        W.b1[o] = b;
        W.tseg[o] = t;
        W.ql[o] = qn - b;
        if (qn > b) W.qh[o] = LNK(j);
        set_tnext(g, t + ((double)tok / P.m.den[b]) / P.m.spre[W.eff[o] - P.m.min_w]);
    }

    __device__ void dispatch_decode(int g, double t, bool at_bnd, bool changed) {
        const int o = g * ws;
        int n = W.a0[o];
        if (n > 0 && !at_bnd) {
            if (get_tnext(g) != t) return;      // mid-step
            W.b0[o] = W.b1[o];                  // join boundary exactly at t
            at_bnd = true;
        }
        int qn = W.ql[o];
        if (!at_bnd && qn == 0) return;
        const bool was_idle = !at_bnd;
        bool joined = false;
        const int step = W.b0[o];
        int mf = W.mfin[o];
        int h = W.qh[o];
        int* hw = heads + (size_t)g * Wh * 32;
        unsigned* bw = bits + (size_t)g * nwords * 32;
        while (n < max_db && qn > 0) {
            const int i = h;
            qn--;
            if (qn > 0) h = LNK(i);
            const int fin = step + (T.out_tok[i] - 1);
            if (PADSIM_JBL) {
                // insert (fin, i) into the sorted list of n members from the back
                unsigned long long* rg = ring + (size_t)g * RB;
                const int f = W.bf[o];
                const unsigned long long e = ((unsigned long long)(unsigned)fin << 32) | (unsigned)i;
                int z = n;
                while (z > 0) {
                    const unsigned long long pv = rg[(f + z - 1) & RBm];
                    if (pv < e) break;
                    rg[(f + z) & RBm] = pv;
                    z--;
                }
                rg[(f + z) & RBm] = e;
            } else {
                const int b = fin & Wm;
                unsigned* wp = bw + (size_t)(b >> 5) * 32;
                const unsigned bit = 1u << (b & 31);
                const unsigned old = *wp;
                LNK(i) = (old & bit) ? hw[(size_t)b * 32] : kNoIdx;
                hw[(size_t)b * 32] = i;
                *wp = old | bit;
            }
            n++;
            if (CX) W.ctx[o] += T.in_tok[i];
            if (CX && gr) W.sj[o] += step;
            mf = fin < mf ? fin : mf;
            joined = true;
        }
        W.ql[o] = qn;
        W.qh[o] = h;
        W.a0[o] = n;
        if (n > 0) {
            const unsigned char f = W.fl[o];
            if (was_idle || joined || changed || (f & JF_DIRTY)) {
                W.tseg[o] = t;
                W.st0[o] = step;
                const int ci = W.eff[o] - P.m.min_w;
                if (!CX) {
                    W.L[o] = P.m.ltab[(size_t)ci * max_db + (n - 1)];
                } else {            // A15 / A40 context of the segment's first step
                    double xv = P.m.dec_fixed + P.m.dec_per_seq * (double)n;
                    long long cc = W.ctx[o];
                    if (CX && gr) cc += (long long)n * (step + 1) - W.sj[o];
                    xv = xv + P.m.dec_per_ctx * (double)cc;
                    W.L[o] = xv / P.m.sdec[ci];
                    if (CX && gr) W.dL[o] = (P.m.dec_per_ctx * (double)n) / P.m.sdec[ci];
                }
                W.fl[o] = f & (unsigned char)~JF_DIRTY;
            }
            W.mfin[o] = mf;
            W.b1[o] = mf;
            if (!PADSIM_JBL) pf_head(hw + (size_t)(mf & Wm) * 32);
            set_tnext(g, bnd(o, mf));
        } else {
            W.mfin[o] = kIntMax;
            set_tnext(g, PAD_INF);
        }
    }

    // ---- dynamic ---------------------------------------------------------
    __device__ void settle(double t) {
#pragma unroll 1
        for (int g = 0; g < N; g++) {
            const int o = g * ws;
            bool changed = false;
            int e = W.eff[o], c = W.cmd[o];
            const int r = W.rse[o];
            if (c < e) { e = c; changed = true; }
            if (r > 0) { e = c = r; W.rse[o] = 0; changed = true; }
            W.eff[o] = e;
            W.cmd[o] = c;
            if (changed && ((dmask >> g) & 1u)) {
                W.fl[o] |= JF_DIRTY;
                if (W.a0[o] > 0) {
                    const int s = first_bnd_ge(o, t);
                    if (s < W.b1[o]) { W.b1[o] = s; set_tnext(g, bnd(o, s)); }
                }
            }
        }
        settle_t = PAD_INF;
        if (t > a0t) {
            w_acc = w_acc + (double)w_sum * (t - w_prev);
            w_prev = t;
        }
        long long wsum_ = 0;
#pragma unroll 1
        for (int g = 0; g < N; g++) wsum_ += W.eff[g * ws];
        w_sum = wsum_;
    }

    __device__ void flip() {
        const int g = flip_g, o = g * ws;
        const bool to_p = ((dmask >> g) & 1u) != 0;
        pmask ^= ((Mask)1) << g;
        dmask ^= ((Mask)1) << g;
        W.fl[o] = 0;
        W.a0[o] = 0; W.ql[o] = 0; W.b0[o] = 0; W.b1[o] = 0; W.st0[o] = 0;
        W.mfin[o] = kIntMax; W.bf[o] = 0;
        if (CX) { W.ctx[o] = 0; W.sj[o] = 0; }
        set_tnext(g, PAD_INF);
        tab.set_p(g, to_p ? 0 : kIntMax);
        tab.set_d(g, to_p ? kIntMax : 0);
        drain_pending = 0;
        flip_g = -1;
        flip_t = PAD_INF;
    }

    // returns 0: cooldown not elapsed (guards not evaluated), 1: evaluated, no
    // move (none or saturated), 2: a move was made
    __device__ int tick(double t, Mask bm_now) {
        int acted = 0;
        if ((t - last_move) > pol.cooldown_s) {
            acted = 1;
            const double lo = t - pol.window_s;
            // expire samples older than the window from both FIFOs in one walk: the
            // next stamp (and flags) of each are loaded together, one round trip per
            // step instead of one per FIFO
            for (;;) {
                const bool ct = w_tlo < w_th, cp = w_plo < w_ph;
                const double a = ct ? wts[w_tlo] : PAD_INF;
                const double b = cp ? X.tst[w_plo] : PAD_INF;
                const unsigned char fa = ct ? wtf[w_tlo] : 0;
                const unsigned char fb = cp ? X.tfl[w_plo] : 0;
                const bool pa = a < lo, pb = b < lo;
                if (!pa && !pb) { wh_t = a; wh_p = b; break; }   // the heads, for skip_ticks
                if (pa) { w_tle -= fa & 1; w_tlt -= fa >> 1; w_tlo++; }
                if (pb) {
                    w_ple0 -= fb & 1; w_plt0 -= (fb >> 1) & 1; w_ple1 -= (fb >> 2) & 1; w_plt1 -= (fb >> 3) & 1;
                    w_plo++;
                }
            }
            const int nt = w_th - w_tlo, np = w_ph - w_plo;
            const int kt = (90 * nt + 99) / 100, kq = (90 * np + 99) / 100;
            CtlSignals sg;
            sg.ttft_gt = w_tle < kt;
            sg.ttft_lt = w_tlt >= kt;
            sg.tpot_gt = (phase2 ? w_ple1 : w_ple0) < kq;
            sg.tpot_lt = (phase2 ? w_plt1 : w_plt0) >= kq;
            int qp = 0;
            for (Mask m = pmask; m; m &= m - 1) qp += W.ql[mffs(m) * ws];
            sg.q_prefill = qp;
            int newcap[NG];
            int gsel, dir;
            JCtlView<Mask> view{&W, pmask, ws};
            const int act = ctl_step(pol, P.m.min_w, P.m.max_w, Bc, N, view, drain_pending != 0,
                                     last_move, t, sg, newcap, &gsel, &dir);
            if (act == ACT_MOVE_POWER || act == ACT_MOVE_GPU) {
                last_move = t;
                if (act == ACT_MOVE_GPU) {
                    const int g = gsel, o = g * ws;
                    W.fl[o] |= JF_DRAIN;
                    drain_pending = 1;
                    flip_g = g;
                    int i = W.qh[o];
                    const int n = W.ql[o];
                    W.ql[o] = 0;
                    if ((pmask >> g) & 1u) {
                        tab.set_p(g, kIntMax);
                        for (int z = 0; z < n; z++) {
                            const int nx = LNK(i);
                            W.a0[o] -= T.in_tok[i];
                            route_prompt(i);
                            i = nx;
                        }
                    } else {
                        tab.set_d(g, kIntMax);
                        for (int z = 0; z < n; z++) {
                            const int nx = LNK(i);
                            route_decode(i, t, bm_now);
                            i = nx;
                        }
                    }
                }
#pragma unroll 1
                for (int g = 0; g < N; g++) {
                    const int o = g * ws;
                    const int tg = newcap[g];
                    if (tg < W.cmd[o]) W.cmd[o] = tg;
                    else if (tg > W.cmd[o]) W.rse[o] = tg;
                }
                settle_t = t + pol.settle_s;
                acted = 2;
            }
        }
        tick_k++;
        tick_t = (double)tick_k * pol.tick_s;
        return acted;
    }

    // first tick index k >= k0 with (double)k * tick_s >= x
    __device__ long long tick_at_or_after(double x, long long k0) const {
        if (!(x < PAD_INF)) return 0x7fffffffffffffffLL;
        long long k = (long long)ceil(x / pol.tick_s);
        if (k < k0) k = k0;
        while ((double)k * pol.tick_s < x) k++;
        while (k - 1 >= k0 && (double)(k - 1) * pol.tick_s >= x) k--;
        return k;
    }
    // first tick index k >= k0 with stamp < (double)k * tick_s − window  (sample expiry)
    __device__ long long expiry_tick(double stamp, long long k0) const {
        long long k = (long long)floor((stamp + pol.window_s) / pol.tick_s);
        if (k < k0) k = k0;
        while (!(stamp < (double)k * pol.tick_s - pol.window_s)) k++;
        while (k - 1 >= k0 && stamp < (double)(k - 1) * pol.tick_s - pol.window_s) k--;
        return k;
    }
    // first tick index k >= k0 with ((double)k * tick_s − last_move) > cooldown
    __device__ long long cooldown_tick(long long k0) const {
        long long k = (long long)floor((last_move + pol.cooldown_s) / pol.tick_s);
        if (k < k0) k = k0;
        while (!(((double)k * pol.tick_s - last_move) > pol.cooldown_s)) k++;
        while (k - 1 >= k0 && ((double)(k - 1) * pol.tick_s - last_move) > pol.cooldown_s) k--;
        return k;
    }

    // Tick skipping (exact): after a tick that changed nothing, no later tick can
    // act before (a) the next pending event changes the state, (b) a sample leaves
    // a metric window, or (c) the cooldown elapses; the decision depends on
    // nothing else.  Jump to the first grid tick that can see one of these.
    __device__ void skip_ticks(int outcome, double next_event) {
        const long long k0 = tick_k;
        long long k;
        if (outcome == 0) {
            k = cooldown_tick(k0);           // no tick before it can act, whatever happens
        } else {
            k = tick_at_or_after(next_event, k0);
            // the oldest stamps were read by this tick's window walk (no sample is
            // added or expired between the tick and here)
            if (w_tlo < w_th) k = min(k, expiry_tick(wh_t, k0));
            if (w_plo < w_ph) k = min(k, expiry_tick(wh_p, k0));
        }
        if (k > k0 && k != 0x7fffffffffffffffLL) {
            tick_k = k;
            tick_t = (double)tick_k * pol.tick_s;
        }
    }

    // the replay in three parts (start / one instant / result) so that a lane can
    // start its next replay inside the same event loop (lane refill, joint_kernel)
    long long events;
    int na;
    double ta;
    float win;

    __device__ ReplayResult run(int c, int q, long long rec) {
        start(c, q, rec);
        while (completed < R) instant();
        return result();
    }

    __device__ void start(int c, int q, long long rec) {
        N = P.N;
        R = T.R;
        max_db = P.m.max_db;
        inv_lam = 1.0 / (P.qps[q] * (double)N);
        rec_base = rec;
        const unsigned char* crole = P.role + (size_t)c * N;
        const int* ccap = P.cap + (size_t)c * N;
        pmask = dmask = 0;
#pragma unroll
        for (int g = 0; g < NG; g++) {
            const int o = g * ws;
            const bool on = g < N;
            const int r = on ? crole[g] : 2;
            if (r == 0) pmask |= ((Mask)1) << g;
            if (r == 1) dmask |= ((Mask)1) << g;
            tab.init(g, r);
            W.tseg[o] = 0.0; W.L[o] = 1.0;
            if (CX) { W.sj[o] = 0; W.dL[o] = 0.0; W.ctx[o] = 0; }
            W.a0[o] = 0; W.qh[o] = kNoIdx; W.qt[o] = kNoIdx; W.ql[o] = 0;
            W.b0[o] = 0; W.b1[o] = 0; W.st0[o] = 0; W.mfin[o] = kIntMax;
            W.eff[o] = W.cmd[o] = on ? ccap[g] : P.m.min_w;
            W.rse[o] = 0; W.fl[o] = 0; W.bf[o] = 0;
        }
        Wh = P.wheel; Wm = Wh - 1; nwords = Wh >> 5;
        if (!PADSIM_JBL)
            for (int z = 0; z < N * nwords; z++) bits[(size_t)z * 32] = 0u;
        tbusy = 0; mk = 0; mid = 0; twh = twt = kNoIdx; twl = 0;
        mte = PAD_INF;
        completed = 0; met = 0; near = 0;
        maxcomp = -PAD_INF;
        if (DYN) {
            pol = P.pol[c];
            Bc = P.cbud[c];
            tick_k = 1;
            tick_t = (double)tick_k * pol.tick_s;
            settle_t = flip_t = PAD_INF;
            last_move = 0.0;
            flip_g = -1; drain_pending = 0; phase2 = 0;
            w_th = w_tlo = w_tle = w_tlt = 0;
            w_ph = w_plo = w_ple0 = w_plt0 = w_ple1 = w_plt1 = 0;
        } else {
            tick_t = settle_t = flip_t = PAD_INF;
        }
        nk = P.sw.n;
#pragma unroll 1
        for (int z = 0; z < nk; z++) metk[z] = 0;
        gr = CX && P.m.ctx_growth != 0 && P.m.dec_per_ctx != 0.0;
        w_sum = P.sw.capsum[c];
        a0t = R > 0 ? arr(0) : 0.0;
        w_acc = 0.0;
        w_prev = a0t;
        {
            double* acc = (double*)(joint_dyn_smem + accoff) +
                          threadIdx.x;
            acc[0] = 0.0;
            acc[TB] = 0.0;
        }
        events = 0;
        na = 0;
        ta = R > 0 ? arr(0) : PAD_INF;
        // keep the simulated clocks of a warp's lanes within sync_win mean
        // inter-arrival times (same trace → shared cache lines); scheduling only,
        // results are independent of it (see stageC_kernel)
        win = P.sync_win > 0.f ? (float)((double)P.sync_win * inv_lam) : 0.f;
    }

    // one DES instant (all events at the next time t, then the dispatch pass)
    __device__ __forceinline__ void instant() {
        {
            double t = tab.tmin(ta < mte ? ta : mte);
            if (DYN) {
                t = tick_t < t ? tick_t : t;
                t = settle_t < t ? settle_t : t;
                t = flip_t < t ? flip_t : t;
            }
            if (win > 0.f) {
                const float tf = (float)t;
                const unsigned mn = __reduce_min_sync(__activemask(), __float_as_uint(tf));
                if (tf > __uint_as_float(mn) + win) return;
            }
            events++;
            touched = 0;
            if (DYN) {
                if (settle_t == t) settle(t);
                if (flip_t == t) flip();
            }
            const Mask bm = tab.eq(t);
            const Mask bp = bm & pmask, bd = bm & dmask;
            for (Mask m = bp; m; m &= m - 1) batch_end(mffs(m), t);
            Mask chg = 0;
            for (Mask m = bd; m; m &= m - 1) {
                const int g = mffs(m);
                if (boundary(g, t)) chg |= ((Mask)1) << g;
            }
            while (tbusy > 0 && mte == t) transfer_end(t, bd);
            while (ta == t) {
                if (DYN && T.phase[na] == 1) phase2 = 1;
                route_prompt(na);
                na++;
                ta = na < R ? arr(na) : PAD_INF;
            }
            int tick_outcome = 2;
            if (DYN && tick_t == t) tick_outcome = tick(t, bd);
            for (Mask m = bm | touched; m; m &= m - 1) {
                const int g = mffs(m);
                if ((pmask >> g) & 1u) dispatch_prefill(g, t);
                else dispatch_decode(g, t, (bd >> g) & 1u, (chg >> g) & 1u);
            }
            if (DYN && flip_g >= 0 && flip_t == PAD_INF) {
                const int o = flip_g * ws;
                const bool empty = ((pmask >> flip_g) & 1u)
                                       ? (get_tnext(flip_g) == PAD_INF && W.ql[o] == 0)
                                       : (W.a0[o] == 0 && W.ql[o] == 0);
                if (empty) flip_t = t + pol.reassign_s;
            }
            if (DYN && tick_outcome < 2) {
                double ne = ta < mte ? ta : mte;
                ne = settle_t < ne ? settle_t : ne;
                ne = flip_t < ne ? flip_t : ne;
                skip_ticks(tick_outcome, tab.tmin(ne));
            }
        }
    }

    __device__ ReplayResult result() {
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

// CTAs bound to one trace (s = blockIdx.x mod S); warps pull 32-replay items.
// MR: register cap — 232 for one-warp CTAs (no spills; measured on cfg 3/4: a
// 168-register variant that fits more warps next to stage C was not faster).
template <bool DYN, int TB, int NG, bool CX, int MR = (TB == 32 ? 232 : 168)>
__global__ void __launch_bounds__(TB) __maxnreg__(MR) joint_kernel(const __grid_constant__ Plan P) {
    constexpr bool kRefill = TB == 32 && NG == 8 && MR == 168;
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    char* wbase = P.scratch + ((size_t)blockIdx.x * (TB / 32) + warp) * P.warp_bytes;
    const size_t accoff = (NG == 64 && P.j_kglob) ? 0 : ((joint_smem_base<NG, TB, CX>() + 15) & ~(size_t)15);
    JWork W;
    int ws;
    if (NG == 8) {           // per-GPU SoA in shared memory
        const int n = kJG * TB;
        unsigned char* p = smem;
        W.tseg = (double*)p + tid; p += n * sizeof(double);
        W.L = (double*)p + tid; p += n * sizeof(double);
        W.sj = nullptr; W.dL = nullptr; W.ctx = nullptr;
        if (CX) {
            W.sj = (long long*)p + tid; p += n * sizeof(long long);
            W.dL = (double*)p + tid; p += n * sizeof(double);
        }
        int* ib = (int*)p;
        W.a0 = ib + 0 * n + tid; W.qh = ib + 1 * n + tid; W.qt = ib + 2 * n + tid;
        W.ql = ib + 3 * n + tid; W.b0 = ib + 4 * n + tid; W.b1 = ib + 5 * n + tid;
        W.st0 = ib + 6 * n + tid; W.mfin = ib + 7 * n + tid; W.eff = ib + 8 * n + tid;
        W.cmd = ib + 9 * n + tid; W.rse = ib + 10 * n + tid; W.bf = ib + 11 * n + tid;
        if (CX) W.ctx = ib + 12 * n + tid;
        p += (CX ? 13 : 12) * n * sizeof(int);
        W.fl = p + tid;
        ws = TB;
    } else {                 // per-GPU SoA in lane-interleaved global scratch
        const int n = NG * 32;
        char* p = wbase + P.off_jw;
        W.tseg = (double*)p + lane; p += n * sizeof(double);
        W.L = (double*)p + lane; p += n * sizeof(double);
        W.sj = (long long*)p + lane; p += n * sizeof(long long);
        W.dL = (double*)p + lane; p += n * sizeof(double);
        int* ib = (int*)p;
        W.a0 = ib + 0 * n + lane; W.qh = ib + 1 * n + lane; W.qt = ib + 2 * n + lane;
        W.ql = ib + 3 * n + lane; W.b0 = ib + 4 * n + lane; W.b1 = ib + 5 * n + lane;
        W.st0 = ib + 6 * n + lane; W.mfin = ib + 7 * n + lane; W.eff = ib + 8 * n + lane;
        W.cmd = ib + 9 * n + lane; W.rse = ib + 10 * n + lane; W.ctx = ib + 11 * n + lane;
        W.bf = ib + 13 * n + lane;
        p += 14 * n * sizeof(int);
        W.fl = (unsigned char*)p + lane;
        ws = 32;
    }
    Scratch X;
    X.link = (int*)(wbase + P.off_link) + lane;
    X.pe = (double*)(wbase + P.off_pe) + lane;
    X.mem = nullptr;
    X.ordt = nullptr;
    // window FIFOs are appended and expired in order: per-lane contiguous, so a
    // lane's consecutive stamps share cache lines
    X.tst = DYN ? (double*)(wbase + P.off_tst) + (size_t)lane * P.Rmax : nullptr;
    X.tfl = DYN ? (unsigned char*)(wbase + P.off_tfl) + (size_t)lane * P.Rmax : nullptr;
    double* tte = (double*)(wbase + P.off_tte) + lane;
    int* tti = (int*)(wbase + P.off_tti) + lane;
    const int s = blockIdx.x % P.S;
    const long long off = P.toff[s];
    TraceView T;
    T.R = P.nreq[s];
    T.s_unit = P.s_unit + off; T.kv = P.kv + off; T.in_tok = P.in_tok + off;
    T.out_tok = P.out_tok + off; T.phase = P.phase + off;
    const int QC = P.Q * P.n_clist;
    if constexpr (kRefill) {
        // Lane refill (the 168-register one-warp variant, which runs next to a large
        // stage C workload): the work counter counts replays; a warp's first lpw lanes
        // start on consecutive replays (u = q·n_clist + c: one arrival stream), and a
        // lane whose replay ends stores it and starts the next replay inside the same
        // event loop instead of idling until the longest replay of its warp is done
        // (for grids smaller than the replay count; at cfg 4's size every lane has
        // exactly one replay).  This variant runs without the lane clock window: next to
        // stage C that is what pays (cfg 4 461 → 452 ms/step), while the joint replays
        // of cfg 3, the whole step there, keep it (270 vs 324 ms without).  Scheduling
        // only: every replay is independent.
        int u;
        {
            int first = 0;
            if (lane == 0) first = (int)atomicAdd(P.work + s, (unsigned)P.lpw);
            u = __shfl_sync(0xffffffffu, first, 0) + lane;
        }
        if (lane >= P.lpw || u >= QC) return;
        int q = u / P.n_clist;
        int c = P.clist[u - q * P.n_clist];
        long long r = ((long long)c * P.Q + q) * P.S + s;
        JReplay<DYN, TB, NG, CX> rp(P, T, X, W);
        rp.ws = ws;
        rp.accoff = accoff;
        if constexpr (NG == 64) {        // next-event / routing keys
            if (P.j_kglob) {             // lane-interleaved global scratch (frees shared memory)
                rp.tab.tn = (double*)(wbase + P.off_keys) + lane;
                rp.tab.kp = (int*)(wbase + P.off_keys + (size_t)NG * 32 * sizeof(double)) + lane;
                rp.tab.kd = rp.tab.kp + NG * 32;
                rp.tab.st = 32;
            } else {                     // shared memory
                rp.tab.tn = (double*)smem + tid;
                rp.tab.kp = (int*)(smem + (size_t)NG * TB * sizeof(double)) + tid;
                rp.tab.kd = rp.tab.kp + NG * TB;
                rp.tab.st = TB;
            }
        }
        rp.metk = P.sw.rep_met + r * kMaxSloSweep;
        rp.tte = tte;
        rp.tti = tti;
        rp.heads = (int*)(wbase + P.off_heads) + lane;
        rp.bits = (unsigned*)(wbase + P.off_bits) + lane;
        rp.RB = P.ring_slots;
        rp.RBm = P.ring_slots - 1;
        rp.ring = (unsigned long long*)(wbase + P.off_ring) + (size_t)lane * NG * P.ring_slots;
        rp.wts = DYN ? (double*)(wbase + P.off_wts) + (size_t)lane * P.Rmax : nullptr;
        rp.wtf = DYN ? (unsigned char*)(wbase + P.off_wtf) + (size_t)lane * P.Rmax : nullptr;
        rp.start(c, q, P.rec_ttft ? r * P.Rmax : -1);
        for (;;) {
            if (rp.completed >= rp.R) {
                const ReplayResult res = rp.result();
                P.rep_met[r] = res.met;
                P.rep_near[r] = res.near;
                P.rep_dur[r] = res.duration;
                P.rep_good[r] = res.goodput;
                P.rep_events[r] = res.events;
                P.sw.rep_watts[r] = res.watts;
                {
                    const double* acc = (const double*)(smem + accoff) + tid;
                    P.sw.rep_sq[r] = acc[0];
                    P.sw.rep_se[r] = acc[TB];
                }
                u = (int)atomicAdd(P.work + s, 1u);
                if (u >= QC) break;
                q = u / P.n_clist;
                c = P.clist[u - q * P.n_clist];
                r = ((long long)c * P.Q + q) * P.S + s;
                rp.metk = P.sw.rep_met + r * kMaxSloSweep;
                rp.start(c, q, P.rec_ttft ? r * P.Rmax : -1);
                continue;
            }
            rp.instant();
        }
    } else {
        for (;;) {
            int item = 0;
            if (lane == 0) item = (int)atomicAdd(P.work + s, 1u);
            item = __shfl_sync(0xffffffffu, item, 0);
            // an item is P.lpw replays: fewer than 32 lanes per warp when the whole
            // workload has too few replays to give every SM several warps
            if (item * P.lpw >= QC) break;
            const int u = item * P.lpw + lane;
            if (lane >= P.lpw || u >= QC) continue;
            const int q = u / P.n_clist;
            const int c = P.clist[u - q * P.n_clist];
            const long long r = ((long long)c * P.Q + q) * P.S + s;
            JReplay<DYN, TB, NG, CX> rp(P, T, X, W);
            rp.ws = ws;
            rp.accoff = accoff;
            if constexpr (NG == 64) {        // next-event / routing keys
                if (P.j_kglob) {             // lane-interleaved global scratch (frees shared memory)
                    rp.tab.tn = (double*)(wbase + P.off_keys) + lane;
                    rp.tab.kp = (int*)(wbase + P.off_keys + (size_t)NG * 32 * sizeof(double)) + lane;
                    rp.tab.kd = rp.tab.kp + NG * 32;
                    rp.tab.st = 32;
                } else {                     // shared memory
                    rp.tab.tn = (double*)smem + tid;
                    rp.tab.kp = (int*)(smem + (size_t)NG * TB * sizeof(double)) + tid;
                    rp.tab.kd = rp.tab.kp + NG * TB;
                    rp.tab.st = TB;
                }
            }
            rp.metk = P.sw.rep_met + r * kMaxSloSweep;
            rp.tte = tte;
            rp.tti = tti;
            rp.heads = (int*)(wbase + P.off_heads) + lane;
            rp.bits = (unsigned*)(wbase + P.off_bits) + lane;
            rp.RB = P.ring_slots;
            rp.RBm = P.ring_slots - 1;
            rp.ring = (unsigned long long*)(wbase + P.off_ring) + (size_t)lane * NG * P.ring_slots;
            rp.wts = DYN ? (double*)(wbase + P.off_wts) + (size_t)lane * P.Rmax : nullptr;
            rp.wtf = DYN ? (unsigned char*)(wbase + P.off_wtf) + (size_t)lane * P.Rmax : nullptr;
            const ReplayResult res = rp.run(c, q, P.rec_ttft ? r * P.Rmax : -1);
            P.rep_met[r] = res.met;
            P.rep_near[r] = res.near;
            P.rep_dur[r] = res.duration;
            P.rep_good[r] = res.goodput;
            P.rep_events[r] = res.events;
            P.sw.rep_watts[r] = res.watts;
            {
                const double* acc = (const double*)(smem + accoff) + tid;
                P.sw.rep_sq[r] = acc[0];
                P.sw.rep_se[r] = acc[TB];
            }
        }
    }
}

constexpr size_t joint_global_bytes_per_warp(int NG) {   // per-GPU SoA for NG = 64
    return NG == 8 ? 0 : (size_t)NG * 32 * (4 * sizeof(double) + 14 * sizeof(int) + 1);
}

}  // namespace padsim
