// coalesced.cuh — the paper's non-disaggregated baseline: every GPU serves both
// phases with chunked prefill ("vLLM in coalesced mode ... generated using
// chunked prefill"; SPEC coalesced_step S:262–269).  SURVEY §8(f) row 3.
//
// Semantics (readings A33–A37): roles ignored, no KV transfer;
// arrivals to the GPU with the least outstanding prompt tokens (lowest id);
// one engine step = ≤ chunk tokens of the head prompt fused with every active
// decode sequence, lat = prefill_lat(c,1,w) + decode_lat(n,C,w); the last
// chunk's step end is the first token, the request then joins the GPU's decode
// batch (pending FIFO when full) for out−1 more steps; runs of decode-only
// steps are constant-composition segments with boundary k at t_seg + (double)k·L.
//
// One thread = one replay (candidate × QPS × trace).  Decode-only runs are
// skipped ahead exactly: a segment is materialised only at its next leave
// (minimum finish step) or, when a prompt arrives, at the first boundary ≥ the
// arrival — nothing can change at the boundaries in between.  Per-GPU state is
// a lane-interleaved SoA in global scratch (stride 32); N ≤ 64.
#pragma once
#include "replay.cuh"

namespace padsim {

enum : int { CF_INSTEP = 1, CF_SEGOK = 2, CF_COMPCHG = 4, CF_BOUNDARY = 8 };

template <bool CTX>
struct CoalReplay {
    const Plan& P;
    TraceView T;
    int N, R, max_db;
    double inv_lam;
    // per-GPU SoA, element g at [g * 32]
    double *tn, *tseg, *L, *hps, *dL;
    long long *outst, *ctx, *sj;     // sj: Σ join steps of the decode members (A40)
    int *qh, *qt, *ql, *ph, *pt, *pl, *done, *nact, *step, *st0, *ts, *mfin, *cid, *ctok, *fl;
    int* act_id;    // [(g * max_db + k) * 32]
    int* act_fin;
    int* link;      // [i * 32]
    double* pe;     // [i * 32]
    int* metk;
    int nk;
    long long rec_base;
    int completed, met, near;
    double maxcomp, sq, se;
    bool gr;                         // A40 context growth

    __device__ CoalReplay(const Plan& p) : P(p) {}

    __device__ __forceinline__ double arr(int i) const { return T.s_unit[i] * inv_lam; }
    __device__ __forceinline__ int& LNK(int i) { return link[(size_t)i * 32]; }
    __device__ __forceinline__ double& PE(int i) { return pe[(size_t)i * 32]; }

    __device__ double dec_lat(int n, long long cx, int cap) const {
        const int ci = cap - P.m.min_w;
        if (!CTX) return P.m.ltab[(size_t)ci * max_db + (n - 1)];
        double xv = P.m.dec_fixed + P.m.dec_per_seq * (double)n;
        xv = xv + P.m.dec_per_ctx * (double)cx;
        return xv / P.m.sdec[ci];
    }

    __device__ void complete(int i, double t, double tpot) {
        completed++;
        const double pei = PE(i);
        const double ttft = pei - arr(i);
        const double tslo = T.phase[i] ? P.tpot_slo1 : P.tpot_slo0;
        met += (ttft <= P.ttft_slo && tpot <= tslo) ? 1 : 0;
        near += (fabs(ttft - P.ttft_slo) <= 1e-9 * P.ttft_slo || fabs(tpot - tslo) <= 1e-9 * tslo) ? 1 : 0;
        maxcomp = fmax(maxcomp, t);
        for (int z = 0; z < nk; z++) {
            const double tz = T.phase[i] ? P.sw.tpot1[z] : P.sw.tpot0[z];
            if (ttft <= P.sw.ttft[z] && tpot <= tz) metk[z]++;
        }
        if (rec_base >= 0) {
            P.rec_ttft[rec_base + i] = ttft;
            P.rec_tpot[rec_base + i] = tpot;
            P.rec_pe[rec_base + i] = pei;
            P.rec_comp[rec_base + i] = t;
            P.rec_te[rec_base + i] = pei;          // A33: no KV transfer
        }
    }

    // boundary k of the current decode-only segment (A37; A40 with growth)
    __device__ __forceinline__ double bnd(int o, int k) const {
        return seg_bnd(tseg[o], L[o], dL[o], k - st0[o], gr);
    }

    // first boundary index > step whose time is ≥ tau (boundaries are monotone in k)
    __device__ int first_bnd_ge(int o, double tau) const {
        return seg_first_ge(tseg[o], L[o], dL[o], st0[o], step[o], tau, gr);
    }

    // decode context of the step after boundary `sn` (A15; A40 with growth)
    __device__ __forceinline__ long long step_ctx(int o, int n, int sn) const {
        return gr ? ctx[o] + (long long)n * (sn + 1) - sj[o] : ctx[o];
    }

    __device__ void step_end(int g, double t) {
        const int o = g * 32;
        const int sn = ts[o];
        step[o] = sn;
        int f = fl[o];
        int n = nact[o];
        if (n > 0 && mfin[o] == sn) {      // sequences emitting their last token
            int mf = kIntMaxC;
            long long cx = ctx[o];
            int k = 0;
            while (k < n) {
                const size_t ak = ((size_t)o * max_db) + (size_t)k * 32;
                const int fin = act_fin[ak];
                if (fin == sn) {
                    const int i = act_id[ak];
                    complete(i, t, (t - PE(i)) / (double)(T.out_tok[i] - 1));
                    cx -= T.in_tok[i];
                    sj[o] -= sn - (T.out_tok[i] - 1);   // its join step
                    const size_t al = ((size_t)o * max_db) + (size_t)(n - 1) * 32;
                    act_id[ak] = act_id[al];
                    act_fin[ak] = act_fin[al];
                    n--;
                } else {
                    mf = fin < mf ? fin : mf;
                    k++;
                }
            }
            nact[o] = n;
            ctx[o] = cx;
            mfin[o] = mf;
            f |= CF_COMPCHG;
        }
        const int i = cid[o];
        if (i >= 0) {                       // the step's prefill chunk (A35/A36)
            const int d = done[o] + ctok[o];
            outst[o] -= ctok[o];
            if (d == T.in_tok[i]) {
                const int nx = LNK(i);
                qh[o] = nx;
                if (--ql[o] == 0) qt[o] = kNoIdx;
                done[o] = 0;
                PE(i) = t;
                se = se + (t - hps[o]);
                if (T.out_tok[i] == 1) {
                    complete(i, t, 0.0);
                } else {                    // pending join FIFO of this GPU
                    LNK(i) = kNoIdx;
                    if (pl[o] == 0) ph[o] = i; else LNK(pt[o]) = i;
                    pt[o] = i;
                    pl[o]++;
                }
            } else {
                done[o] = d;
            }
            cid[o] = kNoIdx;
        }
        fl[o] = (f & ~CF_INSTEP) | CF_BOUNDARY;
        tn[o] = PAD_INF;
    }

    // A34: least outstanding prompt tokens, lowest id; returns true if the GPU is idle
    __device__ bool route(int i, double t, int& gsel) {
        int best = 0;
        long long bl = outst[0];
        for (int g = 1; g < N; g++) {
            const long long v = outst[g * 32];
            if (v < bl) { bl = v; best = g; }
        }
        gsel = best;
        const int o = best * 32;
        outst[o] = bl + T.in_tok[i];
        LNK(i) = kNoIdx;
        const int qn = ql[o];
        if (qn == 0) qh[o] = i; else LNK(qt[o]) = i;
        qt[o] = i;
        ql[o] = qn + 1;
        const int f = fl[o];
        if (!(f & CF_INSTEP)) return true;
        if (qn == 0 && cid[o] < 0) {        // decode-only run: cut at the first boundary ≥ t
            const int s = first_bnd_ge(o, t);
            if (s < ts[o]) {
                ts[o] = s;
                tn[o] = bnd(o, s);
            }
        }
        return false;
    }

    __device__ void dispatch(int g, double t) {
        const int o = g * 32;
        int f = fl[o];
        const bool was_idle = !(f & CF_BOUNDARY);
        bool joined = false;
        int n = nact[o];
        int mf = mfin[o];
        const int sn = step[o];
        while (n < max_db && pl[o] > 0) {
            const int i = ph[o];
            ph[o] = LNK(i);
            pl[o]--;
            const size_t ak = ((size_t)o * max_db) + (size_t)n * 32;
            const int fin = sn + (T.out_tok[i] - 1);
            act_id[ak] = i;
            act_fin[ak] = fin;
            n++;
            ctx[o] += T.in_tok[i];
            sj[o] += sn;
            mf = fin < mf ? fin : mf;
            joined = true;
        }
        nact[o] = n;
        mfin[o] = mf;
        const int cap = P.cap[(size_t)cand * N + g];
        if (ql[o] > 0) {
            const int i = qh[o];
            const int dn = done[o];
            int c = T.in_tok[i] - dn;
            c = c > P.m.chunk ? P.m.chunk : c;
            if (dn == 0) {
                hps[o] = t;
                sq = sq + (t - arr(i));
            }
            double lat = ((double)c / P.m.den[1]) / P.m.spre[cap - P.m.min_w];
            if (n > 0) lat = lat + dec_lat(n, step_ctx(o, n, sn), cap);
            tn[o] = t + lat;
            ts[o] = sn + 1;
            cid[o] = i;
            ctok[o] = c;
            f = (f | CF_INSTEP) & ~CF_SEGOK;
        } else if (n > 0) {
            if (was_idle || joined || (f & CF_COMPCHG) || !(f & CF_SEGOK)) {
                tseg[o] = t;
                st0[o] = sn;
                L[o] = dec_lat(n, step_ctx(o, n, sn), cap);
                dL[o] = gr ? (P.m.dec_per_ctx * (double)n) / P.m.sdec[cap - P.m.min_w] : 0.0;
                f |= CF_SEGOK;
            }
            ts[o] = mf;                     // next leave; nothing changes before it
            tn[o] = bnd(o, mf);
            f |= CF_INSTEP;
        }
        fl[o] = f & ~(CF_BOUNDARY | CF_COMPCHG);
    }

    static constexpr int kIntMaxC = 0x7fffffff;
    int cand;

    __device__ ReplayResult run(int c, int q) {
        cand = c;
        inv_lam = 1.0 / (P.qps[q] * (double)N);
        for (int g = 0; g < N; g++) {
            const int o = g * 32;
            tn[o] = PAD_INF; tseg[o] = 0.0; L[o] = 1.0; hps[o] = 0.0; dL[o] = 0.0;
            outst[o] = 0; ctx[o] = 0; sj[o] = 0;
            qh[o] = kNoIdx; qt[o] = kNoIdx; ql[o] = 0; ph[o] = kNoIdx; pt[o] = kNoIdx; pl[o] = 0;
            done[o] = 0; nact[o] = 0; step[o] = 0; st0[o] = 0; ts[o] = 0; mfin[o] = kIntMaxC;
            cid[o] = kNoIdx; ctok[o] = 0; fl[o] = 0;
        }
        for (int z = 0; z < nk; z++) metk[z] = 0;
        gr = CTX && P.m.ctx_growth != 0;
        completed = 0; met = 0; near = 0;
        maxcomp = -PAD_INF;
        sq = 0.0; se = 0.0;
        long long events = 0;
        int k = 0;
        double ta = R > 0 ? arr(0) : PAD_INF;
        while (completed < R) {
            double t = ta;
            for (int g = 0; g < N; g++) {
                const double v = tn[g * 32];
                t = v < t ? v : t;
            }
            events++;
            unsigned long long disp = 0ull;
            for (int g = 0; g < N; g++) {       // step ends, worker order (A10)
                if (tn[g * 32] == t) {
                    step_end(g, t);
                    disp |= 1ull << g;
                }
            }
            while (ta == t) {                    // arrivals, id order
                int gs;
                if (route(k, t, gs)) disp |= 1ull << gs;
                k++;
                ta = k < R ? arr(k) : PAD_INF;
            }
            for (unsigned long long m = disp; m; m &= m - 1) dispatch(__ffsll((long long)m) - 1, t);
        }
        ReplayResult res;
        res.met = met;
        res.near = near;
        res.duration = R > 0 ? maxcomp - arr(0) : 0.0;
        res.goodput = res.duration > 0 ? (double)met / res.duration : 0.0;
        res.events = events;
        res.watts = (double)P.sw.capsum[c];
        return res;
    }
};

// One warp per CTA; warps stride over 32-replay items (s, q, candidate list).
template <bool CTX>
__global__ void __launch_bounds__(32) coalesced_kernel(const __grid_constant__ Plan P) {
    const int lane = threadIdx.x;
    char* wb = P.scratch + (size_t)blockIdx.x * P.warp_bytes;
    const long long QC = (long long)P.Q * P.n_clist;
    const long long U = QC * P.S;
    for (long long base = (long long)blockIdx.x * 32; base < U; base += (long long)gridDim.x * 32) {
        const long long u = base + lane;
        if (u >= U) continue;
        const int s = (int)(u / QC);
        const long long rem = u - (long long)s * QC;
        const int q = (int)(rem / P.n_clist);
        const int c = P.clist[rem - (long long)q * P.n_clist];
        const long long r = ((long long)c * P.Q + q) * P.S + s;
        CoalReplay<CTX> rp(P);
        rp.N = P.N;
        rp.max_db = P.m.max_db;
        const long long off = P.toff[s];
        rp.R = P.nreq[s];
        rp.T.R = rp.R;
        rp.T.s_unit = P.s_unit + off; rp.T.kv = P.kv + off; rp.T.in_tok = P.in_tok + off;
        rp.T.out_tok = P.out_tok + off; rp.T.phase = P.phase + off;
        const int n = P.N * 32;
        char* p = wb + P.off_jw;
        rp.tn = (double*)p + lane; p += n * sizeof(double);
        rp.tseg = (double*)p + lane; p += n * sizeof(double);
        rp.L = (double*)p + lane; p += n * sizeof(double);
        rp.hps = (double*)p + lane; p += n * sizeof(double);
        rp.dL = (double*)p + lane; p += n * sizeof(double);
        rp.outst = (long long*)p + lane; p += n * sizeof(long long);
        rp.ctx = (long long*)p + lane; p += n * sizeof(long long);
        rp.sj = (long long*)p + lane; p += n * sizeof(long long);
        int* ib = (int*)p;
        int** fields[] = {&rp.qh, &rp.qt, &rp.ql, &rp.ph, &rp.pt, &rp.pl, &rp.done, &rp.nact,
                          &rp.step, &rp.st0, &rp.ts, &rp.mfin, &rp.cid, &rp.ctok, &rp.fl};
#pragma unroll
        for (int z = 0; z < 15; z++) *fields[z] = ib + (size_t)z * n + lane;
        rp.act_id = (int*)(wb + P.off_heads) + lane;
        rp.act_fin = (int*)(wb + P.off_bits) + lane;
        rp.link = (int*)(wb + P.off_link) + lane;
        rp.pe = (double*)(wb + P.off_pe) + lane;
        rp.metk = P.sw.rep_met + r * kMaxSloSweep;
        rp.nk = P.sw.n;
        rp.rec_base = P.rec_ttft ? r * P.Rmax : -1;
        const ReplayResult res = rp.run(c, q);
        P.rep_met[r] = res.met;
        P.rep_near[r] = res.near;
        P.rep_dur[r] = res.duration;
        P.rep_good[r] = res.goodput;
        P.rep_events[r] = res.events;
        P.sw.rep_watts[r] = res.watts;
        P.sw.rep_sq[r] = rp.sq;
        P.sw.rep_se[r] = rp.se;
    }
}

__host__ __device__ constexpr size_t coal_worker_bytes(int N) {
    return (size_t)N * 32 * (5 * sizeof(double) + 3 * sizeof(long long) + 15 * sizeof(int));
}

}  // namespace padsim
