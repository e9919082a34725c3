// group_path.cuh — joint replay on lane groups (rows a4–a7, and a6 for dynamic
// candidates) for nodes of up to 8 simulated GPUs: one lane per simulated GPU,
// 8 lanes per replay, 4 replays per warp (north-star subsystem 2, SURVEY §7
// step 6: "event selection and routing by shuffle-min").
//
// Same semantics as dynamic_path.cuh's joint_kernel (DESIGN.md §3 c.2/c.3; the
// GPU parity tests compare both with the oracle bit for bit), different
// execution model:
//  * lane g of a group holds GPU g's state in registers (next event time,
//    prompt queue / pending joins, batch, segment, caps, flags);
//  * the next instant is a group min (redux.sync on the FP64 bit pattern: all
//    times are ≥ 0), the GPUs with an event at it a ballot, prefill / decode
//    routing a redux-min of the routing keys (derived from the GPU's state:
//    outstanding tokens, active + pending, INT_MAX when not eligible) + ballot;
//  * replay-level state (arrival cursor, KV buffer summary, metric windows,
//    controller, counters) is group-uniform: every lane of the group executes
//    the replay-level code, so the group stays converged; a handler reads GPU
//    g's fields with one shuffle and only lane g writes them;
//  * the per-GPU passes run lane-parallel: the dispatch pass (each touched GPU
//    dispatches its own batch / segment on its own lane), settle instants, the
//    Algorithm 1 guards and MovePower (ballots and group sums over the GPUs);
//  * the ≤ 32 in-flight KV transfers live in registers, 4 per lane; the
//    earliest (te, id) is a group min, not a scan through memory;
//  * no shared memory: occupancy is bounded by registers only.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "controller.cuh"
#include "replay.cuh"

namespace padsim {

constexpr int kGL = 8;                    // lanes per replay group (GPU slots, N ≤ 8)
constexpr int kGPW = 32 / kGL;            // replays per warp
constexpr int kGSlots = PADSIM_MAX_SLOTS / kGL;   // KV slots per lane
constexpr int kGIntMax = 0x7fffffff;

enum : int { GF_DRAIN = 1, GF_DIRTY = 2 };

template <bool DYN, bool CX>
struct GReplay {
    const Plan& P;
    const TraceView& T;
    // group geometry
    unsigned gm;        // lane mask of this group
    int gl, gb;         // lane in group (= GPU id), first lane of the group
    // per-replay scratch
    int* link;          // [i * kGPW]
    double* pe;         // [i * kGPW]
    unsigned long long* ring;   // [g][RB] sorted decode batch lists (fin << 32 | id)
    int RB, RBm;
    double* wts;        // TTFT window stamps
    unsigned char* wtf;
    double* tst;        // TPOT window stamps
    unsigned char* tfl;
    int* metk;
    // ---- this lane's GPU -------------------------------------------------
    double tn;          // next event time
    double tseg, L, dL; // P: batch start | D: segment start, step latency, growth
    long long sj;       // D: Σ join steps of the active members (A40)
    int a0;             // P: outstanding tokens | D: active count
    int qh, qt, ql;     // P: prompt FIFO | D: pending joins
    int b0, b1;         // P: batch head, size | D: last materialised step, next boundary
    int st0, mfin, eff, cmd, rse, cxs, bf, fl;
    double sv[kGSlots]; // KV transfer slots k = gl + 8j: end time, request id
    int si[kGSlots];
    // ---- replay level (group-uniform) ------------------------------------
    int N, R, max_db;
    double inv_lam;
    unsigned pmask, dmask;      // GPU role bits (group-relative)
    int tbusy, mk, mid, twh, twt, twl;
    double mte;
    int completed, met, near;
    double maxcomp;
    long long rec_base;
    double sq, se;              // Fig. 6 decomposition sums
    padsim_policy pol;
    int Bc;
    double tick_t, settle_t, flip_t, last_move;
    long long tick_k;
    int flip_g, drain_pending, phase2;
    int w_th, w_tlo, w_tle, w_tlt, w_ph, w_plo, w_ple0, w_plt0, w_ple1, w_plt1;
    double wh_t, wh_p;
    unsigned touched;
    int nk;
    long long w_sum;
    double w_acc, w_prev, a0t;
    bool gr;

    __device__ GReplay(const Plan& p, const TraceView& t) : P(p), T(t) {}

    // ---- group primitives --------------------------------------------------
    __device__ __forceinline__ unsigned gballot(bool p) const { return (__ballot_sync(gm, p) >> gb) & 0xffu; }
    __device__ __forceinline__ int gsum(int v) const { return (int)__reduce_add_sync(gm, (unsigned)v); }
    __device__ __forceinline__ unsigned gminu(unsigned v) const { return __reduce_min_sync(gm, v); }
    // min of non-negative doubles (or +inf): lexicographic min of the bit pattern
    __device__ __forceinline__ double gmin(double v) const {
        const unsigned long long b = (unsigned long long)__double_as_longlong(v);
        const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
        const unsigned mh = gminu(hi);
        const unsigned ml = gminu(hi == mh ? lo : 0xffffffffu);
        return __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    }
    template <class V> __device__ __forceinline__ V from(V v, int g) const { return __shfl_sync(gm, v, gb + g); }
    // lowest GPU id with the smallest key (keys ≥ 0; kGIntMax = not eligible)
    __device__ __forceinline__ int gargmin(int key) const {
        const unsigned m = gminu((unsigned)key);
        return __ffs(gballot((unsigned)key == m)) - 1;
    }

    __device__ __forceinline__ int& LNK(int i) { return link[(size_t)i * kGPW]; }
    __device__ __forceinline__ double& PE(int i) { return pe[(size_t)i * kGPW]; }
    __device__ __forceinline__ double arr(int i) const { return T.s_unit[i] * inv_lam; }
    __device__ __forceinline__ bool isP() const { return (pmask >> gl) & 1u; }
    __device__ __forceinline__ bool isD() const { return (dmask >> gl) & 1u; }
    // routing keys (A8 / A13): outstanding tokens / active + pending, INT_MAX when
    // the GPU is of the other role, draining or not simulated
    __device__ __forceinline__ int keyP() const { return (isP() && !(fl & GF_DRAIN)) ? a0 : kGIntMax; }
    __device__ __forceinline__ int keyD() const { return (isD() && !(fl & GF_DRAIN)) ? a0 + ql : kGIntMax; }

    // this lane's decode segment (A14 / A40)
    __device__ __forceinline__ double bnd(int s) const { return seg_bnd(tseg, L, gr ? dL : 0.0, s - st0, gr); }
    __device__ __forceinline__ int first_bnd_ge(double tau) const {
        return seg_first_ge(tseg, L, gr ? dL : 0.0, st0, b0, tau, gr);
    }

    // ---- KV transfer slots (registers) --------------------------------------
    __device__ __forceinline__ void slot_set(int k, double v, int id) {
        if (gl == (k & (kGL - 1))) {
            const int j = k / kGL;
#pragma unroll
            for (int z = 0; z < kGSlots; z++) { sv[z] = (z == j) ? v : sv[z]; si[z] = (z == j) ? id : si[z]; }
        }
    }
    __device__ __forceinline__ void slot_get(int k, double& v, int& id) const {
        const int j = k / kGL;
        double x = sv[0];
        int d = si[0];
#pragma unroll
        for (int z = 1; z < kGSlots; z++) { x = (z == j) ? sv[z] : x; d = (z == j) ? si[z] : d; }
        v = from(x, k & (kGL - 1));
        id = from(d, k & (kGL - 1));
    }
    // earliest (te, id) in flight → mte, mid, mk
    __device__ __forceinline__ void slot_min() {
        double bv = PAD_INF;
        int bi = kGIntMax, bk = 0;
#pragma unroll
        for (int z = 0; z < kGSlots; z++) {
            const int k = gl + kGL * z;
            if (k < tbusy && (sv[z] < bv || (sv[z] == bv && si[z] < bi))) { bv = sv[z]; bi = si[z]; bk = k; }
        }
        const double m = gmin(bv);
        const unsigned mi = gminu(bv == m ? (unsigned)bi : 0xffffffffu);
        const int owner = __ffs(gballot(bv == m && (unsigned)bi == mi)) - 1;
        mte = m;
        mid = (int)mi;
        mk = from(bk, owner);
    }

    __device__ void complete(int i, double t, double tpot) {
        completed++;
        const double pv = PE(i);
        const double ttft = pv - arr(i);
        const unsigned char ph = T.phase[i];
        const double ts = ph ? P.tpot_slo1 : P.tpot_slo0;
        met += (ttft <= P.ttft_slo && tpot <= ts) ? 1 : 0;
        near += (fabs(ttft - P.ttft_slo) <= 1e-9 * P.ttft_slo || fabs(tpot - ts) <= 1e-9 * ts) ? 1 : 0;
        maxcomp = fmax(maxcomp, t);
#pragma unroll 1
        for (int z = 0; z < nk; z++) {
            const double tz = ph ? P.sw.tpot1[z] : P.sw.tpot0[z];
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
            tst[w_ph] = t;
            tfl[w_ph] = f;
            w_ph++;
            w_ple0 += f & 1; w_plt0 += (f >> 1) & 1; w_ple1 += (f >> 2) & 1; w_plt1 += (f >> 3) & 1;
        }
        if (rec_base >= 0 && gl == 0) {
            P.rec_ttft[rec_base + i] = ttft;
            P.rec_tpot[rec_base + i] = tpot;
            P.rec_pe[rec_base + i] = pv;
            P.rec_comp[rec_base + i] = t;
        }
    }

    // A8: least outstanding non-draining prefill GPU, lowest id
    __device__ void route_prompt(int i) {
        const int best = gargmin(keyP());
        const int tin = T.in_tok[i];
        LNK(i) = kNoIdx;
        if (gl == best) {
            a0 += tin;
            if (ql == 0) qh = i; else LNK(qt) = i;
            qt = i;
            ql++;
        }
        touched |= 1u << best;
    }

    // A13/A14: fewest active+pending non-draining decode GPU, lowest id; joins at
    // the first step boundary at or after t
    __device__ void route_decode(int i, double t, unsigned bm_now) {
        const int best = gargmin(keyD());
        LNK(i) = kNoIdx;
        if (gl == best) {
            const int qn = ql;
            if (qn == 0) qh = i; else LNK(qt) = i;
            qt = i;
            ql = qn + 1;
            if (a0 > 0 && !((bm_now >> gl) & 1u) && a0 < max_db && qn == 0) {
                const int s = first_bnd_ge(t);
                if (s < b1) { b1 = s; tn = bnd(s); }
            }
        }
        touched |= 1u << best;
    }

    __device__ void batch_end(int g, double t) {
        int i = from(b0, g);
        const int n = from(b1, g);
        const double bstart = from(tseg, g);   // prefill GPUs keep the batch start here
        double bq = 0.0, be = 0.0;             // Fig. 6 decomposition, this batch
        int dec = 0;
        for (int z = 0; z < n; z++) {
            const int nx = LNK(i);
            PE(i) = t;
            dec += T.in_tok[i];
            const double ai = arr(i);
            bq = bq + (bstart - ai);
            be = be + (t - bstart);
            if (DYN && !pol.window_stamp) {    // A22: TTFT known at the first token
                const double ttft = t - ai;
                const unsigned char f = (ttft <= P.ttft_slo ? 1 : 0) | (ttft < P.ttft_slo ? 2 : 0);
                wts[w_th] = t;
                wtf[w_th] = f;
                w_th++;
                w_tle += f & 1;
                w_tlt += f >> 1;
            }
            if (tbusy < P.m.slots) {
                const double te = t + T.kv[i];
                slot_set(tbusy, te, i);
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
        sq = sq + bq;
        se = se + be;
        if (gl == g) { a0 -= dec; b1 = 0; tn = PAD_INF; }
    }

    // decode step boundary of GPU g; true when members left (composition changed)
    __device__ bool boundary(int g, double t) {
        const int s = from(b1, g);
        const int mf0 = from(mfin, g);
        if (gl == g) { b0 = s; tn = PAD_INF; }
        if (s != mf0) return false;
        const int n0 = from(a0, g);
        const unsigned long long* rg = ring + (size_t)g * RB;
        int f = from(bf, g);
        int left = 0, dcx = 0;
        long long dsj = 0;
        unsigned long long e = rg[f];
        for (;;) {
            const int id = (int)(unsigned)e;
            complete(id, t, (t - PE(id)) / (double)(T.out_tok[id] - 1));
            if (CX) dcx += T.in_tok[id];
            if (gr) dsj += s - (T.out_tok[id] - 1);      // its join step (A40)
            left++;
            f = (f + 1) & RBm;
            if (left == n0) break;
            e = rg[f];
            if ((int)(e >> 32) != s) break;
        }
        const int mf = left < n0 ? (int)(e >> 32) : kGIntMax;
        if (gl == g) {
            bf = f;
            a0 = n0 - left;
            mfin = mf;
            if (CX) cxs -= dcx;
            if (gr) sj -= dsj;
        }
        return true;
    }

    __device__ void transfer_end(double t, unsigned bm_now) {
        const int i = mid;
        tbusy--;
        if (mk != tbusy) {
            double v;
            int d;
            slot_get(tbusy, v, d);
            slot_set(mk, v, d);
        }
        if (twl > 0) {
            const int j = twh;
            twh = LNK(j);
            twl--;
            slot_set(tbusy, t + T.kv[j], j);
            tbusy++;
        }
        slot_min();
        if (rec_base >= 0 && gl == 0) P.rec_te[rec_base + i] = t;
        if (T.out_tok[i] == 1) complete(i, t, 0.0);
        else route_decode(i, t, bm_now);
    }

    // ---- dispatch pass: each touched GPU on its own lane ----------------------
    __device__ void dispatch_prefill(double t) {
        const int qn = ql;
        if (tn != PAD_INF || qn == 0) return;
        const int h = qh;
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
        b0 = h;
        b1 = b;
        tseg = t;
        ql = qn - b;
        if (qn > b) qh = LNK(j);
        tn = t + ((double)tok / P.m.den[b]) / P.m.spre[eff - P.m.min_w];
    }

    __device__ void dispatch_decode(double t, bool at_bnd, bool changed) {
        int n = a0;
        if (n > 0 && !at_bnd) {
            if (tn != t) return;          // mid-step
            b0 = b1;                      // join boundary exactly at t
            at_bnd = true;
        }
        int qn = ql;
        if (!at_bnd && qn == 0) return;
        const bool was_idle = !at_bnd;
        bool joined = false;
        const int step = b0;
        int mf = mfin;
        int h = qh;
        unsigned long long* rg = ring + (size_t)gl * RB;
        const int f = bf;
        while (n < max_db && qn > 0) {
            const int i = h;
            qn--;
            if (qn > 0) h = LNK(i);
            const int o = T.out_tok[i];
            const int fin = step + (o - 1);
            // insert (fin, i) into the sorted list of n members from the back
            const unsigned long long e = ((unsigned long long)(unsigned)fin << 32) | (unsigned)i;
            int z = n;
            while (z > 0) {
                const unsigned long long pv = rg[(f + z - 1) & RBm];
                if (pv < e) break;
                rg[(f + z) & RBm] = pv;
                z--;
            }
            rg[(f + z) & RBm] = e;
            n++;
            if (CX) cxs += T.in_tok[i];
            if (gr) sj += step;
            mf = fin < mf ? fin : mf;
            joined = true;
        }
        ql = qn;
        qh = h;
        a0 = n;
        if (n > 0) {
            if (was_idle || joined || changed || (fl & GF_DIRTY)) {
                tseg = t;
                st0 = step;
                const int ci = eff - P.m.min_w;
                if (!CX) {
                    L = P.m.ltab[(size_t)ci * max_db + (n - 1)];
                } else {          // A15 / A40 context of the segment's first step
                    double xv = P.m.dec_fixed + P.m.dec_per_seq * (double)n;
                    long long cc = cxs;
                    if (gr) cc += (long long)n * (step + 1) - sj;
                    xv = xv + P.m.dec_per_ctx * (double)cc;
                    L = xv / P.m.sdec[ci];
                    if (gr) dL = (P.m.dec_per_ctx * (double)n) / P.m.sdec[ci];
                }
                fl &= ~GF_DIRTY;
            }
            mfin = mf;
            b1 = mf;
            tn = bnd(mf);
        } else {
            mfin = kGIntMax;
            tn = PAD_INF;
        }
    }

    // ---- dynamic ---------------------------------------------------------
    __device__ void settle(double t) {
        if (gl < N) {           // every GPU on its own lane
            bool changed = false;
            int e = eff, c = cmd;
            const int r = rse;
            if (c < e) { e = c; changed = true; }
            if (r > 0) { e = c = r; rse = 0; changed = true; }
            eff = e;
            cmd = c;
            if (changed && isD()) {
                fl |= GF_DIRTY;
                if (a0 > 0) {
                    const int s = first_bnd_ge(t);
                    if (s < b1) { b1 = s; tn = bnd(s); }
                }
            }
        }
        settle_t = PAD_INF;
        if (t > a0t) {
            w_acc = w_acc + (double)w_sum * (t - w_prev);
            w_prev = t;
        }
        w_sum = gsum(gl < N ? eff : 0);
    }

    __device__ void flip() {
        const int g = flip_g;
        pmask ^= 1u << g;
        dmask ^= 1u << g;
        if (gl == g) {
            fl = 0; a0 = 0; ql = 0; b0 = 0; b1 = 0; st0 = 0;
            mfin = kGIntMax; cxs = 0; sj = 0; bf = 0;
            tn = PAD_INF;
        }
        drain_pending = 0;
        flip_g = -1;
        flip_t = PAD_INF;
    }

    // Algorithm 1 decision (controller.cuh ctl_step, same rules) with the per-GPU
    // loops as ballots / group sums; newcap = this lane's target
    __device__ int decide(double now, const CtlSignals& sg, int& newcap, int& gsel) const {
        gsel = -1;
        if (pol.kind == 0) return ACT_NONE;                      // static never acts
        if (!((now - last_move) > pol.cooldown_s)) return ACT_NONE;
        int dir;
        if (sg.ttft_gt && sg.q_prefill > pol.queue_threshold && sg.tpot_lt) dir = 0;
        else if (sg.tpot_gt && sg.ttft_lt) dir = 1;
        else return ACT_NONE;
        const int min_w = P.m.min_w;
        const int ceil_to = dir == 0 ? P.m.max_w : pol.decode_ceiling_w;
        const bool live = gl < N && !(fl & GF_DRAIN);
        const bool don = live && (dir == 0 ? isD() : isP());
        const bool rec = live && (dir == 0 ? isP() : isD());
        const int c = rse > 0 ? rse : cmd;
        const int n_don = __popc(gballot(don)), n_rec = __popc(gballot(rec));
        const bool rec_ceil = gballot(rec && c < ceil_to) == 0u;
        const bool don_floor = gballot(don && c > min_w) == 0u;
        const bool limits = rec_ceil || don_floor;
        const bool power_ok = pol.kind == 1 || pol.kind == 3;
        const bool gpu_ok = pol.kind == 2 || pol.kind == 3;
        if (power_ok && !limits) {
            // MovePower: donors −min(step, cap−floor), F = Σ, recipients
            // +min(⌊F/|rec|⌋, ceiling−cap), leftover unallocated
            newcap = c;
            int r = 0;
            if (don) {
                r = c - min_w;
                r = r < pol.power_step_w ? r : pol.power_step_w;
                r = r > 0 ? r : 0;
                newcap = c - r;
            }
            const long long F = gsum(r);
            const long long share = n_rec > 0 ? F / n_rec : 0;
            if (rec) {
                long long r2 = (long long)ceil_to - c;
                r2 = share < r2 ? share : r2;
                r2 = r2 > 0 ? r2 : 0;
                newcap = c + (int)r2;
            }
            return ACT_MOVE_POWER;
        }
        if (gpu_ok && n_don >= 2 && !drain_pending) {
            // MoveGPU: least outstanding work, lowest id; then uniform caps
            gsel = gargmin(don ? a0 + (isP() ? 0 : ql) : kGIntMax);
            int u = Bc / N;                                        // DistributeUniformPower
            u = u < min_w ? min_w : u;
            u = u > P.m.max_w ? P.m.max_w : u;
            newcap = u;
            return ACT_MOVE_GPU;
        }
        return ACT_SATURATED;
    }

    // returns 0: cooldown not elapsed, 1: evaluated, no move, 2: a move was made
    __device__ int tick(double t, unsigned bm_now) {
        int acted = 0;
        if ((t - last_move) > pol.cooldown_s) {
            acted = 1;
            const double lo = t - pol.window_s;
            // expire samples older than the window from both FIFOs in one walk
            for (;;) {
                const bool ct = w_tlo < w_th, cp = w_plo < w_ph;
                const double a = ct ? wts[w_tlo] : PAD_INF;
                const double b = cp ? tst[w_plo] : PAD_INF;
                const unsigned char fa = ct ? wtf[w_tlo] : 0;
                const unsigned char fb = cp ? tfl[w_plo] : 0;
                const bool pa = a < lo, pb = b < lo;
                if (!pa && !pb) { wh_t = a; wh_p = b; break; }
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
            sg.q_prefill = gsum(isP() ? ql : 0);
            int newcap = 0, gsel;
            const int act = decide(t, sg, newcap, gsel);
            if (act == ACT_MOVE_POWER || act == ACT_MOVE_GPU) {
                last_move = t;
                if (act == ACT_MOVE_GPU) {
                    const int g = gsel;
                    int i = from(qh, g);
                    const int n = from(ql, g);
                    const bool wasP = (pmask >> g) & 1u;
                    if (gl == g) { fl |= GF_DRAIN; ql = 0; }
                    drain_pending = 1;
                    flip_g = g;
                    if (wasP) {
                        for (int z = 0; z < n; z++) {
                            const int nx = LNK(i);
                            const int tin = T.in_tok[i];
                            if (gl == g) a0 -= tin;
                            route_prompt(i);
                            i = nx;
                        }
                    } else {
                        for (int z = 0; z < n; z++) {
                            const int nx = LNK(i);
                            route_decode(i, t, bm_now);
                            i = nx;
                        }
                    }
                }
                if (gl < N) {
                    if (newcap < cmd) cmd = newcap;
                    else if (newcap > cmd) rse = newcap;
                }
                settle_t = t + pol.settle_s;
                acted = 2;
            }
        }
        tick_k++;
        tick_t = (double)tick_k * pol.tick_s;
        return acted;
    }

    __device__ long long tick_at_or_after(double x, long long k0) const {
        if (!(x < PAD_INF)) return 0x7fffffffffffffffLL;
        long long k = (long long)ceil(x / pol.tick_s);
        if (k < k0) k = k0;
        while ((double)k * pol.tick_s < x) k++;
        while (k - 1 >= k0 && (double)(k - 1) * pol.tick_s >= x) k--;
        return k;
    }
    __device__ long long expiry_tick(double stamp, long long k0) const {
        long long k = (long long)floor((stamp + pol.window_s) / pol.tick_s);
        if (k < k0) k = k0;
        while (!(stamp < (double)k * pol.tick_s - pol.window_s)) k++;
        while (k - 1 >= k0 && stamp < (double)(k - 1) * pol.tick_s - pol.window_s) k--;
        return k;
    }
    __device__ long long cooldown_tick(long long k0) const {
        long long k = (long long)floor((last_move + pol.cooldown_s) / pol.tick_s);
        if (k < k0) k = k0;
        while (!(((double)k * pol.tick_s - last_move) > pol.cooldown_s)) k++;
        while (k - 1 >= k0 && ((double)(k - 1) * pol.tick_s - last_move) > pol.cooldown_s) k--;
        return k;
    }
    // exact tick skipping (as joint_kernel)
    __device__ void skip_ticks(int outcome, double next_event) {
        const long long k0 = tick_k;
        long long k;
        if (outcome == 0) {
            k = cooldown_tick(k0);
        } else {
            k = tick_at_or_after(next_event, k0);
            if (w_tlo < w_th) k = min(k, expiry_tick(wh_t, k0));
            if (w_plo < w_ph) k = min(k, expiry_tick(wh_p, k0));
        }
        if (k > k0 && k != 0x7fffffffffffffffLL) {
            tick_k = k;
            tick_t = (double)tick_k * pol.tick_s;
        }
    }

    __device__ ReplayResult run(int c, int q, long long rec) {
        N = P.N;
        R = T.R;
        max_db = P.m.max_db;
        inv_lam = 1.0 / (P.qps[q] * (double)N);
        rec_base = rec;
        {
            const bool on = gl < N;
            const int r = on ? P.role[(size_t)c * N + gl] : 2;
            pmask = gballot(r == 0);
            dmask = gballot(r == 1);
            tn = PAD_INF;
            tseg = 0.0; L = 1.0; sj = 0; dL = 0.0;
            a0 = 0; qh = kNoIdx; qt = kNoIdx; ql = 0;
            b0 = 0; b1 = 0; st0 = 0; mfin = kGIntMax;
            eff = cmd = on ? P.cap[(size_t)c * N + gl] : P.m.min_w;
            rse = 0; cxs = 0; fl = 0; bf = 0;
#pragma unroll
            for (int z = 0; z < kGSlots; z++) { sv[z] = PAD_INF; si[z] = kGIntMax; }
        }
        tbusy = 0; mk = 0; mid = 0; twh = twt = kNoIdx; twl = 0;
        mte = PAD_INF;
        completed = 0; met = 0; near = 0;
        maxcomp = -PAD_INF;
        sq = se = 0.0;
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
        if (gl == 0) {
#pragma unroll 1
            for (int z = 0; z < nk; z++) metk[z] = 0;
        }
        __syncwarp(gm);
        gr = CX && P.m.ctx_growth != 0 && P.m.dec_per_ctx != 0.0;
        w_sum = P.sw.capsum[c];
        a0t = R > 0 ? arr(0) : 0.0;
        w_acc = 0.0;
        w_prev = a0t;
        long long events = 0;
        int na = 0;
        double ta = R > 0 ? arr(0) : PAD_INF;
        // lane clock window (scheduling only, results independent): the groups
        // of a warp stay within sync_win mean inter-arrival times of each other
        const float win = P.sync_win > 0.f ? (float)((double)P.sync_win * inv_lam) : 0.f;
        while (completed < R) {
            double t = gmin(tn);
            t = ta < t ? ta : t;
            t = mte < t ? mte : t;
            if (DYN) {
                t = tick_t < t ? tick_t : t;
                t = settle_t < t ? settle_t : t;
                t = flip_t < t ? flip_t : t;
            }
            if (win > 0.f) {
                const float tf = (float)t;
                const unsigned mn = __reduce_min_sync(__activemask(), __float_as_uint(tf));
                if (tf > __uint_as_float(mn) + win) continue;
            }
            events++;
            touched = 0;
            if (DYN) {
                if (settle_t == t) settle(t);
                if (flip_t == t) flip();
            }
            const unsigned bm = gballot(tn == t);
            const unsigned bp = bm & pmask, bd = bm & dmask;
            for (unsigned m = bp; m; m &= m - 1) batch_end(__ffs(m) - 1, t);
            unsigned chg = 0;
            for (unsigned m = bd; m; m &= m - 1) {
                const int g = __ffs(m) - 1;
                if (boundary(g, t)) chg |= 1u << g;
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
            if (((bm | touched) >> gl) & 1u) {
                if (isP()) dispatch_prefill(t);
                else dispatch_decode(t, (bd >> gl) & 1u, (chg >> gl) & 1u);
            }
            __syncwarp(gm);
            if (DYN && flip_g >= 0 && flip_t == PAD_INF) {
                const bool e = isP() ? (tn == PAD_INF && ql == 0) : (a0 == 0 && ql == 0);
                if ((gballot(e) >> flip_g) & 1u) flip_t = t + pol.reassign_s;
            }
            if (DYN && tick_outcome < 2) {
                double ne = ta < mte ? ta : mte;
                ne = settle_t < ne ? settle_t : ne;
                ne = flip_t < ne ? flip_t : ne;
                const double tm = gmin(tn);
                skip_ticks(tick_outcome, tm < ne ? tm : ne);
            }
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

// per-warp scratch of the group kernel: link / pe interleaved over the warp's 4
// replays ([i * 4 + replay]), per-replay contiguous window FIFOs and batch lists
struct GScratch {
    size_t link, pe, wts, wtf, tst, tfl, ring, bytes;
};
__host__ __device__ inline GScratch gscratch_layout(size_t R, int RB, bool dyn) {
    GScratch g{};
    size_t off = 0;
    auto take = [&](size_t b) { const size_t o = off; off += (b + 255) & ~(size_t)255; return o; };
    g.link = take(R * kGPW * sizeof(int));
    g.pe = take(R * kGPW * sizeof(double));
    if (dyn) {
        g.wts = take(R * kGPW * sizeof(double));
        g.wtf = take(R * kGPW);
        g.tst = take(R * kGPW * sizeof(double));
        g.tfl = take(R * kGPW);
    }
    g.ring = take((size_t)kGPW * kGL * RB * sizeof(unsigned long long));
    g.bytes = off;
    return g;
}

// CTAs bound to one trace (s = blockIdx.x mod S); warps pull items of 4 replays
// (one per lane group) from that trace's counter.
template <bool DYN, bool CX, int TB>
__global__ void __launch_bounds__(TB) jointg_kernel(const __grid_constant__ Plan P) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rg = lane / kGL;
    char* wbase = P.scratch + ((size_t)blockIdx.x * (TB / 32) + warp) * P.warp_bytes;
    const GScratch L = gscratch_layout((size_t)(P.Rmax > 0 ? P.Rmax : 1), P.ring_slots, DYN);
    const int s = blockIdx.x % P.S;
    const long long off = P.toff[s];
    TraceView T;
    T.R = P.nreq[s];
    T.s_unit = P.s_unit + off; T.kv = P.kv + off; T.in_tok = P.in_tok + off;
    T.out_tok = P.out_tok + off; T.phase = P.phase + off;
    const int QC = P.Q * P.n_clist;
    const size_t Rm = (size_t)P.Rmax;
    for (;;) {
        int item = 0;
        if (lane == 0) item = (int)atomicAdd(P.work + s, 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if ((long long)item * kGPW >= QC) break;
        const int u = item * kGPW + rg;
        if (u >= QC) continue;
        const int q = u / P.n_clist;
        const int c = P.clist[u - q * P.n_clist];
        const long long r = ((long long)c * P.Q + q) * P.S + s;
        GReplay<DYN, CX> rp(P, T);
        rp.gl = lane & (kGL - 1);
        rp.gb = rg * kGL;
        rp.gm = 0xffu << rp.gb;
        rp.link = (int*)(wbase + L.link) + rg;
        rp.pe = (double*)(wbase + L.pe) + rg;
        rp.ring = (unsigned long long*)(wbase + L.ring) + (size_t)rg * kGL * P.ring_slots;
        rp.RB = P.ring_slots;
        rp.RBm = P.ring_slots - 1;
        if (DYN) {
            rp.wts = (double*)(wbase + L.wts) + rg * Rm;
            rp.wtf = (unsigned char*)(wbase + L.wtf) + rg * Rm;
            rp.tst = (double*)(wbase + L.tst) + rg * Rm;
            rp.tfl = (unsigned char*)(wbase + L.tfl) + rg * Rm;
        }
        rp.metk = P.sw.rep_met + r * kMaxSloSweep;
        const ReplayResult res = rp.run(c, q, P.rec_ttft ? r * P.Rmax : -1);
        if (rp.gl == 0) {
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
}

}  // namespace padsim
