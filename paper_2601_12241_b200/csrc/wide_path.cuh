// wide_path.cuh — the factorized static replay (rows a4 + a5) for wide nodes
// (8 < N ≤ 64 simulated GPUs: cfg 5's 64-GPU, 38.4 kW node; P:98, P:285,
// P:496 "rack scale"), one warp per replay.
//
// Same factorization as static_path.cuh (why it is exact: see there): stage A
// replays the prefill pool + KV buffer of each prefill group (caps of the
// prefill GPUs in P-id order) once per (QPS, trace) and writes the
// transfer-end stream; stage C replays the decode pool of every candidate of
// the group from that stream.  What changes with N: up to 63 workers per
// role do not fit per-thread register arrays, so a replay is one warp —
// lane l owns workers l and l + 32 (state in registers), the next event is a
// warp min (redux.sync on the FP64 bit pattern, all times are ≥ 0), the
// workers with an event at it a ballot, routing a warp argmin of the routing
// keys + ballot (lowest id); replay-level state (arrival / stream cursor, KV
// buffer summary, counters) is warp-uniform, and every handler runs with the
// warp converged, so all collectives take their full-mask fast path.  The
// ≤ 32 KV transfer slots of stage A are one per lane.  Per-worker passes run
// lane-parallel: the dispatch pass (each touched worker forms its batch /
// segment on its own lane).  Queues (prompt FIFOs, KV-wait FIFO, pending
// joins) are linked through a per-replay `link` array; a decode batch is an
// unsorted per-worker array of (finish step, stream index) entries: a join
// appends (one store), a leave scans the array lane-parallel (one coalesced
// load per 32 members), scores the leavers and compacts the rest, and the next
// finish step is a warp min — no sorted insertion, no dependent load chain.
// Same semantics and operation order as the oracle (DESIGN.md §3 c.2).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "replay.cuh"
#include "static_path.cuh"

namespace padsim {

constexpr int kWMax = 64;                  // worker slots (2 per lane)
// resident CTAs per SM the compiler targets (register budget): stage C 8 → 64
// registers, 32 warps per SM (cfg 5: 23.5 → 22.0 s/step against the default 96
// registers / 20 warps; a replay per warp is latency-bound, more warps hide more;
// 10 → 48 registers spills 200 B: 24.3 s); stage A 6 → 80 registers (21.96 s vs
// 22.0-22.5 s at 64 / 130 registers)
#ifndef PADSIM_WIDE_MINB
#define PADSIM_WIDE_MINB 8
#endif
#ifndef PADSIM_WIDEA_MINB
#define PADSIM_WIDEA_MINB 6
#endif
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned long long w_min_u64(unsigned long long v) {
    const unsigned hi = (unsigned)(v >> 32), lo = (unsigned)v;
    const unsigned mh = __reduce_min_sync(kFull, hi);
    const unsigned ml = __reduce_min_sync(kFull, hi == mh ? lo : 0xffffffffu);
    return ((unsigned long long)mh << 32) | ml;
}
// min of non-negative doubles (or +inf) over the warp
__device__ __forceinline__ double w_min_d(double v) {
    return __longlong_as_double((long long)w_min_u64((unsigned long long)__double_as_longlong(v)));
}
// 64-bit mask of the workers (slot 0 = ids 0..31, slot 1 = ids 32..63) with p
__device__ __forceinline__ unsigned long long w_ballot2(bool p0, bool p1) {
    return (unsigned long long)__ballot_sync(kFull, p0) | ((unsigned long long)__ballot_sync(kFull, p1) << 32);
}
// lowest worker id whose key equals the warp minimum (keys ≥ 0, ~0 = ineligible)
__device__ __forceinline__ int w_argmin(unsigned long long k0, unsigned long long k1) {
    const unsigned long long m = w_min_u64(k0 < k1 ? k0 : k1);
    const unsigned long long b = w_ballot2(k0 == m, k1 == m);
    return __ffsll((long long)b) - 1;
}
template <class V> __device__ __forceinline__ V w_sel(const V (&a)[2], int j) { return j ? a[1] : a[0]; }
template <class V> __device__ __forceinline__ void w_put(V (&a)[2], int j, V v) {
    if (j) a[1] = v; else a[0] = v;
}

// per-warp scratch of the wide stages
struct WScratchA { size_t link, bytes; };
struct WScratchC { size_t link, bat, bytes; };
__host__ __device__ inline WScratchA wide_a_layout(size_t R) {
    WScratchA L{};
    L.link = 0;
    L.bytes = (R * sizeof(int) + 255) & ~(size_t)255;
    return L;
}
__host__ __device__ inline WScratchC wide_c_layout(size_t R, int RB) {
    WScratchC L{};
    size_t off = 0;
    auto take = [&](size_t b) { const size_t o = off; off += (b + 255) & ~(size_t)255; return o; };
    L.link = take(R * sizeof(int));
    L.bat = take((size_t)kWMax * RB * sizeof(unsigned long long));
    L.bytes = off;
    return L;
}

// ---------------------------------------------------------------------------
// stage A (wide): prefill workers + KV buffer → transfer-end stream, one warp
// per (prefill group, QPS) of the CTA's trace.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, PADSIM_WIDEA_MINB) stageA_wide_kernel(const __grid_constant__ FPlan P) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sl = blockIdx.x % P.s_count;
    const int s = P.s_begin + sl;
    const long long off = P.toff[s];
    const int R = P.nreq[s];
    const double* su = P.s_unit + off;
    const double* kvl = P.kv + off;
    const int* it = P.in_tok + off;
    const int* ot = P.out_tok + off;
    const unsigned char* ph = P.phase + off;
    char* wb = P.scrA + ((size_t)blockIdx.x * kWarps + warp) * P.a_warp_bytes;
    int* link = (int*)(wb + wide_a_layout((size_t)P.Rmax).link);
    const int QG = P.Q * P.n_groups;
    const int slots = P.m.slots, max_pb = P.m.max_pb, pb_tokens = P.m.pb_tokens;
    for (;;) {
        int item = 0;
        if (lane == 0) item = (int)atomicAdd(P.work + s, 1u);
        item = __shfl_sync(kFull, item, 0);
        if (item >= QG) break;
        const int q = item / P.n_groups;
        const int g = item - q * P.n_groups;
        const long long sb = ((long long)(g * P.Q + q) * P.s_count + sl) * P.Rmax;
        SRec* orec = P.st_rec + sb;
        SHot* ohot = P.st_hot + sb;
        double* spe_w = P.st_pe + sb;        // prefill end of requests waiting for a KV slot
        const double inv_lam = 1.0 / (P.qps[q] * (double)P.N);
        const int x = P.gx[g];
        // this lane's two prefill workers (ids lane, lane + 32)
        double tn[2], bs[2], sp[2];
        unsigned long long a0[2];            // outstanding tokens = routing key (A8); ~0 = no worker
        int qh[2], qt[2], ql[2], bh[2], bn[2];
#pragma unroll
        for (int j = 0; j < 2; j++) {
            const int w = lane + 32 * j;
            tn[j] = PAD_INF; bs[j] = 0.0;
            sp[j] = w < x ? P.m.spre[P.w_gcap[(size_t)g * kWMax + w] - P.m.min_w] : 1.0;
            a0[j] = w < x ? 0ull : ~0ull;
            qh[j] = qt[j] = kNoIdx; ql[j] = 0; bh[j] = kNoIdx; bn[j] = 0;
        }
        // KV transfer slot `lane` (slots are compacted: slot k is lane k)
        double ste = PAD_INF, spe = 0.0;
        int sid = 0x7fffffff;
        int tbusy = 0, mk = 0, mid = 0, twh = kNoIdx, twt = kNoIdx, twl = 0;
        double mte = PAD_INF;
        int na = 0, k = 0;
        double ta = R > 0 ? su[0] * inv_lam : PAD_INF;
        long long inst = 0;
        double sq = 0.0, se = 0.0;
        while (k < R) {
            double t = w_min_d(tn[0] < tn[1] ? tn[0] : tn[1]);
            t = ta < t ? ta : t;
            t = mte < t ? mte : t;
            inst++;
            const unsigned long long bm = w_ballot2(tn[0] == t, tn[1] == t);
            unsigned long long touched = 0;
            // kind 2: prefill batch ends, worker order; members enter the KV buffer
            for (unsigned long long m = bm; m; m &= m - 1) {
                const int w = __ffsll((long long)m) - 1, wl = w & 31, wj = w >> 5;
                int i = __shfl_sync(kFull, w_sel(bh, wj), wl);
                const int n = __shfl_sync(kFull, w_sel(bn, wj), wl);
                const double bstart = __shfl_sync(kFull, w_sel(bs, wj), wl);
                long long dec = 0;
                for (int z = 0; z < n; z++) {
                    const int nx = link[i];
                    dec += it[i];
                    sq = sq + (bstart - su[i] * inv_lam);     // Fig. 6 decomposition
                    se = se + (t - bstart);
                    if (tbusy < slots) {
                        const double te = t + kvl[i];
                        if (lane == tbusy) { ste = te; sid = i; spe = t; }
                        if (tbusy == 0 || te < mte || (te == mte && i < mid)) { mte = te; mid = i; mk = tbusy; }
                        tbusy++;
                    } else {                                   // waits for a KV slot (FIFO)
                        if (lane == 0) {
                            link[i] = kNoIdx;
                            if (twl > 0) link[twt] = i;
                            spe_w[i] = t;
                        }
                        if (twl == 0) twh = i;
                        twt = i;
                        twl++;
                    }
                    i = nx;
                }
                if (lane == wl) { w_put(a0, wj, w_sel(a0, wj) - (unsigned long long)dec); w_put(tn, wj, PAD_INF); }
            }
            __syncwarp();
            // kind 4: transfer ends, earliest (te, id) first → the stream
            while (tbusy > 0 && mte == t) {
                const double pe = __shfl_sync(kFull, spe, mk);
                if (lane == 0) {
                    SRec rc;
                    rc.pe = pe;
                    const double ttft = pe - su[mid] * inv_lam;
                    unsigned fl = (ttft <= P.ttft_slo ? 1u : 0u) |
                                  (fabs(ttft - P.ttft_slo) <= 1e-9 * P.ttft_slo ? 2u : 0u);
                    for (int z = 0; z < P.sw.n; z++) fl |= (ttft <= P.sw.ttft[z] ? 4u : 0u) << z;
                    rc.fl = fl | ((unsigned)mid << kRecIdShift);
                    rc.meta = ot[mid] | ((int)ph[mid] << 31);
                    orec[k] = rc;
                    SHot hc;
                    hc.te = t;
                    hc.meta = rc.meta;
                    hc.id = mid;
                    ohot[k] = hc;
                }
                k++;
                tbusy--;
                {   // move slot tbusy into the freed slot mk
                    const double v = __shfl_sync(kFull, ste, tbusy);
                    const int d = __shfl_sync(kFull, sid, tbusy);
                    const double p = __shfl_sync(kFull, spe, tbusy);
                    if (lane == mk) { ste = v; sid = d; spe = p; }
                }
                if (twl > 0) {
                    const int j = twh;
                    twh = link[j];
                    twl--;
                    const double te = t + kvl[j];
                    const double p = spe_w[j];
                    if (lane == tbusy) { ste = te; sid = j; spe = p; }
                    tbusy++;
                }
                // earliest (te, id) in flight: one slot per lane
                const bool ok = lane < tbusy;
                mte = w_min_d(ok ? ste : PAD_INF);
                mid = (int)__reduce_min_sync(kFull, ok && ste == mte ? (unsigned)sid : 0xffffffffu);
                mk = __ffs(__ballot_sync(kFull, ok && ste == mte && sid == mid)) - 1;
            }
            // kind 5: arrivals → least outstanding prefill worker, lowest id (A8)
            while (ta == t) {
                const int i = na;
                const int best = w_argmin(a0[0], a0[1]);
                const int tin = it[i];
                if (lane == 0) link[i] = kNoIdx;
                if (lane == (best & 31)) {
                    const int j = best >> 5;
                    w_put(a0, j, w_sel(a0, j) + (unsigned long long)tin);
                    if (w_sel(ql, j) == 0) w_put(qh, j, i); else link[w_sel(qt, j)] = i;
                    w_put(qt, j, i);
                    w_put(ql, j, w_sel(ql, j) + 1);
                }
                touched |= 1ull << best;
                na++;
                ta = na < R ? su[na] * inv_lam : PAD_INF;
            }
            __syncwarp();
            // dispatch: idle prefill workers take a FIFO prefix (A9), each on its lane
            const unsigned long long dm = bm | touched;
#pragma unroll
            for (int j = 0; j < 2; j++) {
                if (!((dm >> (lane + 32 * j)) & 1ull)) continue;
                const int qn = ql[j];
                if (tn[j] != PAD_INF || qn == 0) continue;
                const int h = qh[j];
                long long tok = it[h];
                int b = 1, jj = h;
                while (b < max_pb && b < qn) {
                    const int nx = link[jj];
                    const long long tt = tok + it[nx];
                    if (tt > pb_tokens) break;
                    tok = tt;
                    jj = nx;
                    b++;
                }
                bh[j] = h;
                bn[j] = b;
                bs[j] = t;
                ql[j] = qn - b;
                if (qn > b) qh[j] = link[jj];
                tn[j] = t + ((double)tok / P.m.den[b]) / sp[j];
            }
            __syncwarp();
        }
        if (lane == 0) {
            const long long ga = ((long long)g * P.Q + q) * P.S + s;
            P.evA[ga] = inst;
            P.a_sq[ga] = sq;
            P.a_se[ga] = se;
        }
    }
}

// One decode worker of stage C (wide), held in the registers of its lane.
struct WDec {
    double tn, tseg, L;
    int nact, ql, qh, qt, stm, nxs, st0, mfin, ci;
    bool on;
    __device__ __forceinline__ void init(bool o, int cap_idx) {
        on = o; ci = cap_idx;
        tn = PAD_INF; tseg = 0.0; L = 1.0;
        nact = 0; ql = 0; qh = qt = kNoIdx; stm = 0; nxs = 0; st0 = 0; mfin = 0x7fffffff;
    }
    // A13 routing key: active + pending (~0 = no such worker)
    __device__ __forceinline__ unsigned long long key() const {
        return on ? (unsigned long long)(nact + ql) : ~0ull;
    }
    // stream request kk routed here at t; A14: it joins at the first step boundary
    // at or after t
    __device__ __forceinline__ void route(int kk, double t, bool bnd_now, int max_db, int* link) {
        const int qn = ql, na = nact;
        if (qn == 0) qh = kk; else link[qt] = kk;
        qt = kk;
        ql = qn + 1;
        if (na > 0 && !bnd_now && na < max_db && qn == 0) {
            const int sj = seg_first_ge(tseg, L, 0.0, st0, stm, t, false);
            if (sj < nxs) { nxs = sj; tn = seg_bnd(tseg, L, 0.0, sj - st0, false); }
        }
    }
    // dispatch at t (idle, at a boundary, or a join boundary exactly at t): admit
    // pending joins (appended to the worker's unsorted batch array: one store, no
    // load), start a new segment if the batch changed
    __device__ __forceinline__ void dispatch(double t, bool ab, bool changed, int max_db, const int* link,
                                             const SRec* recs, unsigned long long* bw, const double* ltab) {
        int n = nact;
        if (n > 0 && !ab) {
            if (tn != t) return;               // mid-step
            stm = nxs;                         // join boundary exactly at t
            ab = true;
        }
        int qn = ql;
        if (!ab && qn == 0) return;
        const bool was_idle = !ab;
        bool joined = false;
        const int step = stm;
        int mf = mfin;
        int h = qh;
        while (n < max_db && qn > 0) {
            const int kk = h;
            qn--;
            if (qn > 0) h = link[kk];
            const int fin = step + ((recs[kk].meta & 0x7fffffff) - 1);
            bw[n] = ((unsigned long long)(unsigned)fin << 32) | (unsigned)kk;
            n++;
            mf = fin < mf ? fin : mf;
            joined = true;
        }
        ql = qn;
        qh = h;
        nact = n;
        if (n > 0) {
            if (was_idle || joined || changed) {
                tseg = t;
                st0 = step;
                L = ltab[(size_t)ci * max_db + (n - 1)];
            }
            mfin = mf;
            nxs = mf;
            tn = seg_bnd(tseg, L, 0.0, mf - st0, false);
        } else {
            mfin = 0x7fffffff;
            tn = PAD_INF;
        }
    }
};

// ---------------------------------------------------------------------------
// stage C (wide): decode workers consume the transfer-end stream (A13, A14),
// one warp per (candidate, QPS) of the CTA's trace.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, PADSIM_WIDE_MINB) stageC_wide_kernel(const __grid_constant__ FPlan P) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sl = blockIdx.x % P.s_count;
    const int s = P.s_begin + sl;
    const long long off = P.toff[s];
    const int R = P.nreq[s];
    const int RB = P.c_rb;
    const int max_db = P.m.max_db;
    char* wb = P.scrC + ((size_t)blockIdx.x * kWarps + warp) * P.c_warp_bytes;
    const WScratchC L = wide_c_layout((size_t)P.Rmax, RB);
    int* link = (int*)(wb + L.link);
    unsigned long long* bat = (unsigned long long*)(wb + L.bat);   // [worker][RB] (fin << 32 | k), unsorted
    const int QC = P.Q * P.n_cc;
    for (;;) {
        int item = 0;
        if (lane == 0) item = (int)atomicAdd(P.work + s, 1u);
        item = __shfl_sync(kFull, item, 0);
        if (item >= QC) break;
        const int q = item / P.n_cc;
        const int cc = item - q * P.n_cc;
        const int c = P.cc_cand[cc];
        const int g = P.cc_group[cc];
        const int y = P.cc_y[cc];
        const long long r = ((long long)c * P.Q + q) * P.S + s;
        const long long sb = ((long long)(g * P.Q + q) * P.s_count + sl) * P.Rmax;
        const SRec* recs = P.st_rec + sb;
        const SHot* hots = P.st_hot + sb;
        const long long rb = P.rec_ttft ? r * P.Rmax : -1;
        const double inv_lam = 1.0 / (P.qps[q] * (double)P.N);
        // this lane's two decode workers (ids lane, lane + 32): two explicit
        // instances (no run-time indexed arrays, so nothing goes to local memory)
        WDec W0, W1;
        W0.init(lane < y, lane < y ? P.w_dcap[(size_t)cc * kWMax + lane] - P.m.min_w : 0);
        W1.init(lane + 32 < y, lane + 32 < y ? P.w_dcap[(size_t)cc * kWMax + lane + 32] - P.m.min_w : 0);
        const int nk = P.sw.n;
        int* metk = P.sw.rep_met + r * kMaxSloSweep;
        if (lane == 0) {
#pragma unroll 1
            for (int z = 0; z < nk; z++) metk[z] = 0;
        }
        int completed = 0, met = 0, near = 0, k = 0;
        double maxcomp = -PAD_INF;
        SHot nxt;
        if (R > 0) nxt = hots[0]; else { nxt.te = PAD_INF; nxt.meta = 0; nxt.id = 0; }
        double tk = nxt.te;
        long long inst = 0;
        auto complete = [&](const SRec& rc, double t, double tpot) {
            const double ts = (rc.meta < 0) ? P.tpot_slo1 : P.tpot_slo0;
            met += ((rc.fl & 1u) && tpot <= ts) ? 1 : 0;
            if (lane == 0) {
#pragma unroll 1
                for (int z = 0; z < nk; z++) {
                    const double tz = (rc.meta < 0) ? P.sw.tpot1[z] : P.sw.tpot0[z];
                    if (((rc.fl >> (2 + z)) & 1u) && tpot <= tz) metk[z]++;
                }
            }
            near += ((rc.fl & 2u) || fabs(tpot - ts) <= 1e-9 * ts) ? 1 : 0;
            maxcomp = fmax(maxcomp, t);
            completed++;
            if (rb >= 0 && lane == 0) {
                const int id = (int)(rc.fl >> kRecIdShift);
                P.rec_ttft[rb + id] = rc.pe - P.s_unit[off + id] * inv_lam;   // as stage A
                P.rec_tpot[rb + id] = tpot;
                P.rec_pe[rb + id] = rc.pe;
                P.rec_comp[rb + id] = t;
            }
        };
        while (completed < R) {
            double t = w_min_d(W0.tn < W1.tn ? W0.tn : W1.tn);
            t = tk < t ? tk : t;
            inst++;
            const unsigned long long bd = w_ballot2(W0.tn == t, W1.tn == t);
            unsigned long long chg = 0, touched = 0;
            // kind 3: decode step boundaries, worker order
            for (unsigned long long m = bd; m; m &= m - 1) {
                const int w = __ffsll((long long)m) - 1, wl = w & 31, wj = w >> 5;
                const int sN = __shfl_sync(kFull, wj ? W1.nxs : W0.nxs, wl);
                const int mf0 = __shfl_sync(kFull, wj ? W1.mfin : W0.mfin, wl);
                if (lane == wl) {
                    if (wj) { W1.stm = sN; W1.tn = PAD_INF; } else { W0.stm = sN; W0.tn = PAD_INF; }
                }
                if (sN != mf0) continue;
                // the members finishing at step sN leave: the worker's batch array is
                // scanned lane-parallel (32 entries per load), the leavers scored in
                // array order (completion order at one instant changes nothing), the
                // rest compacted to the front, the next finish step a warp min
                const int n0 = __shfl_sync(kFull, wj ? W1.nact : W0.nact, wl);
                unsigned long long* bw = bat + (size_t)w * RB;
                int left = 0;
                unsigned mfm = 0x7fffffffu;
                for (int b0 = 0; b0 < n0; b0 += 32) {
                    const int idx = b0 + lane;
                    const bool ok = idx < n0;
                    const unsigned long long e = ok ? bw[idx] : 0ull;
                    const bool lv = ok && (int)(e >> 32) == sN;
                    const unsigned ml = __ballot_sync(kFull, lv);
                    const unsigned mr = __ballot_sync(kFull, ok && !lv);
                    mfm = min(mfm, __reduce_min_sync(kFull, ok && !lv ? (unsigned)(e >> 32) : 0x7fffffffu));
                    __syncwarp();
                    if (ok && !lv) bw[b0 - left + __popc(mr & ((1u << lane) - 1u))] = e;
                    for (unsigned mm = ml; mm; mm &= mm - 1) {
                        const int kk = __shfl_sync(kFull, (int)(unsigned)e, __ffs(mm) - 1);
                        const SRec rc = recs[kk];
                        complete(rc, t, (t - rc.pe) / (double)((rc.meta & 0x7fffffff) - 1));
                    }
                    left += __popc(ml);
                }
                if (lane == wl) {
                    WDec& X = wj ? W1 : W0;
                    X.nact = n0 - left;
                    X.mfin = n0 - left > 0 ? (int)mfm : 0x7fffffff;
                }
                chg |= 1ull << w;
            }
            __syncwarp();
            // kind 4: transfer ends from the stream, (te, id) order
            while (tk == t) {
                const int kk = k;
                const SHot hc = nxt;
                k++;
                if (k < R) nxt = hots[k]; else nxt.te = PAD_INF;
                tk = nxt.te;
                if (rb >= 0 && lane == 0) P.rec_te[rb + hc.id] = t;
                if ((hc.meta & 0x7fffffff) == 1) {                   // S:280 D4
                    complete(recs[kk], t, 0.0);
                    continue;
                }
                // A13: fewest active + pending, lowest id
                const int best = w_argmin(W0.key(), W1.key());
                if (lane == 0) link[kk] = kNoIdx;
                if (lane == (best & 31)) {
                    if (best >> 5) W1.route(kk, t, (bd >> best) & 1ull, max_db, link);
                    else W0.route(kk, t, (bd >> best) & 1ull, max_db, link);
                }
                touched |= 1ull << best;
            }
            __syncwarp();
            // dispatch over the touched workers, each on its own lane
            const unsigned long long dm = bd | touched;
            if ((dm >> lane) & 1ull)
                W0.dispatch(t, (bd >> lane) & 1ull, (chg >> lane) & 1ull, max_db, link, recs,
                            bat + (size_t)lane * RB, P.m.ltab);
            if ((dm >> (lane + 32)) & 1ull)
                W1.dispatch(t, (bd >> (lane + 32)) & 1ull, (chg >> (lane + 32)) & 1ull, max_db, link, recs,
                            bat + (size_t)(lane + 32) * RB, P.m.ltab);
            __syncwarp();
        }
        if (lane == 0) {
            P.rep_met[r] = met;
            P.rep_near[r] = near;
            const double dur = R > 0 ? maxcomp - P.s_unit[off] * inv_lam : 0.0;
            P.rep_dur[r] = dur;
            P.rep_good[r] = dur > 0 ? (double)met / dur : 0.0;
            P.rep_events[r] = inst;
            const long long ga = ((long long)g * P.Q + q) * P.S + s;
            P.sw.rep_sq[r] = P.a_sq[ga];
            P.sw.rep_se[r] = P.a_se[ga];
            const double cs = (double)P.sw.capsum[c];   // static caps: Σ caps
            const double acc = R > 0 ? cs * dur : 0.0;
            P.sw.rep_watts[r] = dur > 0 ? acc / dur : cs;
        }
        __syncwarp();
    }
}

}  // namespace padsim
