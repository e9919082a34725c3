// static_path.cuh — the factorized static replay (rows a4 + a5) for nodes of
// up to 8 simulated GPUs, with all per-replay worker state in registers.
//
// Why it is exact: for a static candidate nothing on the decode side feeds
// back into prefill routing, batching or the KV buffer (A8, A9, A12: routing
// reads only prefill state, the buffer has no decode back-pressure, the
// controller never acts).  So the joint replay factorises into
//   stage A (prefill + KV buffer), a function of (prefill caps in P-id order,
//            QPS, trace) only — shared by every candidate with the same
//            prefill pool (94 groups for the 955 candidates of cfg 2), and
//   stage C (decode), a function of stage A's transfer-end stream plus the
//            decode caps.
// Same-instant ordering survives the split: in the joint replay prefill ends
// precede transfer ends (A10) and only prefill state touches the KV buffer;
// decode step boundaries precede transfer ends and only decode state sees
// them.  Stage A emits transfer ends in exactly the joint replay's (time, id)
// order.  Parity tests compare both stages against the joint CPU oracle.
//
// Design: one thread per replay; worker state lives in fully unrolled
// per-worker register arrays indexed only by compile-time constants (a
// routed-to worker is updated by a predicated unrolled loop), so no local
// memory is touched; queues are linked through a lane-interleaved per-request
// `link` scratch array; decode batches ({finish step, id}) live in
// lane-interleaved scratch.  Stage C stages its CTA's trace in shared memory
// with cp.async.bulk (TMA) and reads the stream written by stage A.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "replay.cuh"

namespace padsim {

constexpr int kNW = 7;   // ≤ 7 workers per role when N ≤ 8 (each role has ≥ 1 GPU)

// stage C decode-pool classes: y = 1, 2, 3–4, 5, 6–7 decode GPUs → KW = 1, 2, 4, 5, 7
constexpr int kNumKC = 5;
__host__ __device__ constexpr int kc_kw(int k) { return k == 0 ? 1 : k == 1 ? 2 : k == 2 ? 4 : k == 3 ? 5 : kNW; }
__host__ __device__ constexpr int kc_class(int y) { return y <= 1 ? 0 : y <= 2 ? 1 : y <= 4 ? 2 : y <= 5 ? 3 : 4; }

// Register-array helpers: a run-time index selects with predicated moves only
// (no branches, no local memory).
template <int N, class T>
__device__ __forceinline__ void rset(T (&a)[N], int i, T v) {
#pragma unroll
    for (int w = 0; w < N; w++) a[w] = (w == i) ? v : a[w];
}
template <int N, class T>
__device__ __forceinline__ T rget(const T (&a)[N], int i) {
    T v = a[0];
#pragma unroll
    for (int w = 1; w < N; w++) v = (w == i) ? a[w] : v;
    return v;
}
template <int N, class T>
__device__ __forceinline__ void radd(T (&a)[N], int i, T d) {
#pragma unroll
    for (int w = 0; w < N; w++) a[w] += (w == i) ? d : (T)0;
}

// Hot part of a transfer-end record (16 B): read sequentially at transfer ends.
struct __align__(16) SHot {
    double te;      // transfer end
    int meta;       // out_tok | phase << 31
    int id;         // request id
};

// Completion part of a transfer-end record (16 B), read when the request
// completes.  The TTFT tests do not depend on the decode side, so stage A
// evaluates them once per record: bit 0 ttft ≤ TTFT_SLO, bit 1 ttft within
// 1e-9 relative of it (near-boundary), bits 2..9 ttft ≤ sweep SLO z, bits
// 10..31 request id (n_req < 2^22 on the factorized path).
struct __align__(16) SRec {
    double pe;      // prefill end (first token)
    int meta;       // out_tok | phase << 31
    unsigned fl;    // TTFT flags | id << 10
};
constexpr int kRecIdShift = 10;
#ifndef PADSIM_KDEFER
#define PADSIM_KDEFER 1
#endif
constexpr int kDefer = PADSIM_KDEFER;     // stage C completion scoring delay (records in flight)
constexpr int kRecMaxReq = 1 << 22;

struct FPlan {
    DevModel m;
    int N, Q, S, Rmax;
    const long long* toff;
    const int* nreq;
    const double* s_unit;
    const double* kv;
    const int* in_tok;
    const int* out_tok;
    const unsigned char* phase;
    const double* qps;
    double ttft_slo, tpot_slo0, tpot_slo1;
    // prefill groups (stage A)
    int n_groups;
    const int* gx;          // [G] prefill workers
    const int* gcap;        // [G][kNW] their caps, P-id order
    // stage A → C stream, per (g, q, s) block of Rmax records in (te, id) order
    struct SRec* st_rec;
    struct SHot* st_hot;    // same stream, hot 16-B part
    double* st_pe;          // prefill end, indexed by request id (stage A scratch)
    long long* evA;         // [G*Q*S] stage-A instants
    double* a_sq;           // [G*Q*S] Σ queueing delay (prefill start − arrival)
    double* a_se;           // [G*Q*S] Σ prefill exec time (end − start)
    char* scrA;
    size_t a_warp_bytes, a_off_tte, a_off_tid, a_off_tpe, a_off_ring, a_ring_lane;
    int a_blocks_per_trace;   // stage A grid = S × this; a CTA never straddles traces
    int s_begin, s_count;     // traces [s_begin, s_begin + s_count) of this launch (pipelined chunks)
    int a_smem_trace;         // stage A stages its trace in shared memory (TMA bulk)
    // stage C
    int n_cc;
    const int* cc_cand;     // [n_cc] candidate index
    const int* cc_group;    // [n_cc] prefill group
    const int* cc_y;        // [n_cc] decode workers
    const int* cc_dcap;     // [n_cc][kNW] decode caps, D-id order
    int cc_base;            // this launch's candidate class: cc entries [cc_base, cc_base + n_cc)
    int items_per_trace, n_items;
    unsigned* work;
    char* scrC;
    size_t c_warp_bytes, c_off_heads, c_off_bits;
    int wheel;              // decode timing wheel size (power of 2 ≥ max out_tok, ≥ 32)
    int bits_in_smem;       // wheel occupancy bitmap in shared memory (wheel ≤ 256)
    size_t c_off_sdec;      // byte offset of the s_dec(w) table in shared memory
    // decode step latency L[slot][n-1] in shared memory for the caps the candidates
    // use (a3 table; per_ctx = 0 only, small decode-pool classes with smem headroom)
    size_t c_off_ring;      // decode batch lists (BL variant): per lane [kNW][c_rb] u64
    int c_rb;               // ring slots per decode worker (power of 2 ≥ max_db)
    int c_hca_on;           // async head cache in shared memory (KW ≤ 4 classes)
    size_t c_off_hca;       // its byte offset: [KW][kThreads] 32-bit words
    int c_ltab_on;          // this launch reads L from the table (else xv / s_dec)
    int c_lslots;           // distinct decode caps (table rows)
    size_t c_off_ltab;      // byte offset of the table in shared memory
    const int* lsl;         // [c_lslots] cap index (cap - min_w) of each row
    const int* cc_dslot;    // [n_cc][kNW] row of each decode worker's cap
    int c_prefetch;         // prefetch the completion record into L2 at decode join
    float sync_win;         // lane clock window in mean inter-arrival times (0 = off)
    int smem_trace;
    // wide nodes (8 < N ≤ 64, wide_path.cuh): caps of up to 64 workers per role
    const int* w_gcap;      // [G][64] prefill caps of each group, P-id order
    const int* w_dcap;      // [n_cc][64] decode caps of each candidate, D-id order
    // outputs (r = (c*Q + q)*S + s)
    int* rep_met;
    int* rep_near;
    double* rep_dur;
    double* rep_good;
    long long* rep_events;
    double *rec_ttft, *rec_tpot, *rec_pe, *rec_comp, *rec_te;
    SloSweep sw;
};

// ---------------------------------------------------------------------------
// stage A: prefill workers + 32-slot KV request buffer → transfer-end stream
//
// Next event time and routing key (outstanding tokens) per prefill worker are
// register arrays; queue / batch / speedup state is a [field][worker][thread]
// shared-memory SoA so handler bodies are shared across workers (run-time
// worker index, convergent lanes).  Prompt queues are per-worker ring arrays
// of request ids (per-lane contiguous scratch), so forming a batch and ending
// it read the next ≤ max_pb ids with independent loads instead of chasing a
// linked list.  The ≤ 32 in-flight transfers are a small slot array (shared
// memory for 32-thread CTAs) with the earliest (te, id) cached in registers.
// ---------------------------------------------------------------------------
template <int TB>
__host__ __device__ constexpr size_t a_work_bytes() { return (size_t)kNW * TB * (2 * sizeof(double) + 4 * sizeof(int)); }
template <int TB>
__host__ __device__ constexpr size_t a_slot_bytes() {   // KV slots kept in smem for small CTAs
    return TB == 32 ? (size_t)PADSIM_MAX_SLOTS * TB * (2 * sizeof(double) + sizeof(int)) : 0;
}
#ifndef PADSIM_EAGER
#define PADSIM_EAGER 1     // stage C eager joins (see the transfer-end handler)
#endif
#ifndef PADSIM_KPRE
#define PADSIM_KPRE 4
#endif
constexpr int kPre = PADSIM_KPRE;    // ids fetched per batch of independent loads
constexpr int kLtabRows = 16;  // max distinct decode caps of the shared-memory step table
constexpr int kATbBig = 256;   // stage A CTA size for large workloads

template <int TB>
__global__ void __launch_bounds__(TB) stageA_kernel(const __grid_constant__ FPlan P) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ unsigned long long bar;
    const int tid = threadIdx.x;
    const int sl = blockIdx.x / P.a_blocks_per_trace;
    const int s = P.s_begin + sl;
    const int local = (blockIdx.x - sl * P.a_blocks_per_trace) * TB + tid;
    const long long off = P.toff[s];
    const int R = P.nreq[s];
    // the CTA's trace (arrival, kv, prompt tokens): staged once in shared memory
    // by TMA bulk copies, read by every prefill group × QPS replay of the CTA
    const double* su;
    const double* kv;
    const int* it;
    const int* ot = P.out_tok + off;
    const unsigned char* ph = P.phase + off;
    if (P.a_smem_trace) {
        const int Rp = (R + 15) & ~15;
        double* d_su = (double*)(smem + a_work_bytes<TB>() + a_slot_bytes<TB>());
        double* d_kv = d_su + Rp;
        int* d_in = (int*)(d_kv + Rp);
        if (tid == 0) mbar_init(&bar, 1);
        __syncthreads();
        if (tid == 0 && Rp > 0) {
            const unsigned b8 = (unsigned)Rp * 8u, b4 = (unsigned)Rp * 4u;
            mbar_expect_tx(&bar, 2 * b8 + b4);
            bulk_g2s(d_su, P.s_unit + off, b8, &bar);
            bulk_g2s(d_kv, P.kv + off, b8, &bar);
            bulk_g2s(d_in, P.in_tok + off, b4, &bar);
        }
        if (Rp > 0) mbar_wait(&bar, 0);
        su = d_su; kv = d_kv; it = d_in;
    } else {
        su = P.s_unit + off; kv = P.kv + off; it = P.in_tok + off;
    }
    if (local >= P.Q * P.n_groups) return;
    const int q = local / P.n_groups;
    const int g = local - q * P.n_groups;
    const long long u = (long long)blockIdx.x * TB + tid;    // scratch slot
    const int n_sm = kNW * TB;
    double* Wsp = (double*)smem + tid;
    double* Wbs = (double*)smem + n_sm + tid;   // start time of the batch in service
    int* ib = (int*)(smem + (size_t)2 * n_sm * sizeof(double));
    int* Wqh = ib + 0 * n_sm + tid;     // ring index of the queue head
    int* Wql = ib + 1 * n_sm + tid;     // queue length
    int* Wbh = ib + 2 * n_sm + tid;     // ring index of the batch in service
    int* Wbn = ib + 3 * n_sm + tid;     // its size
    const int lane = threadIdx.x & 31;
    char* wb = P.scrA + (size_t)(u >> 5) * P.a_warp_bytes;
    int* ring = (int*)(wb + P.a_off_ring) + (size_t)lane * P.a_ring_lane;   // [w*R + j], per lane
    int* wring = ring + (size_t)kNW * R;                                     // KV-wait FIFO [j]
    double* tte;
    double* tpe;
    int* tidb;
    int ss;
    if (TB == 32) {
        unsigned char* sp = smem + a_work_bytes<TB>();
        tte = (double*)sp + tid;
        tpe = (double*)sp + PADSIM_MAX_SLOTS * TB + tid;
        tidb = (int*)(sp + 2 * PADSIM_MAX_SLOTS * TB * sizeof(double)) + tid;
        ss = TB;
    } else {
        tte = (double*)(wb + P.a_off_tte) + lane;
        tidb = (int*)(wb + P.a_off_tid) + lane;
        tpe = (double*)(wb + P.a_off_tpe) + lane;
        ss = 32;
    }
    const long long sb = ((long long)(g * P.Q + q) * P.S + s) * P.Rmax;
    SRec* orec = P.st_rec + sb;
    SHot* ohot = P.st_hot + sb;
    const double inv_lam = 1.0 / (P.qps[q] * (double)P.N);
    const int x = P.gx[g];
    const int slots = P.m.slots, max_pb = P.m.max_pb, pb_tokens = P.m.pb_tokens;

    double tnext[kNW];
    long long a0[kNW];              // outstanding tokens = routing key (A8)
#pragma unroll
    for (int w = 0; w < kNW; w++) {
        const int o = w * TB;
        tnext[w] = PAD_INF;
        a0[w] = w < x ? 0 : 0x7fffffffffffffffLL;
        Wqh[o] = 0; Wql[o] = 0; Wbh[o] = 0; Wbn[o] = 0;
        Wsp[o] = w < x ? P.m.spre[P.gcap[g * kNW + w] - P.m.min_w] : 1.0;
    }
    auto set_tnext = [&](int wd, double v) { rset<kNW>(tnext, wd, v); };
    int tbusy = 0, mk = 0, mid = 0, twh = 0, twl = 0;
    double mte = PAD_INF;
    int na = 0, k = 0;
    double ta = R > 0 ? su[0] * inv_lam : PAD_INF;
    long long inst = 0;
    double sq = 0.0, se = 0.0;
    while (k < R) {
        double t = ta < mte ? ta : mte;
#pragma unroll
        for (int w = 0; w < kNW; w++) t = tnext[w] < t ? tnext[w] : t;
        inst++;
        unsigned bm = 0, touched = 0;
#pragma unroll
        for (int w = 0; w < kNW; w++) if (tnext[w] == t) bm |= 1u << w;
        // kind 2: prefill batch ends, worker order; members enter the KV buffer
        for (unsigned m = bm; m; m &= m - 1) {
            const int w = __ffs(m) - 1;
            const int o = w * TB;
            const int* rw = ring + (size_t)w * R;
            int j = Wbh[o];
            const int n = Wbn[o];
            const double bstart = Wbs[o];
            long long dec = 0;
            for (int z0 = 0; z0 < n; z0 += kPre) {
                int ids[kPre];
#pragma unroll
                for (int z = 0; z < kPre; z++) {           // independent loads
                    int jj = j + z;
                    jj = jj >= R ? jj - R : jj;
                    ids[z] = z0 + z < n ? rw[jj] : 0;
                }
#pragma unroll
                for (int z = 0; z < kPre; z++) {
                    if (z0 + z >= n) break;
                    const int i = ids[z];
                    dec += it[i];
                    sq = sq + (bstart - su[i] * inv_lam);     // Fig. 6 decomposition
                    se = se + (t - bstart);
                    if (tbusy < slots) {
                        const double te = t + kv[i];
                        tte[tbusy * ss] = te;
                        tidb[tbusy * ss] = i;
                        tpe[tbusy * ss] = t;
                        if (tbusy == 0 || te < mte || (te == mte && i < mid)) { mte = te; mid = i; mk = tbusy; }
                        tbusy++;
                    } else {                                  // waits for a KV slot (FIFO)
                        int wj = twh + twl;
                        wj = wj >= R ? wj - R : wj;
                        wring[wj] = i;
                        P.st_pe[sb + i] = t;
                        twl++;
                    }
                }
                j += kPre;
                j = j >= R ? j - R : j;
            }
            radd<kNW, long long>(a0, w, -dec);
            set_tnext(w, PAD_INF);
        }
        // kind 4: transfer ends, earliest (te, id) first → the stream
        while (tbusy > 0 && mte == t) {
            {
                SRec rc;
                rc.pe = tpe[mk * ss];
                const double ttft = rc.pe - su[mid] * inv_lam;
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
            if (mk != tbusy) {
                tte[mk * ss] = tte[tbusy * ss];
                tidb[mk * ss] = tidb[tbusy * ss];
                tpe[mk * ss] = tpe[tbusy * ss];
            }
            if (twl > 0) {
                const int j = wring[twh];
                twh = twh + 1 >= R ? 0 : twh + 1;
                twl--;
                tte[tbusy * ss] = t + kv[j];
                tidb[tbusy * ss] = j;
                tpe[tbusy * ss] = P.st_pe[sb + j];
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
                    ev[j] = ok ? tte[(z0 + j) * ss] : PAD_INF;
                    dv[j] = ok ? tidb[(z0 + j) * ss] : 0x7fffffff;
                }
#pragma unroll
                for (int j = 0; j < 4; j++)
                    if (ev[j] < mte || (ev[j] == mte && dv[j] < mid)) { mte = ev[j]; mid = dv[j]; mk = z0 + j; }
            }
        }
        // kind 5: arrivals → least outstanding prefill worker, lowest id (A8)
        while (ta == t) {
            const int i = na;
            int best = 0;
            long long bl = a0[0];
#pragma unroll
            for (int w = 1; w < kNW; w++)
                if (a0[w] < bl) { bl = a0[w]; best = w; }
            const int tin = it[i];
            radd<kNW, long long>(a0, best, (long long)tin);
            const int o = best * TB;
            const int qn = Wql[o];
            int jt = Wqh[o] + qn;
            jt = jt >= R ? jt - R : jt;
            ring[(size_t)best * R + jt] = i;
            Wql[o] = qn + 1;
            touched |= 1u << best;
            na++;
            ta = na < R ? su[na] * inv_lam : PAD_INF;
        }
        // dispatch: idle prefill workers take a FIFO prefix (A9)
        for (unsigned m = bm | touched; m; m &= m - 1) {
            const int w = __ffs(m) - 1;
            const int o = w * TB;
            const double tw = rget<kNW>(tnext, w);
            const int qn = Wql[o];
            if (tw != PAD_INF || qn == 0) continue;
            const int* rw = ring + (size_t)w * R;
            const int h = Wqh[o];
            long long tok = 0;
            int b = 0;
            bool stop = false;
            int j = h;
            while (!stop && b < qn && b < max_pb) {
                int ids[kPre];
#pragma unroll
                for (int z = 0; z < kPre; z++) {           // independent loads
                    int jj = j + z;
                    jj = jj >= R ? jj - R : jj;
                    ids[z] = b + z < qn ? rw[jj] : 0;
                }
#pragma unroll
                for (int z = 0; z < kPre; z++) {
                    if (stop || b >= qn || b >= max_pb) { stop = true; break; }
                    const long long tt = tok + it[ids[z]];
                    if (b > 0 && tt > pb_tokens) { stop = true; break; }   // head always admitted
                    tok = tt;
                    b++;
                }
                j += kPre;
                j = j >= R ? j - R : j;
            }
            Wbh[o] = h;
            Wbn[o] = b;
            Wbs[o] = t;
            Wql[o] = qn - b;
            int nh = h + b;
            Wqh[o] = nh >= R ? nh - R : nh;
            set_tnext(w, t + ((double)tok / P.m.den[b]) / Wsp[o]);
        }
    }
    const long long ga = (g * P.Q + q) * (long long)P.S + s;
    P.evA[ga] = inst;
    P.a_sq[ga] = sq;
    P.a_se[ga] = se;
}


// ---------------------------------------------------------------------------
// stage C: decode workers consume the transfer-end stream (A13, A14)
//
// The CTA owns one trace (s = blockIdx.x mod S); its warps pull 32-replay work
// items from that trace's counter (no CTA barrier per item).  Per decode
// worker, the next event time, routing load (active + pending) and cap index
// are register arrays; the rest is a [field][worker][thread] shared-memory SoA
// so handler bodies are shared across workers (run-time index, convergent
// lanes, conflict-free).  Requests are named by their stream index k; the
// stream record carries everything a completion needs (pe, ttft, out, phase).
// Decode batches are a timing wheel: bucket (finish step mod W) holds the
// head k (bit 31 = "more members chained through link[]"), an occupancy
// bitmap (shared memory when W ≤ 256) yields the next finish step.
// ---------------------------------------------------------------------------
struct CWork {            // per-thread shared-memory SoA views (stride kThreads)
    double* tseg;
    double* Ls;
    int* nact; int* qh; int* qt; int* ql; int* stm; int* nxs; int* st0; int* mfin;
    int* bf;                 // BL: ring index of the batch list's front
    long long* ctx;          // CTX: Σ prompt tokens of the active members (A15)
    long long* sj;           // CTX: Σ join steps of the active members (A40)
    double* dL;              // CTX: per-step latency growth of the segment (A40)
};

// stage C shared-memory SoA bytes per decode-worker slot (× KW × kThreads)
constexpr size_t kCWorkSlotBytes = 2 * sizeof(double) + 8 * sizeof(int);
constexpr size_t kCWorkCtxSlotBytes = 2 * sizeof(long long) + sizeof(double);
// IDX: stream-index type of link[] and the wheel heads — uint16_t when
// n_req ≤ 16383 (halves the scratch footprint and its DRAM/L2 traffic),
// else uint32_t; the top bit flags "more members chained through link[]".
// KW: decode-worker slots (2, 4 or 7).  Candidates are launched in classes by
// their decode pool size y ≤ KW, so replays with few decode GPUs run with
// smaller register arrays / shared-memory SoA (fewer instructions per event,
// more resident warps).  168 registers: shared memory caps KW = 7 at 3 CTAs/SM,
// which 168 registers still allow; launched with kThreads threads.
// Async head cache (cp.async, 4 bytes global → shared): the head of a decode
// worker's next finish bucket is copied into shared memory when the bucket
// becomes known and read at the next leave, so the leave does not wait for a
// dependent global load; the copy is asynchronous, so no register waits on it.
__device__ __forceinline__ void hca_issue(unsigned* sdst, const void* gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    const unsigned long long ga = (unsigned long long)__cvta_generic_to_global(gsrc) & ~3ull;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n\tcp.async.commit_group;" :: "r"(sa), "l"(ga) : "memory");
}
__device__ __forceinline__ void hca_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// BL = false: decode batches are a timing wheel (bucket = finish step mod Wh,
// heads + occupancy bitmap).  BL = true: each decode worker's batch is a list
// sorted by (finish step, stream index) in a per-lane ring of u64 entries
// (fin << 32 | k): a leave pops the front entries, a join inserts from the back
// (new members usually finish last), the next finish step is the front's — no
// bitmap in shared memory, and the live entries sit in a few adjacent sectors.
template <bool CTX, typename IDX, int KW, bool BL>
__global__ void __maxnreg__(168) stageC_kernel(const __grid_constant__ FPlan P) {
    constexpr unsigned kMulti = sizeof(IDX) == 2 ? 0x8000u : 0x80000000u;
    // kHalf (the KW = 4 / 5 classes, whose wheel heads were most of stage C's DRAM
    // traffic): the heads have Wh / 2 buckets (bucket = finish step mod Hb); a bucket
    // holds members of at most two finish steps, f and f + Hb (live finish steps lie
    // in (step, step + Wh)), told apart by bit lgH of the finish step, carried in
    // each chain entry (kRound); the occupancy bitmap stays exact (Wh bits).  Halves
    // the heads' footprint (cfg 4 stage C DRAM 221 → ~124 GB) at no cost in time for
    // those classes; the KW = 1 / 2 classes lose time to the extra chain filtering
    // (+20 %), so they keep one bucket per finish step.
    constexpr bool kHalf = KW == 4 || KW == 5;
    constexpr unsigned kRound = sizeof(IDX) == 2 ? 0x4000u : 0x40000000u;
    constexpr unsigned kIdMask = ~(kMulti | kRound);
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    char* wb = P.scrC + ((size_t)blockIdx.x * kWarps + warp) * P.c_warp_bytes;
    IDX* link = (IDX*)wb + lane;                                       // [k*32]
    const int Wm = P.wheel - 1, nwords = P.wheel >> 5;
    const int Hb = kHalf ? P.wheel >> 1 : P.wheel, Hm = Hb - 1, lgH = __ffs(Hb) - 1;
    IDX* heads = (IDX*)(wb + P.c_off_heads) + (size_t)lane * KW * Hb;    // per lane
    const int max_db = P.m.max_db;
    CWork W;
    unsigned* bits;
    int bstride;
    {
        unsigned char* p = smem;
        const int n = KW * kThreads;
        W.tseg = (double*)p + tid; p += n * sizeof(double);
        W.Ls = (double*)p + tid; p += n * sizeof(double);
        int* ib = (int*)p;
        W.nact = ib + 0 * n + tid; W.qh = ib + 1 * n + tid; W.qt = ib + 2 * n + tid;
        W.ql = ib + 3 * n + tid; W.stm = ib + 4 * n + tid; W.nxs = ib + 5 * n + tid;
        W.st0 = ib + 6 * n + tid; W.mfin = ib + 7 * n + tid;
        W.bf = BL ? ib + 8 * n + tid : nullptr;
        p += (BL ? 9 : 8) * n * sizeof(int);
        W.ctx = CTX ? (long long*)p + tid : nullptr;
        W.sj = CTX ? (long long*)p + n + tid : nullptr;
        W.dL = CTX ? (double*)p + 2 * n + tid : nullptr;
        if (CTX) p += 3 * n * sizeof(long long);
        if (P.bits_in_smem) {
            bits = (unsigned*)p + tid;
            bstride = kThreads;
        } else {
            bits = (unsigned*)(wb + P.c_off_bits) + lane;
            bstride = 32;
        }
    }
    // s_dec(w) for every cap in shared memory: a decode segment's step latency is
    // (fixed + per_seq·n) / s_dec(d) computed in place (the same expression as the
    // a3 table, so bit-identical) instead of a dependent global table load
    double* sdt = (double*)(smem + P.c_off_sdec);
    for (int i = tid; i < P.m.ncap; i += kThreads) sdt[i] = P.m.sdec[i];
    double* lts = (double*)(smem + P.c_off_ltab);
    const bool hca = !BL && P.c_hca_on;
    const int RB = P.c_rb, RBm = P.c_rb - 1;
    unsigned long long* ring = BL ? (unsigned long long*)(wb + P.c_off_ring) + (size_t)lane * kNW * RB : nullptr;
    unsigned* hcs = (unsigned*)(smem + P.c_off_hca) + tid;     // [w * kThreads]
    const bool ltab_on = !CTX && P.c_ltab_on;
    if (ltab_on)
        for (int i = tid; i < P.c_lslots * P.m.max_db; i += kThreads)
            lts[i] = P.m.ltab[(size_t)P.lsl[i / P.m.max_db] * P.m.max_db + i % P.m.max_db];
    __syncthreads();
    const int s = P.s_begin + blockIdx.x % P.s_count;
    const long long off = P.toff[s];
    const int R = P.nreq[s];
    const int* itk = P.in_tok + off;
    const int QC = P.Q * P.n_cc;
    for (;;) {
        int item = 0;
        if (lane == 0) item = (int)atomicAdd(P.work + s, 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item * 32 >= QC) break;
        const int u = item * 32 + lane;
        if (u >= QC) continue;
        const int q = u / P.n_cc;
        const int cc = P.cc_base + (u - q * P.n_cc);
        const int c = P.cc_cand[cc];
        const int g = P.cc_group[cc];
        const int y = P.cc_y[cc];
        const long long r = ((long long)c * P.Q + q) * P.S + s;
        const long long sb = ((long long)(g * P.Q + q) * P.S + s) * P.Rmax;
        const SRec* recs = P.st_rec + sb;
        const SHot* hots = P.st_hot + sb;
        const long long rb = P.rec_ttft ? r * P.Rmax : -1;
        const double inv_lam = 1.0 / (P.qps[q] * (double)P.N);
        const bool gr = CTX && P.m.ctx_growth;      // A40 context growth
        // decode cap indices of this candidate, 9 bits per worker (ncap ≤ 512)
        unsigned long long dcx = 0ull;
#pragma unroll
        for (int w = 0; w < KW; w++)
            dcx |= (unsigned long long)(ltab_on ? P.cc_dslot[cc * kNW + w]      // table row
                                                : P.cc_dcap[cc * kNW + w] - P.m.min_w) << (9 * w);
        double tnext[KW];
        int ld[KW];                        // routing load: active + pending (A13)
#pragma unroll
        for (int w = 0; w < KW; w++) {
            const int o = w * kThreads;
            tnext[w] = PAD_INF;
            ld[w] = w < y ? 0 : 0x7fffffff;
            W.tseg[o] = 0.0; W.Ls[o] = 1.0;
            W.nact[o] = 0; W.qh[o] = kNoIdx; W.qt[o] = kNoIdx; W.ql[o] = 0;
            W.stm[o] = 0; W.nxs[o] = 0; W.st0[o] = 0; W.mfin[o] = 0x7fffffff;
            if (BL) W.bf[o] = 0;
            if (CTX) { W.ctx[o] = 0; W.sj[o] = 0; W.dL[o] = 0.0; }
        }
        if (!BL)
            for (int z = 0; z < y * nwords; z++) bits[(size_t)z * bstride] = 0u;
        int completed = 0, met = 0, near = 0, k = 0;
        double maxcomp = -PAD_INF;
        SHot nxt;                          // the next transfer end of the stream
        if (R > 0) nxt = hots[0]; else { nxt.te = PAD_INF; nxt.meta = 0; nxt.id = 0; }
        double tk = nxt.te;
        long long inst = 0;
        auto set_tnext = [&](int wd, double v) { rset<KW>(tnext, wd, v); };
        // SLO-sweep met counts (§8(f) row 1): counted in this replay's global slots
        // (rolled loops; nothing to do when no sweep is set, as in the bench)
        const int nk = P.sw.n;
        int* metk = P.sw.rep_met + r * kMaxSloSweep;
#pragma unroll 1
        for (int z = 0; z < nk; z++) metk[z] = 0;
        int ck0 = -1, cm0 = 0, ck1 = -1, cm1 = 0;   // last two routed (stream index, meta)
        // deferred completions (non-CTX): a kDefer-deep FIFO in registers, shifted
        // with static indices; an entry is scored kDefer completions after its
        // record load was issued, so the load latency is hidden
        SRec drc[kDefer];
        double dt[kDefer];
        int dn = 0;                        // valid entries (0..kDefer)
        // scoring of one completion (`completed` is counted where the member
        // leaves: scoring may be deferred past the end of the event loop)
        auto complete = [&](const SRec& rc, double t, double tpot) {
            const double ts = (rc.meta < 0) ? P.tpot_slo1 : P.tpot_slo0;
            met += ((rc.fl & 1u) && tpot <= ts) ? 1 : 0;
#pragma unroll 1
            for (int z = 0; z < nk; z++) {
                const double tz = (rc.meta < 0) ? P.sw.tpot1[z] : P.sw.tpot0[z];
                if (((rc.fl >> (2 + z)) & 1u) && tpot <= tz) metk[z]++;
            }
            near += ((rc.fl & 2u) || fabs(tpot - ts) <= 1e-9 * ts) ? 1 : 0;
            maxcomp = fmax(maxcomp, t);
            if (rb >= 0) {
                const int id = (int)(rc.fl >> kRecIdShift);
                P.rec_ttft[rb + id] = rc.pe - P.s_unit[off + id] * inv_lam;   // as stage A
                P.rec_tpot[rb + id] = tpot;
                P.rec_pe[rb + id] = rc.pe;
                P.rec_comp[rb + id] = t;
            }
        };
        // lanes of a warp replay the same trace at the same QPS (mostly the same
        // transfer-end stream): keep their simulated clocks within sync_win of
        // each other so their stream / trace reads hit the same cache lines.  A
        // pure scheduling choice — each lane's replay is independent, any
        // interleaving gives identical results; the lane with the smallest clock
        // always proceeds, so there is no deadlock.
        const float win = P.sync_win > 0.f ? P.sync_win / (float)(P.qps[q] * (double)P.N) : 0.f;
        // BL: insert (fin, kk) into worker w's sorted list of n members, shifting
        // later-finishing entries back by one
        auto bl_insert = [&](int w, int n, int fin, int kk) {
            unsigned long long* rg = ring + (size_t)w * RB;
            const int f = W.bf[w * kThreads];
            const unsigned long long e = ((unsigned long long)(unsigned)fin << 32) | (unsigned)kk;
            int i = n;
            while (i > 0) {
                const unsigned long long pv = rg[(f + i - 1) & RBm];
                if (pv < e) break;
                rg[(f + i) & RBm] = pv;
                i--;
            }
            rg[(f + i) & RBm] = e;
        };
        while (completed < R) {
            double t = tk;
#pragma unroll
            for (int w = 0; w < KW; w++) t = tnext[w] < t ? tnext[w] : t;
            if (win > 0.f) {
                const float tf = (float)t;
                const unsigned mn = __reduce_min_sync(__activemask(), __float_as_uint(tf));
                if (tf > __uint_as_float(mn) + win) continue;
            }
            inst++;
            unsigned bnd = 0, touched = 0, eag = 0, hcok = 0;
#pragma unroll
            for (int w = 0; w < KW; w++) if (tnext[w] == t) bnd |= 1u << w;
            // kind 3: materialised step boundaries, worker order
            for (unsigned m = bnd; m; m &= m - 1) {
                const int w = __ffs(m) - 1;
                const int o = w * kThreads;
                const int sN = W.nxs[o];
                W.stm[o] = sN;               // tnext[w] is rewritten by this instant's dispatch
                if (sN == W.mfin[o]) {
                    // one leaving member (stream index kk): score it, now (CTX) or
                    // deferred by kDefer completions
                    auto leave_member = [&](int kk) {
                        if (CTX) {                          // the leave needs the record now
                            const SRec rc = recs[kk];
                            const int o1 = (rc.meta & 0x7fffffff) - 1;
                            complete(rc, t, (t - rc.pe) / (double)o1);
                            completed++;
                            W.ctx[o] -= itk[rc.fl >> kRecIdShift];
                            W.sj[o] -= sN - o1;             // its join step (A40)
                        } else {
                            // deferred scoring: score the previous completion, then
                            // issue this one's record load and use it at the next
                            // completion (or the end of the replay), so the load
                            // latency overlaps the rest of the event processing
                            if (dn == kDefer) {
                                const SRec& e = drc[kDefer - 1];
                                complete(e, dt[kDefer - 1], (dt[kDefer - 1] - e.pe) / (double)((e.meta & 0x7fffffff) - 1));
                            } else {
                                dn++;
                            }
#pragma unroll
                            for (int z = kDefer - 1; z > 0; z--) { drc[z] = drc[z - 1]; dt[z] = dt[z - 1]; }
                            drc[0] = recs[kk];
                            dt[0] = t;
                            completed++;
                        }
                    };
                    int left = 0;
                    int mf = 0x7fffffff;
                    if constexpr (BL) {
                        // pop the front entries with fin == sN; the first entry left
                        // behind is the new front (its fin is the next finish step)
                        const int n0 = W.nact[o];
                        const unsigned long long* rg = ring + (size_t)w * RB;
                        int f = W.bf[o];
                        unsigned long long e = rg[f];
                        for (;;) {
                            leave_member((int)(unsigned)e);
                            left++;
                            f = (f + 1) & RBm;
                            if (left == n0) break;
                            e = rg[f];
                            if ((int)(e >> 32) != sN) break;
                        }
                        W.bf[o] = f;
                        W.nact[o] = n0 - left;
                        if (left < n0) mf = (int)(e >> 32);
                    } else {
                        const int b = sN & Wm;            // bitmap bit of the finish step
                        const int hb = sN & Hm;           // its head bucket
                        const unsigned rr = (kHalf && ((sN >> lgH) & 1)) ? kRound : 0u;
                        unsigned cur;
                        if (hca) {
                            hca_wait();
                            const unsigned wd = hcs[w * kThreads];
                            cur = sizeof(IDX) == 2 ? ((hb & 1) ? (wd >> 16) : (wd & 0xffffu)) : wd;
                        } else {
                            cur = (unsigned)heads[(size_t)w * Hb + hb];
                        }
                        // members of finish step sN leave; those of sN + Hb (other
                        // round bit) are re-chained as the bucket's new list
                        unsigned keep = 0u;
                        bool kept = false;
                        if constexpr (kHalf) {
                            for (;;) {
                                const int kk = (int)(cur & kIdMask);
                                const bool more = (cur & kMulti) != 0u;
                                const unsigned nx = more ? (unsigned)link[(size_t)kk * 32] : 0u;   // IDX → unsigned keeps the flags
                                if ((cur & kRound) == rr) {
                                    leave_member(kk);
                                    left++;
                                } else {
                                    if (kept) link[(size_t)kk * 32] = (IDX)keep;
                                    keep = (unsigned)kk | (cur & kRound) | (kept ? kMulti : 0u);
                                    kept = true;
                                }
                                if (!more) break;
                                cur = nx;
                            }
                        } else {             // one finish step per bucket: every member leaves
                            for (;;) {
                                const int kk = (int)(cur & ~kMulti);
                                leave_member(kk);
                                left++;
                                if (!(cur & kMulti)) break;
                                cur = (unsigned)link[(size_t)kk * 32];   // IDX → unsigned keeps the flag bit
                            }
                        }
                        if (kept) heads[(size_t)w * Hb + hb] = (IDX)keep;
                        unsigned* bw = bits + (size_t)w * nwords * bstride;
                        bw[(size_t)(b >> 5) * bstride] &= ~(1u << (b & 31));
                        const int n = W.nact[o] - left;
                        W.nact[o] = n;
                        if (n > 0) {   // next occupied bucket (finish steps lie in (sN, sN+Wh))
                            const int st = (b + 1) & Wm;
                            int wi = st >> 5;
                            unsigned mword = bw[(size_t)wi * bstride] & (0xffffffffu << (st & 31));
                            while (mword == 0u) {
                                wi = (wi + 1) & (nwords - 1);
                                mword = bw[(size_t)wi * bstride];
                            }
                            mf = sN + ((((wi << 5) + __ffs(mword) - 1) - b) & Wm);
                        }
                        // the kept members finish next (mf = sN + Hb): their new list is the
                        // head of the next bucket — cache it here (the dispatch would
                        // otherwise copy back what this thread just stored)
                        if (hca && kept && (mf & Hm) == hb) {
                            hcs[w * kThreads] = (sizeof(IDX) == 2 && (hb & 1)) ? (keep << 16) : keep;
                            hcok |= 1u << w;
                        }
                    }
                    W.mfin[o] = mf;
                    radd<KW, int>(ld, w, -left);
                    touched |= 1u << (w + 16);          // composition changed
                }
            }
            // kind 4: transfer ends from the stream, (te, id) order
            while (tk == t) {
                const int kk = k;
                const SHot hc = nxt;
                k++;
                if (k < R) nxt = hots[k]; else nxt.te = PAD_INF;
                tk = nxt.te;
                if (rb >= 0) P.rec_te[rb + hc.id] = t;
                if ((hc.meta & 0x7fffffff) == 1) {                   // S:280 D4
                    complete(recs[kk], t, 0.0);
                    completed++;
                    continue;
                }
                int best = 0, bl = ld[0];
#pragma unroll
                for (int w = 1; w < KW; w++) if (ld[w] < bl) { bl = ld[w]; best = w; }
                radd<KW, int>(ld, best, 1);
                const int o = best * kThreads;
                const int qn = W.ql[o];
                const int na = W.nact[o];
                ck1 = ck0; cm1 = cm0; ck0 = kk; cm0 = hc.meta;
                if (qn == 0) W.qh[o] = kk; else link[(size_t)W.qt[o] * 32] = (IDX)kk;
                W.qt[o] = kk;
                W.ql[o] = qn + 1;
                touched |= 1u << best;
                if (na > 0 && !((bnd >> best) & 1u) && na < max_db && qn == 0) {
                    const double ts0 = W.tseg[o], L = W.Ls[o];
                    const double dL = CTX ? W.dL[o] : 0.0;
                    const int s0 = W.st0[o];
                    const int sj = seg_first_ge(ts0, L, dL, s0, W.stm[o], t, gr);
                    if (PADSIM_EAGER && sj < W.mfin[o]) {
                        // Eager join: the request joins at the first boundary sj ≥ t
                        // of the running segment (A14).  When sj precedes the worker's
                        // next leave, nothing else happens to this worker until sj
                        // (routing only reads active + pending, unchanged by a join),
                        // so this instant's dispatch admits it as the boundary instant
                        // would: the new segment starts at sj (time bnd(sj)).  A later
                        // transfer end at or before bnd(sj) finds sj again as its first
                        // boundary and joins the same not-yet-started segment.  Saves
                        // the join-only instant; same state as the DES at bnd(sj).
                        W.nxs[o] = sj;
                        eag |= 1u << best;
                    } else if (sj < W.nxs[o]) {
                        W.nxs[o] = sj;
                        set_tnext(best, seg_bnd(ts0, L, dL, sj - s0, gr));
                    }
                }
            }
            // dispatch over the workers this instant touched, worker order
            for (unsigned m = (bnd | touched) & 0xffffu; m; m &= m - 1) {
                const int w = __ffs(m) - 1;
                const int o = w * kThreads;
                bool ab = (bnd >> w) & 1u;
                const bool eg = (eag >> w) & 1u;         // eager join at boundary W.nxs
                int n = W.nact[o];
                if (n > 0 && !ab && !eg) {
                    if (rget<KW>(tnext, w) != t) continue;   // mid-step
                    W.stm[o] = W.nxs[o];                 // join boundary exactly at t
                    ab = true;
                }
                ab = ab || eg;
                int qn = W.ql[o];
                if (!ab && qn == 0) continue;
                const bool was_idle = !ab;
                bool joined = false;
                bool hset = false;
                unsigned hv = 0u;
                int hb = 0;
                const int step = eg ? W.nxs[o] : W.stm[o];
                int mf = W.mfin[o];
                int h = W.qh[o];
                IDX* hw = heads + (size_t)w * Hb;
                unsigned* bw = bits + (size_t)w * nwords * bstride;
                while (n < max_db && qn > 0) {
                    const int kk = h;
                    qn--;
                    if (qn > 0) h = (int)link[(size_t)kk * 32];
                    // most joiners were routed at one of the last two transfer ends
                    int meta;
                    if (kk == ck0) meta = cm0;
                    else if (kk == ck1) meta = cm1;
                    else meta = hots[kk].meta;
                    const int out = meta & 0x7fffffff;
                    if (P.c_prefetch) asm volatile("prefetch.global.L2 [%0];" :: "l"(recs + kk));
                    const int fin = step + (out - 1);
                    if constexpr (BL) {
                        bl_insert(w, n, fin, kk);
                    } else {
                        const int b = fin & Wm;              // bitmap bit of the finish step
                        const int fb = fin & Hm;             // its head bucket
                        const unsigned ent = (unsigned)kk | ((kHalf && ((fin >> lgH) & 1)) ? kRound : 0u);
                        unsigned* wp = bw + (size_t)(b >> 5) * bstride;
                        const unsigned bit = 1u << (b & 31);
                        const int b2 = b ^ Hb;               // the bucket's other finish step
                        const unsigned old = *wp;
                        const bool occ = (old & bit) ||
                                         (kHalf && (bw[(size_t)(b2 >> 5) * bstride] & (1u << (b2 & 31))));
                        if (occ) {                           // bucket occupied: chain
                            link[(size_t)kk * 32] = hw[fb];
                            hw[fb] = (IDX)(ent | kMulti);
                        } else {
                            hw[fb] = (IDX)ent;
                        }
                        *wp = old | bit;
                        if (fin <= mf || (kHalf && fb == (mf & Hm))) {   // head of the earliest bucket (or of its bucket)
                            hv = occ ? (ent | kMulti) : ent;
                            hb = fb;
                            hset = true;
                        }
                    }
                    n++;
                    if (CTX) { W.ctx[o] += itk[hots[kk].id]; W.sj[o] += step; }
                    mf = fin < mf ? fin : mf;
                    joined = true;
                }
                W.ql[o] = qn;
                W.qh[o] = h;
                W.nact[o] = n;
                if (n > 0) {
                    double ts0 = W.tseg[o], L = W.Ls[o];
                    double dL = CTX ? W.dL[o] : 0.0;
                    int s0 = W.st0[o];
                    if (was_idle || joined || ((touched >> (w + 16)) & 1u)) {
                        // the new segment starts at this instant, or for an eager join
                        // at boundary `step` of the running segment (time bnd(step))
                        ts0 = eg ? seg_bnd(ts0, L, dL, step - s0, gr) : t;
                        if (eg) W.stm[o] = step - 1;         // boundaries ≥ step: new segment
                        s0 = step;
                        const int cix = (int)((dcx >> (9 * w)) & 511u);
                        double xv = P.m.dec_fixed + P.m.dec_per_seq * (double)n;
                        if (CTX) {          // A15 / A40 context of the segment's first step
                            long long cc = W.ctx[o];
                            if (gr) cc += (long long)n * (step + 1) - W.sj[o];
                            xv = xv + P.m.dec_per_ctx * (double)cc;
                        }
                        L = ltab_on ? lts[cix * max_db + n - 1] : xv / sdt[cix];
                        W.tseg[o] = ts0; W.st0[o] = s0; W.Ls[o] = L;
                        if (CTX) {
                            dL = gr ? (P.m.dec_per_ctx * (double)n) / sdt[cix] : 0.0;
                            W.dL[o] = dL;
                        }
                    }
                    W.mfin[o] = mf;
                    W.nxs[o] = mf;
                    if (BL) {
                    } else if (hca) {
                        if (hset) {
                            hca_wait();
                            hcs[w * kThreads] = (sizeof(IDX) == 2 && (hb & 1)) ? (hv << 16) : hv;
                        } else if (((touched >> (w + 16)) & 1u) && !((hcok >> w) & 1u)) {   // after a leave: copy it in
                            hca_issue(hcs + w * kThreads, hw + (mf & Hm));
                        }
                    } else {
                        pf_head(hw + (mf & Hm));
                    }
                    set_tnext(w, seg_bnd(ts0, L, dL, mf - s0, gr));
                } else {
                    W.mfin[o] = 0x7fffffff;
                    set_tnext(w, PAD_INF);
                }
            }
        }
        if (!CTX) {
#pragma unroll
            for (int z = 0; z < kDefer; z++)
                if (z < dn) complete(drc[z], dt[z], (dt[z] - drc[z].pe) / (double)((drc[z].meta & 0x7fffffff) - 1));
        }
        P.rep_met[r] = met;
        P.rep_near[r] = near;
        const double dur = R > 0 ? maxcomp - P.s_unit[off] * inv_lam : 0.0;
        P.rep_dur[r] = dur;
        P.rep_good[r] = dur > 0 ? (double)met / dur : 0.0;
        P.rep_events[r] = inst;
        {
            const long long ga = (g * P.Q + q) * (long long)P.S + s;
            P.sw.rep_sq[r] = P.a_sq[ga];
            P.sw.rep_se[r] = P.a_se[ga];
        }
        {   // static caps: provisioned power is Σ caps over [a_0, last completion]
            const double cs = (double)P.sw.capsum[c];
            const double acc = R > 0 ? cs * dur : 0.0;
            P.sw.rep_watts[r] = dur > 0 ? acc / dur : cs;
        }
    }
}

}  // namespace padsim
