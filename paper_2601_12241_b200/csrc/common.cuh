// common.cuh — device-side plan layout shared by the padsim kernels.
//
// Product code (never includes or links anything under oracle/).  Every
// kernel is compiled with --fmad=false so each FP64 expression keeps the
// operation order pinned in DESIGN.md §3 (c.1): no contraction into FMA,
// IEEE round-to-nearest division and conversion.
#pragma once
#include <cstdint>

#include "../../include/padsim.h"

namespace padsim {

constexpr int kMaxSloSweep = 8;        // extra SLO sets scored per replay
constexpr int kMaxPct = 16;             // percentiles per padsim_fetch_percentiles call (PADSIM_MAX_PCT)
constexpr size_t kPctSmemMax = 128 * 1024;   // bitonic buffer in shared memory up to 16384 values

// Extra SLO sets scored on the same trajectories + per-replay extra outputs.
struct SloSweep {
    int n;
    double ttft[kMaxSloSweep], tpot0[kMaxSloSweep], tpot1[kMaxSloSweep];
    int* rep_met;          // [r * kMaxSloSweep + k]
    double* rep_watts;     // [r] time-weighted mean of Σ effective caps
    const int* capsum;     // [C] Σ initial caps
    double* rep_sq;        // [r] Σ_i (prefill start − arrival)   (Fig. 6)
    double* rep_se;        // [r] Σ_i (prefill end − prefill start)
};

constexpr int kThreads = 128;          // replays per CTA (4 warps)
constexpr int kWarps = kThreads / 32;
constexpr int kNoIdx = -1;

// Device model: scalar parameters + precomputed tables (a3).
struct DevModel {
    int min_w, max_w, ncap;            // ncap = max_w - min_w + 1
    double rate, eff, dec_fixed, dec_per_seq, dec_per_ctx, kvb, bw, ovh;
    int max_pb, pb_tokens, max_db, slots;
    int chunk;                         // coalesced mode: prefill chunk tokens
    int ctx_growth;                    // A40: decode context counts generated tokens
    const double* spre;                // [ncap]  s_pre(w)
    const double* sdec;                // [ncap]  s_dec(w)
    const double* den;                 // [max_pb+1] rate*(1+eff*(b-1))
    const double* ltab;                // [ncap][max_db] decode step latency, n = 1..max_db
};

// Prefetch (to L2) of the timing-wheel head of a decode worker's next finish
// bucket, issued when that bucket becomes known and read at the next leave.
// A/B on one box (tools/call_ab.sh): cfg 4 785 -> 770 ms/step; an L1 prefetch
// (773 ms), keeping the head in registers (807 ms) and deciding the TPOT tests
// without the FP64 division (814 ms) were no better.
__device__ __forceinline__ void pf_head(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" :: "l"(p));
}

// Decode segment boundaries (A14; A40 with context growth): boundary k of a
// segment that started at ts0 with first-step latency L and per-step growth dL.
__device__ __forceinline__ double seg_bnd(double ts0, double L, double dL, int k, bool growth) {
    if (!growth) return ts0 + (double)k * L;
    const long long tri = (long long)k * (long long)(k - 1) / 2;
    return ts0 + ((double)k * L + (double)tri * dL);
}

// Smallest boundary index s > stm of the segment (started at step s0) whose time
// is ≥ tau: a float estimate (linear, or the quadratic root with growth) fixed up
// with the exact FP64 boundary expression (boundaries are increasing in k).
__device__ __forceinline__ int seg_first_ge(double ts0, double L, double dL, int s0, int stm, double tau,
                                            bool growth) {
    const float D = (float)(tau - ts0);
    float kf;
    if (!growth) {
        kf = __fdividef(D, (float)L);
    } else {
        const float B = (float)L - 0.5f * (float)dL;
        kf = 2.f * D / (B + sqrtf(B * B + 2.f * (float)dL * D));
    }
    kf = fminf(fmaxf(kf, 0.f), 1.0e9f);
    int s = s0 + (int)ceilf(kf);
    if (s <= stm) s = stm + 1;
    while (seg_bnd(ts0, L, dL, s - s0, growth) < tau) s++;
    while (s - 1 > stm && seg_bnd(ts0, L, dL, s - 1 - s0, growth) >= tau) s--;
    return s;
}

// Everything a replay kernel launch needs (passed by value as a kernel param).
struct Plan {
    DevModel m;
    int N, C, Q, S, Rmax;
    const int* cbud;                   // [C] node budget per candidate (padsim_budget)
    // traces: SoA, trace s occupies [toff[s], toff[s]+nreq[s]); toff multiple of 16
    const long long* toff;
    const int* nreq;
    const double* s_unit;
    const double* kv;                  // kv_lat(in_tok) per request (a3)
    const int* in_tok;
    const int* out_tok;
    const unsigned char* phase;
    // candidates
    const unsigned char* role;         // [C][N]
    const int* cap;                    // [C][N]
    const padsim_policy* pol;          // [C]
    const double* qps;                 // [Q]
    double ttft_slo, tpot_slo0, tpot_slo1;
    // replay subset for this launch: candidate list
    const int* clist;                  // [n_clist]
    int n_clist;
    int items_per_trace;               // ceil(Q*n_clist / kThreads)
    int n_items;
    unsigned* work;                    // work counter (zeroed before launch)
    // outputs per replay r = (c*Q + q)*S + s
    int* rep_met;
    int* rep_near;
    double* rep_dur;
    double* rep_good;
    long long* rep_events;
    // optional per-request records [r*Rmax + i]
    double *rec_ttft, *rec_tpot, *rec_pe, *rec_comp, *rec_te;
    SloSweep sw;
    // scratch: per CTA slot, lane-interleaved
    char* scratch;
    size_t scratch_per_cta;
    size_t off_link, off_pe, off_mem, off_ordt, off_tst, off_tfl;   // per-warp offsets
    size_t off_tte, off_tti;           // KV-buffer slots (joint8 kernel)
    size_t off_heads, off_bits;        // decode timing wheel (joint8 kernel)
    size_t off_wts, off_wtf;           // TTFT window: stamps + flags (joint kernel)
    size_t off_jw;                     // per-GPU SoA in global scratch (joint kernel, NG = 64)
    size_t off_ring;                   // decode batch lists (joint kernel, PADSIM_JBL): per lane [NG][ring_slots] u64
    int ring_slots;                    // power of 2 ≥ max_decode_batch
    int j_kglob;                       // joint kernel, N > 8: next-event / routing keys in global scratch
    size_t off_keys;                   // their per-warp offset (lane-interleaved [NG][32] f64, i32, i32)
    int wheel;                         // wheel size: power of 2 ≥ max out_tok, ≥ 32
    size_t warp_bytes;
    int smem_trace;                    // stage the trace in shared memory (TMA bulk)
    float sync_win;                    // lane clock window, mean inter-arrival times (0 = off)
    int lpw;                           // replays per warp item (joint kernel; 32, or fewer for small workloads)
    size_t smem_trace_bytes;
};

}  // namespace padsim
