// controller.cuh — Algorithm 1 "Dynamic Resources Scheduling" (PAPER.md
// P:207–251) as a __device__ decision step, used by the dynamic replay
// kernel (row a6) and by padsim_step_controller.
//
// Readings: guards exactly as printed, strict (A20); cooldown
// strict; PowerLimitsReached checked *before* moving (A18):
// if not reached → MovePower, else MoveGPU + DistributeUniformPower (policy
// permitting, donor role keeps ≥1 GPU, no role change pending), else
// "saturated" (no action, last_move unchanged).  Draining GPUs belong
// to neither pool (A26).  The controller never consults the latency model
// (P:294–296): it sees only the window comparisons, |Q_P| and per-GPU load.
#pragma once
#include "common.cuh"

namespace padsim {

enum { ACT_NONE = 0, ACT_MOVE_POWER = 1, ACT_MOVE_GPU = 2, ACT_SATURATED = 3 };

struct CtlSignals {
    bool ttft_gt, ttft_lt, tpot_gt, tpot_lt;   // p90 stat vs SLO (strict)
    int q_prefill;                              // |Q_P|
};

// View: role(g) 0/1, draining(g), target(g) (commanded cap incl. pending
// raise), load(g) (P: outstanding tokens, D: active+pending).
template <class View>
__device__ __forceinline__ int ctl_step(const padsim_policy& pol, int min_w, int max_w, int budget,
                                        int N, const View& v, bool drain_pending, double last_move,
                                        double now, const CtlSignals& sg, int* new_cap,
                                        int* out_gpu, int* out_dir) {
    *out_gpu = -1;
    *out_dir = -1;
    if (pol.kind == 0) return ACT_NONE;                       // static never acts
    if (!((now - last_move) > pol.cooldown_s)) return ACT_NONE;
    int dir;
    if (sg.ttft_gt && sg.q_prefill > pol.queue_threshold && sg.tpot_lt) dir = 0;
    else if (sg.tpot_gt && sg.ttft_lt) dir = 1;
    else return ACT_NONE;
    *out_dir = dir;
    const int from = dir == 0 ? 1 : 0;
    const int to = dir == 0 ? 0 : 1;
    const int ceil_to = to == 0 ? max_w : pol.decode_ceiling_w;
    int n_don = 0, n_rec = 0;
    bool rec_ceil = true, don_floor = true;
#pragma unroll 1
    for (int g = 0; g < N; g++) {
        if (v.draining(g)) continue;
        const int r = v.role(g);
        const int c = v.target(g);
        if (r == from) { n_don++; if (c > min_w) don_floor = false; }
        if (r == to) { n_rec++; if (c < ceil_to) rec_ceil = false; }
    }
    const bool limits = rec_ceil || don_floor;
    const bool power_ok = pol.kind == 1 || pol.kind == 3;
    const bool gpu_ok = pol.kind == 2 || pol.kind == 3;
    if (power_ok && !limits) {
        // MovePower: donors −min(step, cap−floor), F = Σ, recipients
        // +min(⌊F/|rec|⌋, ceiling−cap), leftover unallocated.
        long long F = 0;
#pragma unroll 1
        for (int g = 0; g < N; g++) {
            const int c = v.target(g);
            new_cap[g] = c;
            if (v.draining(g) || v.role(g) != from) continue;
            int r = c - min_w;
            r = r < pol.power_step_w ? r : pol.power_step_w;
            r = r > 0 ? r : 0;
            new_cap[g] = c - r;
            F += r;
        }
        const long long share = n_rec > 0 ? F / n_rec : 0;
#pragma unroll 1
        for (int g = 0; g < N; g++) {
            if (v.draining(g) || v.role(g) != to) continue;
            const int c = v.target(g);
            long long r = (long long)ceil_to - c;
            r = share < r ? share : r;
            r = r > 0 ? r : 0;
            new_cap[g] = c + (int)r;
        }
        return ACT_MOVE_POWER;
    }
    if (gpu_ok && n_don >= 2 && !drain_pending) {
        // MoveGPU: least outstanding work, lowest id; then uniform caps
        int best = -1;
        long long bl = 0;
#pragma unroll 1
        for (int g = 0; g < N; g++) {
            if (v.draining(g) || v.role(g) != from) continue;
            const long long l = v.load(g);
            if (best < 0 || l < bl) { best = g; bl = l; }
        }
        int u = budget / N;                                     // DistributeUniformPower
        u = u < min_w ? min_w : u;
        u = u > max_w ? max_w : u;
#pragma unroll 1
        for (int g = 0; g < N; g++) new_cap[g] = u;
        *out_gpu = best;
        return ACT_MOVE_GPU;
    }
    return ACT_SATURATED;
}

}  // namespace padsim
