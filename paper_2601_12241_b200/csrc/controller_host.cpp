// controller_host.cpp — padsim_step_controller: Algorithm 1 "Dynamic Resources
// Scheduling" as a pure, thread-safe host function over
// the full controller state of one node (include/padsim.h).
//
// Compiled on its own (plain C++, no CUDA): it allocates nothing, touches
// only *st and *act, and never consults the latency model (the
// controller sees the window statistics, |Q_P| and per-GPU load only).  The
// dynamic replay kernel runs the same rules as the __device__ ctl_step of
// controller.cuh; tests/test_controller_host.py replays window-statistics
// sequences recorded from the CPU oracle through this function, and the GPU
// tests compare padsim_controller_decide_device with it.
#include <cmath>
#include <cstdint>

#include "../../include/padsim.h"

namespace {

bool due(double deadline, double now) { return deadline >= 0.0 && deadline <= now; }

// Settle instant: decreases take effect, sinks are raised.
void apply_settle(padsim_ctrl_state* st, int g) {
    if (st->cmd_cap_w[g] < st->eff_cap_w[g]) st->eff_cap_w[g] = st->cmd_cap_w[g];
    if (st->pending_raise_w[g] > 0) {
        st->cmd_cap_w[g] = st->eff_cap_w[g] = st->pending_raise_w[g];
        st->pending_raise_w[g] = 0;
    }
    st->settle_deadline_s[g] = -1.0;
}

// Role change after drain + reassignment latency.
void apply_flip(padsim_ctrl_state* st, int g) {
    st->role[g] ^= 1;
    st->draining[g] = 0;
    st->flip_deadline_s[g] = -1.0;
}

}  // namespace

extern "C" int padsim_step_controller(const padsim_policy* pol, const padsim_budget* budget,
                                      const padsim_model* m, padsim_ctrl_state* st,
                                      const padsim_window_stats* ws, double now, padsim_action* act) {
    if (!pol || !budget || !m || !st || !ws || !act) return PADSIM_EINVAL;
    const int n = st->n_gpus;
    if (n < 2 || n > PADSIM_MAX_GPUS) return PADSIM_EINVAL;
    if (!(m->min_w > 0 && m->min_w < m->max_w)) return PADSIM_EMODEL;
    if (pol->kind < 0 || pol->kind > 3 || pol->window_stamp < 0 || pol->window_stamp > 1)
        return PADSIM_EINVAL;
    if (pol->kind != 0 &&
        !(pol->tick_s > 0 && pol->settle_s > 0 && pol->reassign_s > 0 && pol->cooldown_s >= pol->settle_s &&
          pol->power_step_w > 0 && pol->queue_threshold >= 0 && pol->decode_ceiling_w >= m->min_w &&
          pol->decode_ceiling_w <= m->max_w))
        return PADSIM_EINVAL;
    if (!std::isfinite(now)) return PADSIM_EINVAL;
    for (int g = 0; g < n; g++) {
        if (st->role[g] > 1) return PADSIM_EINVAL;
        if (st->cmd_cap_w[g] < m->min_w || st->cmd_cap_w[g] > m->max_w || st->eff_cap_w[g] < m->min_w ||
            st->eff_cap_w[g] > m->max_w)
            return PADSIM_ERANGE;
    }
    act->kind = 0;
    act->direction = -1;
    act->gpu = -1;

    // 1. transitions due by now (settle before flip at one instant, A10; the two
    //    commute otherwise: one touches caps, the other roles)
    for (int g = 0; g < n; g++)
        if (due(st->settle_deadline_s[g], now)) apply_settle(st, g);
    for (int g = 0; g < n; g++) {
        if (st->draining[g] && st->flip_deadline_s[g] < 0.0 && ws->drained_empty_s[g] >= 0.0)
            st->flip_deadline_s[g] = ws->drained_empty_s[g] + pol->reassign_s;
        if (st->draining[g] && due(st->flip_deadline_s[g], now)) apply_flip(st, g);
    }
    for (int g = 0; g < PADSIM_MAX_GPUS; g++)
        act->new_cap_w[g] = g < n ? (st->pending_raise_w[g] > 0 ? st->pending_raise_w[g] : st->cmd_cap_w[g]) : 0;

    // 2. Alg. 1 body
    if (pol->kind == 0) return PADSIM_OK;                         // static never acts
    if (!((now - st->last_move_s) > pol->cooldown_s)) return PADSIM_OK;
    int dir;
    if (ws->ttft_stat_s > ws->ttft_slo_s && ws->q_prefill > pol->queue_threshold &&
        ws->tpot_stat_s < ws->tpot_slo_s)
        dir = 0;                                                   // D->P
    else if (ws->tpot_stat_s > ws->tpot_slo_s && ws->ttft_stat_s < ws->ttft_slo_s)
        dir = 1;                                                   // P->D
    else
        return PADSIM_OK;
    act->direction = dir;
    const int donor_role = dir == 0 ? 1 : 0;
    const int recv_role = 1 - donor_role;
    const int ceiling = recv_role == 0 ? m->max_w : pol->decode_ceiling_w;
    const int floor_w = m->min_w;
    bool any_pending = false;
    int n_donor = 0, n_recv = 0;
    bool recv_at_ceiling = true, donor_at_floor = true;
    int target[PADSIM_MAX_GPUS];
    for (int g = 0; g < n; g++) {
        target[g] = st->pending_raise_w[g] > 0 ? st->pending_raise_w[g] : st->cmd_cap_w[g];
        any_pending = any_pending || st->draining[g];
        if (st->draining[g]) continue;                              // A26
        if (st->role[g] == donor_role) {
            n_donor++;
            donor_at_floor = donor_at_floor && target[g] <= floor_w;
        } else {
            n_recv++;
            recv_at_ceiling = recv_at_ceiling && target[g] >= ceiling;
        }
    }
    const bool limits = recv_at_ceiling || donor_at_floor;         // PowerLimitsReached
    const bool may_power = pol->kind == 1 || pol->kind == 3;
    const bool may_gpu = pol->kind == 2 || pol->kind == 3;
    int newcap[PADSIM_MAX_GPUS];
    for (int g = 0; g < n; g++) newcap[g] = target[g];
    if (may_power && !limits) {
        long long freed = 0;                                       // MovePower
        for (int g = 0; g < n; g++) {
            if (st->draining[g] || st->role[g] != donor_role) continue;
            int cut = target[g] - floor_w;
            if (cut > pol->power_step_w) cut = pol->power_step_w;
            if (cut < 0) cut = 0;
            newcap[g] = target[g] - cut;
            freed += cut;
        }
        const long long share = n_recv > 0 ? freed / n_recv : 0;  // leftover stays unallocated
        for (int g = 0; g < n; g++) {
            if (st->draining[g] || st->role[g] != recv_role) continue;
            long long add = (long long)ceiling - target[g];
            if (add > share) add = share;
            if (add < 0) add = 0;
            newcap[g] = target[g] + (int)add;
        }
        act->kind = 1;
    } else if (may_gpu && n_donor >= 2 && !any_pending) {
        int pick = -1;                                             // MoveGPU
        for (int g = 0; g < n; g++) {
            if (st->draining[g] || st->role[g] != donor_role) continue;
            if (pick < 0 || ws->load[g] < ws->load[pick]) pick = g;
        }
        const int bud = budget->budget_w;                          // DistributeUniformPower
        int u = bud / n;
        if (u < m->min_w) u = m->min_w;
        if (u > m->max_w) u = m->max_w;
        for (int g = 0; g < n; g++) newcap[g] = u;
        act->kind = 2;
        act->gpu = pick;
        st->draining[pick] = 1;
        st->flip_deadline_s[pick] = -1.0;
    } else {
        act->kind = 3;                                             // saturated: no action
        return PADSIM_OK;
    }
    // 3. source-before-sink: decreases commanded now, raises at the settle instant
    for (int g = 0; g < n; g++) {
        act->new_cap_w[g] = newcap[g];
        if (newcap[g] < st->cmd_cap_w[g]) {
            st->cmd_cap_w[g] = newcap[g];
            st->pending_raise_w[g] = 0;
        } else if (newcap[g] > st->cmd_cap_w[g]) {
            st->pending_raise_w[g] = newcap[g];
        } else {
            st->pending_raise_w[g] = 0;
        }
        st->settle_deadline_s[g] = now + pol->settle_s;
    }
    st->last_move_s = now;
    return PADSIM_OK;
}
