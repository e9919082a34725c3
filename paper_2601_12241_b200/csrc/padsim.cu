// padsim.cu — C ABI (include/padsim.h) of the B200-native what-if evaluator:
// host validation + upload (plan), the model-table kernel (row a3), the
// replay kernels (rows a4–a7, replay.cuh), the seed reduction and the
// per-QPS argmax (row a8), the device controller step (row a6 ABI).
//
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo
//        --fmad=false -Xcompiler -fPIC -shared
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "common.cuh"
#include "controller.cuh"
#include "coalesced.cuh"
#include "replay.cuh"
#include "static_path.cuh"
#include "dynamic_path.cuh"
#include "group_path.cuh"
#include "wide_path.cuh"

#include <map>

using namespace padsim;

struct padsim_ctx {
    int device = 0;
    int n_sm = 0;
    cudaStream_t stream = nullptr;   // stream of the one-shot API (padsim_create)
    padsim_tuning tune{0, 0, -1, 0, -1, 0, -1, 0, -1, -1, 0};   // launch overrides (padsim_set_tuning)
    int n_launches = 0;              // kernels launched by the last padsim_run
    std::string err;
    // plan
    bool planned = false;
    uint32_t flags = 0;
    int N = 0, C = 0, Q = 0, S = 0, Rmax = 0;
    padsim_model model{};
    padsim_slo slo{};
    std::vector<int> static_list, dyn_list, coal_list;
    std::vector<long long> toff;
    std::vector<int> capsum_h;
    // device buffers
    // device buffers of the current plan; a re-plan with the same shapes reuses them
    // in allocation order (no cudaMalloc/cudaFree on the end-to-end path)
    struct Buf { void* p; size_t bytes; };
    std::vector<Buf> bufs;
    size_t buf_cursor = 0;
    long long* d_toff = nullptr;
    int* d_nreq = nullptr;
    double* d_s_unit = nullptr;
    double* d_kv = nullptr;
    int* d_in = nullptr;
    int* d_out = nullptr;
    unsigned char* d_phase = nullptr;
    unsigned char* d_role = nullptr;
    int* d_cap = nullptr;
    int* d_capsum = nullptr;
    int* d_cbud = nullptr;           // [C] per-candidate node budget (padsim_budget)
    padsim_policy* d_pol = nullptr;
    double* d_qps = nullptr;
    int* d_clist_static = nullptr;
    int* d_clist_dyn = nullptr;
    double *d_spre = nullptr, *d_sdec = nullptr, *d_den = nullptr, *d_ltab = nullptr;
    int* d_rep_met = nullptr;
    int* d_rep_near = nullptr;
    double* d_rep_dur = nullptr;
    double* d_rep_good = nullptr;
    long long* d_rep_events = nullptr;
    long long* d_met = nullptr;
    double* d_good = nullptr;
    long long* d_near = nullptr;
    int* d_argmax = nullptr;
    // SLO sweep / provisioned power outputs
    int* d_rep_metk = nullptr;
    double* d_rep_watts = nullptr;
    long long* d_metk = nullptr;     // [C*Q*kMaxSloSweep]
    double* d_qpw = nullptr;         // [C*Q] Σ_s goodput/avg_watts
    double* d_watts = nullptr;       // [C*Q] Σ_s avg_watts
    int* d_max80 = nullptr;          // [C*(1+kMaxSloSweep)]
    // Fig. 6 decomposition and percentiles
    double* d_rep_sq = nullptr;      // [r] Σ_i queueing delay
    double* d_rep_se = nullptr;      // [r] Σ_i prefill exec time
    double* d_qsum = nullptr;        // [C*Q] Σ_s rep_sq
    double* d_esum = nullptr;        // [C*Q] Σ_s rep_se
    int* d_pct = nullptr;            // [kMaxPct] requested percentiles (records mode)
    double* d_pct_out = nullptr;     // [r][2][kMaxPct]
    double* d_pct_scratch = nullptr; // global sort buffers when a trace exceeds shared memory
    int pct_n2 = 0, pct_grid = 0;
    size_t pct_smem = 0;
    long long n_req_total = 0;
    SloSweep sweep{};
    double *d_rec[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    unsigned* d_work = nullptr;
    char* d_scratch_static = nullptr;
    char* d_scratch_dyn = nullptr;
    Plan plan_static{}, plan_dyn{};
    int grid_static = 0, grid_dyn = 0;
    Plan plan_coal{};                // coalesced baseline (policy kind 4)
    int grid_coal = 0;
    int* d_clist_coal = nullptr;
    size_t smem_static = 0, smem_dyn = 0;
    // host staging for the one-shot API
    padsim_ctrl_state* d_ctl_state = nullptr;
    padsim_window_stats* d_ctl_stats = nullptr;
    padsim_action* d_ctl_act = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evA = nullptr, evC = nullptr;
    cudaEvent_t evJ0 = nullptr, evJ1 = nullptr;
    cudaStream_t side = nullptr;     // joint kernel runs concurrently with stages A/C
    cudaEvent_t evC0 = nullptr;
    cudaStream_t sideC[kNumKC] = {};   // stage C classes run concurrently
    cudaEvent_t evCk[kNumKC] = {};    // class joins
    cudaEvent_t evCf = nullptr;                                  // class fork
    bool j_with_a = false;           // experiment knob: joint replays next to stage A
    bool ev_recorded = false;
    // factorized static path (N <= 8)
    bool fact = false;
    FPlan fplan{};
    int fA_grid = 0, fC_grid = 0;
    size_t fC_smem = 0, fA_smem = 0;
    // stage C decode-pool classes (static_path.cuh kc_class): cc range, grid, smem
    int kc_base[kNumKC] = {}, kc_n[kNumKC] = {}, kc_grid[kNumKC] = {};
    size_t kc_smem[kNumKC] = {}, kc_off_sdec[kNumKC] = {};
    int kc_bits_smem[kNumKC] = {};
    int kc_ltab[kNumKC] = {};
    int kc_fine = 0;                   // five decode-pool classes (large workloads)
    bool j_cx = false;                 // joint kernel instantiated with the context term
    bool j_r168 = false;               // joint kernel: 168-register one-warp-CTA variant
    int kc_bl[kNumKC] = {};            // class uses the sorted batch lists (BL) instead of the wheel
    int kc_hca[kNumKC] = {};
    size_t kc_off_hca[kNumKC] = {};
    size_t kc_off_ltab[kNumKC] = {};
    char* kc_scr[kNumKC] = {};
    int fA_tb = kThreads;
    bool fC_idx16 = false;
    int j_tb[2] = {kThreads, kThreads};
    long long* d_evA = nullptr;
    int n_evA = 0;
    unsigned* d_workC = nullptr;
    std::vector<int> max_out;   // per trace
    bool j8[2] = {false, false};   // [static, dynamic] list planned on the joint kernel
    int j_ng = 8;                  // its GPU-slot width (8 or 64)
    bool j_grp = false;            // N ≤ 8 joint replays on lane groups (jointg_kernel)
    // factorized static path for wide nodes (8 < N ≤ 64, wide_path.cuh)
    bool wide = false;
    int w_chunk = 1;               // traces per stage A → C chunk (stream buffers sized for it)
    int wA_grid = 0, wC_grid = 0;  // resident CTAs available to a launch (scratch slots)
    long long wA_items = 0, wC_items = 0;   // warp items per trace (stage A, stage C)
    unsigned* d_workW = nullptr;   // work counters [2][S] (stage A, stage C)
    std::vector<cudaEvent_t> evW;  // per chunk: stage A start/stop, stage C start/stop
    int n_wchunks = 0;             // chunks of the last run
    unsigned* d_workJ[2] = {nullptr, nullptr};
};

static const char* kVersion = "padsim 0.1 (sm_100a)";

static int fail(padsim_ctx* ctx, int code, const char* msg) {
    if (ctx) ctx->err = msg;
    return code;
}
static int cuda_fail(padsim_ctx* ctx, cudaError_t e, const char* where) {
    if (ctx) ctx->err = std::string(where) + ": " + cudaGetErrorString(e);
    return PADSIM_ECUDA;
}
#define CK(call)                                               \
    do {                                                       \
        cudaError_t e_ = (call);                               \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
    } while (0)

template <class T>
static int dalloc(padsim_ctx* ctx, T** p, size_t n) {
    *p = nullptr;
    if (n == 0) n = 1;
    const size_t bytes = n * sizeof(T);
    const size_t k = ctx->buf_cursor++;
    if (k < ctx->bufs.size() && ctx->bufs[k].bytes >= bytes) {
        *p = (T*)ctx->bufs[k].p;
        return PADSIM_OK;
    }
    if (k < ctx->bufs.size()) {
        cudaFree(ctx->bufs[k].p);
        ctx->bufs[k] = {nullptr, 0};
    }
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        ctx->err = std::string("cudaMalloc: ") + cudaGetErrorString(e);
        return PADSIM_ENOMEM;
    }
    if (k < ctx->bufs.size()) ctx->bufs[k] = {q, bytes};
    else ctx->bufs.push_back({q, bytes});
    *p = (T*)q;
    return PADSIM_OK;
}

static void release_buffers(padsim_ctx* ctx) {
    for (auto& b : ctx->bufs) if (b.p) cudaFree(b.p);
    ctx->bufs.clear();
    ctx->buf_cursor = 0;
}

static void free_plan(padsim_ctx* ctx) {
    ctx->buf_cursor = 0;       // buffers are kept for reuse by the next plan
    ctx->planned = false;
    ctx->fact = false;
    ctx->wide = false;
    ctx->j8[0] = ctx->j8[1] = false;
    ctx->static_list.clear();
    ctx->dyn_list.clear();
    ctx->coal_list.clear();
    for (auto& r : ctx->d_rec) r = nullptr;
}

// ---------------------------------------------------------------------------
// row a3: model tables (device).  Same FP64 expressions as DESIGN.md §3 c.1.
// ---------------------------------------------------------------------------
__device__ double dev_speedup(const padsim_curve& c, int w) {
    const int n = c.n;
    if (w == c.w[n - 1]) return c.s[n - 1];
    int j = 0;
    for (int k = 1; k < n - 1; k++)
        if (c.w[k] <= w) j = k;
    const double diff = c.s[j + 1] - c.s[j];
    const double frac = (double)(w - c.w[j]) / (double)(c.w[j + 1] - c.w[j]);
    return c.s[j] + diff * frac;
}

__global__ void tables_kernel(const padsim_model m, double* spre, double* sdec, double* den,
                              double* ltab, const int* in_tok, double* kv, long long n_tok) {
    const int ncap = m.max_w - m.min_w + 1;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long k = tid; k < ncap; k += stride) {
        spre[k] = dev_speedup(m.prefill, m.min_w + (int)k);
        sdec[k] = dev_speedup(m.decode, m.min_w + (int)k);
    }
    for (long long b = tid; b <= m.max_prefill_batch; b += stride) {
        const double be = 1.0 + m.prefill_batch_eff * (double)((int)b - 1);
        den[b] = m.prefill_base_rate * be;
    }
    const long long nl = (long long)ncap * m.max_decode_batch;
    for (long long k = tid; k < nl; k += stride) {
        const int ci = (int)(k / m.max_decode_batch);
        const int n = (int)(k % m.max_decode_batch) + 1;
        const double x = m.decode_fixed_s + m.decode_per_seq_s * (double)n;
        ltab[k] = x / dev_speedup(m.decode, m.min_w + ci);
    }
    for (long long i = tid; i < n_tok; i += stride) {
        kv[i] = m.transfer_overhead_s + ((double)in_tok[i] * m.kv_bytes_per_token) / m.fabric_bw_Bps;
    }
}

// ---------------------------------------------------------------------------
// row a8: seed reduction (ascending trace order) and per-QPS argmax
// ---------------------------------------------------------------------------
__global__ void reduce_kernel(const int* rep_met, const int* rep_near, const double* rep_good,
                              int CQ, int S, long long* met, double* good, long long* near,
                              const int* rep_metk, const double* rep_watts, int nk,
                              long long* metk, double* qpw, double* watts,
                              const double* rep_sq, const double* rep_se, double* qsum, double* esum) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= CQ) return;
    long long m = 0, nn = 0;
    long long mk[kMaxSloSweep] = {0, 0, 0, 0, 0, 0, 0, 0};
    double g = 0.0, qw = 0.0, ws = 0.0, sq = 0.0, se = 0.0;
    const long long base = (long long)k * S;
    for (int s = 0; s < S; s++) {      // ascending trace order (c.4)
        const long long r = base + s;
        m += rep_met[r];
        nn += rep_near[r];
        g += rep_good[r];
        const double w = rep_watts[r];
        qw += w > 0 ? rep_good[r] / w : 0.0;     // QPS/W = goodput / avg provisioned W
        ws += w;
        sq += rep_sq[r];
        se += rep_se[r];
        for (int z = 0; z < nk; z++) mk[z] += rep_metk[r * kMaxSloSweep + z];
    }
    qsum[k] = sq;
    esum[k] = se;
    met[k] = m;
    near[k] = nn;
    good[k] = g;
    qpw[k] = qw;
    watts[k] = ws;
    for (int z = 0; z < kMaxSloSweep; z++) metk[(long long)k * kMaxSloSweep + z] = z < nk ? mk[z] : 0;
}

// Nearest-rank percentiles (1-based rank ceil(p·n/100), integer
// form (p·n+99)/100) of each replay's per-request TTFT and TPOT records
// (records mode). One CTA per replay at a time; bitonic sort of the padded
// power-of-two buffer in shared memory, or in a per-CTA global slice when the
// trace does not fit. Exact: a sort moves values, no arithmetic.
__global__ void __launch_bounds__(512) percentile_kernel(const double* rec_ttft, const double* rec_tpot,
                                                         const int* nreq, int S, int Rmax, int n2,
                                                         long long n_rep, const int* pcts, int np,
                                                         double* out, double* gscratch) {
    extern __shared__ __align__(16) double psm[];
    double* buf = gscratch ? gscratch + (size_t)blockIdx.x * n2 : psm;
    for (long long r = blockIdx.x; r < n_rep; r += gridDim.x) {
        const int R = nreq[r % S];
        for (int m = 0; m < 2; m++) {
            const double* src = (m ? rec_tpot : rec_ttft) + r * Rmax;
            for (int i = threadIdx.x; i < n2; i += blockDim.x) buf[i] = i < R ? src[i] : PAD_INF;
            __syncthreads();
            for (int k = 2; k <= n2; k <<= 1) {
                for (int j = k >> 1; j > 0; j >>= 1) {
                    for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                        const int l = i ^ j;
                        if (l > i) {
                            const double a = buf[i], b = buf[l];
                            if (((i & k) == 0) ? (a > b) : (a < b)) { buf[i] = b; buf[l] = a; }
                        }
                    }
                    __syncthreads();
                }
            }
            for (int z = threadIdx.x; z < np; z += blockDim.x) {
                const int p = pcts[z];
                out[(r * 2 + m) * kMaxPct + z] = R > 0 ? buf[(p * R + 99) / 100 - 1] : __longlong_as_double(0x7ff8000000000000LL);
            }
            __syncthreads();
        }
    }
}

// Max QPS at >= 80% SLO attainment per candidate, for the main SLO
// (column 0) and each sweep SLO (columns 1..nk): the QPS point with the largest
// qps among those with 5·Σmet ≥ 4·Σ_s R_s (integer test), else -1.
__global__ void max80_kernel(const long long* met, const long long* metk, const double* qps, int C, int Q,
                             int nk, long long n_req_total, int* out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    for (int z = 0; z <= nk; z++) {
        int best = -1;
        for (int q = 0; q < Q; q++) {
            const long long m = z == 0 ? met[(long long)c * Q + q]
                                       : metk[((long long)c * Q + q) * kMaxSloSweep + (z - 1)];
            if (5 * m >= 4 * n_req_total && (best < 0 || qps[q] > qps[best])) best = q;
        }
        out[(long long)c * (1 + kMaxSloSweep) + z] = best;
    }
    for (int z = nk + 1; z <= kMaxSloSweep; z++) out[(long long)c * (1 + kMaxSloSweep) + z] = -1;
}

struct Key { long long met; int capsum; int idx; };
__device__ __forceinline__ bool key_better(const Key& a, const Key& b) {
    if (a.met != b.met) return a.met > b.met;            // Σmet ↓
    if (a.capsum != b.capsum) return a.capsum < b.capsum;  // Σcaps ↑ (A25)
    return a.idx < b.idx;                              // index ↑
}

__global__ void argmax_kernel(const long long* met, const int* capsum, int C, int Q, int* argmax) {
    const int q = blockIdx.x;
    Key best{-1, 0x7fffffff, 0x7fffffff};
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        Key k{met[(long long)c * Q + q], capsum[c], c};
        if (key_better(k, best)) best = k;
    }
    for (int o = 16; o > 0; o >>= 1) {
        Key other;
        other.met = __shfl_xor_sync(0xffffffffu, best.met, o);
        other.capsum = __shfl_xor_sync(0xffffffffu, best.capsum, o);
        other.idx = __shfl_xor_sync(0xffffffffu, best.idx, o);
        if (key_better(other, best)) best = other;
    }
    __shared__ Key sk[32];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sk[w] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        Key b = sk[0];
        for (int i = 1; i < (int)(blockDim.x >> 5); i++)
            if (key_better(sk[i], b)) b = sk[i];
        argmax[q] = b.idx;
    }
}

// ---------------------------------------------------------------------------
// row a6: the Alg. 1 decision on the device (same ctl_step as the replay
// kernel), for parity of the kernel's controller with padsim_step_controller
// ---------------------------------------------------------------------------
struct AbiView {
    const padsim_ctrl_state* st;
    const padsim_window_stats* ws;
    __device__ int role(int g) const { return st->role[g]; }
    __device__ bool draining(int g) const { return st->draining[g] != 0; }
    __device__ int target(int g) const {
        return st->pending_raise_w[g] > 0 ? st->pending_raise_w[g] : st->cmd_cap_w[g];
    }
    __device__ long long load(int g) const { return ws->load[g]; }
};

__global__ void controller_kernel(const padsim_policy pol, const int min_w, const int max_w,
                                  const int budget, const padsim_ctrl_state* st,
                                  const padsim_window_stats* ws, const double now,
                                  padsim_action* act) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    CtlSignals sg;
    sg.ttft_gt = ws->ttft_stat_s > ws->ttft_slo_s;
    sg.ttft_lt = ws->ttft_stat_s < ws->ttft_slo_s;
    sg.tpot_gt = ws->tpot_stat_s > ws->tpot_slo_s;
    sg.tpot_lt = ws->tpot_stat_s < ws->tpot_slo_s;
    sg.q_prefill = ws->q_prefill;
    AbiView v{st, ws};
    int newcap[PADSIM_MAX_GPUS];
    int gsel, dir;
    const int N = st->n_gpus;
    bool pending = false;
    for (int g = 0; g < N; g++) pending = pending || st->draining[g];
    const int kind = ctl_step(pol, min_w, max_w, budget, N, v, pending, st->last_move_s, now, sg, newcap,
                              &gsel, &dir);
    act->kind = kind;
    act->direction = dir;
    act->gpu = gsel;
    for (int g = 0; g < PADSIM_MAX_GPUS; g++) act->new_cap_w[g] = g < N ? v.target(g) : 0;
    if (kind == ACT_MOVE_POWER || kind == ACT_MOVE_GPU)
        for (int g = 0; g < N; g++) act->new_cap_w[g] = newcap[g];
}

// ---------------------------------------------------------------------------
// host validation
// ---------------------------------------------------------------------------
static int validate_model(padsim_ctx* ctx, const padsim_model* m) {
    if (!m) return fail(ctx, PADSIM_EINVAL, "model is NULL");
    if (!(m->min_w > 0 && m->min_w < m->max_w)) return fail(ctx, PADSIM_EMODEL, "min_w/max_w");
    if (m->max_w - m->min_w > 511) return fail(ctx, PADSIM_EMODEL, "cap range wider than 511 W");
    const padsim_curve* cs[2] = {&m->prefill, &m->decode};
    for (const padsim_curve* c : cs) {
        if (c->n < 2 || c->n > PADSIM_MAX_ANCHORS) return fail(ctx, PADSIM_EMODEL, "curve anchor count");
        if (c->w[0] != m->min_w || c->w[c->n - 1] != m->max_w)
            return fail(ctx, PADSIM_EMODEL, "curve must span [min_w, max_w]");
        if (c->s[0] != 1.0) return fail(ctx, PADSIM_EMODEL, "speedup at lowest anchor must be 1.0");
        for (int k = 1; k < c->n; k++) {
            if (!(c->w[k] > c->w[k - 1])) return fail(ctx, PADSIM_EMODEL, "anchors not increasing");
            if (!(c->s[k] >= c->s[k - 1]) || !std::isfinite(c->s[k]))
                return fail(ctx, PADSIM_EMODEL, "speedup not monotone");
        }
    }
    if (!(m->prefill_base_rate > 0 && m->prefill_batch_eff >= 0 && m->decode_fixed_s > 0 &&
          m->decode_per_seq_s >= 0 && m->decode_per_ctx_tok_s >= 0 && m->kv_bytes_per_token > 0 &&
          m->fabric_bw_Bps > 0 && m->transfer_overhead_s > 0))
        return fail(ctx, PADSIM_EMODEL, "model parameters must be positive");
    if (m->max_prefill_batch < 1 || m->max_prefill_batch > PADSIM_MAX_PREFILL_BATCH ||
        m->prefill_token_budget < 1 || m->max_decode_batch < 1 ||
        m->max_decode_batch > PADSIM_MAX_DECODE_BATCH || m->transfer_slots < 1 ||
        m->transfer_slots > PADSIM_MAX_SLOTS || m->prefill_chunk_tokens < 1)
        return fail(ctx, PADSIM_EMODEL, "batch / slot / chunk limits");
    if (m->decode_ctx_growth != 0 && m->decode_ctx_growth != 1)
        return fail(ctx, PADSIM_EMODEL, "decode_ctx_growth must be 0/1");
    return PADSIM_OK;
}

static int validate_policy(padsim_ctx* ctx, const padsim_policy* p, const padsim_model* m, int N,
                           int B) {
    if (p->kind < 0 || p->kind > 4) return fail(ctx, PADSIM_EINVAL, "policy kind");
    if (p->window_stamp < 0 || p->window_stamp > 1) return fail(ctx, PADSIM_EINVAL, "window_stamp must be 0/1");
    if (p->kind == 0 || p->kind == 4) return PADSIM_OK;
    if (!(p->tick_s > 0 && p->settle_s > 0 && p->reassign_s > 0 && p->cooldown_s >= p->settle_s &&
          p->window_s >= 0 && p->power_step_w > 0 && p->queue_threshold >= 0 &&
          p->decode_ceiling_w >= m->min_w && p->decode_ceiling_w <= m->max_w &&
          (long long)N * m->min_w <= B && std::isfinite(p->cooldown_s) && std::isfinite(p->window_s)))
        return fail(ctx, PADSIM_EINVAL, "dynamic policy fields");
    return PADSIM_OK;
}

// stage C instantiation for (context term, 16-bit indices, decode-pool class,
// batch-list variant)
template <int KW, bool BL>
static const void* stagec_fn_kwb(bool cm, bool i16) {
    return cm ? (i16 ? (const void*)stageC_kernel<true, unsigned short, KW, BL> : (const void*)stageC_kernel<true, unsigned, KW, BL>)
              : (i16 ? (const void*)stageC_kernel<false, unsigned short, KW, BL> : (const void*)stageC_kernel<false, unsigned, KW, BL>);
}
template <int KW>
static const void* stagec_fn_kw(bool cm, bool i16, bool bl) {
    return bl ? stagec_fn_kwb<KW, true>(cm, i16) : stagec_fn_kwb<KW, false>(cm, i16);
}
static const void* stagec_fn(bool cm, bool i16, int kc, bool bl) {
    return kc == 0 ? stagec_fn_kw<kc_kw(0)>(cm, i16, bl) : kc == 1 ? stagec_fn_kw<kc_kw(1)>(cm, i16, bl)
         : kc == 2 ? stagec_fn_kw<kc_kw(2)>(cm, i16, bl) : kc == 3 ? stagec_fn_kw<kc_kw(3)>(cm, i16, bl)
                   : stagec_fn_kw<kc_kw(4)>(cm, i16, bl);
}
static void stagec_launch(bool cm, bool i16, int kc, bool bl, int grid, size_t smem, cudaStream_t st,
                          const FPlan& F) {
    void* args[] = {(void*)&F};
    (void)cudaLaunchKernel(stagec_fn(cm, i16, kc, bl), dim3(grid), dim3(kThreads), args, smem, st);   // checked by the caller
}

// joint replay instantiation for (dynamic, CTA size, GPU slots, context term)
template <bool D, int TB, int NG>
static const void* joint_fn_t(bool cx) {
    return cx ? (const void*)joint_kernel<D, TB, NG, true> : (const void*)joint_kernel<D, TB, NG, false>;
}
// lane-group joint replay (group_path.cuh) for (dynamic, context term, CTA size)
template <bool D>
static const void* jointg_fn_t(bool cx, int tb) {
    if (tb == kThreads) return cx ? (const void*)jointg_kernel<D, true, kThreads> : (const void*)jointg_kernel<D, false, kThreads>;
    return cx ? (const void*)jointg_kernel<D, true, 32> : (const void*)jointg_kernel<D, false, 32>;
}
static const void* jointg_fn(bool dyn, bool cx, int tb) { return dyn ? jointg_fn_t<true>(cx, tb) : jointg_fn_t<false>(cx, tb); }
static const void* joint_fn(bool dyn, int tb, int ng, bool cx, bool r168 = false) {
    if (ng == 64) return dyn ? joint_fn_t<true, 32, 64>(cx) : joint_fn_t<false, 32, 64>(cx);
    if (tb == kThreads) return dyn ? joint_fn_t<true, kThreads, 8>(cx) : joint_fn_t<false, kThreads, 8>(cx);
    if (r168)        // one-warp CTAs capped at 168 registers: 10 instead of 8 resident warps per SM
        return dyn ? (cx ? (const void*)joint_kernel<true, 32, 8, true, 168> : (const void*)joint_kernel<true, 32, 8, false, 168>)
                   : (cx ? (const void*)joint_kernel<false, 32, 8, true, 168> : (const void*)joint_kernel<false, 32, 8, false, 168>);
    return dyn ? joint_fn_t<true, 32, 8>(cx) : joint_fn_t<false, 32, 8>(cx);
}

// Groups static candidates by their prefill pool (caps of the prefill GPUs in
// GPU-id order) and lays out stage A / stage C (static_path.cuh).
static int plan_factorized(padsim_ctx* ctx, const padsim_model* model, const padsim_slo* slo, int Q,
                           int S, int Rmax, long long tot, const padsim_candidates* cands) {
    const int N = ctx->N;
    std::map<std::vector<int>, int> gid;
    std::vector<int> gx, gcap;
    struct CC { int group, cand, y; int dcap[kNW]; };
    std::vector<CC> ccs;
    for (int c : ctx->static_list) {
        std::vector<int> pc, dc;
        for (int g = 0; g < N; g++) {
            const int w = cands->cap_w[(size_t)c * N + g];
            (cands->role[(size_t)c * N + g] == 0 ? pc : dc).push_back(w);
        }
        auto it = gid.find(pc);
        int gi;
        if (it == gid.end()) {
            gi = (int)gid.size();
            gid.emplace(pc, gi);
            gx.push_back((int)pc.size());
            for (int w = 0; w < kNW; w++) gcap.push_back(w < (int)pc.size() ? pc[w] : model->min_w);
        } else {
            gi = it->second;
        }
        CC e{};
        e.group = gi;
        e.cand = c;
        e.y = (int)dc.size();
        for (int w = 0; w < kNW; w++) e.dcap[w] = w < e.y ? dc[w] : model->min_w;
        ccs.push_back(e);
    }
    // decode-pool classes: one stage C launch per class with register arrays /
    // shared-memory SoA sized to the class (KW = 1, 2, 4, 5, 7 decode-GPU slots);
    // within a class lanes of a warp are consecutive candidates sorted by prefill
    // group.  Small workloads use three classes (y ≤ 2, ≤ 4, ≤ 7): more, smaller
    // launches leave their SMs latency-bound (measured: cfg 2 45.8 → 51.5 ms with
    // five, cfg 4 621 → 609 ms)
    const long long n_static_rep = (long long)ccs.size() * Q * S;
    const int kcs = ctx->tune.stage_c_classes;
    const bool fine = kcs == 5 || (kcs != 3 && n_static_rep >= 400000LL);
    ctx->kc_fine = fine;
    auto kcls = [fine](int y) { return fine ? kc_class(y) : (y <= 2 ? 1 : y <= 4 ? 2 : kNumKC - 1); };
    std::stable_sort(ccs.begin(), ccs.end(), [&](const CC& a, const CC& b) {
        const int ka = kcls(a.y), kb = kcls(b.y);
        return ka != kb ? ka < kb : a.group < b.group;
    });
    const int G = (int)gx.size(), NC = (int)ccs.size();
    for (int k = 0; k < kNumKC; k++) { ctx->kc_base[k] = 0; ctx->kc_n[k] = 0; }
    for (int k = 0; k < NC; k++) ctx->kc_n[kcls(ccs[k].y)]++;
    for (int k = 1; k < kNumKC; k++) ctx->kc_base[k] = ctx->kc_base[k - 1] + ctx->kc_n[k - 1];
    std::vector<int> cc_cand(NC), cc_group(NC), cc_y(NC), cc_dcap((size_t)NC * kNW);
    for (int k = 0; k < NC; k++) {
        cc_cand[k] = ccs[k].cand; cc_group[k] = ccs[k].group; cc_y[k] = ccs[k].y;
        for (int w = 0; w < kNW; w++) cc_dcap[(size_t)k * kNW + w] = ccs[k].dcap[w];
    }
    // rows of the shared-memory decode step table: the distinct decode caps in use
    std::vector<int> lsl, cc_dslot((size_t)NC * kNW, 0);
    {
        std::map<int, int> row;
        for (int k = 0; k < NC; k++)
            for (int w = 0; w < kNW; w++) row.emplace(cc_dcap[(size_t)k * kNW + w], 0);
        int r = 0;
        for (auto& kv : row) { kv.second = r++; lsl.push_back(kv.first - model->min_w); }
        for (size_t i = 0; i < cc_dcap.size(); i++) cc_dslot[i] = row[cc_dcap[i]];
    }
    FPlan& F = ctx->fplan;
    std::memset(&F, 0, sizeof(F));
    F.m.min_w = model->min_w; F.m.max_w = model->max_w; F.m.ncap = model->max_w - model->min_w + 1;
    F.m.rate = model->prefill_base_rate; F.m.eff = model->prefill_batch_eff;
    F.m.dec_fixed = model->decode_fixed_s; F.m.dec_per_seq = model->decode_per_seq_s;
    F.m.dec_per_ctx = model->decode_per_ctx_tok_s; F.m.kvb = model->kv_bytes_per_token;
    F.m.bw = model->fabric_bw_Bps; F.m.ovh = model->transfer_overhead_s;
    F.m.max_pb = model->max_prefill_batch; F.m.pb_tokens = model->prefill_token_budget;
    F.m.max_db = model->max_decode_batch; F.m.slots = model->transfer_slots;
    F.m.ctx_growth = model->decode_ctx_growth;
    F.m.spre = ctx->d_spre; F.m.sdec = ctx->d_sdec; F.m.den = ctx->d_den; F.m.ltab = ctx->d_ltab;
    F.N = N; F.Q = Q; F.S = S; F.Rmax = std::max(Rmax, 1);
    F.toff = ctx->d_toff; F.nreq = ctx->d_nreq; F.s_unit = ctx->d_s_unit; F.kv = ctx->d_kv;
    F.in_tok = ctx->d_in; F.out_tok = ctx->d_out; F.phase = ctx->d_phase; F.qps = ctx->d_qps;
    F.ttft_slo = slo->ttft_s; F.tpot_slo0 = slo->tpot_s[0]; F.tpot_slo1 = slo->tpot_s[1];
    F.n_groups = G;
    F.n_cc = NC;
    F.s_begin = 0;
    F.s_count = S;
    int *d_gx, *d_gcap, *d_ccc, *d_ccg, *d_ccy, *d_ccd;
    double* d_pe;
    SRec* d_rec;
    SHot* d_hot;
    long long* d_evA;
    double *d_asq, *d_ase;
    const long long GQS = (long long)G * Q * S;
    const size_t Rm = (size_t)F.Rmax;
#define AL(p, n) do { int r_ = dalloc(ctx, &(p), (size_t)(n)); if (r_) return r_; } while (0)
    AL(d_gx, G); AL(d_gcap, (size_t)G * kNW); AL(d_ccc, NC); AL(d_ccg, NC); AL(d_ccy, NC);
    AL(d_ccd, (size_t)NC * kNW);
    int *d_lsl, *d_ccsl;
    AL(d_lsl, std::max<size_t>(lsl.size(), 1)); AL(d_ccsl, (size_t)NC * kNW);
    CK(cudaMemcpy(d_lsl, lsl.data(), sizeof(int) * lsl.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ccsl, cc_dslot.data(), sizeof(int) * NC * kNW, cudaMemcpyHostToDevice));
    F.lsl = d_lsl; F.cc_dslot = d_ccsl; F.c_lslots = (int)lsl.size();
    AL(d_rec, GQS * Rm); AL(d_hot, GQS * Rm); AL(d_pe, GQS * Rm); AL(d_evA, GQS);
    AL(d_asq, GQS); AL(d_ase, GQS);
    CK(cudaMemcpy(d_gx, gx.data(), sizeof(int) * G, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_gcap, gcap.data(), sizeof(int) * G * kNW, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ccc, cc_cand.data(), sizeof(int) * NC, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ccg, cc_group.data(), sizeof(int) * NC, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ccy, cc_y.data(), sizeof(int) * NC, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ccd, cc_dcap.data(), sizeof(int) * NC * kNW, cudaMemcpyHostToDevice));
    F.gx = d_gx; F.gcap = d_gcap; F.cc_cand = d_ccc; F.cc_group = d_ccg; F.cc_y = d_ccy; F.cc_dcap = d_ccd;
    F.st_rec = d_rec; F.st_hot = d_hot; F.st_pe = d_pe; F.evA = d_evA;
    F.a_sq = d_asq; F.a_se = d_ase;
    ctx->d_evA = d_evA;
    ctx->n_evA = (int)GQS;
    // stage A scratch per warp: per-lane prompt rings (kNW workers + the KV-wait
    // FIFO, R entries each) and lane-interleaved KV slots (128-thread CTAs)
    {
        size_t off = 0;
        auto take = [&](size_t b) { size_t o = off; off += (b + 255) & ~(size_t)255; return o; };
        F.a_ring_lane = (size_t)(kNW + 1) * Rm;
        F.a_off_ring = take((size_t)32 * F.a_ring_lane * sizeof(int));
        F.a_off_tte = take((size_t)PADSIM_MAX_SLOTS * 32 * sizeof(double));
        F.a_off_tid = take((size_t)PADSIM_MAX_SLOTS * 32 * sizeof(int));
        F.a_off_tpe = take((size_t)PADSIM_MAX_SLOTS * 32 * sizeof(double));
        F.a_warp_bytes = off;
        // small stage-A workloads (e.g. cfg 2: 12k replays) use 32-thread CTAs so every SM
        // gets some of the latency-bound replays; large ones use 128-thread CTAs
        // large ones use 256-thread CTAs: the staged trace is shared by 8 warps
        // and shared memory then holds 16 resident warps per SM instead of 12
        int tb = GQS >= (long long)ctx->n_sm * 2 * kThreads ? kThreads : 32;
        if (tb == kThreads && GQS >= (long long)ctx->n_sm * 2 * 256) tb = kATbBig;
        {
            const int v = ctx->tune.stage_a_threads;             // padsim_set_tuning override
            if (v == 32 || v == kThreads || v == kATbBig) tb = v;
        }
        ctx->fA_tb = tb;
        F.a_blocks_per_trace = (int)(((long long)Q * G + tb - 1) / tb);
        const long long ctas = (long long)F.a_blocks_per_trace * S;
        char* scr;
        AL(scr, (size_t)ctas * (tb / 32) * off);
        F.scrA = scr;
        ctx->fA_grid = (int)ctas;
        const size_t Rp = (Rm + 15) & ~(size_t)15;
        const size_t tb_bytes = Rp * (8 + 8 + 4);
        const size_t wbytes = tb == kATbBig ? a_work_bytes<kATbBig>() + a_slot_bytes<kATbBig>()
                            : tb == kThreads ? a_work_bytes<kThreads>() + a_slot_bytes<kThreads>()
                                             : a_work_bytes<32>() + a_slot_bytes<32>();
        F.a_smem_trace = wbytes + tb_bytes <= 200 * 1024 ? 1 : 0;
        ctx->fA_smem = wbytes + (F.a_smem_trace ? tb_bytes : 0);
        const void* fa = tb == kATbBig ? (const void*)stageA_kernel<kATbBig>
                       : tb == kThreads ? (const void*)stageA_kernel<kThreads> : (const void*)stageA_kernel<32>;
        CK(cudaFuncSetAttribute(fa, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->fA_smem));
    }
    // stage C: CTAs bound to one trace each (staged in smem by TMA bulk copies),
    // warps pull 32-replay items from that trace's counter
    {
        size_t off = 0;
        auto take = [&](size_t b) { size_t o = off; off += (b + 255) & ~(size_t)255; return o; };
        const bool idx16 = Rm <= 16383;          // 14-bit stream index + round + chain flags
        ctx->fC_idx16 = idx16;
        const size_t isz = idx16 ? 2 : 4;
        take(Rm * 32 * isz);
        int maxo = 2;
        for (int s2 = 0; s2 < S; s2++) maxo = std::max(maxo, ctx->max_out[s2]);
        int wheel = 32;
        while (wheel < maxo) wheel <<= 1;        // finish steps lie in (step, step + out − 1]
        F.wheel = wheel;
        F.c_off_heads = take((size_t)32 * kNW * wheel * isz);   // per lane KW × (Wh, or Wh / 2 for KW = 4 / 5)
        F.c_off_bits = take((size_t)kNW * (wheel / 32) * 32 * sizeof(unsigned));
        int rb = 1;
        while (rb < model->max_decode_batch) rb <<= 1;
        F.c_rb = rb;
        F.c_off_ring = take((size_t)32 * kNW * rb * sizeof(unsigned long long));
        F.c_warp_bytes = off;
        unsigned* d_wc;
        AL(d_wc, (size_t)kNumKC * S);             // work counters per (class, trace)
        F.work = d_wc;
        ctx->d_workC = d_wc;
        const bool ctxm = model->decode_per_ctx_tok_s != 0.0;
        F.bits_in_smem = wheel <= 256 ? 1 : 0;
        F.c_prefetch = 1;
        // measured (cfg 4): the lane clock window slows stage C (683 -> 721 ms at
        // 16-64 inter-arrivals, 780 at 4) — its stream reads already coalesce
        // well enough — so it is off here; the joint kernel gains from it
        F.sync_win = 0.f;
        F.smem_trace = 0;
        size_t fr = 0, tm = 0;
        CK(cudaMemGetInfo(&fr, &tm));
        const size_t per_cta = off * kWarps;
        const long long cap_ctas = std::max<long long>(S, (long long)((tm * 3 / 10) / per_cta));
        long long grid_max = S;
        for (int kc = 0; kc < kNumKC; kc++) {
            ctx->kc_grid[kc] = 0;
            if (ctx->kc_n[kc] == 0) continue;
            const int KWc = kc_kw(kc);
            // batch-list variant per class: padsim_tuning.stage_c_batch_lists (bit kc) overrides the default
            // (measured: the KW = 7 class of large workloads gains from the freed shared
            // memory — 16 instead of 12 resident warps per SM: cfg 4 610 → 584 ms; the
            // others lose — all classes 700 ms, cfg 2's KW = 7 class 46.6 → 47.3 ms)
            int blmask = ctx->kc_fine ? (1 << (kNumKC - 1)) : 0;
            if (ctx->tune.stage_c_batch_lists >= 0) blmask = ctx->tune.stage_c_batch_lists;
            const bool blc = (blmask >> kc) & 1;
            ctx->kc_bl[kc] = blc;
            const size_t wbytes = (size_t)KWc * kThreads *
                                  (kCWorkSlotBytes + (blc ? sizeof(int) : 0) + (ctxm ? kCWorkCtxSlotBytes : 0));
            const size_t bbytes = (size_t)KWc * (wheel / 32) * kThreads * sizeof(unsigned);
            const int bsm = blc ? 0 : F.bits_in_smem;
            ctx->kc_bits_smem[kc] = bsm;
            ctx->kc_off_sdec[kc] = wbytes + (bsm ? bbytes : 0);
            const size_t base = ctx->kc_off_sdec[kc] + (size_t)F.m.ncap * sizeof(double);
            const void* fn = stagec_fn(ctxm, idx16, kc, blc);
            auto occ_of = [&](size_t sm) {      // resident CTAs per SM (0: does not fit)
                int o = 0;
                if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess ||
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, kThreads, sm) != cudaSuccess) {
                    (void)cudaGetLastError();
                    return 0;
                }
                return o;
            };
            const int occ0 = occ_of(base);
            // shared-memory extras, each kept only when it costs no resident CTA:
            // the async head cache ([KW][kThreads] words) and the decode step table
            const size_t hbytes = (size_t)KWc * kThreads * sizeof(unsigned);
            const size_t lbytes = (size_t)F.c_lslots * F.m.max_db * sizeof(double);
            size_t sm = base;
            ctx->kc_hca[kc] = occ_of(sm + hbytes) >= occ0;
            ctx->kc_off_hca[kc] = sm;
            if (ctx->kc_hca[kc]) sm += hbytes;
            ctx->kc_ltab[kc] = !ctxm && F.c_lslots <= kLtabRows && occ_of(sm + lbytes) >= occ0;
            ctx->kc_off_ltab[kc] = sm;
            if (ctx->kc_ltab[kc]) sm += lbytes;
            ctx->kc_smem[kc] = sm;
            int occ = occ_of(sm);
            if (occ == 0) return fail(ctx, PADSIM_ECUDA, "stage C shared memory does not fit");
            occ = std::max(occ, 1);
            const long long items = ((long long)Q * ctx->kc_n[kc] + 31) / 32;   // warp items per trace
            long long per_trace = std::max<long long>(1, ((long long)ctx->n_sm * occ) / S);
            per_trace = std::min<long long>(per_trace, (items + kWarps - 1) / kWarps);
            long long grid = std::min<long long>(per_trace * S, (cap_ctas / S) * S);
            grid = std::max<long long>(grid, S);
            ctx->kc_grid[kc] = (int)grid;
            grid_max = std::max(grid_max, grid);
        }
        // classes run concurrently: each has its own scratch slice
        for (int kc = 0; kc < kNumKC; kc++) {
            ctx->kc_scr[kc] = nullptr;
            if (ctx->kc_n[kc] == 0) continue;
            char* scr;
            AL(scr, (size_t)ctx->kc_grid[kc] * per_cta);
            ctx->kc_scr[kc] = scr;
        }
        F.scrC = nullptr;
        ctx->fC_grid = (int)grid_max;
        // the joint replays start with stage A (they do not depend on it): a small
        // stage A (cfg 3) is latency-bound, and next to a large one (cfg 4) the
        // 168-register joint CTAs take the SM slots stage A's waves leave free
        // (measured: cfg 4 524 -> 506 ms/step against starting after stage A)
        ctx->j_with_a = ctx->tune.joint_after_stage_a != 1;
    }
    F.rep_met = ctx->d_rep_met; F.rep_near = ctx->d_rep_near; F.rep_dur = ctx->d_rep_dur;
    F.rep_good = ctx->d_rep_good; F.rep_events = ctx->d_rep_events;
    if (ctx->flags & PADSIM_RECORDS) {
        F.rec_ttft = ctx->d_rec[0]; F.rec_tpot = ctx->d_rec[1]; F.rec_pe = ctx->d_rec[2];
        F.rec_comp = ctx->d_rec[3]; F.rec_te = ctx->d_rec[4];
    }
#undef AL
    (void)tot;
    return PADSIM_OK;
}

// Wide nodes (8 < N ≤ 64): groups static candidates by prefill pool as
// plan_factorized does and lays out the warp-per-replay stages (wide_path.cuh).
// The stage A → C stream (40 B per request per (group, QPS, trace)) is sized
// for a chunk of traces; padsim_run replays the traces chunk by chunk.
static int plan_wide(padsim_ctx* ctx, const padsim_model* model, const padsim_slo* slo, int Q, int S,
                     int Rmax, const padsim_candidates* cands) {
    const int N = ctx->N;
    std::map<std::vector<int>, int> gid;
    std::vector<int> gx, gcap;
    struct CC { int group, cand, y; std::vector<int> dc; };
    std::vector<CC> ccs;
    for (int c : ctx->static_list) {
        std::vector<int> pc, dc;
        for (int g = 0; g < N; g++) {
            const int w = cands->cap_w[(size_t)c * N + g];
            (cands->role[(size_t)c * N + g] == 0 ? pc : dc).push_back(w);
        }
        auto it = gid.find(pc);
        int gi;
        if (it == gid.end()) {
            gi = (int)gid.size();
            gid.emplace(pc, gi);
            gx.push_back((int)pc.size());
            for (int w = 0; w < kWMax; w++) gcap.push_back(w < (int)pc.size() ? pc[w] : model->min_w);
        } else {
            gi = it->second;
        }
        ccs.push_back(CC{gi, c, (int)dc.size(), dc});
    }
    // warps of a CTA take consecutive candidates of one prefill group (same stream)
    std::stable_sort(ccs.begin(), ccs.end(), [](const CC& a, const CC& b) { return a.group < b.group; });
    const int G = (int)gx.size(), NC = (int)ccs.size();
    std::vector<int> cc_cand(NC), cc_group(NC), cc_y(NC), cc_dcap((size_t)NC * kWMax);
    for (int k = 0; k < NC; k++) {
        cc_cand[k] = ccs[k].cand; cc_group[k] = ccs[k].group; cc_y[k] = ccs[k].y;
        for (int w = 0; w < kWMax; w++)
            cc_dcap[(size_t)k * kWMax + w] = w < ccs[k].y ? ccs[k].dc[w] : model->min_w;
    }
    FPlan& F = ctx->fplan;
    std::memset(&F, 0, sizeof(F));
    F.m.min_w = model->min_w; F.m.max_w = model->max_w; F.m.ncap = model->max_w - model->min_w + 1;
    F.m.rate = model->prefill_base_rate; F.m.eff = model->prefill_batch_eff;
    F.m.dec_fixed = model->decode_fixed_s; F.m.dec_per_seq = model->decode_per_seq_s;
    F.m.dec_per_ctx = model->decode_per_ctx_tok_s; F.m.kvb = model->kv_bytes_per_token;
    F.m.bw = model->fabric_bw_Bps; F.m.ovh = model->transfer_overhead_s;
    F.m.max_pb = model->max_prefill_batch; F.m.pb_tokens = model->prefill_token_budget;
    F.m.max_db = model->max_decode_batch; F.m.slots = model->transfer_slots;
    F.m.ctx_growth = model->decode_ctx_growth;
    F.m.spre = ctx->d_spre; F.m.sdec = ctx->d_sdec; F.m.den = ctx->d_den; F.m.ltab = ctx->d_ltab;
    F.N = N; F.Q = Q; F.S = S; F.Rmax = std::max(Rmax, 1);
    F.toff = ctx->d_toff; F.nreq = ctx->d_nreq; F.s_unit = ctx->d_s_unit; F.kv = ctx->d_kv;
    F.in_tok = ctx->d_in; F.out_tok = ctx->d_out; F.phase = ctx->d_phase; F.qps = ctx->d_qps;
    F.ttft_slo = slo->ttft_s; F.tpot_slo0 = slo->tpot_s[0]; F.tpot_slo1 = slo->tpot_s[1];
    F.n_groups = G;
    F.n_cc = NC;
    const size_t Rm = (size_t)F.Rmax;
    const long long GQS = (long long)G * Q * S;
    // traces per chunk: the stream of one trace is G·Q·Rmax·40 B (cfg 5: 26.8 GB)
    size_t fr = 0, tm = 0;
    CK(cudaMemGetInfo(&fr, &tm));
    const size_t per_trace = (size_t)G * Q * Rm * (sizeof(SRec) + sizeof(SHot) + sizeof(double));
    const size_t budget = fr / 2;
    int chunk = (int)std::min<size_t>((size_t)S, std::max<size_t>(1, budget / std::max<size_t>(per_trace, 1)));
    if (ctx->tune.wide_chunk > 0) chunk = std::min(S, (int)ctx->tune.wide_chunk);
    chunk = std::max(chunk, 1);
    if (S > 0) {        // balanced chunks (cfg 5: 2 + 2 traces rather than 3 + 1)
        const int nch = (S + chunk - 1) / chunk;
        chunk = (S + nch - 1) / nch;
    }
    ctx->w_chunk = chunk;
    const long long GQC = (long long)G * Q * chunk;
#define AL(p, n) do { int r_ = dalloc(ctx, &(p), (size_t)(n)); if (r_) return r_; } while (0)
    int *d_gx, *d_gcap, *d_ccc, *d_ccg, *d_ccy, *d_ccd;
    AL(d_gx, G); AL(d_gcap, (size_t)G * kWMax); AL(d_ccc, NC); AL(d_ccg, NC); AL(d_ccy, NC);
    AL(d_ccd, (size_t)NC * kWMax);
    CK(cudaMemcpy(d_gx, gx.data(), sizeof(int) * G, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_gcap, gcap.data(), sizeof(int) * G * kWMax, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ccc, cc_cand.data(), sizeof(int) * NC, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ccg, cc_group.data(), sizeof(int) * NC, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ccy, cc_y.data(), sizeof(int) * NC, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ccd, cc_dcap.data(), sizeof(int) * NC * kWMax, cudaMemcpyHostToDevice));
    F.gx = d_gx; F.w_gcap = d_gcap; F.cc_cand = d_ccc; F.cc_group = d_ccg; F.cc_y = d_ccy; F.w_dcap = d_ccd;
    SRec* d_rec;
    SHot* d_hot;
    double* d_pe;
    long long* d_evA;
    double *d_asq, *d_ase;
    AL(d_rec, GQC * Rm); AL(d_hot, GQC * Rm); AL(d_pe, GQC * Rm);
    AL(d_evA, GQS); AL(d_asq, GQS); AL(d_ase, GQS);
    F.st_rec = d_rec; F.st_hot = d_hot; F.st_pe = d_pe; F.evA = d_evA; F.a_sq = d_asq; F.a_se = d_ase;
    ctx->d_evA = d_evA;
    ctx->n_evA = (int)GQS;
    int rb = 1;
    while (rb < model->max_decode_batch) rb <<= 1;
    F.c_rb = rb;
    F.a_warp_bytes = wide_a_layout(Rm).bytes;
    F.c_warp_bytes = wide_c_layout(Rm, rb).bytes;
    AL(ctx->d_workW, (size_t)2 * S);
    // one warp per replay; CTAs (4 warps) bound to one trace of the chunk, warps pull
    // replays from that trace's counter; scratch per resident warp
    // resident CTAs of a launch (the whole GPU, capped by a scratch budget of 20 % of the
    // free memory, at least one per trace of a chunk); padsim_run splits them over the
    // traces of each chunk, so a short last chunk still fills the GPU
    auto grid_of = [&](const void* fn, size_t warp_bytes, long long& grid) -> int {
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, 0));
        occ = std::max(occ, 1);
        const long long cap = std::max<long long>(1, (long long)((double)fr * 0.2 / ((double)warp_bytes * kWarps)));
        grid = std::max<long long>(chunk, std::min<long long>((long long)ctx->n_sm * occ, cap));
        return PADSIM_OK;
    };
    long long ga = 0, gc = 0;
    if (int r_ = grid_of((const void*)stageA_wide_kernel, F.a_warp_bytes, ga)) return r_;
    if (int r_ = grid_of((const void*)stageC_wide_kernel, F.c_warp_bytes, gc)) return r_;
    ctx->wA_grid = (int)ga;
    ctx->wC_grid = (int)gc;
    ctx->wA_items = (long long)Q * G;
    ctx->wC_items = (long long)Q * NC;
    char *sa, *sc;
    AL(sa, (size_t)ga * kWarps * F.a_warp_bytes);
    AL(sc, (size_t)gc * kWarps * F.c_warp_bytes);
    F.scrA = sa;
    F.scrC = sc;
    F.rep_met = ctx->d_rep_met; F.rep_near = ctx->d_rep_near; F.rep_dur = ctx->d_rep_dur;
    F.rep_good = ctx->d_rep_good; F.rep_events = ctx->d_rep_events;
    if (ctx->flags & PADSIM_RECORDS) {
        F.rec_ttft = ctx->d_rec[0]; F.rec_tpot = ctx->d_rec[1]; F.rec_pe = ctx->d_rec[2];
        F.rec_comp = ctx->d_rec[3]; F.rec_te = ctx->d_rec[4];
    }
#undef AL
    return PADSIM_OK;
}

extern "C" {

const char* padsim_version(void) { return kVersion; }

int padsim_create(int32_t dev, void* stream, padsim_ctx** out) {
    if (!out) return PADSIM_EINVAL;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0 || dev < 0 || dev >= n) {
        cudaGetLastError();
        return PADSIM_ECUDA;
    }
    padsim_ctx* ctx = new (std::nothrow) padsim_ctx();
    if (!ctx) return PADSIM_ENOMEM;
    ctx->device = dev;
    ctx->stream = (cudaStream_t)stream;
    if (cudaSetDevice(dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&ctx->n_sm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        cudaGetLastError();
        delete ctx;
        return PADSIM_ECUDA;
    }
    *out = ctx;
    return PADSIM_OK;
}

void padsim_destroy(padsim_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    free_plan(ctx);
    release_buffers(ctx);
    if (ctx->d_ctl_state) cudaFree(ctx->d_ctl_state);
    if (ctx->d_ctl_act) cudaFree(ctx->d_ctl_act);
    if (ctx->d_ctl_stats) cudaFree(ctx->d_ctl_stats);
    for (auto e : ctx->evW) cudaEventDestroy(e);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->evA) cudaEventDestroy(ctx->evA);
    if (ctx->evC) cudaEventDestroy(ctx->evC);
    if (ctx->evJ0) cudaEventDestroy(ctx->evJ0);
    if (ctx->evJ1) cudaEventDestroy(ctx->evJ1);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->evC0) cudaEventDestroy(ctx->evC0);
    for (auto& x : ctx->sideC) if (x) cudaStreamDestroy(x);
    for (auto& e : ctx->evCk) if (e) cudaEventDestroy(e);
    if (ctx->evCf) cudaEventDestroy(ctx->evCf);
    delete ctx;
}

const char* padsim_last_error(const padsim_ctx* ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

int padsim_enumerate_pool_uniform(int32_t n_gpus, int32_t budget_w, int32_t min_w, int32_t max_w,
                                  int32_t step_w, int32_t exact, int32_t* out_xpd, int32_t cap,
                                  int32_t* n_out) {
    if (!n_out || n_gpus < 2 || n_gpus > PADSIM_MAX_GPUS || step_w <= 0 || min_w <= 0 ||
        min_w > max_w || cap < 0)
        return PADSIM_EINVAL;
    int32_t cnt = 0;
    const int levels = (max_w - min_w) / step_w + 1;
    for (int x = 1; x < n_gpus; x++) {
        const long long y = n_gpus - x;
        for (int a = 0; a < levels; a++) {
            const long long p = min_w + (long long)a * step_w;
            // largest d with x*p + y*d <= B (or == B): a closed-form bound per p
            const long long rem = (long long)budget_w - x * p;
            if (rem < y * min_w) break;            // p increasing: no larger p fits either
            long long dmax = rem / y;
            if (dmax > max_w) dmax = max_w;
            const long long kmax = (dmax - min_w) / step_w;
            for (long long k = 0; k <= kmax; k++) {
                const long long d = min_w + k * step_w;
                if (exact && x * p + y * d != budget_w) continue;
                if (out_xpd && cnt < cap) {
                    out_xpd[3 * cnt + 0] = x;
                    out_xpd[3 * cnt + 1] = (int32_t)p;
                    out_xpd[3 * cnt + 2] = (int32_t)d;
                }
                cnt++;
            }
        }
    }
    *n_out = cnt;
    return PADSIM_OK;
}

int padsim_plan(padsim_ctx* ctx, const padsim_trace* traces, int32_t n_traces,
                const double* qps, int32_t n_qps, const padsim_model* model,
                const padsim_candidates* cands, const padsim_slo* slo,
                const padsim_budget* budget, uint32_t flags, int32_t* bad_index) {
    if (!ctx) return PADSIM_EINVAL;
    if (bad_index) *bad_index = -1;
    CK(cudaSetDevice(ctx->device));
    free_plan(ctx);
    if (!traces || n_traces < 1 || !qps || n_qps < 1 || !cands || !slo || !budget)
        return fail(ctx, PADSIM_EINVAL, "null input or empty dimension");
    int rc = validate_model(ctx, model);
    if (rc) return rc;
    const int N = cands->n_gpus, C = cands->n_cand, B = budget->budget_w;
    const int32_t* cbud = budget->cand_budget_w;     // nullable: one budget per candidate
    if (N < 2 || N > PADSIM_MAX_GPUS || C < 1 || !cands->role || !cands->cap_w || !cands->policy)
        return fail(ctx, PADSIM_EINVAL, "candidates");
    if (!(slo->ttft_s > 0 && slo->tpot_s[0] > 0 && slo->tpot_s[1] > 0))
        return fail(ctx, PADSIM_EINVAL, "SLOs must be > 0");
    for (int q = 0; q < n_qps; q++)
        if (!(qps[q] > 0) || !std::isfinite(qps[q])) return fail(ctx, PADSIM_EINVAL, "qps must be > 0");
    std::vector<int> capsum(C), cbudget(C);
    for (int c = 0; c < C; c++) {
        const int Bc = cbud ? cbud[c] : B;
        cbudget[c] = Bc;
        int np = 0;
        long long cs = 0;
        for (int g = 0; g < N; g++) {
            const int r = cands->role[(size_t)c * N + g];
            const int w = cands->cap_w[(size_t)c * N + g];
            if (r > 1) { if (bad_index) *bad_index = c; return fail(ctx, PADSIM_EROLE, "role must be 0/1"); }
            np += r == 0;
            if (w < model->min_w || w > model->max_w) {
                if (bad_index) *bad_index = c;
                return fail(ctx, PADSIM_ERANGE, "cap outside [min_w, max_w]");
            }
            cs += w;
        }
        const bool coal = cands->policy[c].kind == 4;     // roles ignored (A33)
        if (!coal && (np < 1 || np > N - 1)) {
            if (bad_index) *bad_index = c;
            return fail(ctx, PADSIM_EROLE, "need >= 1 prefill and >= 1 decode GPU");
        }
        if (cs > Bc) {
            if (bad_index) *bad_index = c;
            return fail(ctx, PADSIM_EBUDGET, "sum of caps exceeds the node budget");
        }
        rc = validate_policy(ctx, &cands->policy[c], model, N, Bc);
        if (rc) { if (bad_index) *bad_index = c; return rc; }
        capsum[c] = (int)cs;
    }
    // traces
    std::vector<long long> toff(n_traces + 1);
    int Rmax = 0;
    long long tot = 0;
    for (int s = 0; s < n_traces; s++) {
        const padsim_trace& t = traces[s];
        if (t.n_req < 0 || (t.n_req > 0 && (!t.s_unit || !t.in_tok || !t.out_tok)))
            return fail(ctx, PADSIM_EINVAL, "trace arrays");
        for (int i = 0; i < t.n_req; i++) {
            if (t.in_tok[i] < 1 || t.out_tok[i] < 1) return fail(ctx, PADSIM_EDOMAIN, "token count < 1");
            if (!(t.s_unit[i] >= 0) || !std::isfinite(t.s_unit[i]))
                return fail(ctx, PADSIM_EDOMAIN, "arrival not finite / negative");
            if (i > 0 && !(t.s_unit[i] >= t.s_unit[i - 1])) return fail(ctx, PADSIM_EDOMAIN, "arrivals unsorted");
            if (t.phase && t.phase[i] > 1) return fail(ctx, PADSIM_EINVAL, "phase must be 0/1");
        }
        toff[s] = tot;
        tot += (t.n_req + 15) & ~15;
        Rmax = std::max(Rmax, t.n_req);
    }
    toff[n_traces] = tot;
    ctx->N = N; ctx->C = C; ctx->Q = n_qps; ctx->S = n_traces; ctx->Rmax = Rmax;
    ctx->model = *model;
    ctx->slo = *slo;
    ctx->flags = flags;
    ctx->capsum_h = capsum;
    ctx->toff = toff;
    for (int c = 0; c < C; c++) {
        const int k = cands->policy[c].kind;
        (k == 0 ? ctx->static_list : k == 4 ? ctx->coal_list : ctx->dyn_list).push_back(c);
    }

    // host staging of the padded SoA trace arrays
    std::vector<double> hs(tot, 0.0);
    std::vector<int> hin(tot, 1), hout(tot, 1);
    std::vector<unsigned char> hph(tot, 0);
    std::vector<int> nreq(n_traces);
    ctx->max_out.assign(n_traces, 1);
    for (int s2 = 0; s2 < n_traces; s2++)
        for (int i = 0; i < traces[s2].n_req; i++)
            ctx->max_out[s2] = std::max(ctx->max_out[s2], (int)traces[s2].out_tok[i]);
    for (int s = 0; s < n_traces; s++) {
        const padsim_trace& t = traces[s];
        nreq[s] = t.n_req;
        if (t.n_req == 0) continue;
        std::memcpy(&hs[toff[s]], t.s_unit, sizeof(double) * t.n_req);
        std::memcpy(&hin[toff[s]], t.in_tok, sizeof(int) * t.n_req);
        std::memcpy(&hout[toff[s]], t.out_tok, sizeof(int) * t.n_req);
        if (t.phase) std::memcpy(&hph[toff[s]], t.phase, t.n_req);
    }
    const long long CQ = (long long)C * n_qps, R_all = CQ * n_traces;
    const int ncap = model->max_w - model->min_w + 1;
#define AL(p, n) do { int r_ = dalloc(ctx, &(p), (size_t)(n)); if (r_) return r_; } while (0)
    AL(ctx->d_toff, n_traces + 1);
    AL(ctx->d_nreq, n_traces);
    AL(ctx->d_s_unit, tot);
    AL(ctx->d_kv, tot);
    AL(ctx->d_in, tot);
    AL(ctx->d_out, tot);
    AL(ctx->d_phase, tot);
    AL(ctx->d_role, (size_t)C * N);
    AL(ctx->d_cap, (size_t)C * N);
    AL(ctx->d_capsum, C);
    AL(ctx->d_cbud, C);
    AL(ctx->d_pol, C);
    AL(ctx->d_qps, n_qps);
    AL(ctx->d_clist_static, std::max<size_t>(1, ctx->static_list.size()));
    AL(ctx->d_clist_dyn, std::max<size_t>(1, ctx->dyn_list.size()));
    AL(ctx->d_clist_coal, std::max<size_t>(1, ctx->coal_list.size()));
    AL(ctx->d_spre, ncap);
    AL(ctx->d_sdec, ncap);
    AL(ctx->d_den, model->max_prefill_batch + 1);
    AL(ctx->d_ltab, (size_t)ncap * model->max_decode_batch);
    AL(ctx->d_rep_met, R_all);
    AL(ctx->d_rep_near, R_all);
    AL(ctx->d_rep_dur, R_all);
    AL(ctx->d_rep_good, R_all);
    AL(ctx->d_rep_events, R_all);
    AL(ctx->d_met, CQ);
    AL(ctx->d_good, CQ);
    AL(ctx->d_near, CQ);
    AL(ctx->d_argmax, n_qps);
    AL(ctx->d_rep_metk, R_all * kMaxSloSweep);
    AL(ctx->d_rep_watts, R_all);
    AL(ctx->d_metk, CQ * kMaxSloSweep);
    AL(ctx->d_qpw, CQ);
    AL(ctx->d_watts, CQ);
    AL(ctx->d_max80, (long long)C * (1 + kMaxSloSweep));
    AL(ctx->d_rep_sq, R_all);
    AL(ctx->d_rep_se, R_all);
    AL(ctx->d_qsum, CQ);
    AL(ctx->d_esum, CQ);
    ctx->sweep = SloSweep{};
    ctx->sweep.rep_met = ctx->d_rep_metk;
    ctx->sweep.rep_watts = ctx->d_rep_watts;
    ctx->sweep.rep_sq = ctx->d_rep_sq;
    ctx->sweep.rep_se = ctx->d_rep_se;
    ctx->sweep.capsum = ctx->d_capsum;
    ctx->n_req_total = 0;
    for (int s2 = 0; s2 < n_traces; s2++) ctx->n_req_total += traces[s2].n_req;
    AL(ctx->d_work, 4);
    if (flags & PADSIM_RECORDS) {
        for (auto& r : ctx->d_rec) AL(r, (size_t)R_all * std::max(Rmax, 1));
        AL(ctx->d_pct, kMaxPct);
        AL(ctx->d_pct_out, (size_t)R_all * 2 * kMaxPct);
        int n2 = 1;
        while (n2 < Rmax) n2 <<= 1;
        ctx->pct_n2 = n2;
        if ((size_t)n2 * sizeof(double) <= kPctSmemMax) {
            ctx->pct_smem = (size_t)n2 * sizeof(double);
            ctx->pct_grid = (int)std::min<long long>(R_all, (long long)ctx->n_sm * 8);
            ctx->d_pct_scratch = nullptr;
        } else {
            ctx->pct_smem = 0;
            ctx->pct_grid = (int)std::min<long long>(R_all, (long long)ctx->n_sm * 2);
            AL(ctx->d_pct_scratch, (size_t)ctx->pct_grid * n2);
        }
        CK(cudaFuncSetAttribute(percentile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kPctSmemMax));
    }
    CK(cudaMemcpy(ctx->d_toff, toff.data(), sizeof(long long) * (n_traces + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_nreq, nreq.data(), sizeof(int) * n_traces, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_s_unit, hs.data(), sizeof(double) * tot, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_in, hin.data(), sizeof(int) * tot, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_out, hout.data(), sizeof(int) * tot, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_phase, hph.data(), tot, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_role, cands->role, (size_t)C * N, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_cap, cands->cap_w, sizeof(int) * (size_t)C * N, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_capsum, capsum.data(), sizeof(int) * C, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_cbud, cbudget.data(), sizeof(int) * C, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_pol, cands->policy, sizeof(padsim_policy) * C, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_qps, qps, sizeof(double) * n_qps, cudaMemcpyHostToDevice));
    if (!ctx->static_list.empty())
        CK(cudaMemcpy(ctx->d_clist_static, ctx->static_list.data(), sizeof(int) * ctx->static_list.size(),
                      cudaMemcpyHostToDevice));
    if (!ctx->dyn_list.empty())
        CK(cudaMemcpy(ctx->d_clist_dyn, ctx->dyn_list.data(), sizeof(int) * ctx->dyn_list.size(),
                      cudaMemcpyHostToDevice));
    if (!ctx->coal_list.empty())
        CK(cudaMemcpy(ctx->d_clist_coal, ctx->coal_list.data(), sizeof(int) * ctx->coal_list.size(),
                      cudaMemcpyHostToDevice));
    tables_kernel<<<std::max(1, ctx->n_sm), 256>>>(*model, ctx->d_spre, ctx->d_sdec, ctx->d_den,
                                                    ctx->d_ltab, ctx->d_in, ctx->d_kv, tot);
    CK(cudaGetLastError());

    // factorized static path (stage A prefill groups -> stage C decode) for N <= 8
    // Few static replays (≤ 8 per SM: cfg 1's 13, cfg 3's 160) leave the thread-per-replay
    // stages latency-bound — one serial chain per thread, ~3 µs per request — and they
    // take the warp-per-replay wide path instead (wide_path.cuh works for any N ≤ 64):
    // measured cfg 1 1.40 → 0.83 ms, cfg 3 310 → 271 ms per step (its 160 static
    // replays were a 258 ms stage A → C chain next to the joint replays), cfg 2 (122 k
    // replays) 44 → 197 ms the other way.  padsim_tuning.wide_path = 1 forces it, 0 never.
    const long long n_static_rep = (long long)ctx->static_list.size() * n_qps * n_traces;
    const bool wide_small = N <= 8 && model->decode_per_ctx_tok_s == 0.0 && ctx->tune.wide_path != 0 &&
                            (ctx->tune.wide_path == 1 || n_static_rep <= (long long)ctx->n_sm * 8);
    ctx->fact = N <= 8 && !wide_small && !ctx->static_list.empty() && !(flags & PADSIM_JOINT) &&
                Rmax < kRecMaxReq;
    if (ctx->fact) {
        int r_ = plan_factorized(ctx, model, slo, n_qps, n_traces, Rmax, tot, cands);
        if (r_) return r_;
    }
    // wide nodes: the warp-per-replay factorized path (no context term: with one the
    // static candidates stay on the joint kernel)
    ctx->wide = (N > 8 || wide_small) && N <= kWMax && !ctx->static_list.empty() && !(flags & PADSIM_JOINT) &&
                Rmax < kRecMaxReq && model->decode_per_ctx_tok_s == 0.0 && ctx->tune.wide_path != 0;
    if (ctx->wide) {
        int r_ = plan_wide(ctx, model, slo, n_qps, n_traces, Rmax, cands);
        if (r_) return r_;
    }
    // replay launch plans for the joint kernel (dynamic candidates; static ones when N > 8)
    for (int dyn = 0; dyn < 2; dyn++) {
        if (!dyn && (ctx->fact || ctx->wide)) { std::memset(&ctx->plan_static, 0, sizeof(Plan)); continue; }
        const std::vector<int>& lst = dyn ? ctx->dyn_list : ctx->static_list;
        Plan& P = dyn ? ctx->plan_dyn : ctx->plan_static;
        std::memset(&P, 0, sizeof(P));
        if (lst.empty()) continue;
        P.m.min_w = model->min_w; P.m.max_w = model->max_w; P.m.ncap = ncap;
        P.m.rate = model->prefill_base_rate; P.m.eff = model->prefill_batch_eff;
        P.m.dec_fixed = model->decode_fixed_s; P.m.dec_per_seq = model->decode_per_seq_s;
        P.m.dec_per_ctx = model->decode_per_ctx_tok_s; P.m.kvb = model->kv_bytes_per_token;
        P.m.bw = model->fabric_bw_Bps; P.m.ovh = model->transfer_overhead_s;
        P.m.max_pb = model->max_prefill_batch; P.m.pb_tokens = model->prefill_token_budget;
        P.m.max_db = model->max_decode_batch; P.m.ctx_growth = model->decode_ctx_growth; P.m.slots = model->transfer_slots;
        P.m.spre = ctx->d_spre; P.m.sdec = ctx->d_sdec; P.m.den = ctx->d_den; P.m.ltab = ctx->d_ltab;
        P.N = N; P.C = C; P.Q = n_qps; P.S = n_traces; P.Rmax = Rmax; P.cbud = ctx->d_cbud;
        P.toff = ctx->d_toff; P.nreq = ctx->d_nreq; P.s_unit = ctx->d_s_unit; P.kv = ctx->d_kv;
        P.in_tok = ctx->d_in; P.out_tok = ctx->d_out; P.phase = ctx->d_phase;
        P.role = ctx->d_role; P.cap = ctx->d_cap; P.pol = ctx->d_pol; P.qps = ctx->d_qps;
        P.ttft_slo = slo->ttft_s; P.tpot_slo0 = slo->tpot_s[0]; P.tpot_slo1 = slo->tpot_s[1];
        P.clist = dyn ? ctx->d_clist_dyn : ctx->d_clist_static;
        P.n_clist = (int)lst.size();
        P.items_per_trace = (int)(((long long)n_qps * P.n_clist + kThreads - 1) / kThreads);
        P.n_items = P.items_per_trace * n_traces;
        P.work = ctx->d_work + dyn;
        P.rep_met = ctx->d_rep_met; P.rep_near = ctx->d_rep_near; P.rep_dur = ctx->d_rep_dur;
        P.rep_good = ctx->d_rep_good; P.rep_events = ctx->d_rep_events;
        if (flags & PADSIM_RECORDS) {
            P.rec_ttft = ctx->d_rec[0]; P.rec_tpot = ctx->d_rec[1]; P.rec_pe = ctx->d_rec[2];
            P.rec_comp = ctx->d_rec[3]; P.rec_te = ctx->d_rec[4];
        }
        // scratch layout per warp (lane-interleaved, 32 lanes)
        const size_t R = (size_t)std::max(Rmax, 1);
        const int NG = N <= 8 ? 8 : 64;
        size_t off = 0;
        auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
        P.off_link = take(R * 32 * sizeof(int));
        P.off_pe = take(R * 32 * sizeof(double));
        if (dyn) {
            P.off_tst = take(R * 32 * sizeof(double));
            P.off_tfl = take(R * 32);
            P.off_wts = take(R * 32 * sizeof(double));
            P.off_wtf = take(R * 32);
        }
        P.off_tte = take((size_t)PADSIM_MAX_SLOTS * 32 * sizeof(double));
        P.off_tti = take((size_t)PADSIM_MAX_SLOTS * 32 * sizeof(int));
        int maxo = 2;
        for (int s2 = 0; s2 < n_traces; s2++) maxo = std::max(maxo, ctx->max_out[s2]);
        int wheel = 32;
        while (wheel < maxo) wheel <<= 1;
        P.wheel = wheel;
        if (!PADSIM_JBL) {       // timing wheel
            P.off_heads = take((size_t)NG * wheel * 32 * sizeof(int));
            P.off_bits = take((size_t)NG * (wheel / 32) * 32 * sizeof(unsigned));
        }
        int rslots = 1;
        while (rslots < model->max_decode_batch) rslots <<= 1;
        P.ring_slots = rslots;
        if (PADSIM_JBL) P.off_ring = take((size_t)32 * NG * rslots * sizeof(unsigned long long));
        if (NG == 64) P.off_jw = take(joint_global_bytes_per_warp(64));
        // N > 8: the per-GPU next-event / routing keys in global scratch instead of
        // 32 KB of shared memory per warp, so registers (11 warps/SM) instead of shared
        // memory (7) bound the occupancy: cfg 5 subset (65 k replays) 27.7 -> 23.3 s
        P.j_kglob = NG == 64;
        if (P.j_kglob) P.off_keys = take((size_t)NG * 32 * (sizeof(double) + 2 * sizeof(int)));
        P.warp_bytes = off;
        ctx->j8[dyn] = true;
        ctx->j_ng = NG;
        // N ≤ 8, padsim_set_tuning joint_groups = 1: lane groups (one lane per
        // simulated GPU, 4 replays per warp, group_path.cuh).  Parity-green but
        // measured slower than one thread per replay (cfg 3 386 vs 300 ms, cfg 4
        // 687 vs 487 ms: group collectives under intra-warp divergence take the
        // WARPSYNC.COLLECTIVE slow path, and a DES instant rarely has per-GPU
        // parallel work), so auto keeps the one-thread-per-replay kernel
        ctx->j_grp = NG == 8 && ctx->tune.joint_groups == 1;
        if (ctx->j_grp) P.warp_bytes = gscratch_layout(R, rslots, dyn != 0).bytes;
        unsigned* d_wj;
        AL(d_wj, n_traces);
        ctx->d_workJ[dyn] = d_wj;
        P.work = d_wj;
        P.smem_trace = 0;
        // measured (cfg 3): a 16-inter-arrival lane clock window speeds the joint
        // replays up 15 % (622 -> 529 ms/step): lanes read the same trace lines
        // (round end, with batch lists and the merged window walk: 8 inter-arrivals
        // cfg 3 315 -> 308 ms, 32: 328 ms; cfg 4 unchanged)
        P.sync_win = 8.f;
        const long long UJ = (long long)n_traces * n_qps * P.n_clist;
        int tbj = (NG == 8 && !ctx->j_grp && UJ >= (long long)ctx->n_sm * 3 * kThreads) ? kThreads : 32;
        if (NG == 8 && (ctx->tune.joint_threads == 32 || ctx->tune.joint_threads == kThreads))
            tbj = ctx->tune.joint_threads;
        ctx->j_tb[dyn] = tbj;
        const void* fnj;
        size_t jb;
        const bool cx = model->decode_per_ctx_tok_s != 0.0;
        ctx->j_cx = cx;
        if (NG == 8)
            jb = tbj == kThreads ? (cx ? joint_smem_bytes<8, kThreads, true>() : joint_smem_bytes<8, kThreads, false>())
                                 : (cx ? joint_smem_bytes<8, 32, true>() : joint_smem_bytes<8, 32, false>());
        else jb = P.j_kglob ? 2 * 32 * sizeof(double) : (cx ? joint_smem_bytes<64, 32, true>() : joint_smem_bytes<64, 32, false>());
        // next to a large stage C workload the joint replays run as one-warp CTAs
        // capped at 168 registers so they leave registers to stage C (cfg 4 536 →
        // 522 ms); when they are the bulk of the step (cfg 3) the 232-register
        // variant is faster (327 vs 357 ms).  padsim_tuning.joint_reg_cap overrides.
        ctx->j_r168 = ctx->fact && ctx->kc_fine && NG == 8 && tbj == 32;
        if (ctx->tune.joint_reg_cap >= 0) ctx->j_r168 = ctx->tune.joint_reg_cap != 0 && NG == 8 && tbj == 32;
        fnj = joint_fn(dyn, tbj, NG, cx, ctx->j_r168);
        if (ctx->j_grp) {            // no shared memory; registers bound the occupancy
            ctx->j_r168 = false;
            jb = 0;
            fnj = jointg_fn(dyn != 0, cx, tbj);
        }
        // next to stage C the joint replays run without the lane clock window (cfg 4 461 ->
        // 452 ms; refilled lanes could not keep it anyway), see dynamic_path.cuh
        if (ctx->j_r168) P.sync_win = 0.f;
        P.smem_trace_bytes = jb;
        CK(cudaFuncSetAttribute(fnj, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)jb));
        int occj = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occj, fnj, tbj, jb));
        occj = std::max(occj, 1);
        // replays per warp item: as few as still fit every warp in one wave of
        // resident warps (fewer lanes per warp = less divergence on each latency-bound
        // replay chain; a second wave doubles the step), at least 4, at most 32.
        // Measured on cfg 3 (13.4 k replays, 8 resident one-warp CTAs per SM), back-to-back
        // runs: 16 lanes 270 ms, 12 lanes (1 120 warps, one wave) 245 ms, 10 lanes (1 344
        // warps, two waves) 342 ms; with the bench's L2 flush before each run 267 -> 264 ms.  The 168-register variant next to a large stage C workload
        // (cfg 4) keeps 32: there the joint warps' registers are what stage C waits for
        // (25 lanes: 455 -> 466 ms), and its lanes refill.
        {
            const int wpc0 = tbj / 32;
            const long long per_trace_cap = ((long long)ctx->n_sm * occj) / n_traces;   // CTAs per trace, one wave
            const long long qc = (long long)n_qps * P.n_clist;
            int lpw = 32;
            if (per_trace_cap > 0 && !ctx->j_r168)
                lpw = (int)std::min<long long>(32, std::max<long long>(4, (qc + per_trace_cap * wpc0 - 1) /
                                                                              (per_trace_cap * wpc0)));
            if (ctx->tune.joint_lanes_per_warp > 0) lpw = std::min(32, ctx->tune.joint_lanes_per_warp);
            P.lpw = ctx->j_grp ? kGPW : lpw;
        }
        const long long items = ((long long)n_qps * P.n_clist + P.lpw - 1) / P.lpw;
        const int wpc = tbj / 32;
        long long per_trace = std::max<long long>(1, ((long long)ctx->n_sm * occj) / n_traces);
        per_trace = std::min<long long>(per_trace, (items + wpc - 1) / wpc);
        const size_t per_cta = P.warp_bytes * wpc;
        P.scratch_per_cta = per_cta;
        size_t frj = 0, tmj = 0;
        CK(cudaMemGetInfo(&frj, &tmj));
        // scratch cap: 30 % of device memory
        const double mfr = 0.3;
        const long long cap_ctas = std::max<long long>(n_traces, (long long)((double)tmj * mfr / (double)per_cta));
        long long gridj = std::min<long long>(per_trace * n_traces, (cap_ctas / n_traces) * n_traces);
        gridj = std::max<long long>(gridj, n_traces);
        char* scrj = nullptr;
        AL(scrj, (size_t)gridj * per_cta);
        P.scratch = scrj;
        (dyn ? ctx->grid_dyn : ctx->grid_static) = (int)gridj;
        (dyn ? ctx->smem_dyn : ctx->smem_static) = jb;
    }
    // coalesced baseline replays (policy kind 4): one warp per CTA
    std::memset(&ctx->plan_coal, 0, sizeof(Plan));
    if (!ctx->coal_list.empty()) {
        Plan& P = ctx->plan_coal;
        P.m.min_w = model->min_w; P.m.max_w = model->max_w; P.m.ncap = ncap;
        P.m.rate = model->prefill_base_rate; P.m.eff = model->prefill_batch_eff;
        P.m.dec_fixed = model->decode_fixed_s; P.m.dec_per_seq = model->decode_per_seq_s;
        P.m.dec_per_ctx = model->decode_per_ctx_tok_s;
        P.m.max_db = model->max_decode_batch; P.m.ctx_growth = model->decode_ctx_growth; P.m.chunk = model->prefill_chunk_tokens;
        P.m.spre = ctx->d_spre; P.m.sdec = ctx->d_sdec; P.m.den = ctx->d_den; P.m.ltab = ctx->d_ltab;
        P.N = N; P.C = C; P.Q = n_qps; P.S = n_traces; P.Rmax = Rmax; P.cbud = ctx->d_cbud;
        P.toff = ctx->d_toff; P.nreq = ctx->d_nreq; P.s_unit = ctx->d_s_unit; P.kv = ctx->d_kv;
        P.in_tok = ctx->d_in; P.out_tok = ctx->d_out; P.phase = ctx->d_phase;
        P.role = ctx->d_role; P.cap = ctx->d_cap; P.pol = ctx->d_pol; P.qps = ctx->d_qps;
        P.ttft_slo = slo->ttft_s; P.tpot_slo0 = slo->tpot_s[0]; P.tpot_slo1 = slo->tpot_s[1];
        P.clist = ctx->d_clist_coal;
        P.n_clist = (int)ctx->coal_list.size();
        P.rep_met = ctx->d_rep_met; P.rep_near = ctx->d_rep_near; P.rep_dur = ctx->d_rep_dur;
        P.rep_good = ctx->d_rep_good; P.rep_events = ctx->d_rep_events;
        if (flags & PADSIM_RECORDS) {
            P.rec_ttft = ctx->d_rec[0]; P.rec_tpot = ctx->d_rec[1]; P.rec_pe = ctx->d_rec[2];
            P.rec_comp = ctx->d_rec[3]; P.rec_te = ctx->d_rec[4];
        }
        const size_t R = (size_t)std::max(Rmax, 1);
        size_t off = 0;
        auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
        P.off_link = take(R * 32 * sizeof(int));
        P.off_pe = take(R * 32 * sizeof(double));
        P.off_jw = take(coal_worker_bytes(N));
        P.off_heads = take((size_t)N * model->max_decode_batch * 32 * sizeof(int));   // act_id
        P.off_bits = take((size_t)N * model->max_decode_batch * 32 * sizeof(int));    // act_fin
        P.warp_bytes = off;
        const long long U = (long long)n_traces * n_qps * P.n_clist;
        const long long items = (U + 31) / 32;
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, coalesced_kernel<false>, 32, 0));
        occ = std::max(occ, 1);
        size_t frc = 0, tmc = 0;
        CK(cudaMemGetInfo(&frc, &tmc));
        const long long cap_ctas = std::max<long long>(1, (long long)((tmc / 10) / P.warp_bytes));
        long long gridc = std::min<long long>(items, (long long)ctx->n_sm * occ);
        gridc = std::max<long long>(1, std::min(gridc, cap_ctas));
        char* scr = nullptr;
        AL(scr, (size_t)gridc * P.warp_bytes);
        P.scratch = scr;
        P.scratch_per_cta = P.warp_bytes;
        ctx->grid_coal = (int)gridc;
    }
#undef AL
    ctx->plan_static.sw = ctx->sweep;
    ctx->plan_dyn.sw = ctx->sweep;
    ctx->plan_coal.sw = ctx->sweep;
    ctx->fplan.sw = ctx->sweep;
    CK(cudaDeviceSynchronize());
    ctx->planned = true;
    return PADSIM_OK;
}

int padsim_run(padsim_ctx* ctx, void* stream) {
    if (!ctx) return PADSIM_EINVAL;
    if (!ctx->planned) return fail(ctx, PADSIM_EINVAL, "padsim_run before padsim_plan");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaMemsetAsync(ctx->d_work, 0, 4 * sizeof(unsigned), st));
    if (!ctx->ev0) {
        CK(cudaEventCreate(&ctx->ev0));
        CK(cudaEventCreate(&ctx->ev1));
        CK(cudaEventCreate(&ctx->evA));
        CK(cudaEventCreate(&ctx->evC));
        CK(cudaEventCreate(&ctx->evJ0));
        CK(cudaEventCreate(&ctx->evJ1));
        CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
        CK(cudaEventCreate(&ctx->evC0));
        for (auto& x : ctx->sideC) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
        for (auto& e : ctx->evCk) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->evCf, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(ctx->ev0, st));
    int launches = 0;
    // Schedule (measured on cfg 4): stage A runs first on the whole GPU; the joint
    // replays (dynamic candidates, static ones when N > 8, coalesced baselines) then
    // run on a side stream concurrently with stage C.  Stage C's resident grid is
    // capped by shared memory (3 CTAs/SM), leaving registers and issue slots that
    // the latency-bound joint warps fill; running them next to stage A instead
    // starved stage A of registers and serialised the two stages.
    if (ctx->fact) {
        FPlan F = ctx->fplan;
        F.s_begin = 0;
        F.s_count = ctx->S;
        const int ga = F.a_blocks_per_trace * F.s_count;
        if (ctx->fA_tb == kATbBig) stageA_kernel<kATbBig><<<ga, kATbBig, ctx->fA_smem, st>>>(F);
        else if (ctx->fA_tb == kThreads) stageA_kernel<kThreads><<<ga, kThreads, ctx->fA_smem, st>>>(F);
        else stageA_kernel<32><<<ga, 32, ctx->fA_smem, st>>>(F);
        CK(cudaGetLastError());
        launches++;
    }
    CK(cudaEventRecord(ctx->evA, st));
    const bool any_joint = ctx->plan_dyn.n_clist > 0 || ctx->plan_static.n_clist > 0 ||
                           ctx->plan_coal.n_clist > 0;
    const bool ser = ctx->tune.serialize != 0;     // every kernel on `st`, one after another
    cudaStream_t js = (ctx->fact || ctx->wide) && any_joint && !ser ? ctx->side : st;
    if (js != st) CK(cudaStreamWaitEvent(js, ctx->j_with_a ? ctx->ev0 : ctx->evA, 0));
    CK(cudaEventRecord(ctx->evJ0, js));
    for (int dyn = 0; dyn < 2; dyn++) {
        const Plan& P = dyn ? ctx->plan_dyn : ctx->plan_static;
        if (P.n_clist == 0) continue;
        const int grid = dyn ? ctx->grid_dyn : ctx->grid_static;
        const size_t smem = dyn ? ctx->smem_dyn : ctx->smem_static;
        CK(cudaMemsetAsync(ctx->d_workJ[dyn], 0, (size_t)ctx->S * sizeof(unsigned), js));
        {
            const int tbl = ctx->j_ng == 64 ? 32 : ctx->j_tb[dyn];
            void* args[] = {(void*)&P};
            const void* fn = ctx->j_grp ? jointg_fn(dyn != 0, ctx->j_cx, tbl)
                                        : joint_fn(dyn != 0, tbl, ctx->j_ng, ctx->j_cx, ctx->j_r168);
            CK(cudaLaunchKernel(fn, dim3(grid), dim3(tbl), args, smem, js));
            launches++;
        }
        CK(cudaGetLastError());
    }
    if (ctx->plan_coal.n_clist > 0) {
        if (ctx->model.decode_per_ctx_tok_s != 0.0)
            coalesced_kernel<true><<<ctx->grid_coal, 32, 0, js>>>(ctx->plan_coal);
        else
            coalesced_kernel<false><<<ctx->grid_coal, 32, 0, js>>>(ctx->plan_coal);
        CK(cudaGetLastError());
        launches++;
    }
    CK(cudaEventRecord(ctx->evJ1, js));
    CK(cudaEventRecord(ctx->evC0, st));
    if (ctx->fact) {
        CK(cudaMemsetAsync(ctx->d_workC, 0, (size_t)kNumKC * ctx->S * sizeof(unsigned), st));
        CK(cudaEventRecord(ctx->evCf, st));
        const bool cm = ctx->model.decode_per_ctx_tok_s != 0.0;
        // one launch per decode-pool class, on their own streams so that each
        // class's tail overlaps the others (they share nothing but the stream
        // records written by stage A and the scratch — each class gets its own
        // scratch slice)
        for (int kc = 0; kc < kNumKC; kc++) {
            if (ctx->kc_n[kc] == 0) continue;
            cudaStream_t cs = ser ? st : ctx->sideC[kc];
            if (!ser) CK(cudaStreamWaitEvent(cs, ctx->evCf, 0));
            FPlan F = ctx->fplan;
            F.s_begin = 0;
            F.s_count = ctx->S;
            F.cc_base = ctx->kc_base[kc];
            F.n_cc = ctx->kc_n[kc];
            F.work = ctx->d_workC + (size_t)kc * ctx->S;
            F.c_off_sdec = ctx->kc_off_sdec[kc];
            F.c_ltab_on = ctx->kc_ltab[kc];
            F.c_hca_on = ctx->kc_hca[kc];
            F.c_off_hca = ctx->kc_off_hca[kc];
            F.c_off_ltab = ctx->kc_off_ltab[kc];
            F.bits_in_smem = ctx->kc_bits_smem[kc];
            F.scrC = ctx->kc_scr[kc];
            stagec_launch(cm, ctx->fC_idx16, kc, ctx->kc_bl[kc], ctx->kc_grid[kc], ctx->kc_smem[kc], cs, F);
            CK(cudaGetLastError());
            launches++;
        }
        for (int kc = 0; kc < kNumKC && !ser; kc++) {
            if (ctx->kc_n[kc] == 0) continue;
            CK(cudaEventRecord(ctx->evCk[kc], ctx->sideC[kc]));
            CK(cudaStreamWaitEvent(st, ctx->evCk[kc], 0));
        }
    }
    if (ctx->wide) {          // wide nodes: stage A → stage C per chunk of traces
        CK(cudaMemsetAsync(ctx->d_workW, 0, (size_t)2 * ctx->S * sizeof(unsigned), st));
        const int nch = (ctx->S + ctx->w_chunk - 1) / ctx->w_chunk;
        while ((int)ctx->evW.size() < 4 * nch) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            ctx->evW.push_back(e);
        }
        ctx->n_wchunks = nch;
        for (int kch = 0; kch < nch; kch++) {
            const int s0 = kch * ctx->w_chunk;
            FPlan F = ctx->fplan;
            F.s_begin = s0;
            F.s_count = std::min(ctx->w_chunk, ctx->S - s0);
            // CTAs bound to one trace each: the launch's resident CTAs split over the
            // chunk's traces, no more per trace than its items need
            auto grid_for = [&](int tot, long long items) {
                long long per = std::max<long long>(1, tot / F.s_count);
                per = std::min<long long>(per, std::max<long long>(1, (items + kWarps - 1) / kWarps));
                return (int)(per * F.s_count);
            };
            const int gA = grid_for(ctx->wA_grid, ctx->wA_items);
            const int gC = grid_for(ctx->wC_grid, ctx->wC_items);
            F.work = ctx->d_workW;
            CK(cudaEventRecord(ctx->evW[4 * kch], st));
            stageA_wide_kernel<<<gA, kThreads, 0, st>>>(F);
            CK(cudaGetLastError());
            CK(cudaEventRecord(ctx->evW[4 * kch + 1], st));
            F.work = ctx->d_workW + ctx->S;
            stageC_wide_kernel<<<gC, kThreads, 0, st>>>(F);
            CK(cudaGetLastError());
            CK(cudaEventRecord(ctx->evW[4 * kch + 2], st));
            launches += 2;
        }
    }
    CK(cudaEventRecord(ctx->evC, st));
    if (js != st) CK(cudaStreamWaitEvent(st, ctx->evJ1, 0));   // join
    CK(cudaEventRecord(ctx->ev1, st));
    ctx->ev_recorded = true;
    const int CQ = ctx->C * ctx->Q;
    reduce_kernel<<<(CQ + 255) / 256, 256, 0, st>>>(ctx->d_rep_met, ctx->d_rep_near, ctx->d_rep_good,
                                                    CQ, ctx->S, ctx->d_met, ctx->d_good, ctx->d_near,
                                                    ctx->d_rep_metk, ctx->d_rep_watts, ctx->sweep.n,
                                                    ctx->d_metk, ctx->d_qpw, ctx->d_watts,
                                                    ctx->d_rep_sq, ctx->d_rep_se, ctx->d_qsum, ctx->d_esum);
    CK(cudaGetLastError());
    max80_kernel<<<(ctx->C + 127) / 128, 128, 0, st>>>(ctx->d_met, ctx->d_metk, ctx->d_qps, ctx->C, ctx->Q,
                                                       ctx->sweep.n, ctx->n_req_total, ctx->d_max80);
    CK(cudaGetLastError());
    argmax_kernel<<<ctx->Q, 256, 0, st>>>(ctx->d_met, ctx->d_capsum, ctx->C, ctx->Q, ctx->d_argmax);
    CK(cudaGetLastError());
    ctx->n_launches = launches + 3;     // + reduce, max80, argmax
    return PADSIM_OK;
}

int padsim_replay_records(padsim_ctx* ctx, const padsim_trace* trace, double qps_per_gpu,
                          const padsim_model* model, const padsim_candidates* one,
                          const padsim_slo* slo, const padsim_budget* budget, double* ttft,
                          double* tpot, double* prefill_end, double* completion) {
    if (!ctx || !trace || !one) return PADSIM_EINVAL;
    if (one->n_cand != 1) return fail(ctx, PADSIM_EINVAL, "padsim_replay_records: n_cand must be 1");
    int32_t bad = -1;
    int rc = padsim_plan(ctx, trace, 1, &qps_per_gpu, 1, model, one, slo, budget, PADSIM_RECORDS, &bad);
    if (rc) return rc;
    rc = padsim_run(ctx, ctx->stream);
    if (rc) return rc;
    return padsim_fetch_records(ctx, ctx->stream, ttft, tpot, prefill_end, completion, nullptr, nullptr);
}

int padsim_static_path(padsim_ctx* ctx, int32_t* path) {
    if (!ctx || !path) return PADSIM_EINVAL;
    if (!ctx->planned) return fail(ctx, PADSIM_EINVAL, "no plan");
    *path = ctx->static_list.empty() ? 0 : ctx->fact ? 1 : ctx->wide ? 2 : 3;
    return PADSIM_OK;
}

int padsim_launch_count(padsim_ctx* ctx, int32_t* n) {
    if (!ctx || !n) return PADSIM_EINVAL;
    *n = ctx->n_launches;
    return PADSIM_OK;
}

int padsim_set_tuning(padsim_ctx* ctx, const padsim_tuning* t) {
    if (!ctx) return PADSIM_EINVAL;
    if (!t) { ctx->tune = padsim_tuning{0, 0, -1, 0, -1, 0, -1, 0, -1, -1, 0}; return PADSIM_OK; }
    if ((t->stage_a_threads != 0 && t->stage_a_threads != 32 && t->stage_a_threads != kThreads &&
         t->stage_a_threads != kATbBig) ||
        (t->stage_c_classes != 0 && t->stage_c_classes != 3 && t->stage_c_classes != 5) ||
        t->stage_c_batch_lists < -1 || t->stage_c_batch_lists >= (1 << kNumKC) ||
        (t->joint_threads != 0 && t->joint_threads != 32 && t->joint_threads != kThreads) ||
        t->joint_reg_cap < -1 || t->joint_reg_cap > 1 || t->joint_lanes_per_warp < 0 ||
        t->joint_lanes_per_warp > 32 || t->joint_after_stage_a < -1 || t->joint_after_stage_a > 1 ||
        t->serialize < 0 || t->serialize > 1 || t->joint_groups < -1 || t->joint_groups > 1 ||
        t->wide_path < -1 || t->wide_path > 1 || t->wide_chunk < 0)
        return fail(ctx, PADSIM_EINVAL, "tuning value out of range");
    ctx->tune = *t;
    return PADSIM_OK;
}

int padsim_fetch(padsim_ctx* ctx, void* stream, padsim_result* out) {
    if (!ctx || !out) return PADSIM_EINVAL;
    if (!ctx->planned) return fail(ctx, PADSIM_EINVAL, "fetch before plan");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t CQ = (size_t)ctx->C * ctx->Q;
    if (out->met) CK(cudaMemcpyAsync(out->met, ctx->d_met, CQ * 8, cudaMemcpyDeviceToHost, st));
    if (out->goodput) CK(cudaMemcpyAsync(out->goodput, ctx->d_good, CQ * 8, cudaMemcpyDeviceToHost, st));
    if (out->near_boundary)
        CK(cudaMemcpyAsync(out->near_boundary, ctx->d_near, CQ * 8, cudaMemcpyDeviceToHost, st));
    if (out->argmax)
        CK(cudaMemcpyAsync(out->argmax, ctx->d_argmax, (size_t)ctx->Q * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    out->bad_index = -1;
    return PADSIM_OK;
}

int padsim_get_device_results(padsim_ctx* ctx, padsim_device_results* o) {
    if (!ctx || !o) return PADSIM_EINVAL;
    if (!ctx->planned) return fail(ctx, PADSIM_EINVAL, "no plan");
    o->d_met = (int64_t*)ctx->d_met; o->d_goodput = ctx->d_good; o->d_near = (int64_t*)ctx->d_near;
    o->d_argmax = ctx->d_argmax; o->d_rep_met = ctx->d_rep_met; o->d_rep_near = ctx->d_rep_near;
    o->d_rep_duration = ctx->d_rep_dur; o->d_rep_goodput = ctx->d_rep_good;
    o->d_rep_events = (int64_t*)ctx->d_rep_events;
    o->n_cand = ctx->C; o->n_qps = ctx->Q; o->n_traces = ctx->S;
    o->d_aux_events = (int64_t*)ctx->d_evA;
    o->n_aux_events = (ctx->fact || ctx->wide) ? ctx->n_evA : 0;
    return PADSIM_OK;
}

int padsim_replay_kernel_ms(padsim_ctx* ctx, float* ms) {
    if (!ctx || !ms) return PADSIM_EINVAL;
    if (!ctx->ev_recorded) return fail(ctx, PADSIM_EINVAL, "no run recorded");
    CK(cudaSetDevice(ctx->device));
    CK(cudaEventSynchronize(ctx->ev1));
    CK(cudaEventElapsedTime(ms, ctx->ev0, ctx->ev1));
    return PADSIM_OK;
}

int padsim_set_slo_sweep(padsim_ctx* ctx, const padsim_slo* slos, int32_t n_slo) {
    if (!ctx || n_slo < 0 || n_slo > kMaxSloSweep || (n_slo > 0 && !slos)) return PADSIM_EINVAL;
    if (!ctx->planned) return fail(ctx, PADSIM_EINVAL, "set_slo_sweep before padsim_plan");
    for (int k = 0; k < n_slo; k++)
        if (!(slos[k].ttft_s > 0 && slos[k].tpot_s[0] > 0 && slos[k].tpot_s[1] > 0))
            return fail(ctx, PADSIM_EINVAL, "SLOs must be > 0");
    ctx->sweep.n = n_slo;
    for (int k = 0; k < kMaxSloSweep; k++) {
        ctx->sweep.ttft[k] = k < n_slo ? slos[k].ttft_s : 0.0;
        ctx->sweep.tpot0[k] = k < n_slo ? slos[k].tpot_s[0] : 0.0;
        ctx->sweep.tpot1[k] = k < n_slo ? slos[k].tpot_s[1] : 0.0;
    }
    ctx->plan_static.sw = ctx->sweep;
    ctx->plan_dyn.sw = ctx->sweep;
    ctx->plan_coal.sw = ctx->sweep;
    ctx->fplan.sw = ctx->sweep;
    return PADSIM_OK;
}

int padsim_fetch_extras(padsim_ctx* ctx, void* stream, int64_t* met_sweep, double* qps_per_watt,
                        double* avg_watts, int32_t* max_qps80) {
    if (!ctx) return PADSIM_EINVAL;
    if (!ctx->planned) return fail(ctx, PADSIM_EINVAL, "no plan");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t CQ = (size_t)ctx->C * ctx->Q;
    if (met_sweep)
        CK(cudaMemcpyAsync(met_sweep, ctx->d_metk, CQ * kMaxSloSweep * 8, cudaMemcpyDeviceToHost, st));
    if (qps_per_watt) CK(cudaMemcpyAsync(qps_per_watt, ctx->d_qpw, CQ * 8, cudaMemcpyDeviceToHost, st));
    if (avg_watts) CK(cudaMemcpyAsync(avg_watts, ctx->d_watts, CQ * 8, cudaMemcpyDeviceToHost, st));
    if (max_qps80)
        CK(cudaMemcpyAsync(max_qps80, ctx->d_max80, (size_t)ctx->C * (1 + kMaxSloSweep) * 4,
                           cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return PADSIM_OK;
}

int padsim_fetch_decomposition(padsim_ctx* ctx, void* stream, double* rep_queue, double* rep_exec,
                               double* sum_queue, double* sum_exec) {
    if (!ctx) return PADSIM_EINVAL;
    if (!ctx->planned) return fail(ctx, PADSIM_EINVAL, "no plan");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = (size_t)ctx->C * ctx->Q * ctx->S;
    const size_t CQ = (size_t)ctx->C * ctx->Q;
    if (rep_queue) CK(cudaMemcpyAsync(rep_queue, ctx->d_rep_sq, n * 8, cudaMemcpyDeviceToHost, st));
    if (rep_exec) CK(cudaMemcpyAsync(rep_exec, ctx->d_rep_se, n * 8, cudaMemcpyDeviceToHost, st));
    if (sum_queue) CK(cudaMemcpyAsync(sum_queue, ctx->d_qsum, CQ * 8, cudaMemcpyDeviceToHost, st));
    if (sum_exec) CK(cudaMemcpyAsync(sum_exec, ctx->d_esum, CQ * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return PADSIM_OK;
}

int padsim_fetch_percentiles(padsim_ctx* ctx, void* stream, const int32_t* pcts, int32_t n_pct,
                             double* out) {
    if (!ctx || !pcts || !out) return PADSIM_EINVAL;
    if (!ctx->planned || !(ctx->flags & PADSIM_RECORDS))
        return fail(ctx, PADSIM_EINVAL, "plan without PADSIM_RECORDS");
    if (!ctx->ev_recorded) return fail(ctx, PADSIM_EINVAL, "no run recorded");
    if (n_pct < 1 || n_pct > kMaxPct) return fail(ctx, PADSIM_EINVAL, "n_pct out of range");
    for (int z = 0; z < n_pct; z++)
        if (pcts[z] < 1 || pcts[z] > 100) return fail(ctx, PADSIM_EINVAL, "percentile outside 1..100");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    static_assert(kMaxPct == PADSIM_MAX_PCT, "ABI constant");
    const long long n_rep = (long long)ctx->C * ctx->Q * ctx->S;
    CK(cudaMemcpyAsync(ctx->d_pct, pcts, sizeof(int) * n_pct, cudaMemcpyHostToDevice, st));
    if (n_rep > 0) {
        percentile_kernel<<<ctx->pct_grid, 512, ctx->pct_smem, st>>>(
            ctx->d_rec[0], ctx->d_rec[1], ctx->d_nreq, ctx->S, std::max(ctx->Rmax, 1), ctx->pct_n2, n_rep,
            ctx->d_pct, n_pct, ctx->d_pct_out, ctx->d_pct_scratch);
        CK(cudaGetLastError());
    }
    // compact [r][2][kMaxPct] -> [r][2][n_pct] on the host side of the copy
    CK(cudaMemcpy2DAsync(out, sizeof(double) * n_pct, ctx->d_pct_out, sizeof(double) * kMaxPct,
                         sizeof(double) * n_pct, (size_t)n_rep * 2, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return PADSIM_OK;
}

int padsim_kernel_times_ms(padsim_ctx* ctx, float* ms3) {
    if (!ctx || !ms3) return PADSIM_EINVAL;
    if (!ctx->ev_recorded) return fail(ctx, PADSIM_EINVAL, "no run recorded");
    CK(cudaSetDevice(ctx->device));
    CK(cudaEventSynchronize(ctx->ev1));
    CK(cudaEventElapsedTime(&ms3[0], ctx->ev0, ctx->evA));
    CK(cudaEventElapsedTime(&ms3[1], ctx->evC0, ctx->evC));
    CK(cudaEventElapsedTime(&ms3[2], ctx->evJ0, ctx->evJ1));
    if (ctx->wide) {        // wide nodes: Σ over the chunks' stage A / stage C launches
        ms3[0] = ms3[1] = 0.f;
        for (int k = 0; k < ctx->n_wchunks; k++) {
            float a = 0.f, c = 0.f;
            CK(cudaEventElapsedTime(&a, ctx->evW[4 * k], ctx->evW[4 * k + 1]));
            CK(cudaEventElapsedTime(&c, ctx->evW[4 * k + 1], ctx->evW[4 * k + 2]));
            ms3[0] += a;
            ms3[1] += c;
        }
    }
    return PADSIM_OK;
}

int padsim_fetch_replays(padsim_ctx* ctx, void* stream, int32_t* met, int32_t* near,
                         double* dur, double* good, int64_t* events) {
    if (!ctx) return PADSIM_EINVAL;
    if (!ctx->planned) return fail(ctx, PADSIM_EINVAL, "no plan");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = (size_t)ctx->C * ctx->Q * ctx->S;
    if (met) CK(cudaMemcpyAsync(met, ctx->d_rep_met, n * 4, cudaMemcpyDeviceToHost, st));
    if (near) CK(cudaMemcpyAsync(near, ctx->d_rep_near, n * 4, cudaMemcpyDeviceToHost, st));
    if (dur) CK(cudaMemcpyAsync(dur, ctx->d_rep_dur, n * 8, cudaMemcpyDeviceToHost, st));
    if (good) CK(cudaMemcpyAsync(good, ctx->d_rep_good, n * 8, cudaMemcpyDeviceToHost, st));
    if (events) CK(cudaMemcpyAsync(events, ctx->d_rep_events, n * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return PADSIM_OK;
}

int padsim_fetch_records(padsim_ctx* ctx, void* stream, double* ttft, double* tpot, double* pe,
                         double* comp, double* te, int32_t* r_max) {
    if (!ctx) return PADSIM_EINVAL;
    if (!ctx->planned || !(ctx->flags & PADSIM_RECORDS))
        return fail(ctx, PADSIM_EINVAL, "plan without PADSIM_RECORDS");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = (size_t)ctx->C * ctx->Q * ctx->S * std::max(ctx->Rmax, 1) * 8;
    double* dst[5] = {ttft, tpot, pe, comp, te};
    for (int k = 0; k < 5; k++)
        if (dst[k]) CK(cudaMemcpyAsync(dst[k], ctx->d_rec[k], n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (r_max) *r_max = ctx->Rmax;
    return PADSIM_OK;
}

int padsim_argmax_device(padsim_ctx* ctx, void* stream, const int64_t* d_met, const int32_t* d_capsum,
                         int32_t n_cand, int32_t n_qps, int32_t* d_argmax) {
    if (!ctx || !d_met || !d_argmax || n_cand < 1 || n_qps < 1) return PADSIM_EINVAL;
    if (!d_capsum && (!ctx->planned || n_cand != ctx->C))
        return fail(ctx, PADSIM_EINVAL, "argmax without d_capsum needs the plan's candidate count");
    CK(cudaSetDevice(ctx->device));
    argmax_kernel<<<n_qps, 256, 0, (cudaStream_t)stream>>>((const long long*)d_met,
                                                           d_capsum ? d_capsum : ctx->d_capsum,
                                                           n_cand, n_qps, d_argmax);
    CK(cudaGetLastError());
    return PADSIM_OK;
}

int padsim_evaluate_allocations(padsim_ctx* ctx, const padsim_trace* traces, int32_t n_traces,
                                const double* qps, int32_t n_qps, const padsim_model* model,
                                const padsim_candidates* cands, const padsim_slo* slo,
                                const padsim_budget* budget, padsim_result* out) {
    if (!ctx || !out) return PADSIM_EINVAL;
    int32_t bad = -1;
    int rc = padsim_plan(ctx, traces, n_traces, qps, n_qps, model, cands, slo, budget, 0, &bad);
    out->bad_index = bad;
    if (rc) return rc;
    rc = padsim_run(ctx, ctx->stream);
    if (rc) return rc;
    rc = padsim_fetch(ctx, ctx->stream, out);
    out->bad_index = -1;
    return rc;
}

int padsim_controller_decide_device(padsim_ctx* ctx, const padsim_policy* policy,
                                    const padsim_budget* budget, const padsim_model* model,
                                    const padsim_ctrl_state* st, const padsim_window_stats* ws,
                                    double now, padsim_action* act) {
    if (!ctx || !policy || !budget || !model || !st || !ws || !act) return PADSIM_EINVAL;
    if (st->n_gpus < 2 || st->n_gpus > PADSIM_MAX_GPUS) return fail(ctx, PADSIM_EINVAL, "n_gpus");
    int rc = validate_model(ctx, model);
    if (rc) return rc;
    rc = validate_policy(ctx, policy, model, st->n_gpus, budget->budget_w);
    if (rc) return rc;
    if (policy->kind == 4) return fail(ctx, PADSIM_EINVAL, "coalesced policy has no controller");
    CK(cudaSetDevice(ctx->device));
    if (!ctx->d_ctl_state) {
        CK(cudaMalloc(&ctx->d_ctl_state, sizeof(padsim_ctrl_state)));
        CK(cudaMalloc(&ctx->d_ctl_stats, sizeof(padsim_window_stats)));
        CK(cudaMalloc(&ctx->d_ctl_act, sizeof(padsim_action)));
    }
    cudaStream_t sm = ctx->stream;
    CK(cudaMemcpyAsync(ctx->d_ctl_state, st, sizeof(*st), cudaMemcpyHostToDevice, sm));
    CK(cudaMemcpyAsync(ctx->d_ctl_stats, ws, sizeof(*ws), cudaMemcpyHostToDevice, sm));
    controller_kernel<<<1, 32, 0, sm>>>(*policy, model->min_w, model->max_w, budget->budget_w,
                                        ctx->d_ctl_state, ctx->d_ctl_stats, now, ctx->d_ctl_act);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(act, ctx->d_ctl_act, sizeof(*act), cudaMemcpyDeviceToHost, sm));
    CK(cudaStreamSynchronize(sm));
    return PADSIM_OK;
}

}  // extern "C"
