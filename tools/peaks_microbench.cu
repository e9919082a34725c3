// peaks_microbench.cu — measured issue / FP64 / INT32 throughput of one B200
// (the replay kernels are issue-bound integer +
// FP64 control code, so their roofline denominators are these pipes, not HBM).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a --fmad=true -o peaks tools/peaks_microbench.cu
//   ./peaks > profiles/peaks_rNN.json
//
// Each kernel runs kChains independent dependency chains per thread (enough
// ILP to saturate the pipe), grid = 148 SMs x 8 CTAs x 256 threads, timed with
// CUDA events after a warm-up; the result is thread-ops/s and warp-instr/s.
// The SASS of each loop body is one opcode repeated (checked with cuobjdump).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void k_dfma(double* out, double a, double b) {
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; c++) x[c] = a + c + threadIdx.x;
    for (int i = 0; i < kIters; i++) {
#pragma unroll
        for (int c = 0; c < kChains; c++) x[c] = fma(x[c], b, a);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; c++) s += x[c];
    if (s == 1.2345) out[0] = s;
}

__global__ void k_dadd(double* out, double a, double b) {
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; c++) x[c] = a + c + threadIdx.x;
    for (int i = 0; i < kIters; i++) {
#pragma unroll
        for (int c = 0; c < kChains; c++) x[c] = __dadd_rn(x[c], b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; c++) s += x[c];
    if (s == 1.2345) out[0] = s;
}

__global__ void k_ddiv(double* out, double a, double b) {
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; c++) x[c] = a + c + threadIdx.x;
    for (int i = 0; i < kIters / 16; i++) {
#pragma unroll
        for (int c = 0; c < kChains; c++) x[c] = b / x[c];
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; c++) s += x[c];
    if (s == 1.2345) out[0] = s;
}

__global__ void k_ffma(float* out, float a, float b) {
    float x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; c++) x[c] = a + c + threadIdx.x;
    for (int i = 0; i < kIters; i++) {
#pragma unroll
        for (int c = 0; c < kChains; c++) x[c] = fmaf(x[c], b, a);
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < kChains; c++) s += x[c];
    if (s == 1.2345f) out[0] = s;
}

__global__ void k_iadd(int* out, int a, int b) {
    int x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; c++) x[c] = a + c + threadIdx.x;
    for (int i = 0; i < kIters; i++) {
#pragma unroll
        for (int c = 0; c < kChains; c++) {     // IADD3 then LOP3, kept by asm volatile
            asm volatile("add.s32 %0, %0, %1;" : "+r"(x[c]) : "r"(a));
            asm volatile("xor.b32 %0, %0, %1;" : "+r"(x[c]) : "r"(b));
        }
    }
    int s = 0;
#pragma unroll
    for (int c = 0; c < kChains; c++) s += x[c];
    if (s == 12345) out[0] = s;
}

template <class F>
static double time_ms(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; w++) launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

int main() {
    int sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int grid = sms * 8, tb = 256;
    double* dd;
    cudaMalloc(&dd, 64);
    const double threads = (double)grid * tb;
    const double per_thread = (double)kIters * kChains;
    struct R { const char* name; double ms, thread_ops; };
    R rs[5];
    rs[0] = {"dfma", time_ms([&] { k_dfma<<<grid, tb>>>(dd, 1.0000001, 0.9999999); }), threads * per_thread};
    rs[1] = {"dadd", time_ms([&] { k_dadd<<<grid, tb>>>(dd, 1.0000001, 1e-9); }), threads * per_thread};
    rs[2] = {"ddiv", time_ms([&] { k_ddiv<<<grid, tb>>>(dd, 1.0000001, 1.5); }), threads * per_thread / 16};
    rs[3] = {"ffma", time_ms([&] { k_ffma<<<grid, tb>>>((float*)dd, 1.0001f, 0.9999f); }), threads * per_thread};
    rs[4] = {"iadd_lop", time_ms([&] { k_iadd<<<grid, tb>>>((int*)dd, 3, 0x55); }), threads * per_thread * 2};
    if (cudaGetLastError() != cudaSuccess) { fprintf(stderr, "cuda error\n"); return 1; }
    printf("{\"sms\": %d, \"attr_clock_mhz\": %.0f, \"grid\": %d, \"threads_per_cta\": %d, \"ops\": {", sms,
           clk_khz / 1e3, grid, tb);
    for (int k = 0; k < 5; k++) {
        const double ops_s = rs[k].thread_ops / (rs[k].ms / 1e3);
        printf("%s\"%s\": {\"ms\": %.4f, \"thread_ops_per_s\": %.6e, \"warp_instr_per_s\": %.6e, "
               "\"thread_ops_per_clk_per_sm_at_attr_clock\": %.2f}",
               k ? ", " : "", rs[k].name, rs[k].ms, ops_s, ops_s / 32, ops_s / (sms * (clk_khz * 1e3)));
    }
    printf("}}\n");
    return 0;
}
