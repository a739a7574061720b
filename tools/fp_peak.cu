// fp_peak.cu -- FP pipe microbenchmark for the roofline denominator.
//
// Measures, on one B200 at full occupancy, the sustained throughput of
//   DADD, DMUL (fp64) and FADD, FMUL (fp32) with 8 independent dependency
//   chains per thread (no FMA: the escape loop has none), and
//   the escape-loop body itself (8 FP ops per iteration, no exit test),
// as lane-operations per second and per SM per cycle.  Cycles come from clock64() on
// each CTA: the LONGEST CTA span is the kernel's duration in SM cycles (the warp
// scheduler does not run co-resident CTAs in lockstep -- older warps get priority, so
// CTAs finish staggered and the MEAN span is only ~56% of the kernel; the r01 output
// divided the mean span by the kernel time and printed an "implied_mhz" of ~1100 that
// was this staggering, not the clock).  implied_mhz = longest span / kernel time.
// Prints one JSON object.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/fp_peak tools/fp_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <typename T, int OP>
__global__ void __launch_bounds__(256) chains(T seed, int iters, T* sink, unsigned long long* cyc) {
    T a0 = seed + threadIdx.x, a1 = a0 + T(1), a2 = a0 + T(2), a3 = a0 + T(3);
    T a4 = a0 + T(4), a5 = a0 + T(5), a6 = a0 + T(6), a7 = a0 + T(7);
    const T k = T(1.0000001);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (OP == 0) {
                a0 = a0 + k; a1 = a1 + k; a2 = a2 + k; a3 = a3 + k;
                a4 = a4 + k; a5 = a5 + k; a6 = a6 + k; a7 = a7 + k;
            } else {
                a0 = a0 * k; a1 = a1 * k; a2 = a2 * k; a3 = a3 * k;
                a4 = a4 * k; a5 = a5 * k; a6 = a6 * k; a7 = a7 * k;
            }
        }
    }
    long long t1 = clock64();
    T s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == T(-12345)) sink[0] = s;
    if (threadIdx.x == 0) {
        atomicAdd(&cyc[0], (unsigned long long)(t1 - t0));
        atomicMax(&cyc[1], (unsigned long long)(t1 - t0));
    }
}

// Packed FP32x2 chains (PTX add/mul.rn.f32x2 -> FADD2/FMUL2): 8 packed chains, i.e.
// 16 fp32 lane-ops per packed instruction pair -- does packing raise the FP32 pipe rate?
template <int OP>
__global__ void __launch_bounds__(256) chains_f32x2(int iters, float* sink, unsigned long long* cyc) {
    unsigned long long a[8];
    const float k = 1.0000001f;
    unsigned long long kk;
    asm("mov.b64 %0, {%1, %2};" : "=l"(kk) : "f"(k), "f"(k));
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const float v = 1.0f + threadIdx.x + c;
        asm("mov.b64 %0, {%1, %2};" : "=l"(a[c]) : "f"(v), "f"(v + 0.5f));
    }
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (OP == 0) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[c]) : "l"(kk));
                else asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(a[c]) : "l"(kk));
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[c]));
        s += lo + hi;
    }
    if (s == -12345.f) sink[0] = s;
    if (threadIdx.x == 0) {
        atomicAdd(&cyc[0], (unsigned long long)(t1 - t0));
        atomicMax(&cyc[1], (unsigned long long)(t1 - t0));
    }
}

// The escape-loop body without the exit test (bounded: c = 0.25i keeps |z| < 1).
template <typename T>
__global__ void __launch_bounds__(256) mandel_body(int iters, T* sink, unsigned long long* cyc) {
    T cr = T(-0.1) + T(threadIdx.x) * T(1e-6), ci = T(0.25);
    T x = 0, y = 0, x2 = 0, y2 = 0, s = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            T ny = (x + x) * y + ci;
            T nx = (x2 - y2) + cr;
            x = nx; y = ny;
            x2 = x * x; y2 = y * y;
            s = s + (x2 + y2) * T(0);  // keeps the 8th op (x2 + y2) live
        }
    }
    long long t1 = clock64();
    if (s == T(-12345) || x == T(-12345)) sink[0] = s + x;
    if (threadIdx.x == 0) {
        atomicAdd(&cyc[0], (unsigned long long)(t1 - t0));
        atomicMax(&cyc[1], (unsigned long long)(t1 - t0));
    }
}

struct Timer {
    cudaEvent_t e0, e1;
    Timer() { cudaEventCreate(&e0); cudaEventCreate(&e1); }
};

static void report(const char* name, float ms, const unsigned long long* cyc, int grid, int sms,
                   double ops_per_thread, bool last) {
    double ops = ops_per_thread * 256.0 * grid;
    double mean_span = (double)cyc[0] / grid, max_span = (double)cyc[1];
    int ctas_per_sm = grid / sms;
    double per_sm_cycle = ops_per_thread * 256.0 * ctas_per_sm / max_span;
    printf("  \"%s\": {\"ms\": %.4f, \"tops\": %.4f, \"lane_ops_per_sm_cycle\": %.2f, "
           "\"implied_mhz\": %.1f, \"mean_cta_span_frac\": %.3f}%s\n", name, ms,
           ops / (ms * 1e-3) / 1e12, per_sm_cycle, max_span / (ms * 1e3), mean_span / max_span,
           last ? "" : ",");
}

#define BENCH(NAME, KERNEL, ARGS_WARM, ARGS, OPS, LAST)                         \
    do {                                                                        \
        CK(cudaMemset(cyc, 0, 16));                                             \
        KERNEL<<<grid, 256>>> ARGS_WARM;                                        \
        CK(cudaDeviceSynchronize());                                            \
        CK(cudaMemset(cyc, 0, 16));                                             \
        cudaEventRecord(t.e0);                                                  \
        KERNEL<<<grid, 256>>> ARGS;                                             \
        cudaEventRecord(t.e1);                                                  \
        CK(cudaDeviceSynchronize());                                            \
        float ms = 0;                                                           \
        cudaEventElapsedTime(&ms, t.e0, t.e1);                                  \
        unsigned long long c[2] = {0, 0};                                       \
        cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);                         \
        report(NAME, ms, c, grid, sms, OPS, LAST);                              \
    } while (0)

int main() {
    int sms = 0, dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chains<double, 0>, 256, 0));
    const int grid = sms * occ;
    const int it = 20000;
    double* dsink;
    float* fsink;
    unsigned long long* cyc;
    CK(cudaMalloc(&dsink, 64));
    CK(cudaMalloc(&fsink, 64));
    CK(cudaMalloc(&cyc, 16));
    Timer t;
    printf("{\n  \"sms\": %d, \"ctas_per_sm\": %d, \"threads_per_cta\": 256, \"iters\": %d,\n", sms, occ, it);
    const double chain_ops = (double)it * 32;   // 4 unroll x 8 chains
    const double body_ops = (double)it * 4 * 10; // 4 unroll x (8 FP ops + 2 that keep x2+y2 live)
    BENCH("dadd", (chains<double, 0>), (1.0, it / 10, dsink, cyc), (1.0, it, dsink, cyc), chain_ops, false);
    BENCH("dmul", (chains<double, 1>), (1.0, it / 10, dsink, cyc), (1.0, it, dsink, cyc), chain_ops, false);
    BENCH("fadd", (chains<float, 0>), (1.0f, it / 10, fsink, cyc), (1.0f, it, fsink, cyc), chain_ops, false);
    BENCH("fmul", (chains<float, 1>), (1.0f, it / 10, fsink, cyc), (1.0f, it, fsink, cyc), chain_ops, false);
    BENCH("fadd2_lane_ops", (chains_f32x2<0>), (it / 10, fsink, cyc), (it, fsink, cyc), 2 * chain_ops, false);
    BENCH("fmul2_lane_ops", (chains_f32x2<1>), (it / 10, fsink, cyc), (it, fsink, cyc), 2 * chain_ops, false);
    BENCH("mandel_body_f64", (mandel_body<double>), (it / 10, dsink, cyc), (it, dsink, cyc), body_ops, false);
    BENCH("mandel_body_f32", (mandel_body<float>), (it / 10, fsink, cyc), (it, fsink, cyc), body_ops, true);
    printf("}\n");
    return 0;
}
