// loop_bench.cu -- the escape loop in isolation (no refill, no stores), to separate
// the cost of the per-iteration exit test from the cost of the refill logic.
// Points are chosen inside the main cardioid (never escape), so every warp runs
// `iters` iterations; reported as FP64 (or FP32) pipe fraction at 8 ops/iteration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/loop_bench tools/loop_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <typename T> struct B;
template <> struct B<double> { typedef long long t; static __device__ long long bits(double v) { return __double_as_longlong(v); } };
template <> struct B<float> { typedef int t; static __device__ int bits(float v) { return __float_as_int(v); } };

// MODE 0: no exit test;  MODE 1: 64-bit compare + __any_sync + branch every iteration;
// MODE 2: compare every iteration, __any_sync every 2nd (OR of the two);
// MODE 3: as 1 with a hi-word-only compare;  MODE 4: as 1 with c warp-uniform (kernel args);
// MODE 5: as 3 with c warp-uniform;  MODE 6: as 1 with the compare done in FP (DSETP/FSETP)
template <typename T, int ILP, int MODE>
__global__ void __launch_bounds__(256) loop(int iters, T r2v, T* sink, T ucr, T uci) {
    typedef typename B<T>::t BT;
    const BT r2 = B<T>::bits(r2v);
    const int r2hi = (int)(((long long)B<T>::bits(r2v)) >> (sizeof(T) == 8 ? 32 : 0));
    T x[ILP], y[ILP], x2[ILP], y2[ILP], cr[ILP], ci[ILP];
#pragma unroll
    for (int s = 0; s < ILP; ++s) {
        if (MODE == 4 || MODE == 5) {
            cr[s] = ucr + T(s) * T(1e-3);
            ci[s] = uci;
        } else {
            cr[s] = T(-0.3) + T(1e-7) * T(threadIdx.x + 37 * s);
            ci[s] = T(0.2) + T(1e-7) * T(blockIdx.x);
        }
        x[s] = y[s] = x2[s] = y2[s] = T(0);
    }
    int k = 0;
    bool esc = false;
    for (; k < iters; k += 2) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            bool e = false;
#pragma unroll
            for (int s = 0; s < ILP; ++s) {
                T ny = (x[s] + x[s]) * y[s] + ci[s];
                T nx = (x2[s] - y2[s]) + cr[s];
                x[s] = nx; y[s] = ny;
                x2[s] = x[s] * x[s]; y2[s] = y[s] * y[s];
                if (MODE == 0) x[s] = x[s] + (x2[s] + y2[s]) * T(0);  // keep the 8th op live
                else if (MODE == 3 || MODE == 5) {
                    T sm = x2[s] + y2[s];
                    int hi = sizeof(T) == 8 ? __double2hiint((double)sm) : B<T>::bits(sm);
                    e |= hi > r2hi;
                } else if (MODE == 6) e |= (x2[s] + y2[s]) > r2v;
                else e |= B<T>::bits(x2[s] + y2[s]) > r2;
            }
            esc |= e;
            if (MODE != 0 && MODE != 2 && __any_sync(0xffffffffu, e)) goto out;
        }
        if (MODE == 2 && __any_sync(0xffffffffu, esc)) goto out;
    }
out:
    T acc = T(0);
#pragma unroll
    for (int s = 0; s < ILP; ++s) acc = acc + x[s] + y[s];
    if (acc == T(-12345) || k < 0) sink[0] = acc;
}

template <typename T, int ILP, int MODE>
void run(const char* name, int sms, int ctas_per_sm, int iters, T* sink, bool last) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * ctas_per_sm;
    loop<T, ILP, MODE><<<grid, 256>>>(iters / 10, T(4), sink, T(-0.3), T(0.2));
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    loop<T, ILP, MODE><<<grid, 256>>>(iters, T(4), sink, T(-0.3), T(0.2));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double iter_total = (double)grid * 256 * ILP * iters;
    const double lanes = sizeof(T) == 8 ? 64 : 128;
    const double peak = (double)sms * lanes * 1.965e9 / 8;  // pixel-iterations/s at 8 ops
    printf("  \"%s_ilp%d_mode%d_cta%d\": {\"ms\": %.3f, \"giter_s\": %.1f, \"frac\": %.4f}%s\n", name, ILP,
           MODE, ctas_per_sm, ms, iter_total / (ms * 1e-3) / 1e9, iter_total / (ms * 1e-3) / peak,
           last ? "" : ",");
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* ds;
    float* fs;
    cudaMalloc(&ds, 64);
    cudaMalloc(&fs, 64);
    const int it = 20000;
    printf("{\n");
    run<double, 1, 1>("f64", sms, 8, it, ds, false);
    run<double, 1, 3>("f64", sms, 8, it, ds, false);
    run<double, 1, 4>("f64", sms, 8, it, ds, false);
    run<double, 1, 5>("f64", sms, 8, it, ds, false);
    run<double, 1, 6>("f64", sms, 8, it, ds, false);
    for (int c : {4, 5}) {
        run<double, 2, 1>("f64", sms, c, it, ds, false);
        run<double, 2, 3>("f64", sms, c, it, ds, false);
        run<double, 2, 4>("f64", sms, c, it, ds, false);
        run<double, 2, 5>("f64", sms, c, it, ds, false);
        run<double, 2, 6>("f64", sms, c, it, ds, false);
    }
    run<float, 1, 1>("f32", sms, 8, it, fs, false);
    run<float, 1, 4>("f32", sms, 8, it, fs, false);
    run<float, 1, 6>("f32", sms, 8, it, fs, false);
    run<float, 2, 1>("f32", sms, 6, it, fs, false);
    run<float, 2, 4>("f32", sms, 6, it, fs, false);
    run<float, 4, 1>("f32", sms, 4, it, fs, false);
    run<float, 4, 4>("f32", sms, 4, it, fs, true);
    printf("}\n");
    return 0;
}
