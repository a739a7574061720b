// fp_latency.cu -- dependent-chain latency of DADD / DMUL / FADD / IADD on one warp
// (cudaEvent time x SM clock / chain length), for the escape-loop latency model.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/fp_latency tools/fp_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, int n, double k) {
    double a = out[threadIdx.x];
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (OP == 0) a = __dadd_rn(a, k);
            else if (OP == 1) a = __dmul_rn(a, k);
        }
    }
    out[threadIdx.x] = a;
}
template <int OP>
__global__ void chainf(float* out, int n, float k) {
    float a = out[threadIdx.x];
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (OP == 0) a = __fadd_rn(a, k);
            else a = __fmul_rn(a, k);
        }
    }
    out[threadIdx.x] = a;
}
__global__ void chaini(int* out, int n, int k) {
    int a = out[threadIdx.x];
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) a = (a ^ k) + 3;
    }
    out[threadIdx.x] = a;
}

int main() {
    double* d; float* f; int* q;
    cudaMalloc(&d, 1024); cudaMalloc(&f, 1024); cudaMalloc(&q, 1024);
    cudaMemset(d, 0, 1024); cudaMemset(f, 0, 1024); cudaMemset(q, 0, 1024);
    int mhz = 0; cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0); mhz /= 1000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int n = 200000;
    float ms;
    printf("{\"sm_clock_attr_mhz\": %d", mhz);
#define RUN(NAME, LAUNCH, OPS)                                   \
    LAUNCH; cudaDeviceSynchronize();                              \
    cudaEventRecord(e0); LAUNCH; cudaEventRecord(e1);             \
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);  \
    printf(", \"%s_ns_per_op\": %.3f", NAME, ms * 1e6 / (double)(OPS));
    RUN("dadd", (chain<0><<<1, 32>>>(d, n, 1e-9)), (double)n * 16);
    RUN("dmul", (chain<1><<<1, 32>>>(d, n, 1.0000001)), (double)n * 16);
    RUN("fadd", (chainf<0><<<1, 32>>>(f, n, 1e-9f)), (double)n * 16);
    RUN("fmul", (chainf<1><<<1, 32>>>(f, n, 1.0000001f)), (double)n * 16);
    RUN("int_xor_add", (chaini<<<1, 32>>>(q, n, 5)), (double)n * 32);
    printf("}\n");
    return 0;
}
