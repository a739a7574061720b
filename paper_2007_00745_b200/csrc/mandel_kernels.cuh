// mandel_kernels.cuh -- sm_100a escape-time kernels (hot path of arXiv 2007.00745).
//
// Step a3 + a4 + a5 of the path; a2's dynamic part (FCFS chunk
// claims) and a6 (the gather to rank 0) are fused
// into the same kernel: counts are stored straight into rank 0's image through a
// (possibly peer-mapped) pointer.
//
// Arithmetic (Eq. 1/2; readings R2-R5, R10): from z = 0,
//   y' = (x + x)*y + ci;  x' = (x2 - y2) + cr;  x2 = x'*x';  y2 = y'*y';  n += 1;
//   escape iff x2 + y2 > R2.
// Every operation is an explicit round-to-nearest intrinsic (__dadd_rn, __dmul_rn,
// __fadd_rn, ...), which nvcc never contracts into an FMA, so counts are bit-exact
// against the oracle.  The compare is done on the IEEE bit patterns as integers:
// both x2 + y2 and R2 are non-negative and never NaN on a live lane (DESIGN.md
// "Escape compare"), where integer order equals floating-point order.  That takes
// the compare off the FP64 pipe (9 -> 8 FP64 instructions per iteration).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mandel {

constexpr uint32_t kWarpsPerCta = 8;
constexpr uint32_t kCtaThreads = kWarpsPerCta * 32;
constexpr uint32_t kChunkDone = 0xffffffffu;  // chunk_map entry: counter exhausted
constexpr uint32_t kIdleRem = 0xffffffffu;

enum : uint32_t { kSchemeBlock = 0, kSchemeCyclic = 1, kSchemeFcfs = 2 };

// Per-rank device state; zeroed by the host (cudaMemsetAsync) before every launch.
struct WorkState {
    unsigned int tile_ctr;        // next local tile index
    unsigned int chunks_claimed;  // successful global FCFS claims by this rank
    unsigned int rows_started;    // rows whose first tile this rank drew
    unsigned int pad0;
    unsigned long long sum_iters; // sum of counts stored by this rank
    unsigned long long pixels;    // pixels stored by this rank
    // followed by chunk_map[nchunks + 1] (uint32; 0 = unpublished, g+1 = global chunk g,
    // kChunkDone = exhausted)
};

struct Params {
    double xmin, ymax, dx, dy;       // fp64 mapping constants (host-derived, step a1)
    float xminf, ymaxf, dxf, dyf;    // fp32 mapping constants
    long long r2bits;                // bit pattern of R2 in the working type
    uint32_t W, H, iter_max;
    uint32_t scheme;
    uint32_t tile_w, tiles_per_row;
    // static schemes: slot s -> row s < count0 ? base0 + s*stride0 : base1 + (s - count0)
    uint32_t nslots, base0, stride0, count0, base1;
    uint32_t chunk_rows, nchunks;    // FCFS
    uint32_t* out;                   // rank 0's image, row-major W per row (local or peer)
    WorkState* ws;                   // this rank's state (local memory)
    uint32_t* chunk_map;             // this rank's local->global chunk table (local memory)
    uint32_t* fcfs_ctr;              // shared global chunk counter (GPU 0's memory)
};

template <typename T> struct Arith;
template <> struct Arith<double> {
    typedef long long bits_t;
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ long long bits(double v) { return __double_as_longlong(v); }
    static __device__ __forceinline__ double cvt(uint32_t v) { return __uint2double_rn(v); }
    static __device__ __forceinline__ double xmin(const Params& p) { return p.xmin; }
    static __device__ __forceinline__ double ymax(const Params& p) { return p.ymax; }
    static __device__ __forceinline__ double dx(const Params& p) { return p.dx; }
    static __device__ __forceinline__ double dy(const Params& p) { return p.dy; }
};
template <> struct Arith<float> {
    typedef int bits_t;
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ int bits(float v) { return __float_as_int(v); }
    static __device__ __forceinline__ float cvt(uint32_t v) { return __uint2float_rn(v); }
    static __device__ __forceinline__ float xmin(const Params& p) { return p.xminf; }
    static __device__ __forceinline__ float ymax(const Params& p) { return p.ymaxf; }
    static __device__ __forceinline__ float dx(const Params& p) { return p.dxf; }
    static __device__ __forceinline__ float dy(const Params& p) { return p.dyf; }
};

// One z-update of Eq. 1 and the Eq. 2 escape test, in the oracle's operation order.
#define MANDEL_STEP()                                              \
    do {                                                           \
        T ny_ = A::add(A::mul(A::add(x, x), y), ci);               \
        T nx_ = A::add(A::sub(x2, y2), cr);                        \
        x = nx_;                                                   \
        y = ny_;                                                   \
        x2 = A::mul(x, x);                                         \
        y2 = A::mul(y, y);                                         \
        esc = A::bits(A::add(x2, y2)) > r2;                        \
    } while (0)

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
    return *reinterpret_cast<const volatile uint32_t*>(p);
}
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) {
    *reinterpret_cast<volatile uint32_t*>(p) = v;
}

enum : int { kTileOk = 0, kTileSkip = 1, kTileNone = 2 };

// Draw the next tile of this rank's work (called by one lane).  A tile is the
// column range [j0, j1) of one row.  For FCFS, local chunk k (chunk_rows
// consecutive row slots) is bound to the next global chunk by the warp that
// draws its first tile; claims are issued in local-chunk order so that once the
// global counter is exhausted every later local chunk is too.
__device__ __forceinline__ int draw_tile(const Params& p, uint32_t& row, uint32_t& j0, uint32_t& j1) {
    const uint32_t t = atomicAdd(&p.ws->tile_ctr, 1u);
    const uint32_t slot = t / p.tiles_per_row;
    const uint32_t seg = t - slot * p.tiles_per_row;
    j0 = seg * p.tile_w;
    j1 = min(j0 + p.tile_w, p.W);
    if (p.scheme != kSchemeFcfs) {
        if (slot >= p.nslots) return kTileNone;
        row = slot < p.count0 ? p.base0 + slot * p.stride0 : p.base1 + (slot - p.count0);
        if (seg == 0) atomicAdd(&p.ws->rows_started, 1u);
        return kTileOk;
    }
    const uint32_t k = slot / p.chunk_rows;
    const uint32_t r = slot - k * p.chunk_rows;
    if (k > p.nchunks) return kTileNone;
    uint32_t g;
    if (r == 0 && seg == 0) {
        uint32_t prev = 1;
        if (k > 0) {
            unsigned ns = 32;
            while ((prev = ld_volatile(&p.chunk_map[k - 1])) == 0) {
                __nanosleep(ns);
                ns = min(ns * 2, 1024u);
            }
        }
        if (prev == kChunkDone) {
            g = kChunkDone;
        } else {
            // the claim: one system-scope atomic on the shared counter (GPU 0's HBM)
            const uint32_t c = atomicAdd_system(p.fcfs_ctr, 1u);
            g = c < p.nchunks ? c + 1 : kChunkDone;
            if (c < p.nchunks) atomicAdd(&p.ws->chunks_claimed, 1u);
        }
        st_volatile(&p.chunk_map[k], g);
    } else {
        unsigned ns = 32;
        while ((g = ld_volatile(&p.chunk_map[k])) == 0) {
            __nanosleep(ns);
            ns = min(ns * 2, 1024u);
        }
    }
    if (g == kChunkDone) return kTileNone;
    row = (g - 1) * p.chunk_rows + r;
    if (row >= p.H) return kTileSkip;
    if (seg == 0) atomicAdd(&p.ws->rows_started, 1u);
    return kTileOk;
}

__device__ __forceinline__ void flush_stats(const Params& p, unsigned long long iters,
                                            unsigned long long pix) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        iters += __shfl_xor_sync(0xffffffffu, iters, o);
        pix += __shfl_xor_sync(0xffffffffu, pix, o);
    }
    if ((threadIdx.x & 31) == 0 && pix) {
        atomicAdd(&p.ws->sum_iters, iters);
        atomicAdd(&p.ws->pixels, pix);
    }
}

// ---------------------------------------------------------------------------
// K1/K2: persistent escape kernel with a per-warp tile queue and lane refill.
// Each warp runs the iteration warp-uniformly (no per-lane branch) and leaves
// the inner loop as soon as any lane escapes or reaches iterMax; finished lanes
// store their count and immediately take the next pixel of the warp's tile
// stream, so lanes stay busy through the divergence near the set boundary.
// Per-lane state: z (x, y), x2, y2, c (cr, ci), remaining iterations, output index.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kCtaThreads)
escape_refill_kernel(const Params p) {
    typedef Arith<T> A;
    typedef typename A::bits_t B;
    const unsigned FULL = 0xffffffffu;
    const uint32_t lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const B r2 = (B)p.r2bits;
    const T xmin = A::xmin(p), ymax = A::ymax(p), dx = A::dx(p), dy = A::dy(p);
    const T zero = T(0);

    T x = zero, y = zero, x2 = zero, y2 = zero, cr = zero, ci = zero;
    uint32_t rem = kIdleRem;
    bool active = false;
    uint32_t* dst = p.out;
    unsigned long long my_iters = 0, my_pix = 0;

    uint32_t trow = 0, jcur = 0, jend = 0;  // warp-uniform tile cursor
    bool more = true;
    unsigned need = FULL;

    for (;;) {
        if (need) {
            const uint32_t nd = __popc(need);
            const uint32_t rank = __popc(need & lt_mask);
            const bool mine = (need >> lane) & 1u;
            uint32_t served = 0;
            while (served < nd) {
                if (jcur >= jend) {
                    if (!more) break;
                    int st = 0;
                    uint32_t r_ = 0, a_ = 0, b_ = 0;
                    if (lane == 0) st = draw_tile(p, r_, a_, b_);
                    st = __shfl_sync(FULL, st, 0);
                    if (st == kTileNone) { more = false; break; }
                    if (st == kTileSkip) continue;
                    trow = __shfl_sync(FULL, r_, 0);
                    jcur = __shfl_sync(FULL, a_, 0);
                    jend = __shfl_sync(FULL, b_, 0);
                }
                const uint32_t take = min(jend - jcur, nd - served);
                if (mine && rank >= served && rank < served + take) {
                    const uint32_t j = jcur + (rank - served);
                    cr = A::add(xmin, A::mul(A::cvt(j), dx));    // Cx[j] = xmin + j*dx
                    ci = A::sub(ymax, A::mul(A::cvt(trow), dy)); // Cy[i] = ymax - i*dy
                    x = y = x2 = y2 = zero;
                    rem = p.iter_max;
                    active = true;
                    dst = p.out + ((size_t)trow * p.W + j);
                }
                jcur += take;
                served += take;
            }
        }
        if (!__any_sync(FULL, active)) break;

        const uint32_t kmax = __reduce_min_sync(FULL, rem);
        uint32_t k = 0;
        bool esc = false;
        for (;;) {
            if (kmax - k >= 4) {
                MANDEL_STEP();
                if (__any_sync(FULL, esc)) { k += 1; break; }
                MANDEL_STEP();
                if (__any_sync(FULL, esc)) { k += 2; break; }
                MANDEL_STEP();
                if (__any_sync(FULL, esc)) { k += 3; break; }
                MANDEL_STEP();
                k += 4;
                if (__any_sync(FULL, esc) || k == kmax) break;
            } else {
                MANDEL_STEP();
                k += 1;
                if (__any_sync(FULL, esc) || k == kmax) break;
            }
        }
        bool done = false;
        if (active) {
            rem -= k;
            done = esc || rem == 0;
        }
        if (done) {
            const uint32_t n = p.iter_max - rem;
            *dst = n;                     // a5 (+a6 when dst is rank 0's peer image)
            my_iters += n;
            my_pix += 1;
            active = false;
            x = y = x2 = y2 = cr = ci = zero;  // an idle lane iterates z = 0 forever
            rem = kIdleRem;
        }
        need = __ballot_sync(FULL, done);
    }
    flush_stats(p, my_iters, my_pix);
}

// ---------------------------------------------------------------------------
// Baseline variant: one pixel per thread over a static 2D grid (32 x 8 threads,
// one warp = 32 consecutive pixels of a row), plain per-lane early exit.
// Static schemes only.  Kept for A/B measurement of the refill design.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kCtaThreads)
escape_static_kernel(const Params p) {
    typedef Arith<T> A;
    typedef typename A::bits_t B;
    const B r2 = (B)p.r2bits;
    const uint32_t j = blockIdx.x * 32 + threadIdx.x;
    const uint32_t slot = blockIdx.y * kWarpsPerCta + threadIdx.y;
    unsigned long long my_iters = 0, my_pix = 0;
    if (j < p.W && slot < p.nslots) {
        const uint32_t row = slot < p.count0 ? p.base0 + slot * p.stride0 : p.base1 + (slot - p.count0);
        const T cr = A::add(A::xmin(p), A::mul(A::cvt(j), A::dx(p)));
        const T ci = A::sub(A::ymax(p), A::mul(A::cvt(row), A::dy(p)));
        T x = T(0), y = T(0), x2 = T(0), y2 = T(0);
        bool esc = false;
        uint32_t n = 0;
        while (n < p.iter_max) {
            MANDEL_STEP();
            ++n;
            if (esc) break;
        }
        p.out[(size_t)row * p.W + j] = n;
        my_iters = n;
        my_pix = 1;
        if (threadIdx.x == 0 && j == 0) atomicAdd(&p.ws->rows_started, 1u);
    }
    flush_stats(p, my_iters, my_pix);
}

#undef MANDEL_STEP

}  // namespace mandel
