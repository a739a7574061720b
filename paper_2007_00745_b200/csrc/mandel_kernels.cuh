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
//
// Kernels: escape_refill_kernel (EAGER: persistent CTAs, 2-D warp tiles, lane refill;
// the default loop tests |z|^2 every B updates and replays a hit batch exactly,
// DESIGN.md R18 -- eager_run), escape_lazy_kernel (LAZY: exact test after every
// update, first escape recorded per block of 16 updates, refill when enough lanes
// hold a finished slot; chosen for incoherent views),
// escape_adaptive_kernel (switches between the two per warp), escape_static_kernel
// (one pixel per thread; the A/B baseline).  Arithmetic policies: ArithF64,
// ArithF64Fma (MANDEL_FP64_FMA, R17), ArithF32, ArithF32P (packed FP32x2 loop).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mandel {

// Device-side checks for a debug build (-DMANDEL_DEBUG_CHECKS=1; compute-sanitizer is
// not available on the test pool): a failed check prints and traps the kernel.
#ifndef MANDEL_DEBUG_CHECKS
#define MANDEL_DEBUG_CHECKS 0
#endif
#define MANDEL_DCHECK(cond)                                                                 \
    do {                                                                                    \
        if (MANDEL_DEBUG_CHECKS && !(cond)) {                                               \
            printf("MANDEL_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, \
                   __LINE__, blockIdx.x, threadIdx.x);                                      \
            __trap();                                                                       \
        }                                                                                   \
    } while (0)

// FCFS stress build (-DMANDEL_FCFS_DELAY=1 -> libmandel_delay.so, tests only): random
// sleeps before each claim, between a claim and its binding, at rank start and before
// some stores, so the claim protocol runs under adversarial interleavings (SPEC.md:281
// "injected adversarial per-row delays").
#ifndef MANDEL_FCFS_DELAY
#define MANDEL_FCFS_DELAY 0
#endif
__device__ __forceinline__ void fcfs_delay(uint32_t salt, uint32_t odds_log2 = 1) {
#if MANDEL_FCFS_DELAY
    uint32_t h = salt * 0x9E3779B1u ^ (uint32_t)clock64() ^ (blockIdx.x * 0x85EBCA6Bu) ^
                 (threadIdx.x * 0xC2B2AE35u);
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    if ((h & ((1u << odds_log2) - 1u)) == 0) __nanosleep((h >> 12) & 0x3FFFu);  // up to ~16 us
#else
    (void)salt;
    (void)odds_log2;
#endif
}

// A/B switches of the batch-start backup in the fused-y forms (ArithF64Y, ArithF32Y)
#ifndef MANDEL_F64Y_SAVEX
#define MANDEL_F64Y_SAVEX true
#endif
#ifndef MANDEL_F32Y_SAVEX
#define MANDEL_F32Y_SAVEX true
#endif

#ifndef MANDEL_LAZY_UNROLL
#define MANDEL_LAZY_UNROLL 16
#endif

constexpr uint32_t kWarpsPerCta = 8;
constexpr uint32_t kCtaThreads = kWarpsPerCta * 32;
constexpr uint32_t kChunkDone = 0xffffffffu;  // chunk_map entry: counter exhausted
constexpr uint32_t kIdleRem = 0xffffffffu;

enum : uint32_t { kSchemeBlock = 0, kSchemeCyclic = 1, kSchemeFcfs = 2 };

// Per-rank device state; zeroed before every launch (the previous launch's first CTA,
// zero_next_state).  Every counter the kernel updates atomically sits on its own 128-B
// line: atomics to one line serialise in one L2 slice (~1 per cycle), and on a small
// view the tile draws and the CTAs' closing statistics would otherwise queue behind
// each other (C1: 16.5 us per render at iterMax 1 with one shared line).
struct WorkState {
    unsigned int tile_ctr;        // next local tile index (the tile queue: its own line)
    unsigned int pad_t[31];
    unsigned int chunks_claimed;  // successful global FCFS claims by this rank
    unsigned int rows_started;    // rows whose first tile this rank drew
    unsigned int pad_r[30];
    unsigned long long sum_iters; // sum of counts stored by this rank (one add per CTA)
    unsigned long long pad_s[15];
    unsigned long long pixels;    // pixels stored by this rank (one add per CTA)
    unsigned long long pad_p[15];
    unsigned long long warp_iters; // inner-loop iterations summed over warps (eager/adaptive)
    unsigned long long exits;      // inner-loop exits summed over warps (eager/adaptive)
    unsigned long long pad_l[14];
    unsigned long long clk_cycles; // sum over CTAs of thread 0's SM clock cycles (clock64) ...
    unsigned long long clk_ns;     // ... and of its wall time (%globaltimer): their ratio is the
                                   // SM clock during the kernel (mandel_stats.sm_clock_mhz)
    unsigned long long pad_c[14];
    // followed by chunk_map[nchunks + 1] (uint32; 0 = unpublished, g+1 = global chunk g,
    // kChunkDone = exhausted)
};
static_assert(sizeof(WorkState) == 6 * 128, "WorkState: one 128-B line per atomic counter group");

struct Params {
    double xmin, ymax, dx, dy;       // fp64 mapping constants (host-derived, step a1)
    float xminf, ymaxf, dxf, dyf;    // fp32 mapping constants
    long long r2bits;                // bit pattern of R2 in the working type
    int r2cand;                      // candidate threshold: key(bits(R2) + 1) (see Arith::key)
    uint32_t r2batch;                // batched-check threshold on ukey, below key(R2) (R18)
    uint32_t W, H, iter_max;
    uint32_t scheme;
    uint32_t fused_y;                // 1: warps whose slots are all safe run the fused-y form (R21)
    uint32_t tile_w, tiles_per_row;  // columns per tile; tiles per group of tile_rows row slots
    uint32_t tile_rows;              // row slots per tile (FCFS: divides chunk_rows)
    uint32_t tile_shift;             // log2(tile_rows * 8)
    uint32_t opaque_zero;            // 0: ArithF32P's contraction barrier (XOR operand)
    uint32_t band;                   // 1: out is this rank's compact band (row = local slot)
    uint32_t out_rows;               // rows the out buffer holds (debug checks; H for the image)
    uint32_t stage;                  // 1: stores go through the per-warp staging ring (StageEntry)
    uint32_t vec_ok;                 // 1: out, W and tile_w allow 16-B stores of 4 counts
    // static schemes: slot s -> row s < count0 ? base0 + s*stride0 : base1 + (s - count0)
    uint32_t nslots, base0, stride0, count0, base1;
    uint32_t chunk_rows, nchunks;    // FCFS
    uint32_t claim_batch;            // FCFS: chunks per claim (1 when ranks compete; more for one)
    uint32_t fcfs_sys;               // 1: the counter is shared across devices (system-scope atomics)
    uint32_t refill_lanes;           // lazy refill: leave the loop when this many lanes are free
    uint32_t first_block;            // EAGER batched: a refill of at least this many slots starts with
                                     // one exactly recorded block (0: never)
    uint32_t adapt_lo, adapt_hi;     // adaptive: eager->lazy below adapt_lo iterations per run,
                                     // lazy->eager above adapt_hi
    uint32_t* out;                   // rank 0's image, row-major W per row (local or peer)
    WorkState* ws;                   // this rank's state (local memory)
    uint32_t* chunk_map;             // this rank's local->global chunk table (local memory)
    uint32_t* fcfs_ctr;              // shared global chunk counter (GPU 0's memory)
    // the next render's work state (the other half of the rank's state) and counter word:
    // zeroed by this launch's first CTA, so renders need no host memset between them
    uint32_t* zero_next;
    uint32_t zero_words;
    uint32_t* zero_ctr;
};

// Arithmetic policies: the storage type T, its RN operations, the escape-test bit
// pattern, and one z-update in the oracle's exact operation order (step) with its
// |z|^2 (sumsq).  The kernels are templated on the policy.
struct ArithF64 {
    typedef double T;
    typedef long long bits_t;
    static constexpr bool kPacked = false;
    // the batched loop keeps the batch-start x as a copy (sx) instead of as x + x (t0)
    static constexpr bool kSaveX = false;
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ long long bits(double v) { return __double_as_longlong(v); }
    static __device__ __forceinline__ double cvt(uint32_t v) { return __uint2double_rn(v); }
    // 32-bit escape-candidate key: the high word of the bit pattern.  key(s) >= r2cand
    // (= high word of bits(R2) + 1) is necessary for s > R2; exits verify exactly.
    static __device__ __forceinline__ int key(double v) { return __double2hiint(v); }
    // unsigned key for the batched check: NaN (either sign) and inf compare above any
    // finite threshold
    static __device__ __forceinline__ uint32_t ukey(double v) { return (uint32_t)__double2hiint(v); }
    static __device__ __forceinline__ double xmin(const Params& p) { return p.xmin; }
    static __device__ __forceinline__ double ymax(const Params& p) { return p.ymax; }
    static __device__ __forceinline__ double dx(const Params& p) { return p.dx; }
    static __device__ __forceinline__ double dy(const Params& p) { return p.dy; }
    // Eq. 1: y' = (x + x) y + ci;  x' = (x2 - y2) + cr;  x2 = x'x';  y2 = y'y'  (8 ops with sumsq)
    static __device__ __forceinline__ void step(double& x, double& y, double& x2, double& y2,
                                                double cr, double ci) {
        const double ny = add(mul(add(x, x), y), ci);
        const double nx = add(sub(x2, y2), cr);
        x = nx;
        y = ny;
        x2 = mul(x, x);
        y2 = mul(y, y);
    }
    static __device__ __forceinline__ double sumsq(double, double, double x2, double y2) { return add(x2, y2); }
    // step() with x + x supplied (the batched loop keeps it: x = t * 0.5 exactly restores x)
    static __device__ __forceinline__ void step_t(double t, double& x, double& y, double& x2, double& y2,
                                                  double cr, double ci) {
        const double ny = add(mul(t, y), ci);
        const double nx = add(sub(x2, y2), cr);
        x = nx;
        y = ny;
        x2 = mul(x, x);
        y2 = mul(y, y);
    }
    static __device__ __forceinline__ double half(double t) { return mul(t, 0.5); }
    // the carried squares of a restored z (what step() left next to it)
    static __device__ __forceinline__ void resq(double x, double y, double& x2, double& y2) {
        x2 = mul(x, x);
        y2 = mul(y, y);
    }
};

// MANDEL_FP64_FMA: the same recurrence with fused multiply-adds (R17):
//   y' = fma(x + x, y, ci);  x' = fma(x, x, -y2) + cr;  y2 = y'y';  |z|^2 = fma(x', x', y2)
// -- 6 FP64 instructions per iteration instead of 8; a different map (own oracle).
struct ArithF64Fma : ArithF64 {
    static __device__ __forceinline__ double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
    static __device__ __forceinline__ void step(double& x, double& y, double& x2, double& y2,
                                                double cr, double ci) {
        const double ny = fma(add(x, x), y, ci);
        const double nx = add(fma(x, x, -y2), cr);
        x = nx;
        y = ny;
        y2 = mul(y, y);
        x2 = 0.0;  // not carried (dead)
    }
    static __device__ __forceinline__ double sumsq(double x, double, double, double y2) { return fma(x, x, y2); }
    static __device__ __forceinline__ void step_t(double t, double& x, double& y, double& x2, double& y2,
                                                  double cr, double ci) {
        const double ny = fma(t, y, ci);
        const double nx = add(fma(x, x, -y2), cr);
        x = nx;
        y = ny;
        y2 = mul(y, y);
        x2 = 0.0;
    }
    static __device__ __forceinline__ void resq(double, double y, double& x2, double& y2) {
        x2 = 0.0;
        y2 = mul(y, y);
    }
};

struct ArithF32 {
    typedef float T;
    typedef int bits_t;
    static constexpr bool kPacked = false;
    static constexpr bool kSaveX = false;
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ int bits(float v) { return __float_as_int(v); }
    static __device__ __forceinline__ float cvt(uint32_t v) { return __uint2float_rn(v); }
    static __device__ __forceinline__ int key(float v) { return __float_as_int(v); }  // exact
    static __device__ __forceinline__ uint32_t ukey(float v) { return (uint32_t)__float_as_int(v); }
    static __device__ __forceinline__ float xmin(const Params& p) { return p.xminf; }
    static __device__ __forceinline__ float ymax(const Params& p) { return p.ymaxf; }
    static __device__ __forceinline__ float dx(const Params& p) { return p.dxf; }
    static __device__ __forceinline__ float dy(const Params& p) { return p.dyf; }
    static __device__ __forceinline__ void step(float& x, float& y, float& x2, float& y2, float cr, float ci) {
        const float ny = add(mul(add(x, x), y), ci);
        const float nx = add(sub(x2, y2), cr);
        x = nx;
        y = ny;
        x2 = mul(x, x);
        y2 = mul(y, y);
    }
    static __device__ __forceinline__ float sumsq(float, float, float x2, float y2) { return add(x2, y2); }
    static __device__ __forceinline__ void step_t(float t, float& x, float& y, float& x2, float& y2, float cr,
                                                  float ci) {
        const float ny = add(mul(t, y), ci);
        const float nx = add(sub(x2, y2), cr);
        x = nx;
        y = ny;
        x2 = mul(x, x);
        y2 = mul(y, y);
    }
    static __device__ __forceinline__ float half(float t) { return mul(t, 0.5f); }
    static __device__ __forceinline__ void resq(float x, float y, float& x2, float& y2) {
        x2 = mul(x, x);
        y2 = mul(y, y);
    }
};

// ---------------------------------------------------------------------------
// "Fused-y" forms of the fp64 / fp32 policies (R21): the same map, one FP
// instruction fewer per update.  Eq. 1's y' = RN(RN((x + x) y) + ci) is computed as
// fma(RN(x y), 2, ci) = RN(2 RN(x y) + ci): x + x is exact, and RN(2p) = 2 RN(p) for
// any product p in the normal range, so the two agree whenever x y is 0 or normal and
// 2 RN(x y) does not overflow.  A slot may run this form only when its pixel is "safe":
// cr != 0 with |cr| >= 2^-400 and (ci = 0 or |ci| >= 2^-400) [fp32: 2^-32], and R^2 <= 2^256
// [fp32: 2^64].  Then every iterate component before the escape is 0 or at least
// 2^-454 (the sum of two doubles >= 2^-401 in magnitude is 0 or a multiple of their
// common ulp), so |x y| is 0 or >= 2^-908 (normal), and |x y| <= R^2 (no overflow).
// The kernels check the pixels of a warp at every refill (fast_slot) and run a warp's
// loop in this form only when all of its live slots are safe; the replay of a hit batch
// uses the same form (exact before the escape, so the recorded escape is the oracle's).
// ---------------------------------------------------------------------------
struct ArithF64Y : ArithF64 {
    // x + x is no part of the fused update, so the batch start keeps a copy of x (two
    // register moves, off the FP64 pipe) instead of computing x + x (one DADD per slot and
    // batch on the pipe that bounds the loop)
    static constexpr bool kSaveX = MANDEL_F64Y_SAVEX;
    static __device__ __forceinline__ void step(double& x, double& y, double& x2, double& y2,
                                                double cr, double ci) {
        const double ny = __fma_rn(mul(x, y), 2.0, ci);
        const double nx = add(sub(x2, y2), cr);
        x = nx;
        y = ny;
        x2 = mul(x, x);
        y2 = mul(y, y);
    }
    static __device__ __forceinline__ bool fast_slot(double cr, double ci) {
        return fabs(cr) >= 0x1p-400 && (ci == 0.0 || fabs(ci) >= 0x1p-400);
    }
};
struct ArithF32Y : ArithF32 {
    // fp32 is issue-bound: a move costs the same issue slot as the x + x FADD, but not the
    // FP32 pipe (C3 +0.4 %, profiles/r02al_c3_*.jsonl)
    static constexpr bool kSaveX = MANDEL_F32Y_SAVEX;
    static __device__ __forceinline__ void step(float& x, float& y, float& x2, float& y2, float cr, float ci) {
        const float ny = __fmaf_rn(mul(x, y), 2.0f, ci);
        const float nx = add(sub(x2, y2), cr);
        x = nx;
        y = ny;
        x2 = mul(x, x);
        y2 = mul(y, y);
    }
    static __device__ __forceinline__ bool fast_slot(float cr, float ci) {
        return fabsf(cr) >= 0x1p-32f && (ci == 0.0f || fabsf(ci) >= 0x1p-32f);
    }
};
// The fused-y partner of a policy (itself where there is none).
template <typename A> struct FusedY { typedef A type; static constexpr bool kHas = false; };
template <> struct FusedY<ArithF64> { typedef ArithF64Y type; static constexpr bool kHas = true; };
template <> struct FusedY<ArithF32> { typedef ArithF32Y type; static constexpr bool kHas = true; };

// MANDEL_FP32 with the batched loop on packed pairs of slots (NEXT-4b): FADD2/FMUL2
// (PTX add/sub/mul.rn.f32x2, sm_100a) do two slots' RN operations per instruction,
// bit-identical to the scalar ones.  ptxas contracts a packed multiply feeding a
// packed add into FFMA2 even with .rn and -fmad=false, so every product passes
// through an opaque integer XOR with a runtime zero (one LOP3 on its high half)
// that ptxas cannot see through; the SASS gate test checks no FFMA2 remains.
struct ArithF32P : ArithF32 {
    static constexpr bool kPacked = true;
    static constexpr bool kSaveX = true;
    typedef unsigned long long u64;
    static __device__ __forceinline__ u64 pk(float a, float b) {
        u64 r;
        asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
        return r;
    }
    static __device__ __forceinline__ void upk(u64 v, float& a, float& b) {
        asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
    }
    static __device__ __forceinline__ u64 add2(u64 a, u64 b) {
        u64 r;
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
        return r;
    }
    static __device__ __forceinline__ u64 sub2(u64 a, u64 b) {
        u64 r;
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
        return r;
    }
    static __device__ __forceinline__ u64 mul2(u64 a, u64 b) {
        u64 r;
        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
        return r;
    }
    // contraction barrier: v with its high half XOR-ed with oz (== 0 at run time)
    static __device__ __forceinline__ u64 opq(u64 v, uint32_t oz) {
        uint32_t lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(v));
        hi ^= oz;
        u64 r;
        asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
        return r;
    }
    // Eq. 1 on two slots at once, in the oracle's operation order
    static __device__ __forceinline__ void step2(float& xa, float& xb, float& ya, float& yb, float& x2a,
                                                 float& x2b, float& y2a, float& y2b, float cra, float crb,
                                                 float cia, float cib, uint32_t oz) {
        const u64 X = pk(xa, xb), Y = pk(ya, yb), X2 = pk(x2a, x2b), Y2 = pk(y2a, y2b);
        const u64 NY = add2(opq(mul2(add2(X, X), Y), oz), pk(cia, cib));
        const u64 NX = add2(sub2(X2, Y2), pk(cra, crb));
        upk(NX, xa, xb);
        upk(NY, ya, yb);
        upk(opq(mul2(NX, NX), oz), x2a, x2b);
        upk(opq(mul2(NY, NY), oz), y2a, y2b);
    }
};

// One z-update of Eq. 1 and the Eq. 2 escape test, in the oracle's operation order.
#define MANDEL_STEP()                                              \
    do {                                                           \
        A::step(x, y, x2, y2, cr, ci);                             \
        esc = A::bits(A::sumsq(x, y, x2, y2)) > r2;                \
    } while (0)

// The same update on slot s of the per-lane arrays (refill kernel).
#define MANDEL_STEP_SLOT(s)                                                \
    do {                                                                   \
        A::step(x[s], y[s], x2[s], y2[s], cr[s], ci[s]);                   \
        esc[s] = A::key(A::sumsq(x[s], y[s], x2[s], y2[s])) >= r2c;        \
    } while (0)

// chunk_map is private to one rank's kernel (its own HBM): device-scope relaxed
// accesses suffice and stay in L2 (a volatile access compiles to a system-scope
// strong load, measured at ~2500 cycles per tile draw on B200).
__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

enum : int { kTileOk = 0, kTileSkip = 1, kTileNone = 2 };

// Draw the next tile of this rank's work (called by one lane).  A tile is the
// column range [j0, j1) of one row.  For FCFS, local chunk k (chunk_rows
// consecutive row slots) is bound to the next global chunk by the warp that
// draws its first tile; claims are issued in local-chunk order so that once the
// global counter is exhausted every later local chunk is too.
// One FCFS claim ("the master node sends the next row number"):
// an atomic on the shared counter in GPU 0's HBM -- system scope when ranks on other
// GPUs claim from it too (NVLink), device scope otherwise.  Returns the chunk_map
// entry: global chunk + 1, or kChunkDone once every chunk is taken.
// Bind local chunks [k0, k0 + claim_batch) (up to nchunks) with one claim of that many
// global chunks -- or to kChunkDone without a claim once the counter is known exhausted.
// claim_batch is 1 whenever ranks compete for the counter (a claim reserves only the
// next chunk, so the FCFS tail stays one chunk); a single claimant binds 16 at a time,
// which shortens the chain of one-ahead bindings (each link an atomic round trip) that
// bounds small views (C1: 50 chunks of cheap rows).  Called by one lane.
__device__ __forceinline__ void bind_chunks(const Params& p, uint32_t k0, bool exhausted) {
    const uint32_t nb = p.claim_batch;
    uint32_t c = 0;
    if (!exhausted) {
        fcfs_delay(1);
        c = p.fcfs_sys ? atomicAdd_system(p.fcfs_ctr, nb) : atomicAdd(p.fcfs_ctr, nb);
    }
    uint32_t got = 0;
    for (uint32_t i = 0; i < nb && k0 + i <= p.nchunks; ++i) {
        const bool ok = !exhausted && c + i < p.nchunks;
        got += ok ? 1u : 0u;
        if (i == 0) fcfs_delay(3);  // the claim is made, its binding not yet visible
        st_volatile(&p.chunk_map[k0 + i], ok ? c + i + 1 : kChunkDone);
    }
    if (got) atomicAdd(&p.ws->chunks_claimed, got);
}

// Wait until local chunk k is bound (warp-collective: lane 0 reads, every lane loops on
// the broadcast value, so no lane spins alone while the others wait at a warp barrier).
__device__ __forceinline__ uint32_t wait_bound(const Params& p, uint32_t k) {
    const unsigned FULL = 0xffffffffu;
    unsigned ns = 32;
    for (;;) {
        uint32_t g = 0;
        if ((threadIdx.x & 31) == 0) g = ld_volatile(&p.chunk_map[k]);
        g = __shfl_sync(FULL, g, 0);
        if (g != 0) return g;
        __nanosleep(ns);
        ns = min(ns * 2, 256u);
    }
}

// A tile: `nrows` row slots x `cols` columns starting at column j0.  `base` is the
// first slot of the group (static schemes; rows come from the plan) or the first
// image row (FCFS; the group's rows are consecutive inside one chunk).  Its pixels
// are streamed in 8-column sub-blocks, row-major inside each (tile_pixel), so the
// pixels a warp holds at once are a compact 2-D patch: neighbours escape at nearly
// the same update, which makes escapes -- and the batched test's hits -- coincide.
struct Tile {
    uint32_t base, nrows, j0, cols;
    uint32_t slot;  // the rank's local slot of the first row (its band row in band mode)
};

// Pixel q of tile t -> image (row, col) and the row of the output buffer it is stored
// to: the image row, or (band mode) the rank-local band row = its local slot.
__device__ __forceinline__ void tile_pixel(const Params& p, const Tile& t, uint32_t q, uint32_t& row,
                                           uint32_t& col, uint32_t& orow, uint32_t& sub, uint32_t& w) {
    // full groups (the common case) have a power-of-two height: shift instead of divide
    const uint32_t band = t.nrows << 3;
    sub = t.nrows == p.tile_rows ? q >> p.tile_shift : q / band;
    w = q - sub * band;
    const uint32_t bw = min(8u, t.cols - (sub << 3));
    uint32_t dy, dx;
    if (bw == 8u) {
        dy = w >> 3;
        dx = w & 7u;
    } else {
        dy = w / bw;
        dx = w - dy * bw;
    }
    col = t.j0 + (sub << 3) + dx;
    MANDEL_DCHECK(q < t.nrows * t.cols && dy < t.nrows && col < t.j0 + t.cols && col < p.W);
    const uint32_t sl = t.base + dy;
    row = p.scheme == kSchemeFcfs ? sl
                                  : (sl < p.count0 ? p.base0 + sl * p.stride0 : p.base1 + (sl - p.count0));
    orow = p.band ? t.slot + dy : row;
    MANDEL_DCHECK(row < p.H && (p.out_rows == 0 || orow < p.out_rows));
}
__device__ __forceinline__ void tile_pixel(const Params& p, const Tile& t, uint32_t q, uint32_t& row,
                                           uint32_t& col, uint32_t& orow) {
    uint32_t sub, w;
    tile_pixel(p, t, q, row, col, orow, sub, w);
}

// ---------------------------------------------------------------------------
// Store staging (a5, and a6 when out is rank 0's peer-mapped map): coalesced,
// vectorised output stores.  A warp hands its tile stream out in blocks -- the 8-column
// sub-blocks of tile_pixel, up to 8 rows x 8 columns.  Each block in flight owns an
// entry of a per-warp ring of kStageEntries in shared memory, zeroed when opened; a
// retiring slot writes its count there (one STS instead of the scattered 4-B global
// store).  When the stream needs the entry again, kStageEntries blocks later, the block
// is stored: if every count is there (all nonzero -- counts are >= 1) as whole 32-B rows,
// two lanes per row with one 16-B vector store each (STG.E.128); otherwise (a slow
// interior pixel still computing) its retired counts one by one, and the slots still
// computing its pixels switch to direct stores (kStageDirect).  No atomics: nothing is
// tracked per retirement.  The warp stores what is left in its ring when it ends.
// ---------------------------------------------------------------------------
constexpr uint32_t kStageEntries = 8;
constexpr uint32_t kStageDirect = 0xffffffffu;

struct __align__(16) StageEntry {
    uint32_t npx;             // pixels of the block; 0 = the entry is free
    uint32_t base, slot;      // the tile's base (tile_pixel) and first band slot
    uint32_t col0;            // first image column of the block
    uint32_t shape;           // rows | columns << 8
    uint32_t pad[3];
    uint32_t counts[64];      // row-major inside the block (tile_pixel's w); 0 = not retired
};

__device__ __forceinline__ uint32_t stage_orow(const Params& p, uint32_t base, uint32_t slot, uint32_t dy) {
    const uint32_t sl = base + dy;
    const uint32_t row = p.scheme == kSchemeFcfs ? sl
                                                 : (sl < p.count0 ? p.base0 + sl * p.stride0 : p.base1 + (sl - p.count0));
    const uint32_t orow = p.band ? slot + dy : row;
    MANDEL_DCHECK(row < p.H && (p.out_rows == 0 || orow < p.out_rows));
    return orow;
}

// Store the retired counts of an open entry (warp-collective, warp-uniform en) and free
// it.  Returns true when the block was complete.
__device__ __forceinline__ bool stage_store(const Params& p, StageEntry& en, uint32_t lane) {
    __syncwarp();  // every lane's count is in shared memory
    const uint32_t nr = en.shape & 0xffu, bw = en.shape >> 8;
    const unsigned FULL = 0xffffffffu;
    bool whole = false;
    if (bw == 8u && p.vec_ok) {
        // lane 2*dy + h holds columns 4h..4h+3 of row dy: counts[4*lane .. 4*lane + 3]
        const bool mine = lane < 2 * nr;
        uint4 v = make_uint4(1u, 1u, 1u, 1u);
        if (mine) v = *reinterpret_cast<const uint4*>(&en.counts[4 * lane]);
        whole = __all_sync(FULL, v.x != 0u && v.y != 0u && v.z != 0u && v.w != 0u);
        if (whole && mine) {
            const uint32_t dy = lane >> 1, h = lane & 1u;
            uint32_t* dst = p.out + ((size_t)stage_orow(p, en.base, en.slot, dy) * p.W + en.col0 + h * 4);
            MANDEL_DCHECK((reinterpret_cast<uintptr_t>(dst) & 15u) == 0);
            *reinterpret_cast<uint4*>(dst) = v;
        }
    }
    if (!whole) {
        // narrow edge blocks, misaligned maps and incomplete blocks: count by count, row-major
        bool all = true;
        for (uint32_t w = lane; w < nr * bw; w += 32) {
            const uint32_t n = en.counts[w];
            if (n != 0u) {
                const uint32_t dy = w / bw, dx = w - dy * bw;
                MANDEL_DCHECK(en.col0 + dx < p.W && n <= p.iter_max);
                p.out[(size_t)stage_orow(p, en.base, en.slot, dy) * p.W + en.col0 + dx] = n;
            } else {
                all = false;
            }
        }
        whole = __all_sync(FULL, all);
    }
    __syncwarp();
    if (lane == 0) en.npx = 0u;
    __syncwarp();
    return whole;
}

// Open ring entry e for sub-block `sub` of tile t (warp-uniform).  The block still in the
// entry is stored first; if it was incomplete, the slots computing its pixels (tag entry
// e) switch to direct stores -- their global address is formed here from the entry (a
// staged slot never needs it otherwise).
template <int ILP>
__device__ __forceinline__ void stage_open(const Params& p, StageEntry* ring, uint32_t e, const Tile& t,
                                           uint32_t sub, uint32_t lane, uint32_t (&stag)[ILP],
                                           uint32_t* (&dst)[ILP]) {
    StageEntry& en = ring[e];
    if (en.npx != 0u && !stage_store(p, en, lane)) {
        const uint32_t bw = en.shape >> 8;
#pragma unroll
        for (int s = 0; s < ILP; ++s) {
            if (stag[s] != kStageDirect && (stag[s] >> 6) == e) {
                const uint32_t w = stag[s] & 63u, dy = w / bw, dx = w - dy * bw;
                dst[s] = p.out + ((size_t)stage_orow(p, en.base, en.slot, dy) * p.W + en.col0 + dx);
                stag[s] = kStageDirect;
            }
        }
    }
    if (lane < 16) *reinterpret_cast<uint4*>(&en.counts[lane * 4]) = make_uint4(0u, 0u, 0u, 0u);
    if (lane == 0) {
        const uint32_t bw = min(8u, t.cols - (sub << 3));
        en.npx = t.nrows * bw;
        en.base = t.base;
        en.slot = t.slot;
        en.col0 = t.j0 + (sub << 3);
        en.shape = t.nrows | (bw << 8);
    }
    __syncwarp();
}

// A slot retires count n: into its block's entry, or directly when it is not staged.
__device__ __forceinline__ void stage_retire(StageEntry* ring, uint32_t tag, uint32_t* dst, uint32_t n) {
    if (tag == kStageDirect) *dst = n;
    else ring[tag >> 6].counts[tag & 63u] = n;
}

// At the warp's end: store every block still in the ring (all complete by then, except
// blocks some of whose pixels were handed out unstaged).
__device__ __forceinline__ void stage_drain(const Params& p, StageEntry* ring, uint32_t lane) {
    __syncwarp();
#pragma unroll 1
    for (uint32_t e = 0; e < kStageEntries; ++e)
        if (ring[e].npx != 0u) stage_store(p, ring[e], lane);
}

// (ck, cg) caches lane 0's last local->global chunk binding, so only the first
// draw in each chunk reads chunk_map (an L2 round trip) -- init ck = 0xffffffff.
// tn: each warp's first tile is its own index in the grid -- no atomic, so the launch
// does not start with every warp of the rank hitting the one counter at once; later
// draws take counter values from the warp count on (init tn = first_tile(), then
// kTileFirstDone).  (Requesting the next index one tile ahead was tried: the tiles
// reserved by busy warps lengthened the tail, C2 -3%.)
constexpr uint32_t kTileFirstDone = 0xffffffffu;
__device__ __forceinline__ uint32_t first_tile() { return blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5); }
__device__ __forceinline__ int draw_tile(const Params& p, Tile& tl, uint32_t& ck, uint32_t& cg, uint32_t& tn) {
    // warp-collective: lane 0 issues the atomics, every lane computes the (uniform) tile
    const unsigned FULL = 0xffffffffu;
    const bool l0 = (threadIdx.x & 31) == 0;
    uint32_t t = 0;
    if (tn != kTileFirstDone) {
        t = tn;  // the warp's first tile
        tn = kTileFirstDone;
    } else {
        if (l0) t = atomicAdd(&p.ws->tile_ctr, 1u) + gridDim.x * kWarpsPerCta;
        t = __shfl_sync(FULL, t, 0);
    }
    const uint32_t grp = t / p.tiles_per_row;
    const uint32_t seg = t - grp * p.tiles_per_row;
    const uint32_t slot = grp * p.tile_rows;
    if (p.scheme != kSchemeFcfs) {
        if (slot >= p.nslots) return kTileNone;
        tl.j0 = seg * p.tile_w;
        tl.cols = min(p.tile_w, p.W - tl.j0);
        tl.base = slot;
        tl.slot = slot;
        tl.nrows = min(p.tile_rows, p.nslots - slot);
        if (l0 && seg == 0) atomicAdd(&p.ws->rows_started, tl.nrows);
        return kTileOk;
    }
    const uint32_t k = slot / p.chunk_rows;
    const uint32_t r = slot - k * p.chunk_rows;
    if (k > p.nchunks) return kTileNone;
    uint32_t g;
    if (k == ck) {
        g = cg;
    } else {
        if (r == 0 && seg == 0) {
            // first tile of local chunk k: bind the first batch if k == 0; the first chunk
            // of each batch binds the next batch one batch ahead (claims stay in
            // local-chunk order, so once the counter is exhausted every later local chunk
            // is too; a batch is bound before its tiles are drawn, so warps rarely wait)
            const uint32_t nb = p.claim_batch;
            if (k == 0 && l0) bind_chunks(p, 0, false);
            g = wait_bound(p, k);
            if (k % nb == 0 && k + nb <= p.nchunks && l0) bind_chunks(p, k + nb, g == kChunkDone);
        } else {
            g = wait_bound(p, k);
        }
    }
    ck = k;
    cg = g;
    if (g == kChunkDone) return kTileNone;
    const uint32_t row = (g - 1) * p.chunk_rows + r;
    if (row >= p.H) return kTileSkip;
    tl.j0 = seg * p.tile_w;
    tl.cols = min(p.tile_w, p.W - tl.j0);
    tl.base = row;
    tl.slot = slot;
    tl.nrows = min(p.tile_rows, p.H - row);
    if (l0 && seg == 0) atomicAdd(&p.ws->rows_started, tl.nrows);
    return kTileOk;
}

// The SM clock as the kernel saw it: thread 0 of each CTA reads its SM cycle counter and
// the global nanosecond timer at start and end (kept in shared memory, not registers);
// the host divides the sums.
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void cta_clock_start(unsigned long long* sm) {
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        sm[1] = global_ns();
        sm[0] = (unsigned long long)clock64();
    }
}
#define MANDEL_CTA_CLOCK_START()                       \
    __shared__ unsigned long long mandel_clk_sm_[2];   \
    cta_clock_start(mandel_clk_sm_)

// The first CTA zeroes the next render's state half and counter word (Params::zero_next).
__device__ __forceinline__ void zero_next_state(const Params& p) {
    if (blockIdx.x == 0 && blockIdx.y == 0) {
        const uint32_t tid = threadIdx.y * blockDim.x + threadIdx.x, nt = blockDim.x * blockDim.y;
        for (uint32_t i = tid; i < p.zero_words; i += nt) p.zero_next[i] = 0u;
        if (tid == 0 && p.zero_ctr) *p.zero_ctr = 0u;
    }
}

// Development timeline (-DMANDEL_TRACE=1 -> libmandel_trace.so, read by
// tools/trace_view.py only): one record per warp -- its SM, first and last
// %globaltimer, tiles drawn, pixels retired and their iterations.
#ifndef MANDEL_TRACE
#define MANDEL_TRACE 0
#endif
#if MANDEL_TRACE
struct TraceRec {
    unsigned long long t0, t1, iters;
    unsigned int smid, tiles, pixels, warp;
};
constexpr uint32_t kTraceRecs = 1u << 16;
__device__ TraceRec g_trace[kTraceRecs];
__device__ __forceinline__ void trace_warp(unsigned long long t0, uint32_t tiles, unsigned long long iters,
                                           unsigned long long pix) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        iters += __shfl_xor_sync(0xffffffffu, iters, o);
        pix += __shfl_xor_sync(0xffffffffu, pix, o);
    }
    const uint32_t w = (blockIdx.y * gridDim.x + blockIdx.x) * kWarpsPerCta +
                       ((threadIdx.y * blockDim.x + threadIdx.x) >> 5);
    if ((threadIdx.x & 31) == 0 && w < kTraceRecs) {
        unsigned int sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        g_trace[w] = TraceRec{t0, global_ns(), iters, sm, tiles, (unsigned int)pix, w};
    }
}
#define MANDEL_TRACE_START() const unsigned long long trace_t0_ = global_ns(); uint32_t trace_tiles_ = 0
#define MANDEL_TRACE_TILE() (++trace_tiles_)
#define MANDEL_TRACE_END() trace_warp(trace_t0_, trace_tiles_, my_iters, my_pix)
#else
#define MANDEL_TRACE_START() do {} while (0)
#define MANDEL_TRACE_TILE() do {} while (0)
#define MANDEL_TRACE_END() do {} while (0)
#endif

// The CTA's closing statistics: each warp reduces its lanes' sums by shuffles, warp sums
// meet in shared memory, and thread 0 adds the CTA's totals -- one atomic per counter
// per CTA (per warp before: C1's 3552 warps x 2 adds on one line cost ~5 us), then the
// CTA's clock span (cta_clock_start; read after the barrier, so it is the CTA's whole
// lifetime).  witers / exits are warp-uniform (lane 0's values are the warp's).
template <bool LOOP>
__device__ __forceinline__ void cta_flush(const Params& p, unsigned long long iters, unsigned long long pix,
                                          uint32_t witers, uint32_t exits, const unsigned long long* clk) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        iters += __shfl_xor_sync(0xffffffffu, iters, o);
        pix += __shfl_xor_sync(0xffffffffu, pix, o);
    }
    __shared__ unsigned long long red[kWarpsPerCta][4];
    const uint32_t tid = threadIdx.y * blockDim.x + threadIdx.x;
    if ((tid & 31) == 0) {
        red[tid >> 5][0] = iters;
        red[tid >> 5][1] = pix;
        if constexpr (LOOP) {
            red[tid >> 5][2] = witers;
            red[tid >> 5][3] = exits;
        }
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long a = 0, b = 0, c = 0, d = 0;
#pragma unroll
        for (uint32_t w = 0; w < kWarpsPerCta; ++w) {
            a += red[w][0];
            b += red[w][1];
            if constexpr (LOOP) {
                c += red[w][2];
                d += red[w][3];
            }
        }
        if (b) {
            atomicAdd(&p.ws->sum_iters, a);
            atomicAdd(&p.ws->pixels, b);
        }
        if (LOOP && d) {
            atomicAdd(&p.ws->warp_iters, c);
            atomicAdd(&p.ws->exits, d);
        }
        const long long c1 = clock64();
        const unsigned long long t1 = global_ns();
        atomicAdd(&p.ws->clk_cycles, (unsigned long long)c1 - clk[0]);
        atomicAdd(&p.ws->clk_ns, t1 - clk[1]);
    }
}

// Batched check (BT z-updates, then one |z|^2): true if one of this thread's slots has
// a final |z|^2 key reaching r2b (below key(R2); R18).  The warp-wide hit is
// the vote of this predicate (batch_hit).
template <typename A, int ILP, int BT, typename T>
__device__ __forceinline__ bool batch_key_hit(T (&x)[ILP], T (&y)[ILP], T (&x2)[ILP], T (&y2)[ILP],
                                          const T (&cr)[ILP], const T (&ci)[ILP], uint32_t r2b,
                                          uint32_t oz, const T (&t0)[ILP]) {
#pragma unroll
    for (int u = 0; u < BT; ++u) {
        if constexpr (!A::kSaveX) {
            if (u == 0) {  // the first update takes the caller's x + x (kept for the restore)
#pragma unroll
                for (int s = 0; s < ILP; ++s) A::step_t(t0[s], x[s], y[s], x2[s], y2[s], cr[s], ci[s]);
                continue;
            }
        }
        if constexpr (A::kPacked) {
#pragma unroll
            for (int s = 0; s + 1 < ILP; s += 2)
                A::step2(x[s], x[s + 1], y[s], y[s + 1], x2[s], x2[s + 1], y2[s], y2[s + 1], cr[s], cr[s + 1],
                         ci[s], ci[s + 1], oz);
            if (ILP & 1) A::step(x[ILP - 1], y[ILP - 1], x2[ILP - 1], y2[ILP - 1], cr[ILP - 1], ci[ILP - 1]);
        } else {
#pragma unroll
            for (int s = 0; s < ILP; ++s) A::step(x[s], y[s], x2[s], y2[s], cr[s], ci[s]);
        }
    }
    uint32_t m = 0;
#pragma unroll
    for (int s = 0; s < ILP; ++s) m = max(m, A::ukey(A::sumsq(x[s], y[s], x2[s], y2[s])));
    return m >= r2b;
}

// The exact replay of one slot S of a hit batch: restore its batch-start z (x from the kept
// x + x, or sx when packed), rebuild the squares with the same operations, and run the BT
// updates with the Eq. 2 test after each, recording the first escaping update in e[S].
template <typename A, int ILP, int BT, int S, typename T, typename B>
__device__ __forceinline__ void replay_slot(T (&x)[ILP], T (&y)[ILP], T (&x2)[ILP], T (&y2)[ILP],
                                            const T (&cr)[ILP], const T (&ci)[ILP], const T (&t0)[ILP],
                                            const T (&sx)[ILP], const T (&sy)[ILP], B r2, uint32_t (&e)[ILP]) {
    if constexpr (A::kSaveX) x[S] = sx[S];
    else x[S] = A::half(t0[S]);
    y[S] = sy[S];
    A::resq(x[S], y[S], x2[S], y2[S]);
#pragma unroll
    for (int u = 0; u < BT; ++u) {
        A::step(x[S], y[S], x2[S], y2[S], cr[S], ci[S]);
        if (A::bits(A::sumsq(x[S], y[S], x2[S], y2[S])) > r2) e[S] = min(e[S], (uint32_t)u);
    }
}

// ---------------------------------------------------------------------------
// One EAGER run of a warp: iterate Eq. 1 on every slot until some slot finishes
// (or the smallest remaining budget kmax runs out).  Returns the run length k;
// fin[s] marks finished slots and kx[s] the iterations slot s performed in the run.
// ---------------------------------------------------------------------------
template <typename A, int ILP, int BT, typename T>
__device__ __forceinline__ uint32_t eager_run(const Params& p, T (&x)[ILP], T (&y)[ILP], T (&x2)[ILP],
                                              T (&y2)[ILP], const T (&cr)[ILP], const T (&ci)[ILP],
                                              const uint32_t (&rem)[ILP], bool (&fin)[ILP],
                                              uint32_t (&kx)[ILP], uint32_t kmax) {
    typedef typename A::bits_t B;
    const unsigned FULL = 0xffffffffu;
    const B r2 = (B)p.r2bits;
    const int r2c = p.r2cand;
    const uint32_t r2b = p.r2batch;
    bool esc[ILP];
    // ---- iterate: Eq. 1 on every slot until some slot is finished.  BT = 1: the loop
    // tests a 32-bit candidate key (one compare per slot) after every update; on a
    // candidate the warp leaves the loop and verifies the exact 64-bit test, resuming
    // on a false alarm.  BT > 1 (batched check, R18): BT z-updates per test and |z|^2 only
    // after the last one, against a threshold below R2 that every slot which escaped
    // inside the batch still exceeds (|z| grows after an escape when R >= 2); on a
    // hit the warp restores the batch-start state and replays the batch with the
    // exact per-update test, so each recorded count is the slot's first escaping
    // update.  Budget tails shorter than BT run the per-update loop below.
    uint32_t k = 0;
    bool lazy_exit = false;
    for (;;) {
        if (BT > 1) {
            // only z is kept at the batch start (x as x + x, which the first update
            // consumes anyway; y copied); on a hit A::resq rebuilds the carried squares
            // from it with the same operations (identical bits), and the whole batch is
            // replayed with the exact per-update test, each slot's first escaping update
            // recorded; every slot that escaped in the batch is then retired at once
            while (kmax - k >= BT) {
                T sx[ILP], sy[ILP];
                bool hit;
                // the hot loop: BT updates, one test; a down-counter of whole batches is
                // its only loop state (k is advanced once, after the loop)
                const uint32_t nb0 = (kmax - k) / BT;
                uint32_t nb = nb0;
                T t0[ILP];  // x + x of the batch start: its first update's operand and x's backup
                for (;;) {
#pragma unroll
                    for (int s = 0; s < ILP; ++s) {
                        if constexpr (A::kSaveX) sx[s] = x[s];
                        else t0[s] = A::add(x[s], x[s]);
                        sy[s] = y[s];
                    }
                    // one vote and one branch leave the loop on a hit or at the budget
                    const bool h = batch_key_hit<A, ILP, BT>(x, y, x2, y2, cr, ci, r2b, p.opaque_zero, t0);
                    --nb;
                    if (__any_sync(FULL, h || nb == 0)) {
                        hit = __any_sync(FULL, h);
                        break;
                    }
                }
                k += (nb0 - nb) * BT;  // batches run, the hit batch included ...
                if (hit) k -= BT;      // ... which is counted after its replay
                if (!hit) break;
                uint32_t e[ILP];  // the slot's first escaping update in the batch (BT: none)
                // per slot index: R18 holds slot by slot (a slot whose final key stayed below
                // r2b did not escape in the batch), so with ILP 2 a hit confined to one slot
                // index replays that slot alone -- the other keeps its batch-end state
                bool hs[ILP];
#pragma unroll
                for (int s = 0; s < ILP; ++s) {
                    hs[s] = ILP == 1 || __any_sync(FULL, A::ukey(A::sumsq(x[s], y[s], x2[s], y2[s])) >= r2b);
                    e[s] = BT;
                }
                if (ILP == 2 && !(hs[0] && hs[1])) {
                    if (hs[0]) replay_slot<A, ILP, BT, 0>(x, y, x2, y2, cr, ci, t0, sx, sy, r2, e);
                    else replay_slot<A, ILP, BT, ILP - 1>(x, y, x2, y2, cr, ci, t0, sx, sy, r2, e);
                } else {
#pragma unroll
                    for (int s = 0; s < ILP; ++s) {
                        if constexpr (A::kSaveX) x[s] = sx[s];
                        else x[s] = A::half(t0[s]);  // (x + x) * 0.5 = x exactly
                        y[s] = sy[s];
                        A::resq(x[s], y[s], x2[s], y2[s]);
                    }
#pragma unroll
                    for (int u = 0; u < BT; ++u) {
#pragma unroll
                        for (int s = 0; s < ILP; ++s) {
                            A::step(x[s], y[s], x2[s], y2[s], cr[s], ci[s]);
                            if (A::bits(A::sumsq(x[s], y[s], x2[s], y2[s])) > r2) e[s] = min(e[s], (uint32_t)u);
                        }
                    }
                }
                bool any_esc = false;
#pragma unroll
                for (int s = 0; s < ILP; ++s) {
                    // idle slots (z = c = 0) never escape; R3 counts the escaping update
                    fin[s] = rem[s] != kIdleRem && e[s] < (uint32_t)BT;
                    kx[s] = k + e[s] + 1u;
                    any_esc |= fin[s];
                }
                k += BT;
                if (__any_sync(FULL, any_esc)) {
                    lazy_exit = true;
                    break;
                }
                // a false alarm (no slot escaped): keep batching from the batch end
            }
            if (lazy_exit) break;
        }
        const uint32_t lim = kmax;
        // per-update test up to the end of the budget (tails shorter than BT, BT = 1)
        while (k < lim) {
            if (lim - k >= 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    bool e = false;
#pragma unroll
                    for (int s = 0; s < ILP; ++s) MANDEL_STEP_SLOT(s);
#pragma unroll
                    for (int s = 0; s < ILP; ++s) e |= esc[s];
                    if (__any_sync(FULL, e)) { k += u + 1; goto left_loop; }
                }
                k += 4;
            } else {
                bool e = false;
#pragma unroll
                for (int s = 0; s < ILP; ++s) MANDEL_STEP_SLOT(s);
#pragma unroll
                for (int s = 0; s < ILP; ++s) e |= esc[s];
                k += 1;
                if (__any_sync(FULL, e)) break;
            }
        }
    left_loop:
        bool any_fin = false;
#pragma unroll
        for (int s = 0; s < ILP; ++s) {
            // exact Eq. 2 test on the candidate's own |z|^2 (same operands, same bits);
            // idle slots hold z = 0 and never pass it
            fin[s] = A::bits(A::sumsq(x[s], y[s], x2[s], y2[s])) > r2;
            any_fin |= fin[s];
        }
        if (k == kmax || __any_sync(FULL, any_fin)) break;
    }
#pragma unroll
    for (int s = 0; s < ILP; ++s)
        if (!(lazy_exit && fin[s])) kx[s] = k;

    return k;
}

// ---------------------------------------------------------------------------
// K1/K2: persistent escape kernel with a per-warp tile queue and lane refill.
// Each lane holds ILP independent pixels ("slots"); their z-updates are
// interleaved so the FP64 dependency chains of one warp overlap.  The warp
// iterates warp-uniformly (no per-lane branch) and leaves the inner loop as
// soon as any slot escapes or the smallest remaining budget runs out; finished
// slots store their count and immediately take the next pixels of the warp's
// tile stream, so lanes stay busy through the divergence near the set boundary.
// Per-slot state: z (x, y), x2, y2, c (cr, ci), remaining iterations, output ptr.
// ---------------------------------------------------------------------------
// LSTATS: count loop exits and iterations per warp (the kernel-choice probe only:
// the two counters cost ~3% on C2 in production, measured A/B).
// STAGE: stores go through the per-warp staging ring (the instantiation the host picks
// when p.stage is set; without it the kernel keeps no staging state at all).
#ifndef MANDEL_FIRST_BLOCK
#define MANDEL_FIRST_BLOCK 8
#endif
constexpr int kFirstBlock = MANDEL_FIRST_BLOCK;  // updates of the first block after a large refill
template <typename AR, int ILP, int LU, typename T>
__device__ __forceinline__ void lazy_block(T (&x)[ILP], T (&y)[ILP], T (&x2)[ILP], T (&y2)[ILP],
                                           const T (&cr)[ILP], const T (&ci)[ILP],
                                           typename AR::bits_t r2, uint32_t (&e)[ILP]);

template <typename AR, int ILP, int MINB, int BT = 1, bool LSTATS = false, bool STAGE = false>
__global__ void __launch_bounds__(kCtaThreads, MINB)
escape_refill_kernel(const Params p) {
    MANDEL_DCHECK((reinterpret_cast<uintptr_t>(p.ws) & 7u) == 0 && p.tile_rows >= 1 && p.tile_w >= 1);
    MANDEL_CTA_CLOCK_START();
    MANDEL_TRACE_START();
    zero_next_state(p);
    typedef AR A;
    typedef typename AR::T T;
    const unsigned FULL = 0xffffffffu;
    const uint32_t lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const T xmin = A::xmin(p), ymax = A::ymax(p), dx = A::dx(p), dy = A::dy(p);
    const T zero = T(0);

    // per-slot state; rem == kIdleRem marks an idle slot (z = c = 0: never a candidate)
    T x[ILP], y[ILP], x2[ILP], y2[ILP], cr[ILP], ci[ILP];
    uint32_t rem[ILP];
    uint32_t* dst[ILP];
    uint32_t stag[ILP];  // the slot's staging tag (entry * 64 + pixel of the block) or kStageDirect
    bool fs[ILP];        // the slot may run the fused-y form (FusedY; idle slots may)
    typedef typename FusedY<A>::type AF;
#pragma unroll
    for (int s = 0; s < ILP; ++s) {
        x[s] = y[s] = x2[s] = y2[s] = cr[s] = ci[s] = zero;
        fs[s] = true;
        rem[s] = kIdleRem;
        dst[s] = p.out;
        stag[s] = kStageDirect;
    }
    unsigned long long my_iters = 0, my_pix = 0;
    uint32_t w_iters = 0, w_exits = 0;  // warp-uniform loop statistics (wrap-free below 2^32)

    // this warp's store-staging ring (StageEntry)
    __shared__ StageEntry stage_ring[STAGE ? kWarpsPerCta : 1][STAGE ? kStageEntries : 1];
    StageEntry* const ring = stage_ring[STAGE ? threadIdx.x >> 5 : 0];
    if (STAGE && lane < kStageEntries) ring[lane].npx = 0u;
    __syncwarp();
    uint32_t tile_e0 = 0, sub_open = 0;  // ring entry of the tile's sub-block 0; sub-blocks opened

    // warp-uniform tile cursor: pixels [tq, tqend) of tile tl
    Tile tl = {0u, 0u, 0u, 0u, 0u};
    uint32_t tq = 0, tqend = 0;
    bool more = true;
    uint32_t ck_ = 0xffffffffu, cg_ = 0;  // the warp's chunk-binding cache (draw_tile)
    uint32_t tn_ = first_tile();          // the warp's first tile (draw_tile)
    fcfs_delay(4);
    unsigned need[ILP];
#pragma unroll
    for (int s = 0; s < ILP; ++s) need[s] = FULL;

    for (;;) {
        // ---- refill: hand the next pixels of the tile stream to the free slots
        uint32_t nd = 0, rank[ILP];
#pragma unroll
        for (int s = 0; s < ILP; ++s) {
            rank[s] = nd + __popc(need[s] & lt_mask);
            nd += __popc(need[s]);
        }
        if (nd) {
            uint32_t served = 0;
            uint32_t opens = 0;  // ring entries opened this round: at most kStageEntries - 1, so
                                 // the blocks one round hands out never share an entry
            for (;;) {
                if (tq >= tqend) {
                    if (!more) break;
                    const int st = draw_tile(p, tl, ck_, cg_, tn_);  // warp-uniform
                    if (st == kTileNone) { more = false; break; }
                    if (st == kTileSkip) continue;
                    MANDEL_TRACE_TILE();
                    tq = 0;
                    tqend = tl.nrows * tl.cols;
                    tile_e0 = (tile_e0 + sub_open) & (kStageEntries - 1);
                    sub_open = 0;
                }
                const uint32_t take = min(tqend - tq, nd - served);
                if (STAGE) {
                    // open the ring entries of the sub-blocks this round hands out (pixels of a
                    // sub-block left unopened -- tiny blocks only -- store directly)
                    const uint32_t qe = tq + take - 1;
                    const uint32_t last = tl.nrows == p.tile_rows ? qe >> p.tile_shift : qe / (tl.nrows << 3);
                    for (; sub_open <= last && opens < kStageEntries - 1; ++sub_open, ++opens)
                        stage_open<ILP>(p, ring, (tile_e0 + sub_open) & (kStageEntries - 1), tl, sub_open, lane, stag, dst);
                }
#pragma unroll
                for (int s = 0; s < ILP; ++s) {
                    const uint32_t q = rank[s] - served;
                    if (((need[s] >> lane) & 1u) && q < take) {
                        uint32_t i, j, o, sb, w;
                        tile_pixel(p, tl, tq + q, i, j, o, sb, w);
                        cr[s] = A::add(xmin, A::mul(A::cvt(j), dx));      // Cx[j] = xmin + j*dx
                        ci[s] = A::sub(ymax, A::mul(A::cvt(i), dy));      // Cy[i] = ymax - i*dy
                        if constexpr (FusedY<A>::kHas) fs[s] = AF::fast_slot(cr[s], ci[s]);
                        x[s] = y[s] = x2[s] = y2[s] = zero;
                        rem[s] = p.iter_max;
                        const bool stg = STAGE && sb < sub_open;
                        stag[s] = stg ? ((((tile_e0 + sb) & (kStageEntries - 1)) << 6) | w) : kStageDirect;
                        if (!stg) dst[s] = p.out + ((size_t)o * p.W + j);
                    }
                }
                tq += take;
                served += take;
                if (served == nd) break;
            }
            if (served < nd) {
                // the work is exhausted: unserved free slots go idle
#pragma unroll
                for (int s = 0; s < ILP; ++s) {
                    if (((need[s] >> lane) & 1u) && rank[s] >= served) {
                        x[s] = y[s] = x2[s] = y2[s] = cr[s] = ci[s] = zero;
                        fs[s] = true;
                        rem[s] = kIdleRem;
                    }
                }
            }
        }
        uint32_t mrem = kIdleRem;
#pragma unroll
        for (int s = 0; s < ILP; ++s) mrem = min(mrem, rem[s]);
        const uint32_t kmax = __reduce_min_sync(FULL, mrem);
        if (kmax == kIdleRem) break;  // every slot of the warp is idle: done

        bool fin[ILP];
        uint32_t kx[ILP];  // per-slot iterations of this run (differs from k for batch-replay escapes)
        // the fused-y form when every slot of the warp is safe for it (ArithF64Y)
        bool fast = false;
        if constexpr (FusedY<A>::kHas) {
            bool ok = p.fused_y != 0u;
#pragma unroll
            for (int s = 0; s < ILP; ++s) ok = ok && fs[s];
            fast = __all_sync(FULL, ok);
        }
        uint32_t k;
        if (BT > 1 && !LSTATS && nd >= p.first_block && kmax >= (uint32_t)kFirstBlock) {
            // ---- first block: a refill that handed out many fresh pixels (the warp is in the
            // exterior, where counts are a few updates) runs kFirstBlock updates with the exact
            // Eq. 2 test recorded after each (lazy_block) instead of a batch that would hit and
            // be replayed: half the updates per escape there.  Slots that did not escape keep
            // their exact state and go on in the batched loop.
            uint32_t e[ILP];
            const typename A::bits_t r2 = (typename A::bits_t)p.r2bits;
            if (fast) lazy_block<AF, ILP, kFirstBlock>(x, y, x2, y2, cr, ci, r2, e);
            else lazy_block<A, ILP, kFirstBlock>(x, y, x2, y2, cr, ci, r2, e);
#pragma unroll
            for (int s = 0; s < ILP; ++s) {
                fin[s] = rem[s] != kIdleRem && e[s] < (uint32_t)kFirstBlock;  // R3: count the escaping update
                kx[s] = fin[s] ? e[s] + 1u : (uint32_t)kFirstBlock;
            }
            k = kFirstBlock;
        } else {
            k = fast ? eager_run<AF, ILP, BT>(p, x, y, x2, y2, cr, ci, rem, fin, kx, kmax)
                     : eager_run<A, ILP, BT>(p, x, y, x2, y2, cr, ci, rem, fin, kx, kmax);
        }

        if (LSTATS) {
            w_iters += k;
            w_exits += 1;
        }

        // ---- retire finished slots (a5, +a6 when dst is rank 0's peer image): into the
        // staging ring, completed blocks stored whole with vector stores
#pragma unroll
        for (int s = 0; s < ILP; ++s) {
            bool done = false;
            if (rem[s] != kIdleRem) {
                rem[s] -= kx[s];
                done = fin[s] || rem[s] == 0;
            }
            if (done) {
                const uint32_t n = p.iter_max - rem[s];
                fcfs_delay(5, 5);
                if (STAGE) stage_retire(ring, stag[s], dst[s], n);
                else *dst[s] = n;
                my_iters += n;
                my_pix += 1;
            }
            need[s] = __ballot_sync(FULL, done);
        }
    }
    if (STAGE) stage_drain(p, ring, lane);
    MANDEL_TRACE_END();
    cta_flush<LSTATS>(p, my_iters, my_pix, w_iters, w_exits, mandel_clk_sm_);
}

// ---------------------------------------------------------------------------
// K1/K2 (lazy refill): like escape_refill_kernel, but a slot that escapes does not
// end the inner loop.  The warp runs blocks of LU z-updates on all slots with the
// exact Eq. 2 test after every update; the test only records e[s], the slot's first
// escaping update in the block -- one 64-bit compare (two ISETPs) and one predicated
// min per slot-update, no per-update count or live flag.  At the block end each live
// slot's count advances by e+1 (it escaped: R3 counts the escaping update) or by LU,
// capped at iterMax, so the count is min(first escape, iterMax) exactly as Eq. 1-2
// define it: updates past the escape or past iterMax inside the block change nothing.
// A finished slot stops counting and waits (its z keeps running, unread); the warp
// leaves the run only when `refill_lanes` lanes hold a finished slot, then retires
// and refills all of them in one pass over its tile stream.  This amortises the
// refill over several finished pixels -- the eager variant leaves the loop on every
// escape, which dominates where neighbouring counts differ (C4's zoom: one escape
// every ~2 warp-updates).  The block form replaced a per-update `n += live; live &=
// in` (1.5 more instructions per slot-update): C4 1739 -> 1770 Giter/s
// (profiles/r01w_sweep_lazy_record.jsonl).
// ---------------------------------------------------------------------------
// LU: updates between two exit tests; the exit is a refill decision only, so the
// interval changes no count.  C4 (refill_lanes 16): LU 2 -> 1543, 4 -> 1664,
// 8 -> 1696, 16 -> 1728 Giter/s (per-update form; profiles/r01g_sweep_lazy_unroll.jsonl).
template <typename AR, int ILP, int LU, typename T = typename AR::T>
__device__ __forceinline__ void lazy_block(T (&x)[ILP], T (&y)[ILP], T (&x2)[ILP], T (&y2)[ILP],
                                           const T (&cr)[ILP], const T (&ci)[ILP],
                                           typename AR::bits_t r2, uint32_t (&e)[ILP]) {
#pragma unroll
    for (int s = 0; s < ILP; ++s) e[s] = LU;
#pragma unroll
    for (int u = 0; u < LU; ++u) {
#pragma unroll
        for (int s = 0; s < ILP; ++s) {
            AR::step(x[s], y[s], x2[s], y2[s], cr[s], ci[s]);
            if (AR::bits(AR::sumsq(x[s], y[s], x2[s], y2[s])) > r2) e[s] = min(e[s], (uint32_t)u);
        }
    }
}

// Development instrumentation (-DMANDEL_LAZY_PROF=1 -> libmandel_prof.so, read by
// tools/lazy_prof.py only): slot-updates of the LAZY loop by slot state -- [live,
// past its escape inside the block, finished or idle] x [filling, draining] -- and the
// number of runs per mode; printed by the last CTA of a launch.
#ifndef MANDEL_LAZY_PROF
#define MANDEL_LAZY_PROF 0
#endif
#if MANDEL_LAZY_PROF
__device__ unsigned long long g_lazy_prof[8];
__device__ unsigned int g_lazy_prof_done;
#endif

template <typename AR, int ILP, int MINB, bool STAGE = false>
__global__ void __launch_bounds__(kCtaThreads, MINB)
escape_lazy_kernel(const Params p) {
    MANDEL_DCHECK((reinterpret_cast<uintptr_t>(p.ws) & 7u) == 0 && p.tile_rows >= 1 && p.tile_w >= 1);
    MANDEL_CTA_CLOCK_START();
    MANDEL_TRACE_START();
    zero_next_state(p);
    typedef AR A;
    typedef typename AR::T T;
    typedef typename A::bits_t B;
    constexpr uint32_t LU = MANDEL_LAZY_UNROLL;
    const unsigned FULL = 0xffffffffu;
    const uint32_t lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const B r2 = (B)p.r2bits;
    const T xmin = A::xmin(p), ymax = A::ymax(p), dx = A::dx(p), dy = A::dy(p);
    const T zero = T(0);
    const int refill_at = (int)p.refill_lanes;  // leave the run when this many lanes hold a finished slot

    T x[ILP], y[ILP], x2[ILP], y2[ILP], cr[ILP], ci[ILP];
    uint32_t n[ILP];
    bool live[ILP];  // the slot's pixel has not finished (its count still advances)
    bool has[ILP];   // the slot holds a pixel not yet stored (else idle: z = c = 0)
    uint32_t* dst[ILP];
    uint32_t stag[ILP];  // staging tag (as escape_refill_kernel)
    bool fs[ILP];        // the slot may run the fused-y form (FusedY; idle slots may)
    typedef typename FusedY<A>::type AF;
#pragma unroll
    for (int s = 0; s < ILP; ++s) {
        x[s] = y[s] = x2[s] = y2[s] = cr[s] = ci[s] = zero;
        fs[s] = true;
        n[s] = 0;
        live[s] = has[s] = false;
        dst[s] = p.out;
        stag[s] = kStageDirect;
    }
    __shared__ StageEntry stage_ring[STAGE ? kWarpsPerCta : 1][STAGE ? kStageEntries : 1];
    StageEntry* const ring = stage_ring[STAGE ? threadIdx.x >> 5 : 0];
    if (STAGE && lane < kStageEntries) ring[lane].npx = 0u;
    __syncwarp();
    uint32_t tile_e0 = 0, sub_open = 0;
    unsigned long long my_iters = 0, my_pix = 0;
    Tile tl = {0u, 0u, 0u, 0u, 0u};  // warp-uniform tile cursor (as escape_refill_kernel)
    uint32_t tq = 0, tqend = 0;
    bool more = true;
    uint32_t ck_ = 0xffffffffu, cg_ = 0;  // the warp's chunk-binding cache (draw_tile)
    uint32_t tn_ = first_tile();          // the warp's first tile (draw_tile)
#if MANDEL_LAZY_PROF
    unsigned long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
    fcfs_delay(4);

    for (;;) {
        // ---- refill free slots from the warp's tile stream
        unsigned need[ILP];
        uint32_t nd = 0, rank[ILP];
#pragma unroll
        for (int s = 0; s < ILP; ++s) {
            need[s] = __ballot_sync(FULL, !has[s]);
            rank[s] = nd + __popc(need[s] & lt_mask);
            nd += __popc(need[s]);
        }
        uint32_t served = 0;
        uint32_t opens = 0;  // ring entries opened this round (see escape_refill_kernel)
        while (served < nd) {
            if (tq >= tqend) {
                if (!more) break;
                const int st = draw_tile(p, tl, ck_, cg_, tn_);  // warp-uniform
                if (st == kTileNone) { more = false; break; }
                if (st == kTileSkip) continue;
                MANDEL_TRACE_TILE();
                tq = 0;
                tqend = tl.nrows * tl.cols;
                tile_e0 = (tile_e0 + sub_open) & (kStageEntries - 1);
                sub_open = 0;
            }
            const uint32_t take = min(tqend - tq, nd - served);
            if (STAGE) {
                const uint32_t qe = tq + take - 1;
                const uint32_t last = tl.nrows == p.tile_rows ? qe >> p.tile_shift : qe / (tl.nrows << 3);
                for (; sub_open <= last && opens < kStageEntries - 1; ++sub_open, ++opens)
                    stage_open<ILP>(p, ring, (tile_e0 + sub_open) & (kStageEntries - 1), tl, sub_open, lane, stag, dst);
            }
#pragma unroll
            for (int s = 0; s < ILP; ++s) {
                if (((need[s] >> lane) & 1u) && rank[s] >= served && rank[s] < served + take) {
                    uint32_t i, j, o, sb, w;
                    tile_pixel(p, tl, tq + (rank[s] - served), i, j, o, sb, w);
                    cr[s] = A::add(xmin, A::mul(A::cvt(j), dx));  // Cx[j] = xmin + j*dx
                    ci[s] = A::sub(ymax, A::mul(A::cvt(i), dy));  // Cy[i] = ymax - i*dy
                    if constexpr (FusedY<A>::kHas) fs[s] = AF::fast_slot(cr[s], ci[s]);
                    x[s] = y[s] = x2[s] = y2[s] = zero;
                    n[s] = 0;
                    live[s] = has[s] = true;
                    const bool stg = STAGE && sb < sub_open;
                    stag[s] = stg ? ((((tile_e0 + sb) & (kStageEntries - 1)) << 6) | w) : kStageDirect;
                    if (!stg) dst[s] = p.out + ((size_t)o * p.W + j);
                }
            }
            tq += take;
            served += take;
        }
        bool any_live = false;
#pragma unroll
        for (int s = 0; s < ILP; ++s) any_live |= live[s];
        if (!__any_sync(FULL, any_live)) break;  // tiles exhausted and every slot retired
        // the fused-y form when every live slot of the warp is safe for it (ArithF64Y);
        // finished slots iterate unread and idle ones hold z = c = 0
        bool fast = false;
        if constexpr (FusedY<A>::kHas) {
            bool ok = p.fused_y != 0u;
#pragma unroll
            for (int s = 0; s < ILP; ++s) ok = ok && (fs[s] || !live[s]);
            fast = __all_sync(FULL, ok);
        }
#if MANDEL_LAZY_PROF
        prof[more ? 6 : 7] += 1;
#endif

        // ---- blocks of LU updates until enough slots have finished
        for (;;) {
            uint32_t e[ILP];
            if (fast) lazy_block<AF, ILP, LU>(x, y, x2, y2, cr, ci, r2, e);
            else lazy_block<A, ILP, LU>(x, y, x2, y2, cr, ci, r2, e);
            bool fin[ILP];
#pragma unroll
            for (int s = 0; s < ILP; ++s) {
                // live: n < iterMax, so the cap keeps n <= iterMax (no uint32 overflow)
                const uint32_t inc = min(e[s] < LU ? e[s] + 1u : LU, p.iter_max - n[s]);
#if MANDEL_LAZY_PROF
                prof[(more ? 0 : 3) + (live[s] ? 0 : 2)] += live[s] ? inc : LU;
                if (live[s]) prof[more ? 1 : 4] += LU - inc;
#endif
                if (live[s]) n[s] += inc;
                fin[s] = live[s] && (e[s] < LU || n[s] == p.iter_max);
            }
#pragma unroll
            for (int s = 0; s < ILP; ++s) live[s] = live[s] && !fin[s];
            if (more) {
                bool want = false;
#pragma unroll
                for (int s = 0; s < ILP; ++s) want |= !live[s];
                if (__popc(__ballot_sync(FULL, want)) >= refill_at) break;
            } else {  // draining: run until every slot is done
                bool go = false;
#pragma unroll
                for (int s = 0; s < ILP; ++s) go |= live[s];
                if (!__any_sync(FULL, go)) break;
            }
        }

        // ---- retire the finished slots (a5, +a6 when dst is rank 0's peer image) through
        // the staging ring (escape_refill_kernel)
#pragma unroll
        for (int s = 0; s < ILP; ++s) {
            if (has[s] && !live[s]) {
                fcfs_delay(5, 5);
                if (STAGE) stage_retire(ring, stag[s], dst[s], n[s]);
                else *dst[s] = n[s];
                my_iters += n[s];
                my_pix += 1;
                has[s] = false;
                fs[s] = true;
                x[s] = y[s] = x2[s] = y2[s] = cr[s] = ci[s] = zero;  // idle: z = 0 forever
            }
        }
    }
    if (STAGE) stage_drain(p, ring, lane);
#if MANDEL_LAZY_PROF
    for (int q = 0; q < 8; ++q) {
        unsigned long long v = q < 6 ? prof[q] : (lane == 0 ? prof[q] : 0ull);
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        if (lane == 0) atomicAdd(&g_lazy_prof[q], v);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&g_lazy_prof_done, 1u) == gridDim.x - 1) {
            printf("LAZY_PROF live %llu past_escape %llu finished_or_idle %llu | drain live %llu past_escape %llu "
                   "finished_or_idle %llu | runs %llu drain_runs %llu\n",
                   g_lazy_prof[0], g_lazy_prof[1], g_lazy_prof[2], g_lazy_prof[3], g_lazy_prof[4],
                   g_lazy_prof[5], g_lazy_prof[6], g_lazy_prof[7]);
            for (int q = 0; q < 8; ++q) g_lazy_prof[q] = 0;
            g_lazy_prof_done = 0;
        }
    }
#endif
    MANDEL_TRACE_END();
    cta_flush<false>(p, my_iters, my_pix, 0u, 0u, mandel_clk_sm_);
}

// ---------------------------------------------------------------------------
// K1/K2 (adaptive): the eager kernel's state and exits, plus the lazy kernel's
// in-loop escape bookkeeping, chosen per warp and per run.  A warp whose eager
// runs average (EMA, weight 1/4) fewer than adapt_lo iterations (escapes are
// dense and incoherent, e.g. C4's zoom) switches to adapt_hi lazy runs, which
// retire and refill only when refill_lanes lanes hold a finished pixel, and
// then probes eager runs again (sparse, coherent escapes: C2, C5).
// Lazy per-slot bookkeeping: `rem -= lv` and `lv = in ? lv : 0` every iteration
// with the exact 64-bit Eq. 2 test (rem = iterations still allowed; lv = live).
// ---------------------------------------------------------------------------
#define ADAPT_LAZY_STEP_SLOT(s)                                            \
    do {                                                                   \
        A::step(x[s], y[s], x2[s], y2[s], cr[s], ci[s]);                   \
        const bool in_ = !(A::bits(A::sumsq(x[s], y[s], x2[s], y2[s])) > r2); \
        rem[s] -= lv[s];                                                   \
        lv[s] = in_ ? lv[s] : 0u;                                          \
    } while (0)

template <typename AR, int ILP, int MINB, int BT = 1>
__global__ void __launch_bounds__(kCtaThreads, MINB)
escape_adaptive_kernel(const Params p) {
    MANDEL_DCHECK((reinterpret_cast<uintptr_t>(p.ws) & 7u) == 0 && p.tile_rows >= 1 && p.tile_w >= 1);
    MANDEL_CTA_CLOCK_START();
    MANDEL_TRACE_START();
    zero_next_state(p);
    typedef AR A;
    typedef typename AR::T T;
    typedef typename A::bits_t B;
    const unsigned FULL = 0xffffffffu;
    const uint32_t lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const B r2 = (B)p.r2bits;
    const T xmin = A::xmin(p), ymax = A::ymax(p), dx = A::dx(p), dy = A::dy(p);
    const T zero = T(0);
    const int max_live_full = 32 - (int)p.refill_lanes;

    T x[ILP], y[ILP], x2[ILP], y2[ILP], cr[ILP], ci[ILP];
    uint32_t rem[ILP];
    uint32_t* dst[ILP];
#pragma unroll
    for (int s = 0; s < ILP; ++s) {
        x[s] = y[s] = x2[s] = y2[s] = cr[s] = ci[s] = zero;
        rem[s] = kIdleRem;
        dst[s] = p.out;
    }
    unsigned long long my_iters = 0, my_pix = 0;
    Tile tl = {0u, 0u, 0u, 0u, 0u};  // warp-uniform tile cursor (as escape_refill_kernel)
    uint32_t tq = 0, tqend = 0;
    bool more = true;
    uint32_t ck_ = 0xffffffffu, cg_ = 0;  // the warp's chunk-binding cache (draw_tile)
    uint32_t tn_ = first_tile();          // the warp's first tile (draw_tile)
    bool lazy = false;           // warp-uniform run mode
    uint32_t ema = 4 * p.adapt_lo + 64;  // EMA of eager run lengths (x4, fixed point)
    uint32_t lazy_left = 0;      // lazy runs left before the next eager probe
    unsigned need[ILP];
#pragma unroll
    for (int s = 0; s < ILP; ++s) need[s] = FULL;

    for (;;) {
        // ---- refill (as escape_refill_kernel)
        uint32_t nd = 0, rank[ILP];
#pragma unroll
        for (int s = 0; s < ILP; ++s) {
            rank[s] = nd + __popc(need[s] & lt_mask);
            nd += __popc(need[s]);
        }
        if (nd) {
            uint32_t served = 0;
            for (;;) {
                if (tq >= tqend) {
                    if (!more) break;
                    const int st = draw_tile(p, tl, ck_, cg_, tn_);  // warp-uniform
                    if (st == kTileNone) { more = false; break; }
                    if (st == kTileSkip) continue;
                    MANDEL_TRACE_TILE();
                    tq = 0;
                    tqend = tl.nrows * tl.cols;
                }
                const uint32_t take = min(tqend - tq, nd - served);
#pragma unroll
                for (int s = 0; s < ILP; ++s) {
                    const uint32_t q = rank[s] - served;
                    if (((need[s] >> lane) & 1u) && q < take) {
                        uint32_t i, j, o;
                        tile_pixel(p, tl, tq + q, i, j, o);
                        cr[s] = A::add(xmin, A::mul(A::cvt(j), dx));      // Cx[j] = xmin + j*dx
                        ci[s] = A::sub(ymax, A::mul(A::cvt(i), dy));      // Cy[i] = ymax - i*dy
                        x[s] = y[s] = x2[s] = y2[s] = zero;
                        rem[s] = p.iter_max;
                        dst[s] = p.out + ((size_t)o * p.W + j);
                    }
                }
                tq += take;
                served += take;
                if (served == nd) break;
            }
            if (served < nd) {
#pragma unroll
                for (int s = 0; s < ILP; ++s) {
                    if (((need[s] >> lane) & 1u) && rank[s] >= served) {
                        x[s] = y[s] = x2[s] = y2[s] = cr[s] = ci[s] = zero;
                        rem[s] = kIdleRem;
                    }
                }
            }
        }
        uint32_t mrem = kIdleRem;
#pragma unroll
        for (int s = 0; s < ILP; ++s) mrem = min(mrem, rem[s]);
        const uint32_t kmax = __reduce_min_sync(FULL, mrem);
        if (kmax == kIdleRem) break;

        uint32_t k = 0;
        bool fin[ILP];
        if (!lazy) {
            // ---- eager run (per-update or batched test; see eager_run)
            uint32_t kx[ILP];
            k = eager_run<A, ILP, BT>(p, x, y, x2, y2, cr, ci, rem, fin, kx, kmax);
#pragma unroll
            for (int s = 0; s < ILP; ++s)
                if (rem[s] != kIdleRem) rem[s] -= kx[s];
            ema = ema - (ema >> 2) + k;  // ema/4 tracks the eager run length
            if ((ema >> 2) < p.adapt_lo) {
                lazy = true;
                lazy_left = p.adapt_hi;
            }
        } else {
            // ---- lazy run: per-slot exact bookkeeping, leave when enough lanes are free
            uint32_t lv[ILP];
#pragma unroll
            for (int s = 0; s < ILP; ++s) lv[s] = rem[s] != kIdleRem ? 1u : 0u;
            const int thr = more ? max_live_full : 0;
            for (;;) {
                if (kmax - k >= 2) {
#pragma unroll
                    for (int s = 0; s < ILP; ++s) ADAPT_LAZY_STEP_SLOT(s);
#pragma unroll
                    for (int s = 0; s < ILP; ++s) ADAPT_LAZY_STEP_SLOT(s);
                    k += 2;
                } else {
#pragma unroll
                    for (int s = 0; s < ILP; ++s) ADAPT_LAZY_STEP_SLOT(s);
                    k += 1;
                }
                uint32_t acc = more ? 1u : 0u;
#pragma unroll
                for (int s = 0; s < ILP; ++s) acc = more ? (acc & lv[s]) : (acc | lv[s]);
                const int c = __popc(__ballot_sync(FULL, acc != 0u));
                if (k == kmax || c <= thr) break;
            }
#pragma unroll
            for (int s = 0; s < ILP; ++s) fin[s] = lv[s] == 0u;  // escaped (or idle)
            if (--lazy_left == 0) {
                lazy = false;            // probe eager again
                ema = 4 * p.adapt_lo + 16;
            }
        }

        // ---- retire finished slots (a5, +a6 when dst is rank 0's peer image)
#pragma unroll
        for (int s = 0; s < ILP; ++s) {
            bool done = false;
            if (rem[s] != kIdleRem) done = fin[s] || rem[s] == 0;
            if (done) {
                const uint32_t n = p.iter_max - rem[s];
                *dst[s] = n;
                my_iters += n;
                my_pix += 1;
            }
            need[s] = __ballot_sync(FULL, done);
        }
    }
    MANDEL_TRACE_END();
    cta_flush<false>(p, my_iters, my_pix, 0u, 0u, mandel_clk_sm_);
}

#undef ADAPT_LAZY_STEP_SLOT

// ---------------------------------------------------------------------------
// Baseline variant: one pixel per thread over a static 2D grid (32 x 8 threads,
// one warp = 32 consecutive pixels of a row), plain per-lane early exit.
// Static schemes only.  Kept for A/B measurement of the refill design.
// ---------------------------------------------------------------------------
template <typename AR>
__global__ void __launch_bounds__(kCtaThreads)
escape_static_kernel(const Params p) {
    MANDEL_CTA_CLOCK_START();
    MANDEL_TRACE_START();
    zero_next_state(p);
    typedef AR A;
    typedef typename AR::T T;
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
        // band mode (options.band_out): the rank's compact band, band row = its local slot
        p.out[(size_t)(p.band ? slot : row) * p.W + j] = n;
        my_iters = n;
        my_pix = 1;
        if (threadIdx.x == 0 && j == 0) atomicAdd(&p.ws->rows_started, 1u);
    }
    MANDEL_TRACE_END();
    cta_flush<false>(p, my_iters, my_pix, 0u, 0u, mandel_clk_sm_);
}

#undef MANDEL_STEP
#undef MANDEL_STEP_SLOT

}  // namespace mandel
