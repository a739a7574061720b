// mandel.cu -- host runtime and C ABI (include/mandel.h) of the B200 escape-time library.
//
// Layers: L1 device kernels (mandel_kernels.cuh) <- L2 this host runtime
// (validation, step a1 constants, partition plans, per-device contexts, launches,
// statistics) <- L3 the extern "C" functions at the bottom.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false
//        -Xcompiler -fPIC,-ffp-contract=off -shared -Iinclude -o libmandel.so mandel.cu
#include <algorithm>
#include <atomic>
#include <chrono>
#include <map>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "mandel.h"
#include "mandel_kernels.cuh"
#include "mandel_image.cuh"

namespace {

thread_local std::string g_detail;

int fail(int code, const std::string& what) {
    g_detail = what;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    g_detail = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    if (e == cudaErrorMemoryAllocation) return MANDEL_ENOMEM;
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return MANDEL_ENODEV;
    return MANDEL_ECUDA;
}

#define CK(call)                                              \
    do {                                                      \
        cudaError_t e_ = (call);                              \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);   \
    } while (0)

// ---------------------------------------------------------------------------
// Step a1: validation and derived constants (SURVEY.md §8(a) a1, §8(b) errors).
// dx = (xmax - xmin)/W, dy = (ymax - ymin)/H, R2 = R*R, each one IEEE operation in
// the working type; fp32 first rounds the bounds and R to float (R9).
// ---------------------------------------------------------------------------
struct Derived {
    double xmin, ymax, dx, dy;
    float xminf, ymaxf, dxf, dyf;
    long long r2bits;
    bool r2_ge4;  // R2 >= 4 in the working type: the batched escape check is valid (R18)
};

int derive(double xmin, double xmax, double ymin, double ymax, uint32_t W, uint32_t H,
           uint32_t iter_max, double R, int dtype, Derived& d) {
    if (W == 0 || H == 0) return fail(MANDEL_EINVAL, "W and H must be >= 1");
    if ((uint64_t)W * (uint64_t)H > (uint64_t)(SIZE_MAX / 4)) return fail(MANDEL_EINVAL, "W*H*4 overflows size_t");
    if (iter_max == 0) return fail(MANDEL_EINVAL, "iterMax must be >= 1");
    // the kernels mark an idle slot with a remaining budget of 0xffffffff
    if (iter_max == 0xffffffffu) return fail(MANDEL_EINVAL, "iterMax must be < 2^32 - 1");
    if (dtype != MANDEL_FP64 && dtype != MANDEL_FP32 && dtype != MANDEL_FP64_FMA)
        return fail(MANDEL_EINVAL, "dtype out of range");
    if (!std::isfinite(xmin) || !std::isfinite(xmax) || !std::isfinite(ymin) || !std::isfinite(ymax))
        return fail(MANDEL_EINVAL, "window bounds must be finite");
    if (!(xmin < xmax) || !(ymin < ymax)) return fail(MANDEL_EINVAL, "need xmin < xmax and ymin < ymax");
    if (!std::isfinite(R) || !(R > 0.0)) return fail(MANDEL_EINVAL, "R must be finite and > 0");
    std::memset(&d, 0, sizeof(d));
    if (dtype == MANDEL_FP64 || dtype == MANDEL_FP64_FMA) {
        volatile double r2 = R * R;
        if (!std::isfinite((double)r2) || !(r2 > 0.0)) return fail(MANDEL_EINVAL, "R*R not finite/positive in fp64");
        volatile double dx = (xmax - xmin) / (double)W;
        volatile double dy = (ymax - ymin) / (double)H;
        if (!(dx > 0.0) || !(dy > 0.0) || !std::isfinite((double)dx) || !std::isfinite((double)dy))
            return fail(MANDEL_EINVAL, "window collapses (dx or dy not positive/finite)");
        d.xmin = xmin;
        d.ymax = ymax;
        d.dx = dx;
        d.dy = dy;
        double r2v = r2;
        std::memcpy(&d.r2bits, &r2v, 8);
        d.r2_ge4 = r2v >= 4.0;
        return MANDEL_OK;
    }
    volatile float xa = (float)xmin, xb = (float)xmax, ya = (float)ymin, yb = (float)ymax, Rf = (float)R;
    if (!std::isfinite((float)xa) || !std::isfinite((float)xb) || !std::isfinite((float)ya) ||
        !std::isfinite((float)yb) || !std::isfinite((float)Rf))
        return fail(MANDEL_EINVAL, "bounds or R not finite in fp32");
    if (!(xa < xb) || !(ya < yb)) return fail(MANDEL_EINVAL, "window collapses after rounding to fp32");
    if (!(Rf > 0.0f)) return fail(MANDEL_EINVAL, "R rounds to 0 in fp32");
    volatile float r2 = Rf * Rf;
    if (!std::isfinite((float)r2) || !(r2 > 0.0f)) return fail(MANDEL_EINVAL, "R*R not finite/positive in fp32");
    volatile float dx = (xb - xa) / (float)W;
    volatile float dy = (yb - ya) / (float)H;
    if (!(dx > 0.0f) || !(dy > 0.0f) || !std::isfinite((float)dx) || !std::isfinite((float)dy))
        return fail(MANDEL_EINVAL, "window collapses in fp32 (dx or dy == 0)");
    d.xminf = xa;
    d.ymaxf = yb;
    d.dxf = dx;
    d.dyf = dy;
    float r2v = r2;
    int32_t b;
    std::memcpy(&b, &r2v, 4);
    d.r2bits = b;
    d.r2_ge4 = r2v >= 4.0f;
    return MANDEL_OK;
}

// ---------------------------------------------------------------------------
// Step a2: static partition plans (§III).  A plan is a slot->row map
//   row(s) = s < count0 ? base0 + s*stride0 : base1 + (s - count0),  s < nslots.
// ---------------------------------------------------------------------------
struct Plan {
    uint32_t nslots, base0, stride0, count0, base1;
};

bool is_dynamic(int scheme) { return scheme == MANDEL_FCFS || scheme == MANDEL_FCFS_MASTER; }

int make_plan(int scheme, uint32_t H, int n, int r, Plan& pl) {
    if (n < 1) return fail(MANDEL_EINVAL, "ngpus must be >= 1");
    if (r < 0 || r >= n) return fail(MANDEL_EINVAL, "rank out of range");
    const uint32_t N = (uint32_t)n, R = (uint32_t)r;
    if (scheme == MANDEL_BLOCK || scheme == MANDEL_CYCLIC) {
        if (H < N) return fail(MANDEL_EINVAL, "static schemes need H >= ngpus");
        const uint32_t q = H / N;  // Eq. 16, rows per task
        if (scheme == MANDEL_BLOCK) {
            // Eq. 14: S_r = q*r;  Eq. 15 (read (r+1)): E_r = q*(r+1) - 1;  Eq. 17: last rank += H mod N
            const uint32_t rows = q + (R == N - 1 ? H % N : 0);
            pl = Plan{rows, q * R, 1, rows, 0};
        } else {
            // Alternating: r, r+N, ... below q*N; the master (rank 0) takes the tail [q*N, H)
            const uint32_t tail = (R == 0) ? H - q * N : 0;
            pl = Plan{q + tail, R, N, q, q * N};
        }
        return MANDEL_OK;
    }
    if (scheme == MANDEL_FCFS) {
        pl = Plan{0, 0, 0, 0, 0};
        return MANDEL_OK;
    }
    if (scheme == MANDEL_FCFS_MASTER) {
        if (N < 2) return fail(MANDEL_EINVAL, "FCFS_MASTER needs a master and at least one worker");
        pl = Plan{0, 0, 0, 0, 0};
        return MANDEL_OK;
    }
    return fail(MANDEL_EINVAL, "scheme out of range");
}

// ---------------------------------------------------------------------------
// Per-device and per-rank resources (cached across calls; freed by mandel_shutdown).
// ---------------------------------------------------------------------------
typedef void (*KernelFn)(mandel::Params);

struct DeviceCtx {
    bool init = false;
    int sms = 0;
    std::map<KernelFn, int> occ_cache;  // CTAs/SM per instantiated kernel (variant, ilp, budget,
                                        // batch length and packing all change the registers)
    bool peer_to0 = false;
    uint32_t* scratch = nullptr;  // the view probe's compact sample band (every 16th row)
    size_t scratch_bytes = 0;
    void* pstate = nullptr;       // the view probe's own work state
    size_t pstate_bytes = 0;
};

struct RankCtx {
    int device = -1;
    cudaStream_t stream = nullptr;
    cudaEvent_t k0 = nullptr, k1 = nullptr;
    // recorded after every launch that reads or writes `state`; the next call's reset of
    // the state waits on it, so enqueue-only renders on different streams never share it
    // mid-flight (the caller may pass a different stream per call)
    cudaEvent_t used = nullptr;
    // two halves of state_bytes each (WorkState + chunk_map): render n uses half par, and its
    // kernel zeroes the other half for render n + 1 -- no host memset between renders
    void* state = nullptr;
    size_t state_bytes = 0;
    int par = 0;
    size_t zeroed[2] = {0, 0};  // bytes of each half known to be zero
    void* half(int k) const { return static_cast<char*>(state) + (size_t)k * state_bytes; }
    // the per-device host hand-off (options.host_handoff): this rank's rows, stored on its
    // own device and copied to the host over its own link
    uint32_t* band = nullptr;
    size_t band_bytes = 0;
    cudaEvent_t d2h = nullptr;
};

constexpr int kMaxBands = 32;

struct Root {
    uint32_t* image = nullptr;  // library-owned map on device 0
    size_t image_bytes = 0;
    uint32_t* fcfs_ctr = nullptr;  // two counter words (0 and 32): render n claims from word
    int ctr_par = 0;               // ctr_par, its rank-0 kernel zeroes the other for render n+1
    bool ctr_zeroed[2] = {false, false};
    cudaEvent_t start = nullptr, done = nullptr, d2h = nullptr;
    // pipelined one-GPU hand-off: band states, a second compute stream, a copy stream
    void* band_state = nullptr;
    size_t band_state_bytes = 0;
    cudaStream_t band_stream = nullptr, copy_stream = nullptr;
    cudaEvent_t band_k0[kMaxBands] = {}, band_k1[kMaxBands] = {}, band_cp[kMaxBands] = {};
    cudaEvent_t copy_done = nullptr;
    // asynchronous pipelined renders (options.async_host): two library maps and band-state
    // sets used by alternate calls, a compute stream of their own, and per-set copy events
    uint32_t* pp_image[2] = {nullptr, nullptr};
    size_t pp_image_bytes = 0;
    void* pp_state[2] = {nullptr, nullptr};
    size_t pp_state_bytes = 0;
    cudaStream_t async_stream = nullptr;
    cudaEvent_t entry = nullptr, pp_done[2] = {nullptr, nullptr};
    int pp_next = 0;
};

std::mutex g_mu;
std::vector<uint32_t> g_band_rows;  // image row of each band row of the last band-mode render
std::atomic<bool> g_busy{false};
std::vector<DeviceCtx> g_dev;
RankCtx g_rank[MANDEL_MAX_GPUS];
Root g_root;

struct BusyGuard {
    bool ok;
    BusyGuard() { bool f = false; ok = g_busy.compare_exchange_strong(f, true); }
    ~BusyGuard() { if (ok) g_busy.store(false); }
};

constexpr int kVariantProbe = 99;  // internal: eager + loop statistics (kernel-choice probe)

// Register-budget instantiations (min CTAs per SM in __launch_bounds__).
constexpr int kMinbVals[6] = {1, 3, 4, 5, 6, 8};
int minb_index(int v) {
    for (int i = 0; i < 6; ++i)
        if (kMinbVals[i] == v) return i;
    return -1;
}

#define MANDEL_MINB_ROW(K, T, I) \
    {K<T, I, 1>, K<T, I, 3>, K<T, I, 4>, K<T, I, 5>, K<T, I, 6>, K<T, I, 8>}

// kernel_fn(dtype, variant, ilp, minb index); nullptr if not instantiated.
// dtype index: 0 = MANDEL_FP64, 1 = MANDEL_FP32, 2 = MANDEL_FP64_FMA.
#define MANDEL_ILP4_ROWS(K, A)                                                              \
    {MANDEL_MINB_ROW(K, A, 1), MANDEL_MINB_ROW(K, A, 2), MANDEL_MINB_ROW(K, A, 3),        \
     MANDEL_MINB_ROW(K, A, 4)}
#define MANDEL_ILP2_ROWS(K, A) {MANDEL_MINB_ROW(K, A, 1), MANDEL_MINB_ROW(K, A, 2)}
// batched-check EAGER kernels (R18): check every BT z-updates; min CTAs 1 or 3 only
#define MANDEL_BT_ROW(T, I, BT) {escape_refill_kernel<T, I, 1, BT>, escape_refill_kernel<T, I, 3, BT>}
#define MANDEL_BT_ROWS(T, BT) \
    {MANDEL_BT_ROW(T, 1, BT), MANDEL_BT_ROW(T, 2, BT), MANDEL_BT_ROW(T, 3, BT), MANDEL_BT_ROW(T, 4, BT)}
// Store-staging instantiations (STAGE = true): the batched EAGER loop (check every 8) and
// LAZY, ILP 1..4 / 1..2, register budgets 1 and 3 CTAs per SM; nullptr otherwise.
#define MANDEL_BT8S_ROW(T, I) {escape_refill_kernel<T, I, 1, 8, false, true>, escape_refill_kernel<T, I, 3, 8, false, true>}
#define MANDEL_BT8S_ROWS(T) {MANDEL_BT8S_ROW(T, 1), MANDEL_BT8S_ROW(T, 2), MANDEL_BT8S_ROW(T, 3), MANDEL_BT8S_ROW(T, 4)}
#define MANDEL_LAZYS_ROWS(T) \
    {{escape_lazy_kernel<T, 1, 1, true>, escape_lazy_kernel<T, 1, 3, true>}, \
     {escape_lazy_kernel<T, 2, 1, true>, escape_lazy_kernel<T, 2, 3, true>}}
KernelFn kernel_fn_staged(int fp32, int variant, int ilp, int mi, int bt) {
    using namespace mandel;
    static const KernelFn e8[4][4][2] = {MANDEL_BT8S_ROWS(ArithF64), MANDEL_BT8S_ROWS(ArithF32),
                                         MANDEL_BT8S_ROWS(ArithF64Fma), MANDEL_BT8S_ROWS(ArithF32P)};
    static const KernelFn lz[3][2][2] = {MANDEL_LAZYS_ROWS(ArithF64), MANDEL_LAZYS_ROWS(ArithF32),
                                         MANDEL_LAZYS_ROWS(ArithF64Fma)};
    if (mi < 0 || mi > 5) return nullptr;
    const int bi = kMinbVals[mi] == 1 ? 0 : (kMinbVals[mi] == 3 ? 1 : -1);
    if (bi < 0 || fp32 < 0 || fp32 > 3) return nullptr;
    if (variant == MANDEL_KERNEL_EAGER && bt == 8 && ilp >= 1 && ilp <= 4) return e8[fp32][ilp - 1][bi];
    if (fp32 == 3) fp32 = 1;
    if (variant == MANDEL_KERNEL_LAZY && ilp >= 1 && ilp <= 2) return lz[fp32][ilp - 1][bi];
    return nullptr;
}

KernelFn kernel_fn(int fp32, int variant, int ilp, int mi, int bt = 1) {
    using namespace mandel;
    static const KernelFn eager[3][4][6] = {MANDEL_ILP4_ROWS(escape_refill_kernel, ArithF64),
                                            MANDEL_ILP4_ROWS(escape_refill_kernel, ArithF32),
                                            MANDEL_ILP4_ROWS(escape_refill_kernel, ArithF64Fma)};
    static const KernelFn lazy[3][2][6] = {MANDEL_ILP2_ROWS(escape_lazy_kernel, ArithF64),
                                           MANDEL_ILP2_ROWS(escape_lazy_kernel, ArithF32),
                                           MANDEL_ILP2_ROWS(escape_lazy_kernel, ArithF64Fma)};
    static const KernelFn adaptive[3][2][6] = {MANDEL_ILP2_ROWS(escape_adaptive_kernel, ArithF64),
                                               MANDEL_ILP2_ROWS(escape_adaptive_kernel, ArithF32),
                                               MANDEL_ILP2_ROWS(escape_adaptive_kernel, ArithF64Fma)};
    static const KernelFn statics[3] = {escape_static_kernel<ArithF64>, escape_static_kernel<ArithF32>,
                                        escape_static_kernel<ArithF64Fma>};
    if (fp32 < 0 || fp32 > 3) return nullptr;
    if (fp32 == 3 && !(variant == MANDEL_KERNEL_EAGER && bt > 1)) fp32 = 1;  // packing: batched loop only
    if (variant == MANDEL_KERNEL_STATIC) return statics[fp32];
    if (variant == kVariantProbe) {  // the per-update-check eager kernels with loop statistics
        static const KernelFn probe[3] = {escape_refill_kernel<ArithF64, 2, 1, 1, true>,
                                          escape_refill_kernel<ArithF32, 4, 3, 1, true>,
                                          escape_refill_kernel<ArithF64Fma, 2, 1, 1, true>};
        return probe[fp32];
    }
    if (mi < 0 || mi > 5) return nullptr;
    if (variant == MANDEL_KERNEL_EAGER && bt > 1) {
        // row 3: fp32 on packed slot pairs (ArithF32P, NEXT-4b)
        static const KernelFn b4[4][4][2] = {MANDEL_BT_ROWS(ArithF64, 4), MANDEL_BT_ROWS(ArithF32, 4),
                                             MANDEL_BT_ROWS(ArithF64Fma, 4), MANDEL_BT_ROWS(ArithF32P, 4)};
        static const KernelFn b8[4][4][2] = {MANDEL_BT_ROWS(ArithF64, 8), MANDEL_BT_ROWS(ArithF32, 8),
                                             MANDEL_BT_ROWS(ArithF64Fma, 8), MANDEL_BT_ROWS(ArithF32P, 8)};
        const int bi = kMinbVals[mi] == 1 ? 0 : (kMinbVals[mi] == 3 ? 1 : -1);
        if (bi < 0 || ilp < 1 || ilp > 4) return nullptr;
        static const KernelFn b16[2][4][2] = {MANDEL_BT_ROWS(ArithF64, 16), MANDEL_BT_ROWS(ArithF64Fma, 16)};
        if (bt == 4) return b4[fp32][ilp - 1][bi];
        if (bt == 8) return b8[fp32][ilp - 1][bi];
        if (bt == 16 && (fp32 == 0 || fp32 == 2)) return b16[fp32 == 2 ? 1 : 0][ilp - 1][bi];
        return nullptr;
    }
    if (variant == MANDEL_KERNEL_EAGER && ilp >= 1 && ilp <= 4) return eager[fp32][ilp - 1][mi];
    if (variant == MANDEL_KERNEL_LAZY && ilp >= 1 && ilp <= 2) return lazy[fp32][ilp - 1][mi];
    if (variant == MANDEL_KERNEL_ADAPTIVE && bt > 1) {  // ADAPTIVE on the batched EAGER runs
        static const KernelFn ab[3][2][2][2] = {
            {{{escape_adaptive_kernel<ArithF64, 1, 1, 4>, escape_adaptive_kernel<ArithF64, 1, 3, 4>},
              {escape_adaptive_kernel<ArithF64, 1, 1, 8>, escape_adaptive_kernel<ArithF64, 1, 3, 8>}},
             {{escape_adaptive_kernel<ArithF64, 2, 1, 4>, escape_adaptive_kernel<ArithF64, 2, 3, 4>},
              {escape_adaptive_kernel<ArithF64, 2, 1, 8>, escape_adaptive_kernel<ArithF64, 2, 3, 8>}}},
            {{{escape_adaptive_kernel<ArithF32, 1, 1, 4>, escape_adaptive_kernel<ArithF32, 1, 3, 4>},
              {escape_adaptive_kernel<ArithF32, 1, 1, 8>, escape_adaptive_kernel<ArithF32, 1, 3, 8>}},
             {{escape_adaptive_kernel<ArithF32, 2, 1, 4>, escape_adaptive_kernel<ArithF32, 2, 3, 4>},
              {escape_adaptive_kernel<ArithF32, 2, 1, 8>, escape_adaptive_kernel<ArithF32, 2, 3, 8>}}},
            {{{escape_adaptive_kernel<ArithF64Fma, 1, 1, 4>, escape_adaptive_kernel<ArithF64Fma, 1, 3, 4>},
              {escape_adaptive_kernel<ArithF64Fma, 1, 1, 8>, escape_adaptive_kernel<ArithF64Fma, 1, 3, 8>}},
             {{escape_adaptive_kernel<ArithF64Fma, 2, 1, 4>, escape_adaptive_kernel<ArithF64Fma, 2, 3, 4>},
              {escape_adaptive_kernel<ArithF64Fma, 2, 1, 8>, escape_adaptive_kernel<ArithF64Fma, 2, 3, 8>}}}};
        const int bi = kMinbVals[mi] == 1 ? 0 : (kMinbVals[mi] == 3 ? 1 : -1);
        if (bi < 0 || ilp < 1 || ilp > 2 || (bt != 4 && bt != 8) || fp32 > 2) return nullptr;
        return ab[fp32][ilp - 1][bt == 8][bi];
    }
    if (variant == MANDEL_KERNEL_ADAPTIVE && ilp >= 1 && ilp <= 2) return adaptive[fp32][ilp - 1][mi];
    return nullptr;
}

// MANDEL_KERNEL_REFILL resolves to these configurations (the measured fastest).
struct KernelChoice {
    int variant, ilp, minb;
    int bt;          // EAGER: z-updates per escape check (1 = every update; 4, 8, 16 = batched, R18)
    int packed = 0;  // fp32 batched loop on FADD2/FMUL2 slot pairs (set by build_params)
    int ctas = 0;    // resident CTAs per SM cap (0: the occupancy maximum)
    int lanes = 0;   // LAZY refill_lanes (0: kDefaultRefillLanes; options.refill_lanes wins)
};
// ILP2 runs with ptxas' unconstrained schedule (74 registers, 3 CTAs of 256 threads per SM).
// Batched escape check with a whole-batch replay on a hit (R18), measured per config
// (profiles/r01_sweep_batch.jsonl, Giter/s): fp64 C2 check-every-8 ILP2 2061 (per-update
// check 1722), C5 2360 (1962); fp32 C3 check-every-8 ILP1 3346 (per-update ILP4 2504).
// fp32 stops at 8 updates per test: R18's drift bound covers no more (16 measured 3438).
// fp32 ILP1 fits 5 CTAs of 256 threads per SM (48 registers); 4 resident CTAs run C3 at
// 3584 Giter/s against 3491 with 5 (profiles/r02m_sweep.jsonl), so the default caps it.
constexpr KernelChoice kDefaultChoice[3] = {{MANDEL_KERNEL_EAGER, 2, 3, 8, 0, 0},    // fp64
                                            {MANDEL_KERNEL_EAGER, 1, 3, 8, 0, 4},    // fp32
                                            {MANDEL_KERNEL_EAGER, 2, 3, 8, 0, 0}};   // fp64 FMA
constexpr uint32_t kDefaultFirstBlock = 2;    // options.first_block (lanes)
constexpr uint32_t kDefaultRefillLanes = 16;  // LAZY on C4: 8 -> 1509, 16 -> 1555 Giter/s
constexpr uint32_t kDefaultAdaptLo = 8, kDefaultAdaptHi = 16;  // C2 1653, C4 1546, C5 1824 Giter/s
constexpr double kDefaultBandTaper = 0.7;  // band pair p holds a 0.7^p share of the rows
constexpr int kDefaultBands = 8;  // C2: 4 -> 8.50 ms, 8 -> 8.29 ms, 16 -> 8.86 ms per render (e2e_probe)  // pipelined device->host hand-off (one GPU, host output)

int device_count(int& n) {
    n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n <= 0) {
        cudaGetLastError();
        n = 0;
        return fail(MANDEL_ENODEV, std::string("no CUDA device: ") + cudaGetErrorString(e));
    }
    if ((int)g_dev.size() < n) g_dev.resize(n);
    return MANDEL_OK;
}

int ensure_device(int dev) {
    DeviceCtx& d = g_dev[dev];
    if (d.init) return MANDEL_OK;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
    d.init = true;
    return MANDEL_OK;
}

int ensure_peer(int dev) {
    if (dev == 0) return MANDEL_OK;
    DeviceCtx& d = g_dev[dev];
    if (d.peer_to0) return MANDEL_OK;
    int can = 0;
    CK(cudaDeviceCanAccessPeer(&can, dev, 0));
    if (!can) return fail(MANDEL_ENODEV, "peer access from device " + std::to_string(dev) + " to device 0 unavailable");
    CK(cudaSetDevice(dev));
    cudaError_t e = cudaDeviceEnablePeerAccess(0, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
    d.peer_to0 = true;
    return MANDEL_OK;
}

int ensure_rank(int r, int dev, size_t state_bytes, cudaStream_t user_stream) {
    RankCtx& rc = g_rank[r];
    if (rc.device != dev) {
        if (rc.device >= 0) {
            cudaSetDevice(rc.device);
            if (rc.stream) cudaStreamDestroy(rc.stream);
            if (rc.k0) cudaEventDestroy(rc.k0);
            if (rc.k1) cudaEventDestroy(rc.k1);
            if (rc.used) cudaEventDestroy(rc.used);
            if (rc.d2h) cudaEventDestroy(rc.d2h);
            if (rc.state) cudaFree(rc.state);
            if (rc.band) cudaFree(rc.band);
            rc = RankCtx();
        }
        rc.device = dev;
    }
    CK(cudaSetDevice(dev));
    // blocking streams: ordered after work the caller queued on the legacy default stream
    // (e.g. torch.zeros of the destination) when no stream0 is passed
    if (!rc.stream) CK(cudaStreamCreateWithFlags(&rc.stream, cudaStreamDefault));
    if (!rc.k0) CK(cudaEventCreate(&rc.k0));
    if (!rc.k1) CK(cudaEventCreate(&rc.k1));
    if (!rc.used) CK(cudaEventCreateWithFlags(&rc.used, cudaEventDisableTiming));
    if (rc.state_bytes < state_bytes) {
        // an enqueued render may still use the old buffer
        if (rc.state) CK(cudaEventSynchronize(rc.used));
        if (rc.state) CK(cudaFree(rc.state));
        rc.state = nullptr;
        rc.state_bytes = 0;
        CK(cudaMalloc(&rc.state, 2 * state_bytes));
        CK(cudaMemset(rc.state, 0, 2 * state_bytes));
        rc.state_bytes = state_bytes;
        rc.par = 0;
        rc.zeroed[0] = rc.zeroed[1] = state_bytes;
    }
    (void)user_stream;
    return MANDEL_OK;
}

constexpr uint32_t kDefaultTile = 256;     // pixels per tile (large views; small ones use less)
constexpr uint32_t kDefaultTileRows = 8;   // rows per tile: 8 x 32 px, streamed as 8 x 8 blocks
constexpr uint32_t kDefaultChunk = 16;

struct LaunchSpec {
    mandel::Params p;
    dim3 grid, block;
    KernelFn fn;
    KernelChoice kc;
    size_t smem = 0;  // dynamic shared memory (only to pin one CTA per SM, options.max_sms)
};

int occupancy(int device, KernelFn fn, int& occ) {
    int& c = g_dev[device].occ_cache[fn];
    if (c == 0) {
        CK(cudaSetDevice(device));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, fn, mandel::kCtaThreads, 0));
        if (c <= 0) c = 1;
    }
    occ = c;
    return MANDEL_OK;
}

// FCFS rows per claim: options.chunk_rows, else 16 (BASELINE.json C5) or, for the
// paper's master/worker protocol, one row.  Sizes the chunk map too.
uint32_t effective_chunk(int scheme, const mandel_options* o) {
    if (o && o->chunk_rows) return o->chunk_rows;
    return scheme == MANDEL_FCFS_MASTER ? 1u : kDefaultChunk;
}

int build_params(const Derived& d, uint32_t W, uint32_t H, uint32_t iter_max, int dtype, int scheme,
                 int nranks, int rank, const mandel_options* o, uint32_t* out, void* state,
                 size_t state_cap, uint32_t* fcfs_ctr, bool fcfs_sys, int device, LaunchSpec& ls,
                 const Plan* band = nullptr, const KernelChoice* force = nullptr, bool remote = false) {
    // FCFS runs its claims even with a single claimant (the counter then hands out chunks
    // 0, 1, 2, ... in order; chunks_claimed is the device's own count, Eq. 19).
    // FCFS_MASTER: rank 0 computes nothing (an empty plan, its kernel exits at once);
    // the workers run the FCFS claim path with single-row chunks by default.
    int kscheme = scheme;
    Plan pl;
    int rc = make_plan(kscheme, H, nranks, rank, pl);
    if (rc) return rc;
    if (band) {  // a row band of a one-GPU render (pipelined hand-off): rows in order
        kscheme = MANDEL_BLOCK;
        pl = *band;
    }
    if (kscheme == MANDEL_FCFS_MASTER) {
        if (rank == 0) {
            kscheme = MANDEL_BLOCK;
            pl = Plan{0, 0, 1, 0, 0};
        } else {
            kscheme = MANDEL_FCFS;
        }
    }
    const int kernel = o ? o->kernel : MANDEL_KERNEL_REFILL;
    if (kernel < MANDEL_KERNEL_REFILL || kernel > MANDEL_KERNEL_ADAPTIVE)
        return fail(MANDEL_EINVAL, "options.kernel out of range");
    if (kernel == MANDEL_KERNEL_STATIC && is_dynamic(scheme))
        return fail(MANDEL_EINVAL, "the static kernel has no work queue: FCFS needs the refill kernel");
    const uint32_t chunk = effective_chunk(scheme, o);
    // 2-D tiles: tile_rows row slots x (tile_px / tile_rows) columns; an
    // FCFS tile must stay inside one chunk, so its rows are cut to a power of two
    // dividing chunk_rows
    uint32_t trows = (o && o->tile_rows) ? (uint32_t)o->tile_rows : kDefaultTileRows;
    if (trows > 64 || (trows & (trows - 1)) != 0)
        return fail(MANDEL_EINVAL, "options.tile_rows must be a power of two <= 64");
    if (kscheme == MANDEL_FCFS)
        while (chunk % trows) trows >>= 1;
    // cyclic slots are stride0 rows apart: keep a tile's rows within ~8 image rows
    if (!(o && o->tile_rows) && kscheme == MANDEL_CYCLIC && pl.stride0 > 1)
        while (trows > 1 && trows * pl.stride0 > kDefaultTileRows) trows >>= 1;
    // default tile: 256 px, smaller when a rank has few pixels per resident warp (the
    // first tile draw then decides the critical path: C1 800^2 kernel 79 -> 38 us at 64 px)
    uint32_t tpx = (o && o->tile_px) ? o->tile_px : kDefaultTile;
    if (!(o && o->tile_px)) {
        const uint64_t px_rank = (uint64_t)W * H / (uint64_t)(nranks > 0 ? nranks : 1);
        const uint64_t warps = (uint64_t)(g_dev[device].sms > 0 ? g_dev[device].sms : 148) * 24;
        const uint64_t per_warp = px_rank / warps;
        tpx = per_warp >= 4096 ? 256u : (per_warp >= 1024 ? 128u : 64u);
    }
    uint32_t tile = tpx / trows > 0 ? tpx / trows : 1u;
    if (tile > W) tile = W;
    mandel::Params& p = ls.p;
    std::memset(&p, 0, sizeof(p));
    p.xmin = d.xmin; p.ymax = d.ymax; p.dx = d.dx; p.dy = d.dy;
    p.xminf = d.xminf; p.ymaxf = d.ymaxf; p.dxf = d.dxf; p.dyf = d.dyf;
    p.r2bits = d.r2bits;
    // candidate key threshold: fp64 -> high word of bits(R2)+1; fp32 -> bits(R2)+1 (exact)
    p.r2cand = dtype != MANDEL_FP32 ? (int)(((unsigned long long)d.r2bits + 1ull) >> 32)
                                    : (int)(d.r2bits + 1);
    // batched-check threshold (R18): key(R2) lowered by a relative margin far above the
    // rounding drift of an escaped orbit over 8 updates -- 2^-12 (fp64), 2^-2 (fp32)
    p.r2batch = dtype != MANDEL_FP32 ? (uint32_t)((unsigned long long)d.r2bits >> 32) - 0x100u
                                     : (uint32_t)d.r2bits - (1u << 21);
    p.W = W; p.H = H; p.iter_max = iter_max;
    p.scheme = (uint32_t)kscheme;
    p.tile_w = tile;
    p.tiles_per_row = (W + tile - 1) / tile;
    p.tile_rows = trows;
    p.tile_shift = 3;
    while ((1u << p.tile_shift) < trows * 8) ++p.tile_shift;
    p.nslots = pl.nslots; p.base0 = pl.base0; p.stride0 = pl.stride0; p.count0 = pl.count0; p.base1 = pl.base1;
    p.chunk_rows = chunk;
    p.nchunks = (uint32_t)(((uint64_t)H + chunk - 1) / chunk);
    // one claimant (N = 1, not the paper's master/worker) claims 16 chunks at a time
    p.claim_batch = (nranks == 1 && scheme == MANDEL_FCFS) ? 16u : 1u;
    if (kscheme == MANDEL_FCFS) {
        uint64_t tiles = (uint64_t)(p.nchunks + 1) * (chunk / trows) * p.tiles_per_row;
        if (tiles >= 0xF0000000ull) return fail(MANDEL_EINVAL, "FCFS tile space exceeds 32 bits; raise tile_px");
    } else if ((uint64_t)p.nslots * p.tiles_per_row >= 0xF0000000ull) {
        return fail(MANDEL_EINVAL, "tile space exceeds 32 bits; raise tile_px");
    }
    p.out = out;
    if (sizeof(mandel::WorkState) + ((size_t)p.nchunks + 2) * sizeof(uint32_t) > state_cap)
        return fail(MANDEL_ECUDA, "internal: chunk map larger than the rank state buffer");
    p.ws = reinterpret_cast<mandel::WorkState*>(state);
    p.chunk_map = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(state) + sizeof(mandel::WorkState));
    p.fcfs_ctr = fcfs_ctr;
    p.fcfs_sys = fcfs_sys ? 1u : 0u;
    const DeviceCtx& dc = g_dev[device];
    const int fi = dtype == MANDEL_FP32 ? 1 : (dtype == MANDEL_FP64_FMA ? 2 : 0);
    KernelChoice kc = kDefaultChoice[fi];
    if (force) {
        kc = *force;
        // the per-view choice fixes the kernel; an explicit ilp / min_ctas still applies
        // (mandel_render_ex and mandel_render_rank honour them alike)
        if (kernel == MANDEL_KERNEL_REFILL && kc.variant != kVariantProbe && o) {
            if (o->ilp) kc.ilp = o->ilp;
            if (o->min_ctas) kc.minb = o->min_ctas;
        }
    } else if (kernel != MANDEL_KERNEL_REFILL) {
        kc.variant = kernel;
        kc.ilp = (o && o->ilp) ? o->ilp : 2;
        kc.minb = (o && o->min_ctas) ? o->min_ctas : 1;
        kc.bt = 1;  // an explicit EAGER checks every update unless check_every says otherwise
    } else if (o && (o->ilp || o->min_ctas)) {
        if (o->ilp) kc.ilp = o->ilp;
        if (o->min_ctas) kc.minb = o->min_ctas;
    }
    // escape-check batching (R18): EAGER only, valid only when R2 >= 4 in the dtype.
    // Requested (check_every) -> errors if impossible; defaulted -> falls back to 1.
    const int ce = o ? o->check_every : 0;
    if (ce < 0 || (ce > 1 && ce != 4 && ce != 8 && ce != 16))
        return fail(MANDEL_EINVAL, "options.check_every must be 0, 1, 4, 8 or 16");
    if (kc.variant != MANDEL_KERNEL_EAGER && kc.variant != MANDEL_KERNEL_ADAPTIVE) {
        if (ce > 1 && !force) return fail(MANDEL_EINVAL, "check_every > 1 needs the EAGER or ADAPTIVE kernel");
        kc.bt = 1;
    } else if (ce) {
        if (ce > 1 && !d.r2_ge4) return fail(MANDEL_EINVAL, "a batched escape check needs R >= 2");
        if (ce > 8 && dtype == MANDEL_FP32)
            return fail(MANDEL_EINVAL, "fp32 allows check_every <= 8 (the R18 drift bound)");
        kc.bt = ce;
    } else if (!d.r2_ge4 || (kc.minb != 1 && kc.minb != 3)) {
        kc.bt = 1;
    }
    const int mi = minb_index(kc.minb);
    // fp32 batched loops run on packed slot pairs (FADD2/FMUL2) unless options.no_pack
    const bool packed = dtype == MANDEL_FP32 && kc.variant == MANDEL_KERNEL_EAGER && kc.bt > 1 &&
                        kc.ilp >= 2 && !(o && o->no_pack);
    kc.packed = packed ? 1 : 0;
    ls.kc = kc;
    // store staging (options.stage; DESIGN.md §6 "Store staging"): staged 8 x 8 blocks stored
    // with 16-B vector stores.  Default: staged when the map is another GPU's (the fused
    // gather's peer stores cross NVLink), direct 4-B stores into local HBM, where the L2
    // already merges them into whole lines (staging costs 1-4% there, measured)
    const int so = o ? o->stage : 0;
    if (so < -1 || so > 1) return fail(MANDEL_EINVAL, "options.stage must be -1, 0 or 1");
    bool stage = so == 1 || (so == 0 && remote);
    ls.fn = stage ? kernel_fn_staged(packed ? 3 : fi, kc.variant, kc.ilp, mi, kc.bt) : nullptr;
    if (!ls.fn) {  // no staged instantiation of this variant: direct stores
        stage = false;
        ls.fn = kernel_fn(packed ? 3 : fi, kc.variant, kc.ilp, mi, kc.bt);
    }
    p.opaque_zero = 0u;
    // fused-y form (R21): exact while |x y| <= R^2 cannot overflow 2 RN(x y) --
    // R^2 <= 2^256 (fp64) / 2^64 (fp32); the kernels add the per-pixel condition
    const int fy = o ? o->fused_y : 0;
    if (fy < -1 || fy > 1) return fail(MANDEL_EINVAL, "options.fused_y must be -1, 0 or 1");
    double r2v;
    if (dtype == MANDEL_FP32) {
        float f;
        const int32_t b = (int32_t)d.r2bits;
        std::memcpy(&f, &b, 4);
        r2v = f;
    } else {
        std::memcpy(&r2v, &d.r2bits, 8);
    }
    p.fused_y = (fy >= 0 && r2v <= (dtype == MANDEL_FP32 ? 0x1p64 : 0x1p256)) ? 1u : 0u;
    p.band = (o && o->band_out) ? 1u : 0u;
    p.stage = stage ? 1u : 0u;
    p.vec_ok = ((reinterpret_cast<uintptr_t>(out) & 15u) == 0 && (W & 3u) == 0 && (tile & 3u) == 0) ? 1u : 0u;
    p.out_rows = p.band ? 0u : H;  // a band's capacity is the caller's (not known here)
    if (!ls.fn) return fail(MANDEL_EINVAL, "no kernel instantiated for this variant/ilp/min_ctas");
    const bool persistent = kc.variant != MANDEL_KERNEL_STATIC;  // (the probe variant is persistent)
    int rl = (o && o->refill_lanes) ? o->refill_lanes
                                    : (kc.lanes ? kc.lanes : (int)kDefaultRefillLanes);
    if (rl < 1 || rl > 32) return fail(MANDEL_EINVAL, "options.refill_lanes must be in 1..32");
    p.refill_lanes = (uint32_t)rl;
    // first block (mandel_kernels.cuh): lanes' worth of fresh slots
    // that start one (C2: off 5.17, 1 -> 5.00, 4 -> 5.01, 16 -> 5.03, 32 -> 5.06 ms; profiles/r02as_*, r02at_*)
    const int fb = o ? o->first_block : 0;
    if (fb < -1 || fb > 32) return fail(MANDEL_EINVAL, "options.first_block must be -1 or in 0..32");
    p.first_block = fb < 0 ? 0xffffffffu : (uint32_t)((fb ? fb : (int)kDefaultFirstBlock) * kc.ilp);
    p.adapt_lo = (o && o->adapt_lo > 0) ? (uint32_t)o->adapt_lo : kDefaultAdaptLo;
    p.adapt_hi = (o && o->adapt_hi > 0) ? (uint32_t)o->adapt_hi : kDefaultAdaptHi;
    ls.block = persistent ? dim3(mandel::kCtaThreads) : dim3(32, mandel::kWarpsPerCta);
    if (persistent) {
        int occ = 1;
        int rc2 = occupancy(device, ls.fn, occ);
        if (rc2) return rc2;
        // options.max_sms: the rank is a slice of exactly that many SMs (the paper's task
        // on one core, tools/paper_tables.py): one CTA per SM -- a dynamic shared memory
        // request above half an SM's keeps any second CTA (this rank's or another's) off
        if (o && o->max_sms > 0) {
            int smem_sm = 0;
            CK(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device));
            ls.smem = (size_t)smem_sm / 2 + 1024;
            ls.grid = dim3((unsigned)std::min(o->max_sms, dc.sms));
        } else {
            if (o && o->ctas_per_sm < 0) return fail(MANDEL_EINVAL, "options.ctas_per_sm must be >= 0");
            const int cap = (o && o->ctas_per_sm > 0) ? o->ctas_per_sm : kc.ctas;
            if (cap > 0 && cap < occ) occ = cap;
            ls.grid = dim3((unsigned)(occ * dc.sms));
        }
    } else {
        ls.grid = dim3((W + 31) / 32, (pl.nslots + mandel::kWarpsPerCta - 1) / mandel::kWarpsPerCta);
        if (pl.nslots == 0) ls.grid.y = 1;
    }
    return MANDEL_OK;
}

// true when ptr is memory of device dev (a pointer another process mapped with CUDA IPC
// reports the device that owns the memory)
bool same_device(const void* ptr, int dev) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice && a.device == dev;
}

int store_mode(const mandel::Params& p) { return p.stage ? (p.vec_ok ? 2 : 1) : 0; }

// mandel_stats.first_block: the threshold in lanes, 0 when the launch runs no first block
int first_block_lanes(const LaunchSpec& ls) {
    const bool on = ls.kc.variant == MANDEL_KERNEL_EAGER && ls.kc.bt > 1 && ls.p.first_block != 0xffffffffu;
    return on ? (int)(ls.p.first_block / (uint32_t)std::max(ls.kc.ilp, 1)) : 0;
}

// SM clock over a set of kernel states (mandel_stats.sm_clock_mhz): sum of cycles / sum of ns
double clock_mhz(const mandel::WorkState* ws, int n) {
    double cyc = 0, ns = 0;
    for (int i = 0; i < n; ++i) {
        cyc += (double)ws[i].clk_cycles;
        ns += (double)ws[i].clk_ns;
    }
    return ns > 0 ? cyc / ns * 1e3 : 0.0;
}

size_t state_bytes_for(int scheme, uint32_t H, const mandel_options* o) {
    const uint32_t chunk = effective_chunk(scheme, o);
    const uint64_t nchunks = ((uint64_t)H + chunk - 1) / chunk;
    // rounded to 256 B: the pipelined hand-off packs one state per band back to back,
    // and each WorkState holds 64-bit counters updated with 64-bit atomics
    const size_t raw = sizeof(mandel::WorkState) + (nchunks + 2) * sizeof(uint32_t);
    return (raw + 255) & ~(size_t)255;
}

int launch(const LaunchSpec& ls, cudaStream_t s) {
    if (ls.smem > 48 * 1024)
        CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(ls.fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)ls.smem));
    ls.fn<<<ls.grid, ls.block, ls.smem, s>>>(ls.p);
    CK(cudaGetLastError());
    return MANDEL_OK;
}

double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

// ---------------------------------------------------------------------------
// MANDEL_KERNEL_REFILL chooses, once per view, between the EAGER and LAZY kernels:
// both render every 16th row (a strided sample of the same image, written to the
// destination -- the real render rewrites those rows with identical values), the
// faster one is cached for the view.  Eager wins on smooth views (C2, C5), lazy
// where neighbouring counts differ (deep zooms, C4).
// ---------------------------------------------------------------------------
struct ViewKey {
    double b[5];
    uint32_t W, H, it;
    int dtype;
    bool operator<(const ViewKey& o) const {
        if (dtype != o.dtype) return dtype < o.dtype;
        if (W != o.W) return W < o.W;
        if (H != o.H) return H < o.H;
        if (it != o.it) return it < o.it;
        for (int i = 0; i < 5; ++i)
            if (b[i] != o.b[i]) return b[i] < o.b[i];
        return false;
    }
};
std::map<ViewKey, KernelChoice> g_auto;
std::map<ViewKey, float> g_view_ms;  // last compute time of a view (one GPU), for the band split

// Pipelined hand-off shape for a view whose last compute took `ms` (< 0: unknown) and
// whose map takes ~copy_ms over PCIe: copy-bound views want equal bands (copies start
// early), compute-bound ones thin late bands (short exposed tail); long renders afford
// more bands.  Measured (profiles/r01k_e2e_bands.jsonl): C2 8 bands taper 0.4-0.55,
// C3 (copy-bound) equal bands, C4 (balanced) 12 / 0.7, C5 12-16 / 0.5.
void band_shape(float ms, double copy_ms, int& bands, double& taper) {
    bands = kDefaultBands;
    taper = kDefaultBandTaper;
    if (ms < 0) return;
    const double r = ms / copy_ms;
    taper = r >= 1.15 ? 0.5 : (r <= 0.9 ? 1.0 : 0.7);
    bands = ms > 10.0 ? 12 : (ms < 0.5 ? 1 : 8);  // sub-0.5 ms renders: launches cost more than overlap saves
}
float g_probe[2] = {0, 0};  // last probe: eager sample time (ms), eager iterations per exit
// LAZY below 23 eager iterations per loop exit: calibrated over 44 views with the
// batched EAGER default (tools/probe_calibrate.py, profiles/r01t_probe_calibration.jsonl);
// the previous threshold (10, set against the per-update EAGER loop) lost up to 1.7x.
constexpr float kLazyBelowItersPerExit = 23.0f;
constexpr uint32_t kProbeStride = 16;
constexpr uint64_t kTunePixels = 1ull << 21;  // views up to 2 M pixels are tuned by timing

// The probe renders its sample rows into a compact band in library-owned scratch memory
// on the probing device (band mode: band row = sample index), never into the caller's
// map -- under mandel_render_rank that map is rank 0's shared image on another GPU.
// The probe's device buffers: a compact output band of sbytes and its own work state.
int ensure_probe_buffers(DeviceCtx& dc, size_t sbytes, size_t state_cap) {
    if (dc.scratch_bytes < sbytes) {
        if (dc.scratch) {
            CK(cudaDeviceSynchronize());
            CK(cudaFree(dc.scratch));
        }
        dc.scratch = nullptr;
        dc.scratch_bytes = 0;
        CK(cudaMalloc(&dc.scratch, sbytes));
        dc.scratch_bytes = sbytes;
    }
    if (dc.pstate_bytes < state_cap) {  // the probe's own work state (the ranks' halves are theirs)
        if (dc.pstate) {
            CK(cudaDeviceSynchronize());
            CK(cudaFree(dc.pstate));
        }
        dc.pstate = nullptr;
        dc.pstate_bytes = 0;
        CK(cudaMalloc(&dc.pstate, state_cap));
        dc.pstate_bytes = state_cap;
    }
    return MANDEL_OK;
}

// Small views (<= kTunePixels): render the whole view once with each candidate kernel into
// the probe's scratch (whole GPU, row order, one rank), twice each, and keep the fastest.
// A small render is latency- and tail-bound, so the iterations-per-exit statistic that
// picks EAGER or LAZY on large views does not predict it, and a 1/16 sample does not either
// (DESIGN.md); the whole view costs only a few of its own renders, once per view.  The
// candidates: the batched EAGER default, EAGER with the other slot count, LAZY ILP 2
// (refill at 16 free lanes), LAZY ILP 1 refilling only whole warps (32) -- measured over six
// small views, each is the best on some (profiles/r02af_small_views.jsonl).  Any choice
// computes the same counts.
int tune_small(const Derived& d, uint32_t W, uint32_t H, uint32_t iter_max, int dtype,
               const mandel_options* o, size_t state_cap, int device, cudaStream_t s, KernelChoice& out) {
    const int fi = dtype == MANDEL_FP32 ? 1 : (dtype == MANDEL_FP64_FMA ? 2 : 0);
    DeviceCtx& dc = g_dev[device];
    CK(cudaSetDevice(device));
    int rc = ensure_probe_buffers(dc, (size_t)W * H * sizeof(uint32_t), state_cap);
    if (rc) return rc;
    const Plan pl{H, 0, 1, H, 0};
    KernelChoice cand[4] = {kDefaultChoice[fi], kDefaultChoice[fi], {MANDEL_KERNEL_LAZY, 2, 1, 1},
                            {MANDEL_KERNEL_LAZY, 1, 1, 1}};
    cand[1].ilp = kDefaultChoice[fi].ilp == 1 ? 2 : 1;
    cand[1].minb = 1;
    cand[1].ctas = 0;
    cand[2].lanes = (int)kDefaultRefillLanes;
    cand[3].lanes = 32;
    mandel_options po{};
    if (o) po = *o;
    po.max_sms = 0;   // the view, not the launch geometry (as the probe)
    po.band_out = 1;  // view row k -> scratch row k
    cudaEvent_t ev[8];
    for (int i = 0; i < 8; ++i) CK(cudaEventCreate(&ev[i]));
    float best[4] = {1e30f, 1e30f, 1e30f, 1e30f};
    for (int round = 0; round < 3 && rc == MANDEL_OK; ++round) {
        for (int c = 0; c < 4 && rc == MANDEL_OK; ++c) {
            LaunchSpec ls;
            rc = build_params(d, W, H, iter_max, dtype, MANDEL_BLOCK, 1, 0, &po, dc.scratch, dc.pstate, state_cap,
                              nullptr, false, device, ls, &pl, &cand[c]);
            if (rc) break;
            if (cudaMemsetAsync(dc.pstate, 0, state_cap, s) != cudaSuccess) { rc = cuda_fail(cudaGetLastError(), "tune memset"); break; }
            cudaEventRecord(ev[2 * c], s);
            rc = launch(ls, s);
            cudaEventRecord(ev[2 * c + 1], s);
        }
        if (rc) break;
        if (cudaStreamSynchronize(s) != cudaSuccess) { rc = cuda_fail(cudaGetLastError(), "tune sync"); break; }
        for (int c = 0; c < 4 && round > 0; ++c) {  // round 0 warms every candidate
            float ms = 0;
            cudaEventElapsedTime(&ms, ev[2 * c], ev[2 * c + 1]);
            best[c] = std::min(best[c], ms);
        }
    }
    for (int i = 0; i < 8; ++i) cudaEventDestroy(ev[i]);
    if (rc) return rc;
    int k = 0;
    for (int c = 1; c < 4; ++c)
        if (best[c] < best[k]) k = c;
    out = cand[k];
    g_probe[0] = best[k];
    g_probe[1] = 0.f;  // no iterations-per-exit statistic: timed
    return MANDEL_OK;
}

int auto_choice(const Derived& d, const double* bounds, uint32_t W, uint32_t H, uint32_t iter_max,
                int dtype, const mandel_options* o, size_t state_cap, int device, cudaStream_t s,
                KernelChoice& out) {
    const int fi = dtype == MANDEL_FP32 ? 1 : (dtype == MANDEL_FP64_FMA ? 2 : 0);
    out = kDefaultChoice[fi];
    if (o && (o->kernel != MANDEL_KERNEL_REFILL || o->ilp || o->min_ctas > 1)) return MANDEL_OK;
    ViewKey key{{bounds[0], bounds[1], bounds[2], bounds[3], bounds[4]}, W, H, iter_max, dtype};
    auto it = g_auto.find(key);
    if (it != g_auto.end()) {
        out = it->second;
        return MANDEL_OK;
    }
    // small views: time the candidates on the view itself, once (tune_small)
    if ((uint64_t)W * H <= kTunePixels) {
        int rc = tune_small(d, W, H, iter_max, dtype, o, state_cap, device, s, out);
        if (rc) return rc;
        g_auto[key] = out;
        return MANDEL_OK;
    }
    if (H < 32 * kProbeStride) return MANDEL_OK;
    const uint32_t n = (H + kProbeStride - 1) / kProbeStride;
    const Plan pl{n, 0, kProbeStride, n, 0};
    DeviceCtx& dc = g_dev[device];
    const size_t sbytes = (size_t)n * W * sizeof(uint32_t);
    CK(cudaSetDevice(device));
    int rc0 = ensure_probe_buffers(dc, sbytes, state_cap);
    if (rc0) return rc0;
    void* const pst = dc.pstate;
    const KernelChoice cand[2] = {{kVariantProbe, kDefaultChoice[fi].ilp, kDefaultChoice[fi].minb, 1},
                                  {MANDEL_KERNEL_LAZY, 2, 1, 1}};
    mandel_options po{};
    if (o) po = *o;
    // the probe characterises the view, not the launch: it always runs on the whole
    // GPU, the geometry its threshold was calibrated in (on an SM slice, options.max_sms,
    // the sample has no drain phase and reads fewer iterations per exit -- the paper
    // grid on 4 SMs picked LAZY, 16% slower than EAGER there)
    po.max_sms = 0;
    po.band_out = 1;  // sample row k -> scratch row k
    // one eager launch over the sample: its iterations per loop exit measure how
    // incoherent the escapes are (C2 ~29, C5 ~68, C4's zoom ~3 at ILP2)
    cudaEvent_t e0, e1;
    CK(cudaSetDevice(device));
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    LaunchSpec ls;
    int rc = build_params(d, W, H, iter_max, dtype, MANDEL_BLOCK, 1, 0, &po, dc.scratch, pst, state_cap,
                          nullptr, false, device, ls, &pl, &cand[0]);
    if (rc) { cudaEventDestroy(e0); cudaEventDestroy(e1); return rc; }
    CK(cudaMemsetAsync(pst, 0, state_cap, s));
    CK(cudaEventRecord(e0, s));
    rc = launch(ls, s);
    if (rc) { cudaEventDestroy(e0); cudaEventDestroy(e1); return rc; }
    CK(cudaEventRecord(e1, s));
    mandel::WorkState ws;
    CK(cudaMemcpyAsync(&ws, pst, sizeof(ws), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const float ipe = ws.exits ? (float)((double)ws.warp_iters / (double)ws.exits) : 1e9f;
    g_probe[0] = ms;
    g_probe[1] = ipe;
    out = ipe < kLazyBelowItersPerExit ? cand[1] : kDefaultChoice[fi];
    g_auto[key] = out;
    return MANDEL_OK;
}

// One GPU with a host destination: split the rows into `bands` bands, launch them
// alternately on two streams (a band's kernel fills the previous band's tail), and
// copy each finished band to the host on a copy stream while later bands compute --
// the paper's master file write overlapped with generation.
int render_banded(const Derived& d, uint32_t W, uint32_t H, uint32_t iter_max, int dtype, int scheme,
                  const mandel_options* opts, uint32_t* image, uint32_t* out_host, void* stream0v,
                  mandel_stats* stats, int bands, size_t sbytes, double t_call,
                  const KernelChoice* choice, double taper_auto, float* compute_ms_out,
                  int async_set = -1) {
    int rc = ensure_rank(0, 0, sbytes, nullptr);
    if (rc) return rc;
    CK(cudaSetDevice(0));
    const size_t need = sbytes * (size_t)bands;
    if (async_set >= 0) {
        // asynchronous: this call's map and band states are set `async_set` of two
        const size_t bytes = (size_t)W * H * sizeof(uint32_t);
        if (g_root.pp_image_bytes < bytes || g_root.pp_state_bytes < need) {
            CK(cudaDeviceSynchronize());  // earlier asynchronous calls may still use them
            for (int k = 0; k < 2; ++k) {
                if (g_root.pp_image[k]) CK(cudaFree(g_root.pp_image[k]));
                if (g_root.pp_state[k]) CK(cudaFree(g_root.pp_state[k]));
                g_root.pp_image[k] = nullptr;
                g_root.pp_state[k] = nullptr;
            }
            g_root.pp_image_bytes = g_root.pp_state_bytes = 0;
            for (int k = 0; k < 2; ++k) {
                CK(cudaMalloc(&g_root.pp_image[k], bytes));
                CK(cudaMalloc(&g_root.pp_state[k], need));
            }
            g_root.pp_image_bytes = bytes;
            g_root.pp_state_bytes = need;
        }
        image = g_root.pp_image[async_set];
        if (!g_root.async_stream) CK(cudaStreamCreateWithFlags(&g_root.async_stream, cudaStreamNonBlocking));
        if (!g_root.entry) CK(cudaEventCreateWithFlags(&g_root.entry, cudaEventDisableTiming));
        for (int k = 0; k < 2; ++k)
            if (!g_root.pp_done[k]) CK(cudaEventCreateWithFlags(&g_root.pp_done[k], cudaEventDisableTiming));
    } else if (g_root.band_state_bytes < need) {
        if (g_root.band_state) CK(cudaFree(g_root.band_state));
        g_root.band_state = nullptr;
        g_root.band_state_bytes = 0;
        CK(cudaMalloc(&g_root.band_state, need));
        g_root.band_state_bytes = need;
    }
    if (!g_root.band_stream) CK(cudaStreamCreateWithFlags(&g_root.band_stream, cudaStreamDefault));
    if (!g_root.copy_stream) CK(cudaStreamCreateWithFlags(&g_root.copy_stream, cudaStreamDefault));
    if (!g_root.copy_done) CK(cudaEventCreateWithFlags(&g_root.copy_done, cudaEventDisableTiming));
    for (int b = 0; b < bands; ++b) {
        if (!g_root.band_k0[b]) CK(cudaEventCreate(&g_root.band_k0[b]));
        if (!g_root.band_k1[b]) CK(cudaEventCreate(&g_root.band_k1[b]));
        if (!g_root.band_cp[b]) CK(cudaEventCreate(&g_root.band_cp[b]));
    }
    // bands in issue order, outside-in (top, bottom, next top, ...): the edges of a view
    // are usually its cheap rows, so their copies drain while the costly middle still
    // computes.  Band pair p gets a share taper^p of the rows, so the bands issued last
    // (the middle, finishing last) are thin and their exposed copies short.
    const double taper = (opts && opts->band_taper > 0) ? opts->band_taper / 100.0 : taper_auto;
    std::vector<double> w(bands);
    double wsum = 0;
    for (int i = 0; i < bands; ++i) wsum += (w[i] = std::pow(taper, i / 2));
    std::vector<LaunchSpec> specs(bands);
    std::vector<uint32_t> r0(bands), nr(bands);
    uint32_t top = 0, bot = H;
    for (int b = 0; b < bands; ++b) {
        uint32_t n = (uint32_t)std::llround((double)H * w[b] / wsum);
        if (b == bands - 1 || n > bot - top) n = bot - top;
        if (n == 0) n = bot - top > 0 ? 1 : 0;
        if (b & 1) {
            bot -= n;
            r0[b] = bot;
        } else {
            r0[b] = top;
            top += n;
        }
        nr[b] = n;
        Plan pl{nr[b], r0[b], 1, nr[b], 0};
        char* st = reinterpret_cast<char*>(async_set >= 0 ? g_root.pp_state[async_set] : g_root.band_state) +
                   sbytes * b;
        rc = build_params(d, W, H, iter_max, dtype, scheme, 1, 0, opts, image, st, sbytes,
                          g_root.fcfs_ctr, false, 0, specs[b], &pl, choice);
        if (rc) return rc;
    }
    cudaStream_t s0 = stream0v ? (cudaStream_t)stream0v : g_rank[0].stream;
    cudaStream_t cp = g_root.copy_stream;
    if (async_set >= 0) {
        // after the caller's earlier work on stream0, and after the copies of the call
        // that last used this set's map (two calls ago); stream0 is not made to wait
        cudaStream_t a0 = g_root.async_stream, a1 = g_root.band_stream;
        CK(cudaEventRecord(g_root.entry, s0));
        for (cudaStream_t x : {a0, a1, cp}) {
            CK(cudaStreamWaitEvent(x, g_root.entry, 0));
            CK(cudaStreamWaitEvent(x, g_root.pp_done[async_set], 0));
        }
        CK(cudaMemsetAsync(g_root.pp_state[async_set], 0, need, a0));
        CK(cudaEventRecord(g_root.start, a0));
        CK(cudaStreamWaitEvent(a1, g_root.start, 0));
        cudaStream_t cs[2] = {a0, a1};
        for (int b = 0; b < bands; ++b) {
            cudaStream_t x = cs[b & 1];
            rc = launch(specs[b], x);
            if (rc) return rc;
            CK(cudaEventRecord(g_root.band_k1[b], x));
            if (nr[b] == 0) continue;
            CK(cudaStreamWaitEvent(cp, g_root.band_k1[b], 0));
            const size_t off = (size_t)r0[b] * W;
            CK(cudaMemcpyAsync(out_host + off, image + off, (size_t)nr[b] * W * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, cp));
        }
        CK(cudaEventRecord(g_root.pp_done[async_set], cp));  // copies are in order on cp
        return MANDEL_OK;
    }
    cudaStream_t cs[2] = {s0, g_root.band_stream};
    CK(cudaMemsetAsync(g_root.band_state, 0, need, s0));
    CK(cudaEventRecord(g_root.start, s0));
    CK(cudaStreamWaitEvent(cs[1], g_root.start, 0));
    CK(cudaStreamWaitEvent(cp, g_root.start, 0));
    for (int i = 0; i < bands; ++i) {
        const int b = i;
        cudaStream_t s = cs[i & 1];
        CK(cudaEventRecord(g_root.band_k0[b], s));
        rc = launch(specs[b], s);
        if (rc) return rc;
        CK(cudaEventRecord(g_root.band_k1[b], s));
        if (nr[b] == 0) continue;
        CK(cudaStreamWaitEvent(cp, g_root.band_k1[b], 0));
        const size_t off = (size_t)r0[b] * W;
        CK(cudaMemcpyAsync(out_host + off, image + off, (size_t)nr[b] * W * sizeof(uint32_t),
                           cudaMemcpyDeviceToHost, cp));
        CK(cudaEventRecord(g_root.band_cp[b], cp));
    }
    CK(cudaEventRecord(g_root.copy_done, cp));  // the copy stream is in order: all copies done
    // s0 (the caller's stream) is done when every band kernel and every copy is
    for (int b = 0; b < bands; ++b) CK(cudaStreamWaitEvent(s0, g_root.band_k1[b], 0));
    CK(cudaStreamWaitEvent(s0, g_root.copy_done, 0));
    CK(cudaEventRecord(g_root.d2h, s0));
    std::vector<mandel::WorkState> ws(bands);
    for (int b = 0; b < bands; ++b)
        CK(cudaMemcpyAsync(&ws[b], reinterpret_cast<char*>(g_root.band_state) + sbytes * b,
                           sizeof(mandel::WorkState), cudaMemcpyDeviceToHost, s0));
    CK(cudaStreamSynchronize(s0));
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        float ms = 0, kend = 0;
        for (int b = 0; b < bands; ++b) {
            CK(cudaEventElapsedTime(&ms, g_root.start, g_root.band_k1[b]));
            if (ms > kend) kend = ms;
            stats->sum_iters += ws[b].sum_iters;
            stats->pixels += ws[b].pixels;
            stats->rank_rows[0] += ws[b].rows_started;
            stats->warp_iters += ws[b].warp_iters;
            stats->loop_exits += ws[b].exits;
        }
        stats->device_ms = kend;
        *compute_ms_out = kend;
        stats->kernel_ms[0] = kend;
        stats->kernel_ms_max = kend;
        CK(cudaEventElapsedTime(&ms, g_root.start, g_root.d2h));
        stats->d2h_ms = ms - kend;  // the part of the hand-off not hidden behind compute
        stats->rank_iters[0] = stats->sum_iters;
        stats->rank_pixels[0] = stats->pixels;
        stats->chunks_claimed = 0;  // the bands are row ranges: no claims
        stats->kernel_scheme = MANDEL_BLOCK;
        stats->sm_clock_mhz = clock_mhz(ws.data(), bands);
        stats->transfers = 0;
        stats->kernel_launches = (uint32_t)bands;
        stats->ngpus = 1;
        stats->ndevices = 1;
        stats->kernel_variant = specs[0].kc.variant;
        stats->kernel_ilp = specs[0].kc.ilp;
        stats->kernel_batch = specs[0].kc.bt;
        stats->kernel_packed = specs[0].kc.packed;
        stats->store_mode = store_mode(specs[0].p);
        stats->fused_y = (int32_t)specs[0].p.fused_y;
        stats->first_block = first_block_lanes(specs[0]);
        stats->probe[0] = g_probe[0];
        stats->probe[1] = g_probe[1];
        stats->total_ms = now_ms() - t_call;
    }
    return MANDEL_OK;
}

// The per-device host hand-off (options.host_handoff): enqueue, on every rank's stream
// after its kernel, the copies of its band's rows into their image rows of out_host, and
// record the rank's d2h event after them.  Static schemes: the plan is known before the
// kernel runs -- slots [0, count0) are rows base0 + s * stride0 (one strided 2-D copy),
// slots [count0, nslots) rows base1 + ... (one contiguous copy).  FCFS: local chunk k
// holds global chunk chunk_map[k] - 1 (bound in local order; 0 / kChunkDone end the
// list), read back once the rank's kernel is done; runs of consecutive global chunks are
// copied as one block of rows.  copies counts the copies enqueued.
int copy_bands_to_host(const std::vector<LaunchSpec>& specs, int ngpus, cudaStream_t s0, uint32_t W,
                       uint32_t H, uint32_t* out_host, uint32_t& copies) {
    const size_t row_bytes = (size_t)W * sizeof(uint32_t);
    std::vector<std::vector<uint32_t>> cmap(ngpus);
    // FCFS chunk maps first, so that each rank's read waits only for its own kernel
    for (int r = 0; r < ngpus; ++r) {
        const mandel::Params& p = specs[r].p;
        if (p.scheme != MANDEL_FCFS) continue;
        RankCtx& rk = g_rank[r];
        CK(cudaSetDevice(rk.device));
        cmap[r].resize((size_t)p.nchunks + 1);
        CK(cudaMemcpyAsync(cmap[r].data(), p.chunk_map, cmap[r].size() * sizeof(uint32_t),
                           cudaMemcpyDeviceToHost, r == 0 ? s0 : rk.stream));
    }
    for (int r = 0; r < ngpus; ++r) {
        const mandel::Params& p = specs[r].p;
        RankCtx& rk = g_rank[r];
        cudaStream_t s = r == 0 ? s0 : rk.stream;
        CK(cudaSetDevice(rk.device));
        if (p.scheme == MANDEL_FCFS) {
            CK(cudaStreamSynchronize(s));
            const uint32_t c = p.chunk_rows;
            uint32_t k = 0;
            while (k <= p.nchunks) {
                const uint32_t g = cmap[r][k];
                if (g == 0 || g == mandel::kChunkDone) break;
                uint32_t n = 1;  // a run of local chunks bound to consecutive global chunks
                while (k + n <= p.nchunks && cmap[r][k + n] == g + n) ++n;
                const uint64_t row0 = (uint64_t)(g - 1) * c;
                const uint64_t rows = std::min<uint64_t>((uint64_t)n * c, H - row0);
                CK(cudaMemcpyAsync(out_host + row0 * W, p.out + (size_t)k * c * W, rows * row_bytes,
                                   cudaMemcpyDeviceToHost, s));
                ++copies;
                k += n;
            }
        } else {
            if (p.count0 > 0) {
                CK(cudaMemcpy2DAsync(out_host + (size_t)p.base0 * W, (size_t)p.stride0 * row_bytes, p.out,
                                     row_bytes, row_bytes, p.count0, cudaMemcpyDeviceToHost, s));
                ++copies;
            }
            if (p.nslots > p.count0) {
                CK(cudaMemcpyAsync(out_host + (size_t)p.base1 * W, p.out + (size_t)p.count0 * W,
                                   (size_t)(p.nslots - p.count0) * row_bytes, cudaMemcpyDeviceToHost, s));
                ++copies;
            }
        }
        CK(cudaEventRecord(rk.d2h, s));
    }
    return MANDEL_OK;
}

int render_impl(double xmin, double xmax, double ymin, double ymax, uint32_t W, uint32_t H,
                uint32_t iter_max, double R, int dtype, int scheme, int ngpus,
                const mandel_options* opts, uint32_t* out_host, uint32_t* out_dev0,
                void* stream0v, mandel_stats* stats) {
    const double t_call = now_ms();
    Derived d;
    int rc = derive(xmin, xmax, ymin, ymax, W, H, iter_max, R, dtype, d);
    if (rc) return rc;
    if (scheme < MANDEL_BLOCK || scheme > MANDEL_FCFS_MASTER) return fail(MANDEL_EINVAL, "scheme out of range");
    if (!out_host && !out_dev0) return fail(MANDEL_EINVAL, "need out_host or out_dev0");
    if (scheme == MANDEL_FCFS_MASTER && ngpus < 2) return fail(MANDEL_EINVAL, "FCFS_MASTER needs ngpus >= 2");
    if (ngpus < 1 || ngpus > MANDEL_MAX_GPUS) return fail(MANDEL_ENODEV, "ngpus out of range");
    if (!is_dynamic(scheme) && H < (uint32_t)ngpus) return fail(MANDEL_EINVAL, "static schemes need H >= ngpus");
    if (opts && opts->kernel == MANDEL_KERNEL_STATIC && is_dynamic(scheme))
        return fail(MANDEL_EINVAL, "the static kernel has no work queue: FCFS needs the refill kernel");
    if (opts && opts->band_out) return fail(MANDEL_EINVAL, "band_out is a mandel_render_rank option");
    int ndev = 0;
    rc = device_count(ndev);
    if (rc) return rc;
    const bool logical = opts && opts->logical_ranks;
    if (ngpus > ndev && !logical) return fail(MANDEL_ENODEV, "ngpus exceeds the visible device count");
    const int nphys = ngpus < ndev ? ngpus : ndev;
    for (int g = 0; g < nphys; ++g) {
        rc = ensure_device(g);
        if (rc) return rc;
        rc = ensure_peer(g);
        if (rc) return rc;
    }
    const size_t bytes = (size_t)W * H * sizeof(uint32_t);
    CK(cudaSetDevice(0));
    if (!g_root.start) {
        CK(cudaEventCreate(&g_root.start));
        CK(cudaEventCreate(&g_root.done));
        CK(cudaEventCreate(&g_root.d2h));
    }
    if (!g_root.fcfs_ctr) {
        CK(cudaMalloc(&g_root.fcfs_ctr, 256));
        CK(cudaMemset(g_root.fcfs_ctr, 0, 256));
        g_root.ctr_zeroed[0] = g_root.ctr_zeroed[1] = true;
    }
    uint32_t* image = out_dev0;
    if (!image) {
        if (g_root.image_bytes < bytes) {
            if (g_root.image) CK(cudaFree(g_root.image));
            g_root.image = nullptr;
            g_root.image_bytes = 0;
            CK(cudaMalloc(&g_root.image, bytes));
            g_root.image_bytes = bytes;
        }
        image = g_root.image;
    }
    const size_t sbytes = state_bytes_for(scheme, H, opts);
    // kernel choice for this view (MANDEL_KERNEL_REFILL: probed once on device 0)
    KernelChoice kc;
    {
        const double bounds[5] = {xmin, xmax, ymin, ymax, R};
        rc = ensure_rank(0, 0, sbytes, nullptr);
        if (rc) return rc;
        cudaStream_t sp = stream0v ? (cudaStream_t)stream0v : g_rank[0].stream;
        rc = auto_choice(d, bounds, W, H, iter_max, dtype, opts, sbytes, 0, sp, kc);
        if (rc) return rc;
    }
    const bool auto_k = !opts || opts->kernel == MANDEL_KERNEL_REFILL;
    const KernelChoice* kcp = auto_k ? &kc : nullptr;
    const ViewKey vkey{{xmin, xmax, ymin, ymax, R}, W, H, iter_max, dtype};
    int bands_auto = kDefaultBands;
    double taper_auto = kDefaultBandTaper;
    {
        auto vm = g_view_ms.find(vkey);
        band_shape(vm == g_view_ms.end() ? -1.f : vm->second, (double)bytes / 5.0e7, bands_auto, taper_auto);
    }
    const int bands = opts && opts->bands ? opts->bands : bands_auto;
    if (opts && opts->async_host) {
        // asynchronous pipelined host output (one GPU, library-owned maps, no statistics)
        if (!out_host || out_dev0 || stats || ngpus != 1 || scheme == MANDEL_FCFS_MASTER)
            return fail(MANDEL_EINVAL, "async_host needs out_host, no out_dev0, no stats, one GPU");
        // frames overlap each other, so the bands only need to start the copies early:
        // four equal bands (tools/async_bands.py: C2 5.84, C3 4.68, C4 22.0 ms per frame
        // against 5.83 / 4.77 / 22.6 with the synchronous shape), one for tiny renders
        int want = opts->bands ? opts->bands : (bands_auto == 1 ? 1 : 4);
        const double taper = opts->band_taper ? taper_auto : 1.0;
        const int nb = std::max(1, std::min(want, std::min((int)kMaxBands, (int)(H / 2 > 0 ? H / 2 : 1))));
        const int set = g_root.pp_next;
        g_root.pp_next ^= 1;
        return render_banded(d, W, H, iter_max, dtype, scheme, opts, image, out_host, stream0v, nullptr, nb,
                             sbytes, t_call, kcp, taper, nullptr, set);
    }
    if (out_host && ngpus == 1 && bands > 1 && H >= 2 * (uint32_t)bands && scheme != MANDEL_FCFS_MASTER) {
        mandel_stats local;
        float cms = -1.f;
        rc = render_banded(d, W, H, iter_max, dtype, scheme, opts, image, out_host, stream0v,
                           stats ? stats : &local, bands > kMaxBands ? kMaxBands : bands, sbytes, t_call,
                           kcp, taper_auto, &cms);
        if (rc == MANDEL_OK && cms > 0) g_view_ms[vkey] = cms;
        return rc;
    }
    // Host hand-off of a multi-rank render (options.host_handoff).  Through GPU 0: every
    // rank stores into GPU 0's map (the fused gather) and GPU 0 copies W*H*4 bytes to the
    // host over its one link.  Per device (the default when the ranks span several GPUs):
    // every rank stores its rows into a band in its own HBM (band mode, local stores) and
    // its own device copies them into out_host -- the copies of N GPUs run over N links
    // and each starts when its rank's kernel ends (PAPER.md:151 sends each task's rows to
    // the master; here the host is the master).
    const int hh = opts ? opts->host_handoff : 0;
    if (hh < -1 || hh > 1) return fail(MANDEL_EINVAL, "options.host_handoff must be -1, 0 or 1");
    const bool per_dev = out_host && !out_dev0 && (hh == 1 || (hh == 0 && nphys > 1));
    mandel_options bopt;
    if (opts) bopt = *opts;
    else std::memset(&bopt, 0, sizeof(bopt));
    bopt.band_out = 1;
    const mandel_options* ropts = per_dev ? &bopt : opts;
    std::vector<LaunchSpec> specs(ngpus);
    const int cp = g_root.ctr_par;  // the counter word this render claims from
    for (int r = 0; r < ngpus; ++r) {
        const int dev = r % ndev;
        rc = ensure_rank(r, dev, sbytes, nullptr);
        if (rc) return rc;
        RankCtx& rk = g_rank[r];
        rc = build_params(d, W, H, iter_max, dtype, scheme, ngpus, r, ropts, per_dev ? nullptr : image,
                          rk.half(rk.par), rk.state_bytes, g_root.fcfs_ctr + 32 * cp, nphys > 1, dev, specs[r],
                          nullptr, kcp, !per_dev && dev != 0);
        if (rc) return rc;
        if (per_dev) {
            // the band holds the rank's row slots: static schemes the plan's rows, FCFS up to
            // every chunk (band row k * chunk_rows + r = local chunk k, row r)
            const mandel::Params& p = specs[r].p;
            const uint64_t rows = p.scheme == MANDEL_FCFS ? (uint64_t)p.nchunks * p.chunk_rows : p.nslots;
            const size_t need = std::max<size_t>((size_t)(rows * W * sizeof(uint32_t)), 256);
            if (rk.band_bytes < need) {
                CK(cudaEventSynchronize(rk.used));  // an earlier render may still copy from it
                if (rk.band) CK(cudaFree(rk.band));
                rk.band = nullptr;
                rk.band_bytes = 0;
                CK(cudaMalloc(&rk.band, need));
                rk.band_bytes = need;
            }
            if (!rk.d2h) CK(cudaEventCreateWithFlags(&rk.d2h, cudaEventDisableTiming));
            specs[r].p.out = rk.band;
        }
        // the kernel zeroes the rank's other half (and rank 0 the other counter word) for the
        // next render
        specs[r].p.zero_next = static_cast<uint32_t*>(rk.half(rk.par ^ 1));
        specs[r].p.zero_words = (uint32_t)(sbytes / sizeof(uint32_t));
        specs[r].p.zero_ctr = r == 0 ? g_root.fcfs_ctr + 32 * (cp ^ 1) : nullptr;
    }
    cudaStream_t s0 = stream0v ? (cudaStream_t)stream0v : g_rank[0].stream;
    // events: only when the call times or waits (statistics, host output) or orders ranks
    const bool timed = stats || out_host || ngpus > 1;
    // rank 0 orders everything: start event, then every rank waits on it
    CK(cudaSetDevice(0));
    // the counter words and the rank states are library-owned and reused: an earlier
    // enqueued render (possibly on another stream) must be done with them first
    for (int r = 0; r < ngpus; ++r) CK(cudaStreamWaitEvent(s0, g_rank[r].used, 0));
    if (!g_root.ctr_zeroed[cp]) CK(cudaMemsetAsync(g_root.fcfs_ctr + 32 * cp, 0, sizeof(uint32_t), s0));
    if (g_rank[0].zeroed[g_rank[0].par] < sbytes) CK(cudaMemsetAsync(g_rank[0].half(g_rank[0].par), 0, sbytes, s0));
    if (timed) CK(cudaEventRecord(g_root.start, s0));
    for (int r = 1; r < ngpus; ++r) {
        RankCtx& rk = g_rank[r];
        CK(cudaSetDevice(rk.device));
        CK(cudaStreamWaitEvent(rk.stream, g_root.start, 0));
        if (rk.zeroed[rk.par] < sbytes) CK(cudaMemsetAsync(rk.half(rk.par), 0, sbytes, rk.stream));
    }
    int launches = 0;
    for (int r = 0; r < ngpus; ++r) {
        RankCtx& rk = g_rank[r];
        cudaStream_t s = r == 0 ? s0 : rk.stream;
        CK(cudaSetDevice(rk.device));
        if (timed) CK(cudaEventRecord(rk.k0, s));
        rc = launch(specs[r], s);
        if (rc) return rc;
        ++launches;
        if (timed) CK(cudaEventRecord(rk.k1, s));
        rk.zeroed[rk.par] = 0;
        rk.zeroed[rk.par ^ 1] = sbytes;
        rk.par ^= 1;
    }
    g_root.ctr_zeroed[cp] = false;
    g_root.ctr_zeroed[cp ^ 1] = true;
    g_root.ctr_par = cp ^ 1;
    CK(cudaSetDevice(0));
    for (int r = 1; r < ngpus; ++r) CK(cudaStreamWaitEvent(s0, g_rank[r].k1, 0));
    if (timed) CK(cudaEventRecord(g_root.done, s0));
    uint32_t d2h_copies = 0;
    if (per_dev) {
        // each rank's copies follow its own kernel on its own stream (rank 0's follow the
        // done event on s0, so device_ms stays the compute); the map is complete on the
        // host once GPU 0's stream has waited for every rank's last copy
        rc = copy_bands_to_host(specs, ngpus, s0, W, H, out_host, d2h_copies);
        if (rc) return rc;
        CK(cudaSetDevice(0));
        for (int r = 0; r < ngpus; ++r) CK(cudaStreamWaitEvent(s0, g_rank[r].d2h, 0));
    }
    // every rank's state and the counter are free once GPU 0's stream passes here
    for (int r = 0; r < ngpus; ++r) {
        CK(cudaSetDevice(g_rank[r].device));
        CK(cudaEventRecord(g_rank[r].used, r == 0 ? s0 : g_rank[r].stream));
    }
    CK(cudaSetDevice(0));
    // device output without statistics: enqueued only (stream0 orders everything after it)
    if (!stats && !out_host) return MANDEL_OK;
    if (out_host) {
        if (!per_dev) CK(cudaMemcpyAsync(out_host, image, bytes, cudaMemcpyDeviceToHost, s0));
        CK(cudaEventRecord(g_root.d2h, s0));
    }
    // read back per-rank statistics (small, ordered after each rank's kernel)
    std::vector<mandel::WorkState> ws(ngpus);
    for (int r = 0; r < ngpus; ++r) {
        RankCtx& rk = g_rank[r];
        CK(cudaSetDevice(rk.device));
        CK(cudaMemcpyAsync(&ws[r], specs[r].p.ws, sizeof(mandel::WorkState), cudaMemcpyDeviceToHost,
                           r == 0 ? s0 : rk.stream));
    }
    for (int r = 0; r < ngpus; ++r) {
        RankCtx& rk = g_rank[r];
        CK(cudaSetDevice(rk.device));
        CK(cudaStreamSynchronize(r == 0 ? s0 : rk.stream));
    }
    CK(cudaSetDevice(0));
    if (ngpus == 1) {
        float vms = 0;
        CK(cudaEventElapsedTime(&vms, g_root.start, g_root.done));
        g_view_ms[vkey] = vms;
    }
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, g_root.start, g_root.done));
        stats->device_ms = ms;
        if (out_host) {
            CK(cudaEventElapsedTime(&ms, g_root.done, g_root.d2h));
            stats->d2h_ms = ms;
        }
        uint32_t claims = 0, transfers = 0;
        for (int r = 0; r < ngpus; ++r) {
            CK(cudaEventElapsedTime(&ms, g_rank[r].k0, g_rank[r].k1));
            stats->kernel_ms[r] = ms;
            if (ms > stats->kernel_ms_max) stats->kernel_ms_max = ms;
            stats->rank_iters[r] = ws[r].sum_iters;
            stats->rank_pixels[r] = ws[r].pixels;
            stats->rank_rows[r] = ws[r].rows_started;
            stats->sum_iters += ws[r].sum_iters;
            stats->pixels += ws[r].pixels;
            stats->warp_iters += ws[r].warp_iters;
            stats->loop_exits += ws[r].exits;
            claims += ws[r].chunks_claimed;
            if (r != 0) transfers += is_dynamic(scheme) ? ws[r].rows_started : 1u;
        }
        stats->chunks_claimed = claims;
        stats->kernel_scheme = scheme;
        stats->sm_clock_mhz = clock_mhz(ws.data(), ngpus);
        // per-device hand-off: no gather to rank 0; the transfers are the copies to the host
        stats->transfers = per_dev ? d2h_copies : transfers;
        stats->host_handoff = per_dev ? 1 : 0;
        stats->kernel_launches = (uint32_t)launches;
        stats->ngpus = (uint32_t)ngpus;
        stats->ndevices = (uint32_t)nphys;
        stats->kernel_variant = specs[0].kc.variant;
        stats->kernel_ilp = specs[0].kc.ilp;
        stats->kernel_batch = specs[0].kc.bt;
        stats->kernel_packed = specs[0].kc.packed;
        stats->store_mode = store_mode(specs[0].p);
        stats->fused_y = (int32_t)specs[0].p.fused_y;
        stats->first_block = first_block_lanes(specs[0]);
        stats->probe[0] = g_probe[0];
        stats->probe[1] = g_probe[1];
        stats->total_ms = now_ms() - t_call;
    }
    return MANDEL_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int mandel_abi_version(void) { return MANDEL_ABI_VERSION; }

const char* mandel_strerror(int code) {
    switch (code) {
        case MANDEL_OK: return "ok";
        case MANDEL_EINVAL: return "invalid argument";
        case MANDEL_ENODEV: return "no usable CUDA device / peer access";
        case MANDEL_ENOMEM: return "out of memory";
        case MANDEL_ECUDA: return "CUDA runtime error";
        case MANDEL_ECOMM: return "inter-GPU communication error";
        case MANDEL_EBUSY: return "library busy (concurrent call)";
        case MANDEL_EIO: return "file write failed";
        default: return "unknown status";
    }
}

const char* mandel_last_error(void) { return g_detail.c_str(); }

int mandel_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int mandel_plan_rows(int scheme, uint32_t H, int ngpus, int rank, uint32_t* rows_out, uint32_t* count) {
    if (!count) return fail(MANDEL_EINVAL, "count must not be NULL");
    if (is_dynamic(scheme)) return fail(MANDEL_EINVAL, "FCFS is dynamic: no static plan");
    if (scheme != MANDEL_BLOCK && scheme != MANDEL_CYCLIC) return fail(MANDEL_EINVAL, "scheme out of range");
    Plan pl;
    int rc = make_plan(scheme, H, ngpus, rank, pl);
    if (rc) return rc;
    if (rows_out) {
        if (*count < pl.nslots) {
            *count = pl.nslots;
            return fail(MANDEL_EINVAL, "rows_out capacity too small");
        }
        for (uint32_t s = 0; s < pl.nslots; ++s)
            rows_out[s] = s < pl.count0 ? pl.base0 + s * pl.stride0 : pl.base1 + (s - pl.count0);
    }
    *count = pl.nslots;
    return MANDEL_OK;
}

int mandel_render_ex(double xmin, double xmax, double ymin, double ymax, uint32_t W, uint32_t H,
                     uint32_t iterMax, double R, int dtype, int scheme, int ngpus,
                     const mandel_options* opts, uint32_t* out_host, uint32_t* out_dev0,
                     void* stream0, mandel_stats* stats) {
    BusyGuard busy;
    if (!busy.ok) return fail(MANDEL_EBUSY, "another mandel call is in progress");
    std::lock_guard<std::mutex> lk(g_mu);
    int prev = 0;
    cudaGetDevice(&prev);
    cudaGetLastError();
    int rc = render_impl(xmin, xmax, ymin, ymax, W, H, iterMax, R, dtype, scheme, ngpus, opts,
                         out_host, out_dev0, stream0, stats);
    cudaSetDevice(prev);
    cudaGetLastError();
    return rc;
}

int mandel_render(double xmin, double xmax, double ymin, double ymax, uint32_t W, uint32_t H,
                  uint32_t iterMax, double R, int dtype, int scheme, int ngpus, uint32_t* out_u32) {
    if (!out_u32) return fail(MANDEL_EINVAL, "out_u32 must not be NULL");
    return mandel_render_ex(xmin, xmax, ymin, ymax, W, H, iterMax, R, dtype, scheme, ngpus,
                            nullptr, out_u32, nullptr, nullptr, nullptr);
}

int mandel_render_rank(double xmin, double xmax, double ymin, double ymax, uint32_t W, uint32_t H,
                       uint32_t iterMax, double R, int dtype, int scheme, int rank, int nranks,
                       const mandel_options* opts, uint32_t* out_root, uint32_t* fcfs_counter,
                       void* streamv, mandel_stats* stats) {
    BusyGuard busy;
    if (!busy.ok) return fail(MANDEL_EBUSY, "another mandel call is in progress");
    std::lock_guard<std::mutex> lk(g_mu);
    Derived d;
    int rc = derive(xmin, xmax, ymin, ymax, W, H, iterMax, R, dtype, d);
    if (rc) return rc;
    if (scheme < MANDEL_BLOCK || scheme > MANDEL_FCFS_MASTER) return fail(MANDEL_EINVAL, "scheme out of range");
    if (scheme == MANDEL_FCFS_MASTER && nranks < 2) return fail(MANDEL_EINVAL, "FCFS_MASTER needs nranks >= 2");
    if (nranks < 1 || nranks > MANDEL_MAX_GPUS || rank < 0 || rank >= nranks)
        return fail(MANDEL_EINVAL, "rank/nranks out of range");
    if (!out_root) return fail(MANDEL_EINVAL, "out_root must not be NULL");
    if (is_dynamic(scheme) && !fcfs_counter) return fail(MANDEL_EINVAL, "FCFS needs fcfs_counter");
    if (!is_dynamic(scheme) && H < (uint32_t)nranks) return fail(MANDEL_EINVAL, "static schemes need H >= nranks");
    int ndev = 0;
    rc = device_count(ndev);
    if (rc) return rc;
    // the device this rank runs on: the caller's stream's device, else the current device
    int dev = 0;
    if (streamv) CK(cudaStreamGetDevice((cudaStream_t)streamv, &dev));
    else CK(cudaGetDevice(&dev));
    if (dev < 0 || dev >= ndev) return fail(MANDEL_ENODEV, "stream device out of range");
    rc = ensure_device(dev);
    if (rc) return rc;
    const size_t sbytes = state_bytes_for(scheme, H, opts);
    // slot 0 of the rank table holds this process's single rank
    rc = ensure_rank(0, dev, sbytes, nullptr);
    if (rc) return rc;
    RankCtx& rk = g_rank[0];
    cudaStream_t s = streamv ? (cudaStream_t)streamv : rk.stream;
    // MANDEL_KERNEL_REFILL: the per-view EAGER/LAZY choice, probed once per view on this
    // rank's own device (scratch sample band; cached) -- as mandel_render_ex does
    KernelChoice kc;
    const bool auto_k = (!opts || opts->kernel == MANDEL_KERNEL_REFILL) &&
                        !(scheme == MANDEL_FCFS_MASTER && rank == 0);  // the master computes nothing
    if (auto_k) {
        const double bounds[5] = {xmin, xmax, ymin, ymax, R};
        rc = auto_choice(d, bounds, W, H, iterMax, dtype, opts, sbytes, dev, s, kc);
        if (rc) return rc;
    }
    LaunchSpec ls;
    // across processes the counter is (in general) on another GPU: system scope
    // the fused gather: a rank other than 0 stores into rank 0's map on another GPU (its
    // band, with options.band_out, is local)
    const bool remote = rank != 0 && !(opts && opts->band_out) && !same_device(out_root, dev);
    void* const cur = rk.half(rk.par);
    rc = build_params(d, W, H, iterMax, dtype, scheme, nranks, rank, opts, out_root, cur,
                      rk.state_bytes, fcfs_counter, nranks > 1, dev, ls, nullptr, auto_k ? &kc : nullptr, remote);
    if (rc) return rc;
    ls.p.zero_next = static_cast<uint32_t*>(rk.half(rk.par ^ 1));  // the next render's state half
    ls.p.zero_words = (uint32_t)(sbytes / sizeof(uint32_t));
    const double t0 = now_ms();
    CK(cudaStreamWaitEvent(s, rk.used, 0));  // an earlier enqueued render may still use the state
    if (rk.zeroed[rk.par] < sbytes) CK(cudaMemsetAsync(cur, 0, sbytes, s));
    const bool band = opts && opts->band_out;
    if (stats || band) CK(cudaEventRecord(rk.k0, s));
    rc = launch(ls, s);
    if (rc) return rc;
    if (stats || band) CK(cudaEventRecord(rk.k1, s));
    CK(cudaEventRecord(rk.used, s));
    rk.zeroed[rk.par] = 0;
    rk.zeroed[rk.par ^ 1] = sbytes;
    rk.par ^= 1;
    if (!stats && !band) return MANDEL_OK;  // asynchronous: enqueued on the stream, not awaited
    mandel::WorkState ws;
    CK(cudaMemcpyAsync(&ws, cur, sizeof(ws), cudaMemcpyDeviceToHost, s));
    std::vector<uint32_t> cmap;
    if (band && ls.p.scheme == MANDEL_FCFS) {
        cmap.resize((size_t)ls.p.nchunks + 1);
        CK(cudaMemcpyAsync(cmap.data(), ls.p.chunk_map, cmap.size() * sizeof(uint32_t),
                           cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    if (band) {
        // the band's row list (K4's input): static schemes -> the plan, slot by slot;
        // FCFS -> local chunk k holds global chunk cmap[k]-1 (bound in local order)
        g_band_rows.clear();
        if (ls.p.scheme == MANDEL_FCFS) {
            const uint32_t c = ls.p.chunk_rows;
            for (uint32_t k = 0; k <= ls.p.nchunks; ++k) {
                const uint32_t g = cmap[k];
                if (g == 0 || g == mandel::kChunkDone) break;
                for (uint32_t r = 0; r < c; ++r) {
                    const uint64_t row = (uint64_t)(g - 1) * c + r;
                    g_band_rows.push_back(row < H ? (uint32_t)row : 0xffffffffu);
                }
            }
        } else {
            for (uint32_t sl = 0; sl < ls.p.nslots; ++sl)
                g_band_rows.push_back(sl < ls.p.count0 ? ls.p.base0 + sl * ls.p.stride0
                                                      : ls.p.base1 + (sl - ls.p.count0));
        }
    }
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, rk.k0, rk.k1));
        stats->kernel_ms[0] = ms;
        stats->kernel_ms_max = ms;
        stats->device_ms = ms;
        stats->rank_iters[0] = ws.sum_iters;
        stats->rank_pixels[0] = ws.pixels;
        stats->rank_rows[0] = ws.rows_started;
        stats->sum_iters = ws.sum_iters;
        stats->pixels = ws.pixels;
        stats->warp_iters = ws.warp_iters;
        stats->loop_exits = ws.exits;
        stats->chunks_claimed = ws.chunks_claimed;
        stats->kernel_scheme = scheme;
        stats->sm_clock_mhz = clock_mhz(&ws, 1);
        stats->transfers = rank == 0 ? 0u : (is_dynamic(scheme) ? ws.rows_started : 1u);
        stats->kernel_launches = 1;
        stats->ngpus = 1;
        stats->ndevices = 1;
        stats->kernel_variant = ls.kc.variant;
        stats->kernel_ilp = ls.kc.ilp;
        stats->kernel_batch = ls.kc.bt;
        stats->kernel_packed = ls.kc.packed;
        stats->store_mode = store_mode(ls.p);
        stats->fused_y = (int32_t)ls.p.fused_y;
        stats->first_block = first_block_lanes(ls);
        stats->probe[0] = g_probe[0];
        stats->probe[1] = g_probe[1];
        stats->total_ms = now_ms() - t0;
    }
    return MANDEL_OK;
}

int mandel_band_rows(uint32_t* rows_out, uint32_t* count) {
    if (!count) return fail(MANDEL_EINVAL, "count must not be NULL");
    std::lock_guard<std::mutex> lk(g_mu);
    const uint32_t n = (uint32_t)g_band_rows.size();
    if (rows_out) {
        if (*count < n) {
            *count = n;
            return fail(MANDEL_EINVAL, "rows_out capacity too small");
        }
        std::memcpy(rows_out, g_band_rows.data(), (size_t)n * sizeof(uint32_t));
    }
    *count = n;
    return MANDEL_OK;
}

int mandel_scatter_rows(const uint32_t* band_dev, const uint32_t* rows_dev, uint32_t nrows, uint32_t W,
                        uint32_t* image_dev, void* stream) {
    if (nrows == 0) return MANDEL_OK;
    if (!band_dev || !rows_dev || !image_dev || W == 0)
        return fail(MANDEL_EINVAL, "scatter_rows needs device pointers and W >= 1");
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    if (s) CK(cudaStreamGetDevice(s, &dev));
    else {
        cudaPointerAttributes a;
        CK(cudaPointerGetAttributes(&a, image_dev));
        dev = a.device;
    }
    CK(cudaSetDevice(dev));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const unsigned grid = (unsigned)std::min<uint64_t>(nrows, (uint64_t)sms * 8);
    mandel::scatter_rows_kernel<<<grid, 256, 0, s>>>(band_dev, rows_dev, nrows, W, image_dev);
    CK(cudaGetLastError());
    return MANDEL_OK;
}

int mandel_dev_alloc(int device, size_t bytes, void** dev_ptr) {
    if (!dev_ptr || bytes == 0) return fail(MANDEL_EINVAL, "dev_alloc needs a pointer and bytes > 0");
    int prev = 0;
    cudaGetDevice(&prev);
    CK(cudaSetDevice(device));
    cudaError_t e = cudaMalloc(dev_ptr, bytes);
    cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    return MANDEL_OK;
}

int mandel_dev_free(void* dev_ptr) {
    if (!dev_ptr) return MANDEL_OK;
    CK(cudaFree(dev_ptr));
    return MANDEL_OK;
}

int mandel_ipc_handle(void* dev_ptr, void* handle_out) {
    if (!dev_ptr || !handle_out) return fail(MANDEL_EINVAL, "ipc_handle needs pointers");
    static_assert(sizeof(cudaIpcMemHandle_t) == MANDEL_IPC_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, dev_ptr);
    if (e != cudaSuccess) { cuda_fail(e, "cudaIpcGetMemHandle"); return MANDEL_ECOMM; }
    std::memcpy(handle_out, &h, sizeof(h));
    return MANDEL_OK;
}

int mandel_ipc_open(int device, const void* handle, void** dev_ptr_out) {
    if (!handle || !dev_ptr_out) return fail(MANDEL_EINVAL, "ipc_open needs pointers");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    CK(cudaSetDevice(device));
    cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) { cuda_fail(e, "cudaIpcOpenMemHandle"); return MANDEL_ECOMM; }
    return MANDEL_OK;
}

int mandel_ipc_close(void* dev_ptr) {
    if (!dev_ptr) return fail(MANDEL_EINVAL, "ipc_close needs a pointer");
    cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    if (e != cudaSuccess) { cuda_fail(e, "cudaIpcCloseMemHandle"); return MANDEL_ECOMM; }
    return MANDEL_OK;
}

int mandel_colorize(const uint32_t* counts_dev, uint8_t* rgb_dev, uint32_t W, uint32_t H,
                    uint32_t iterMax, int mode, void* stream) {
    if (!counts_dev || !rgb_dev) return fail(MANDEL_EINVAL, "colorize needs device pointers");
    if (W == 0 || H == 0 || iterMax == 0) return fail(MANDEL_EINVAL, "colorize needs W, H, iterMax >= 1");
    if (mode != MANDEL_COLOUR_GRAY && mode != MANDEL_COLOUR_CLASSIC) return fail(MANDEL_EINVAL, "unknown colour mode");
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    if (s) CK(cudaStreamGetDevice(s, &dev));
    else {
        cudaPointerAttributes a;
        CK(cudaPointerGetAttributes(&a, counts_dev));
        dev = a.device;
    }
    CK(cudaSetDevice(dev));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const uint64_t npix = (uint64_t)W * H;
    const bool aligned = ((uintptr_t)counts_dev % 16 == 0) && ((uintptr_t)rgb_dev % 4 == 0);
    const unsigned grid = (unsigned)(sms * 8);  // 8 x 256-thread CTAs per SM, grid-stride
    const float scale = iterMax > 1 ? (float)(255.0 / (double)(iterMax - 1)) : 0.0f;  // any estimate works:
    // the kernel corrects it exactly (mandel_image.cuh, colour_rgb)
    if (aligned) mandel::colourize_kernel<<<grid, 256, 0, s>>>(counts_dev, rgb_dev, npix, iterMax, mode, scale);
    else mandel::colourize_scalar_kernel<<<grid, 256, 0, s>>>(counts_dev, rgb_dev, npix, iterMax, mode, scale);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    return MANDEL_OK;
}

int mandel_write_ppm(const char* path, const uint8_t* rgb_host, uint32_t W, uint32_t H,
                     uint64_t* bytes_written) {
    if (!path || !rgb_host || W == 0 || H == 0) return fail(MANDEL_EINVAL, "write_ppm needs a path, data and W, H >= 1");
    char hdr[64];
    const int hl = std::snprintf(hdr, sizeof(hdr), "P6\n%u %u\n255\n", W, H);
    FILE* f = std::fopen(path, "wb");
    if (!f) return fail(MANDEL_EIO, std::string("cannot open ") + path);
    const size_t body = (size_t)W * H * 3;
    bool ok = std::fwrite(hdr, 1, (size_t)hl, f) == (size_t)hl && std::fwrite(rgb_host, 1, body, f) == body;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) return fail(MANDEL_EIO, std::string("write failed: ") + path);
    if (bytes_written) *bytes_written = (uint64_t)hl + body;
    return MANDEL_OK;
}

int mandel_finish(void) {
    BusyGuard busy;
    if (!busy.ok) return fail(MANDEL_EBUSY, "another mandel call is in progress");
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_dev.empty()) return MANDEL_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    CK(cudaSetDevice(0));
    if (g_root.copy_stream) CK(cudaStreamSynchronize(g_root.copy_stream));
    if (g_root.async_stream) CK(cudaStreamSynchronize(g_root.async_stream));
    if (g_root.band_stream) CK(cudaStreamSynchronize(g_root.band_stream));
    cudaSetDevice(prev);
    return MANDEL_OK;
}

int mandel_sync(void* stream) {
    if (stream) CK(cudaStreamSynchronize((cudaStream_t)stream));
    else CK(cudaDeviceSynchronize());
    return MANDEL_OK;
}

int mandel_dev_zero(void* dev_ptr, size_t bytes, void* stream) {
    if (!dev_ptr) return fail(MANDEL_EINVAL, "dev_zero needs a pointer");
    cudaStream_t s = (cudaStream_t)stream;
    if (s) {
        int dev = 0;
        CK(cudaStreamGetDevice(s, &dev));
        CK(cudaSetDevice(dev));
    }
    CK(cudaMemsetAsync(dev_ptr, 0, bytes, s));
    CK(cudaStreamSynchronize(s));
    return MANDEL_OK;
}

void mandel_shutdown(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (int r = 0; r < MANDEL_MAX_GPUS; ++r) {
        RankCtx& rc = g_rank[r];
        if (rc.device < 0) continue;
        cudaSetDevice(rc.device);
        if (rc.stream) cudaStreamDestroy(rc.stream);
        if (rc.k0) cudaEventDestroy(rc.k0);
        if (rc.k1) cudaEventDestroy(rc.k1);
        if (rc.used) {
            cudaEventSynchronize(rc.used);
            cudaEventDestroy(rc.used);
        }
        if (rc.d2h) {
            cudaEventSynchronize(rc.d2h);
            cudaEventDestroy(rc.d2h);
        }
        if (rc.state) cudaFree(rc.state);
        if (rc.band) cudaFree(rc.band);
        rc = RankCtx();
    }
    if (!g_dev.empty()) {
        cudaSetDevice(0);
        if (g_root.image) cudaFree(g_root.image);
        if (g_root.fcfs_ctr) cudaFree(g_root.fcfs_ctr);
        if (g_root.start) cudaEventDestroy(g_root.start);
        if (g_root.done) cudaEventDestroy(g_root.done);
        if (g_root.d2h) cudaEventDestroy(g_root.d2h);
        if (g_root.band_state) cudaFree(g_root.band_state);
        if (g_root.band_stream) cudaStreamDestroy(g_root.band_stream);
        if (g_root.copy_stream) cudaStreamDestroy(g_root.copy_stream);
        if (g_root.copy_done) cudaEventDestroy(g_root.copy_done);
        cudaDeviceSynchronize();  // asynchronous renders may still be in flight
        for (int k = 0; k < 2; ++k) {
            if (g_root.pp_image[k]) cudaFree(g_root.pp_image[k]);
            if (g_root.pp_state[k]) cudaFree(g_root.pp_state[k]);
            if (g_root.pp_done[k]) cudaEventDestroy(g_root.pp_done[k]);
        }
        if (g_root.entry) cudaEventDestroy(g_root.entry);
        if (g_root.async_stream) cudaStreamDestroy(g_root.async_stream);
        for (int b = 0; b < kMaxBands; ++b) {
            if (g_root.band_k0[b]) cudaEventDestroy(g_root.band_k0[b]);
            if (g_root.band_k1[b]) cudaEventDestroy(g_root.band_k1[b]);
            if (g_root.band_cp[b]) cudaEventDestroy(g_root.band_cp[b]);
        }
    }
    for (size_t dv = 0; dv < g_dev.size(); ++dv) {
        cudaSetDevice((int)dv);
        if (g_dev[dv].scratch) cudaFree(g_dev[dv].scratch);
        if (g_dev[dv].pstate) cudaFree(g_dev[dv].pstate);
        g_dev[dv].scratch = nullptr;
        g_dev[dv].scratch_bytes = 0;
        g_dev[dv].pstate = nullptr;
        g_dev[dv].pstate_bytes = 0;
    }
    g_root = Root();
    g_auto.clear();
    g_view_ms.clear();
    for (auto& d : g_dev) d.init = false;
    cudaGetLastError();
}

#if MANDEL_TRACE
// Development only (libmandel_trace.so; not in include/mandel.h): copy the first n warp
// records of the last traced launch on the current device (tools/trace_view.py), then
// clear them.
int mandel_dev_trace(void* host, unsigned n) {
    const size_t bytes = (size_t)std::min<unsigned>(n, mandel::kTraceRecs) * sizeof(mandel::TraceRec);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpyFromSymbol(host, mandel::g_trace, bytes));
    static std::vector<char> zeros(sizeof(mandel::TraceRec) * mandel::kTraceRecs, 0);
    CK(cudaMemcpyToSymbol(mandel::g_trace, zeros.data(), zeros.size()));
    return MANDEL_OK;
}
#endif

}  // extern "C"
