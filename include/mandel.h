/*
 * mandel.h -- C ABI of the B200-native escape-time Mandelbrot library
 * (paper_2007_00745_b200/libmandel.so), the boundary of the hot path of
 * arXiv 2007.00745, "Efficient Generation of Mandelbrot Set using Message
 * Passing Interface" (Gamage & Baskaran).
 *
 * Every step of the path (pixel -> c mapping, escape iteration, store, the
 * FCFS chunk claims and the gather to rank 0) runs in this library's sm_100a
 * kernels.  There is no CPU fallback: without a usable CUDA device every
 * compute entry point returns MANDEL_ENODEV.
 *
 * Operation (Eq. 1 and Eq. 2; PAPER.md:179 Cx/Cy arrays):
 *   dx = (xmax - xmin) / W,   dy = (ymax - ymin) / H,   R2 = R * R   (host, one IEEE op each)
 *   c(i, j) = (xmin + j*dx, ymax - i*dy)          row 0 is ymax (top-left-corner sampling)
 *   z0 = 0;  z_{n+1} = z_n^2 + c;  count(i, j) = first n >= 1 with |z_n|^2 > R2, else iterMax
 *   out[i*W + j] = count(i, j),  1 <= count <= iterMax
 * Every floating-point operation is a single round-to-nearest-even operation
 * in the working type, in the order  y' = (x + x)*y + ci;  x' = (x2 - y2) + cr;
 * x2 = x'*x';  y2 = y'*y';  escape iff x2 + y2 > R2  -- no FMA contraction.
 * The result is therefore one exact uint32 map per argument set, identical for
 * every scheme, GPU count and chunk size (Bernstein conditions).
 *
 * dtype MANDEL_FP32 computes everything in float: the bounds and R are first
 * rounded to float, then dx, dy, R2 and the mapping are float operations
 * (reading R9).
 *
 * Partition schemes (§III, 150-225) distribute rows over ngpus GPUs:
 *   MANDEL_BLOCK   "Naive" rows, Eq. 14-17: rank r owns [q*r, q*(r+1)-1],
 *                  q = floor(H/N); the last rank also owns the H mod N tail.
 *   MANDEL_CYCLIC  "Alternating" rows: rank r owns rows
 *                  r, r+N, ... below floor(H/N)*N; rank 0 owns the tail.
 *   MANDEL_FCFS    "First Come First Served": GPUs claim
 *                  chunk_rows-row chunks from one atomic counter in GPU 0's
 *                  memory (system-scope atomics over NVLink); no master GPU.
 *   MANDEL_FCFS_MASTER the paper's own FCFS: rank 0 computes nothing, the others
 *                  claim single rows (Eq. 19: T_m = 2 iYmax messages) -- needs N >= 2.
 * Each GPU's kernel stores its counts directly into GPU 0's image (peer
 * stores over NVLink): the paper's "send to master" without a
 * separate gather or the alternating scheme's reconstruction pass.
 *
 * Threading: calls are serialised inside the library; a call that finds
 * another in progress returns MANDEL_EBUSY.  All calls are synchronous: they
 * return when the map is complete in the requested destination.
 */
#ifndef MANDEL_H
#define MANDEL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MANDEL_ABI_VERSION 10
#define MANDEL_MAX_GPUS 64          /* logical ranks (physical GPUs <= device count) */
#define MANDEL_IPC_HANDLE_BYTES 64  /* size of a cudaIpcMemHandle_t                  */

enum mandel_dtype {
    MANDEL_FP64 = 0,     /* the reference map: every operation a separate RN double op          */
    MANDEL_FP32 = 1,     /* the same in float (bounds and R rounded to float first)             */
    MANDEL_FP64_FMA = 2  /* double with fused multiply-adds in the iteration (R17):
                            y' = fma(x+x, y, ci); x' = fma(x, x, -y^2) + cr; |z|^2 = fma(x', x', y'^2)
                            -- 6 instead of 8 FP64 instructions; a different, equally exact map */
};

enum mandel_scheme {
    MANDEL_BLOCK = 0,   /* paper "Naive" row segmentation, Eq. 14-17     */
    MANDEL_CYCLIC = 1,  /* paper "Alternating" row segmentation          */
    MANDEL_FCFS = 2,    /* paper "First Come First Served" (chunked)     */
    MANDEL_FCFS_MASTER = 3  /* paper-faithful FCFS: rank 0 only
                               dispatches and computes no rows; ranks 1..N-1 claim
                               chunk_rows rows at a time (default 1 row); N >= 2 */
};

enum mandel_status {
    MANDEL_OK = 0,
    MANDEL_EINVAL = -1,  /* an argument is out of its documented domain                */
    MANDEL_ENODEV = -2,  /* no CUDA device, too few devices, or no peer access         */
    MANDEL_ENOMEM = -3,  /* device or pinned allocation failed                         */
    MANDEL_ECUDA = -4,   /* a CUDA runtime call failed (detail: mandel_last_error)      */
    MANDEL_ECOMM = -5,   /* inter-GPU / inter-process plumbing failed (IPC, peer map)   */
    MANDEL_EBUSY = -6,   /* another call is in progress                                */
    MANDEL_EIO = -7      /* a file could not be written (mandel_write_ppm)             */
};

enum mandel_colour { MANDEL_COLOUR_GRAY = 0, MANDEL_COLOUR_CLASSIC = 1 };

enum mandel_kernel {
    MANDEL_KERNEL_REFILL = 0,  /* default: EAGER, or LAZY when an EAGER render of a strided 1/16
                                  row sample of the view (once per view, cached) leaves its loop
                                  more often than once per 23 iterations (incoherent escapes)  */
    MANDEL_KERNEL_STATIC = 1,  /* one pixel per thread, static grid (baseline; BLOCK/CYCLIC only)  */
    MANDEL_KERNEL_EAGER = 2,   /* persistent CTAs, warp tile queue, lane refill on every escape   */
    MANDEL_KERNEL_LAZY = 3,    /* the same, refill batched: escapes recorded in-loop, the warp
                                  refills when refill_lanes lanes hold a finished pixel          */
    MANDEL_KERNEL_ADAPTIVE = 4 /* per warp and run: EAGER while escapes are sparse, LAZY while
                                  they are dense (runs shorter than adapt_lo iterations)         */
};

/* Per-call statistics (all fields written when stats != NULL and the call succeeds). */
typedef struct mandel_stats {
    double   device_ms;            /* synchronised start on all GPUs -> GPU 0 holds the full map     */
    double   kernel_ms_max;        /* max over ranks of the escape kernel's CUDA-event time          */
    double   kernel_ms[MANDEL_MAX_GPUS];
    double   d2h_ms;               /* device -> host copy of the map (0 if out_host == NULL)         */
    double   total_ms;             /* host wall time of the whole call                               */
    uint64_t sum_iters;            /* sum of all counts = pixel-iterations performed                 */
    uint64_t pixels;               /* pixels written (W*H when complete)                             */
    uint64_t rank_iters[MANDEL_MAX_GPUS];  /* per-rank pixel-iterations                            */
    uint64_t rank_pixels[MANDEL_MAX_GPUS]; /* per-rank pixels                                      */
    uint32_t rank_rows[MANDEL_MAX_GPUS];   /* per-rank rows started (FCFS: claimed chunk rows)     */
    uint32_t chunks_claimed;       /* FCFS successful global claims counted on the device by the
                                      claiming kernels (= ceil(H/chunk_rows) when complete; Eq. 19).
                                      0 when the kernels ran a static row order (kernel_scheme)   */
    uint32_t transfers;            /* results sent to rank 0: static schemes one band per rank != 0
                                      (N-1, Eq. 18/20); FCFS schemes the rows computed by ranks != 0
                                      (FCFS_MASTER: every row; Eq. 19 counts claim + reply = 2 H)   */
    uint32_t kernel_launches;      /* kernels this call launched                                    */
    uint32_t ngpus;                /* ranks used                                                    */
    uint32_t ndevices;             /* distinct physical devices used                                */
    int32_t  kernel_variant;       /* enum mandel_kernel actually run (EAGER/LAZY/ADAPTIVE/STATIC)   */
    int32_t  kernel_ilp;           /* pixels per lane of that kernel                                */
    float    probe[2];             /* last view probe (MANDEL_KERNEL_REFILL): eager sample time (ms),
                                      eager iterations per loop exit (< 23 selects LAZY)           */
    uint64_t warp_iters;           /* kernel-choice probe only (else 0): loop iterations over warps */
    uint64_t loop_exits;           /* kernel-choice probe only (else 0): loop exits over warps      */
    int32_t  kernel_batch;         /* EAGER: z-updates per escape check actually run (1, 4, 8, 16)  */
    int32_t  kernel_packed;        /* 1: the fp32 batched loop ran on FADD2/FMUL2 slot pairs        */
    double   sm_clock_mhz;         /* SM clock during the escape kernels, measured in them: the sum
                                      over CTAs of SM cycles (clock64) / the sum of wall ns
                                      (%globaltimer), x 1e3; over every rank and band of the call  */
    int32_t  kernel_scheme;        /* the row order the kernels actually ran (enum mandel_scheme):
                                      the requested scheme, except MANDEL_BLOCK for the row bands of
                                      the pipelined one-GPU host hand-off (each band a row range)  */
    int32_t  store_mode;           /* how rank 0's kernels stored counts: 0 each count directly (4-B
                                      stores), 1 staged 8 x 8 blocks stored count by count, 2 staged
                                      blocks stored with 16-B vector stores (map 16-B aligned, W and
                                      the tile width multiples of 4)                               */
    int32_t  fused_y;              /* 1: the fused-y form was enabled for rank 0's launch (its warps
                                      use it where their pixels allow, options.fused_y)         */
    int32_t  host_handoff;         /* 1: the per-device host hand-off ran (options.host_handoff):
                                      d2h_ms is then from the last kernel's end to the last rank's
                                      last copy, and transfers counts the device->host copies     */
    int32_t  first_block;          /* lanes' worth of fresh slots that start an exactly recorded first
                                      block in rank 0's launch (options.first_block); 0: none (the
                                      kernel is not a batched EAGER one, or -1 was asked)          */
} mandel_stats;

/* Optional knobs for mandel_render_ex / mandel_render_rank (NULL = defaults). */
typedef struct mandel_options {
    uint32_t chunk_rows;     /* FCFS rows per claim; 0 -> 16 (BASELINE.json C5)                   */
    uint32_t tile_px;        /* pixels per warp tile (persistent kernels); 0 -> 256, or 128 / 64
                                when a rank has < 4096 / < 1024 pixels per resident warp        */
    int      kernel;         /* enum mandel_kernel                                                */
    int      logical_ranks;  /* nonzero: allow ngpus > device count, rank g runs on device
                                g % count on its own stream (tests; ranks never wait on each other) */
    int      refill_lanes;   /* LAZY: lanes with a finished pixel that trigger a refill (1..32);
                                0 -> library default                                               */
    int      ilp;            /* pixels per lane (EAGER 1..4, LAZY/ADAPTIVE 1..2); 0 -> default     */
    int      min_ctas;       /* register budget as CTAs per SM (1,3,4,5,6,8); 0 -> default           */
    int      adapt_lo;       /* ADAPTIVE: eager->lazy when the mean eager run is shorter; 0 -> default */
    int      adapt_hi;       /* ADAPTIVE: lazy runs before probing eager again; 0 -> default         */
    int      bands;          /* one GPU + out_host: row bands whose device->host copies overlap
                                the later bands' compute (0 -> 8, 1 -> no pipelining, max 32)     */
    int      band_taper;     /* pipelined bands: band pair p (outside-in) holds a share taper^p
                                of the rows, in percent (100 = equal bands); 0 -> 70            */
    int      tile_rows;      /* persistent kernels: row slots per warp tile (power of two <= 64;
                                a tile is tile_rows x tile_px/tile_rows pixels, handed to the
                                warp in 8-column blocks); FCFS cuts it to divide chunk_rows;
                                0 -> 8                                                           */
    int      band_out;       /* mandel_render_rank only (the NCCL gather path):
                                out_root is this rank's own compact band on its device, band row
                                b = the rank's b-th row slot (static: the plan's order; FCFS: local
                                chunk k row r at b = k*chunk_rows + r); mandel_band_rows then gives
                                each band row's image row, and mandel_scatter_rows (K4) places a
                                gathered band in the image.  Capacity: static schemes the plan's
                                row count x W; FCFS ceil(H/chunk_rows)*chunk_rows x W (a rank may
                                claim every chunk).  mandel_render_ex -> MANDEL_EINVAL            */
    int      no_pack;        /* fp32: nonzero keeps the batched loop scalar (default: packed
                                FADD2/FMUL2 on slot pairs when ilp >= 2; bit-identical)           */
    int      max_sms;        /* persistent kernels: run each rank on exactly this many SMs, one
                                CTA per SM (a rank as a fixed slice of the GPU; ranks sharing a
                                GPU then never share an SM); 0 -> every SM, full occupancy      */
    int      async_host;     /* mandel_render_ex with out_host, one GPU, no out_dev0 and no stats:
                                return once the render and its banded device->host copy are
                                enqueued; consecutive calls overlap (alternate library maps), and
                                out_host is complete after mandel_finish().  Do not touch out_host
                                of an unfinished call.  0 -> synchronous                          */
    int      check_every;    /* EAGER: z-updates per escape test.  1 -> every update (Eq. 2 as
                                written); 4, 8 or 16 -> batched (R18): |z|^2 is tested
                                after every 4th/8th/16th update against a threshold just below
                                R^2; a batch that reaches it is replayed from its saved start
                                with the exact per-update test, so counts are unchanged.  Needs
                                R >= 2 (an escaped orbit then keeps growing); fp32 allows <= 8.
                                0 -> default (8 when valid, else 1); otherwise MANDEL_EINVAL       */
    int      stage;          /* output stores (EAGER check-every-8 and LAZY kernels, budgets 1/3):
                                1 -> staged: each warp collects its 8 x 8 pixel blocks in shared
                                memory and stores each whole block as 32-B rows with 16-B vector
                                stores (map 16-B aligned, W a multiple of 4; else count by
                                count); -1 -> every count stored directly (4-B stores);
                                0 -> default: staged when the map is on another GPU (the fused
                                gather's NVLink peer stores), direct into the rank's own HBM    */
    int      ctas_per_sm;    /* persistent kernels: at most this many resident CTAs per SM (grid =
                                min(this, occupancy) x SMs); 0 -> the occupancy maximum            */
    int      fused_y;        /* fp64 / fp32, EAGER and LAZY kernels: how y' = (x + x) y + ci is
                                evaluated (R21).  0 or 1 -> fma(RN(x y), 2, ci) for the
                                warps whose pixels are all "safe" (cr != 0, |cr| and any nonzero
                                |ci| >= 2^-400 [fp32 2^-32]) when R^2 <= 2^256 [fp32 2^64]: the
                                same rounded value, one instruction fewer per update; other
                                warps and views use the three-operation form.  -1 -> always the
                                three-operation form.  Counts are identical either way.        */
    int      host_handoff;   /* mandel_render / _ex with out_host and ngpus > 1: how the map reaches
                                the host.  -1 -> through GPU 0: every rank stores into GPU 0's map
                                (the fused gather) and GPU 0 copies W*H*4 bytes to out_host;
                                1 -> per device: every rank stores its rows into a band in its own
                                device memory and its device copies them to their rows of
                                out_host (N links in parallel, each copy starting when its rank's
                                kernel ends; FCFS: after reading back the rank's chunk map);
                                0 -> default: per device when the ranks span more than one GPU.
                                Ignored with one rank or without out_host.                      */
    int      first_block;    /* EAGER batched kernels (check_every > 1): a refill that hands fresh
                                pixels to at least this many lanes' worth of the warp's slots
                                (1..32) starts with one block of 8 z-updates whose Eq. 2 test is
                                recorded exactly after every update (as the LAZY kernel does)
                                instead of a batch that would hit and be replayed -- the warp is
                                in the exterior, where counts are a few updates.  Counts are
                                identical either way.  0 -> default
                                (2); -1 -> never; otherwise MANDEL_EINVAL                         */
} mandel_options;

/*
 * mandel_render -- BASELINE.json north_star entry point.
 *   xmin < xmax, ymin < ymax : the complex window (finite doubles)
 *   W, H      : image width (columns, real axis) and height (rows, imaginary axis), >= 1
 *   iterMax   : iteration cap ("iterationMax"), 1 <= iterMax <= 2^32 - 2
 *   R         : escape RADIUS (> 0, R*R finite in dtype); escape is |z|^2 > R*R.
 *               The paper's "Escape Radius 400" is R = 20 (R1).
 *   dtype     : enum mandel_dtype
 *   scheme    : enum mandel_scheme
 *   ngpus     : GPUs 0..ngpus-1 (1 <= ngpus <= device count)
 *   out_u32   : HOST buffer of W*H uint32, row-major, caller-owned (pinned recommended)
 * Returns MANDEL_OK or a negative mandel_status; on error out_u32 is unspecified.
 * EINVAL: W or H == 0; W*H*4 overflows size_t; iterMax == 0 or 2^32 - 1; R <= 0 or non-finite or
 *   R*R non-finite (in dtype); any bound non-finite (in dtype); xmin >= xmax or
 *   ymin >= ymax (after rounding, for fp32); dx or dy == 0 in dtype; dtype/scheme out of
 *   range; out_u32 == NULL; BLOCK/CYCLIC with H < ngpus; FCFS_MASTER with ngpus < 2.
 * ENODEV: ngpus < 1, ngpus > devices, no CUDA device, or peer access unavailable.
 */
int mandel_render(double xmin, double xmax, double ymin, double ymax,
                  uint32_t W, uint32_t H, uint32_t iterMax, double R,
                  int dtype, int scheme, int ngpus, uint32_t *out_u32);

/*
 * mandel_render_ex -- mandel_render with options, statistics and device output.
 *   out_host : nullable HOST destination (W*H uint32); copied device->host at the end.
 *   out_dev0 : nullable DEVICE pointer on device 0 (caller-owned, >= W*H*4 bytes,
 *              4-byte aligned) that receives the map; if NULL the library uses a
 *              cached buffer it owns.  At least one of out_host / out_dev0 is required.
 *   stream0  : nullable cudaStream_t on device 0; rank 0's work (and the D2H copy) is
 *              ordered on it, so a caller can time the call with events on that stream.
 *   opts     : nullable options;  stats : nullable statistics.
 * With out_host == NULL and stats == NULL the render is only ENQUEUED (the call returns
 * without waiting; work ordered on stream0 runs after it); otherwise it returns when the
 * map is in place.
 * Errors as mandel_render; EINVAL also when both outputs are NULL.
 */
int mandel_render_ex(double xmin, double xmax, double ymin, double ymax,
                     uint32_t W, uint32_t H, uint32_t iterMax, double R,
                     int dtype, int scheme, int ngpus,
                     const mandel_options *opts,
                     uint32_t *out_host, uint32_t *out_dev0, void *stream0,
                     mandel_stats *stats);

/*
 * mandel_render_rank -- one rank of a multi-PROCESS render (one process per GPU,
 * e.g. under torchrun).  The caller's process runs rank `rank` of `nranks` on the
 * current CUDA device and:
 *   out_root     : DEVICE pointer, valid in this process, to rank 0's W*H uint32 image
 *                  (rank 0: its own buffer; others: mapped with mandel_ipc_open).
 *   fcfs_counter : DEVICE pointer to a uint32 chunk counter shared by all ranks (rank 0's
 *                  memory, IPC-mapped elsewhere); must be 0 before any rank starts and is
 *                  only used by MANDEL_FCFS (may be NULL otherwise).  Every render needs a
 *                  counter no rank still claims from (a fresh zeroed one, or a barrier).
 *   stream       : nullable cudaStream_t; the rank runs on the stream's device (else on the
 *                  calling thread's current device).
 * With stats != NULL (or options.band_out) the call returns when this rank's rows are
 * stored and stats receives this rank's kernel_ms / rank_iters[0] / rank_pixels[0] /
 * chunks_claimed.  With stats == NULL the render is only ENQUEUED on the stream (no host
 * synchronisation): the caller orders later work with the stream.
 * Errors: as mandel_render_ex, plus EINVAL for rank outside [0, nranks) or a NULL out_root,
 * or FCFS with a NULL fcfs_counter.
 */
int mandel_render_rank(double xmin, double xmax, double ymin, double ymax,
                       uint32_t W, uint32_t H, uint32_t iterMax, double R,
                       int dtype, int scheme, int rank, int nranks,
                       const mandel_options *opts,
                       uint32_t *out_root, uint32_t *fcfs_counter, void *stream,
                       mandel_stats *stats);

/*
 * Device memory shared across processes (CUDA IPC).  mandel_dev_alloc returns a
 * cudaMalloc'd block on `device` (so IPC handles address it at offset 0);
 * mandel_ipc_handle writes MANDEL_IPC_HANDLE_BYTES bytes describing it;
 * mandel_ipc_open maps another process's block into this process for use on `device`
 * (peer access enabled lazily); mandel_ipc_close unmaps it.
 * Errors: EINVAL on NULL arguments, ENOMEM, ECOMM when the IPC call fails.
 */
int mandel_dev_alloc(int device, size_t bytes, void **dev_ptr);
int mandel_dev_free(void *dev_ptr);
int mandel_ipc_handle(void *dev_ptr, void *handle_out);
int mandel_ipc_open(int device, const void *handle, void **dev_ptr_out);
int mandel_ipc_close(void *dev_ptr);
/* Zero `bytes` bytes at dev_ptr (any device pointer valid in this process) on `stream`
 * (nullable = the legacy default stream of the current device) and wait for it.
 * Used to reset the shared FCFS counter between multi-process renders. */
int mandel_dev_zero(void *dev_ptr, size_t bytes, void *stream);
/* Wait until every asynchronous (options.async_host) render's host output is complete. */
int mandel_finish(void);
/* Wait for everything enqueued on stream (NULL: the whole current device), e.g. after
 * asynchronous mandel_render_rank calls (stats == NULL). */
int mandel_sync(void *stream);

/*
 * mandel_plan_rows -- host-only planner of the static schemes (no GPU needed).
 * Writes the rows rank `rank` of `ngpus` owns under `scheme` (BLOCK: Eq. 14-17;
 * CYCLIC: PAPER.md:217-218), ascending, to rows_out (nullable: then only *count is
 * written).  *count must hold the capacity of rows_out on entry when rows_out != NULL.
 * EINVAL: scheme FCFS (dynamic) or out of range, ngpus < 1, H < ngpus, rank outside
 * [0, ngpus), count NULL, or capacity too small (then *count = rows needed).
 */
int mandel_plan_rows(int scheme, uint32_t H, int ngpus, int rank,
                     uint32_t *rows_out, uint32_t *count);

/*
 * Output stage (after the hot path; "The iteration is then used to determine
 * the pixel color", PAPER.md:179 the master writes the image file).  The paper names no
 * palette: MANDEL_COLOUR_GRAY is SPEC.md:313-321's ramp (interior n == iterMax black,
 * escaped v = round-half-up(255 (n-1)/(iterMax-1)) in all three channels);
 * MANDEL_COLOUR_CLASSIC is (7n, 13n, 29n) mod 256 for escaped pixels, interior black.
 * mandel_colorize: counts_dev (W*H uint32, device) -> rgb_dev (3*W*H bytes, device,
 *   r, g, b per pixel, row-major), on `stream` (nullable: legacy default stream of the
 *   pointer's device); returns when done.  EINVAL on NULL pointers, W or H == 0,
 *   iterMax == 0 or an unknown mode.
 * mandel_write_ppm: binary PPM (P6) "P6\n<W> <H>\n255\n" + rgb_host (3*W*H bytes, host)
 *   to `path`; *bytes_written (nullable) = header + 3*W*H.  EINVAL / EIO.
 */
int mandel_colorize(const uint32_t *counts_dev, uint8_t *rgb_dev, uint32_t W, uint32_t H,
                    uint32_t iterMax, int mode, void *stream);
int mandel_write_ppm(const char *path, const uint8_t *rgb_host, uint32_t W, uint32_t H,
                     uint64_t *bytes_written);

/* Static description of a status code (never NULL). */
const char *mandel_strerror(int code);
/* Detail string of the calling thread's last failure ("" if none). */
const char *mandel_last_error(void);
/* Number of visible CUDA devices (0 when none or the driver is unusable). */
int mandel_device_count(void);
/* Frees cached device buffers, streams and events on every device. */
void mandel_shutdown(void);
/*
 * mandel_band_rows -- after a band_out mandel_render_rank call (SURVEY.md §8(e) NCCL path):
 * the image row of every band row of that render, in band order; 0xffffffff marks a
 * band row no pixel was written to (FCFS slots past the last image row).  Host memory;
 * rows_out NULL queries *count.  EINVAL if *count is too small (*count is set).
 */
int mandel_band_rows(uint32_t *rows_out, uint32_t *count);

/*
 * mandel_scatter_rows -- K4: image[rows[b]] = band[b] for b < nrows, W uint32 per row;
 * rows[b] == 0xffffffff skipped.  band_dev, rows_dev and image_dev are device pointers on
 * stream's device (stream NULL: image_dev's device, legacy stream).  Asynchronous on
 * stream.  The de-interleave step after the NCCL gather of cyclic / FCFS bands
 * ("reconstructs the image").
 */
int mandel_scatter_rows(const uint32_t *band_dev, const uint32_t *rows_dev, uint32_t nrows, uint32_t W,
                        uint32_t *image_dev, void *stream);

/* MANDEL_ABI_VERSION of the loaded library. */
int mandel_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* MANDEL_H */
