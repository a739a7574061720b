/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the escape-time
 * Mandelbrot map of arXiv 2007.00745 ("Efficient Generation of Mandelbrot Set
 * using Message Passing Interface").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this
 * library.  The product path (paper_2007_00745_b200/) never links, loads or
 * imports it, and shares no code, header, table or constant generator with it.
 *
 * Build (see __graft_entry__.build and tests/conftest.py):
 *   gcc -std=c11 -O2 -ffp-contract=off -fno-fast-math -fPIC -shared \
 *       -o oracle/liboracle.so oracle/oracle.c -lm
 * -ffp-contract=off forbids fusing a*b+c into one FMA; on x86-64 all float and
 * double arithmetic is SSE (FLT_EVAL_METHOD == 0), so every operation below is
 * one IEEE-754 round-to-nearest-even operation in its own type.
 *
 * What it computes (SURVEY.md §8(c) "C-def"):
 *   Eq. 1  (§I):  f(z) = z^2 + c, applied repeatedly from z = 0.
 *   Eq. 2  (§I):  I_{i,j} = Iteration_{i,j}, "the Iteration at
 *          which either the magnitude (z^2) exceeding the escape radius or the
 *          iterationMax, is recorded".
 *   Cx/Cy  (§III-A): "all of the nodes will generate the Cy and Cx
 *          arrays" -- the per-column real part and per-row imaginary part.
 * Readings (R1..R11): escape is |z|^2 > R*R (strict), tested after each
 * update on the new z; the count is the number of z-updates performed (1-based,
 * in [1, iterMax]); Cx[j] = xmin + j*dx, Cy[i] = ymax - i*dy with dx, dy
 * divided once; fp32 rounds the bounds and R to float first and then works in
 * float only.
 *
 * Pins (tests/test_oracle_pins.py): closed-form orbits, hand-iterated escapes,
 * exact-rational brute force on an 8x8 grid, pixel-exact pin points on the
 * configured grids, mirror symmetry, power-of-two decimation, iterMax
 * monotonicity, and an independent numpy re-implementation.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

#define ORACLE_FP64 0
#define ORACLE_FP32 1
#define ORACLE_FP64_FMA 2

/* ---------------------------------------------------------------------------
 * Eq. 1 + Eq. 2 for one point c = cr + i*ci, in double.
 * z = x + i*y; z^2 + c = (x^2 - y^2 + cr) + i*(2*x*y + ci).
 * x2 = x*x and y2 = y*y are carried from the previous update (both 0 at z = 0).
 * ------------------------------------------------------------------------- */
uint32_t oracle_escape_f64(double cr, double ci, uint32_t iterMax, double R2)
{
    double x = 0.0, y = 0.0, x2 = 0.0, y2 = 0.0;
    uint32_t n = 0;
    while (n < iterMax) {
        double two_x = x + x;          /* 2x                         */
        double xy2 = two_x * y;        /* 2xy                        */
        double new_y = xy2 + ci;       /* Im(z^2 + c) = 2xy + ci     */
        double d = x2 - y2;            /* x^2 - y^2                  */
        double new_x = d + cr;         /* Re(z^2 + c) = x^2-y^2 + cr */
        x = new_x;
        y = new_y;
        x2 = x * x;
        y2 = y * y;
        n = n + 1;
        double mag2 = x2 + y2;         /* |z|^2                      */
        if (mag2 > R2)                 /* escape radius exceeded     */
            break;
    }
    return n;
}

/* The same computation with every variable and operation in float. */
uint32_t oracle_escape_f32(float cr, float ci, uint32_t iterMax, float R2)
{
    float x = 0.0f, y = 0.0f, x2 = 0.0f, y2 = 0.0f;
    uint32_t n = 0;
    while (n < iterMax) {
        float two_x = x + x;
        float xy2 = two_x * y;
        float new_y = xy2 + ci;
        float d = x2 - y2;
        float new_x = d + cr;
        x = new_x;
        y = new_y;
        x2 = x * x;
        y2 = y * y;
        n = n + 1;
        float mag2 = x2 + y2;
        if (mag2 > R2)
            break;
    }
    return n;
}

/* ---------------------------------------------------------------------------
 * The fused-multiply-add variant of the same recurrence (reading R17):
 *   y' = fma(x + x, y, ci);  x' = fma(x, x, -y^2) + cr;  y2' = y' * y';
 *   |z'|^2 = fma(x', x', y2')
 * C99 fma() is one correctly rounded fused multiply-add (ISO C 7.12.13.1).
 * ------------------------------------------------------------------------- */
uint32_t oracle_escape_f64fma(double cr, double ci, uint32_t iterMax, double R2)
{
    double x = 0.0, y = 0.0, y2 = 0.0;
    uint32_t n = 0;
    while (n < iterMax) {
        double two_x = x + x;
        double new_y = fma(two_x, y, ci);     /* 2xy + ci, one rounding        */
        double d = fma(x, x, -y2);            /* x^2 - y^2, one rounding       */
        double new_x = d + cr;
        x = new_x;
        y = new_y;
        y2 = y * y;
        n = n + 1;
        double mag2 = fma(x, x, y2);          /* x^2 + y^2, one rounding       */
        if (mag2 > R2)
            break;
    }
    return n;
}

/* ---------------------------------------------------------------------------
 * Step a1: derived constants.  dx = (xmax - xmin)/W, dy = (ymax - ymin)/H,
 * R2 = R*R, each one IEEE operation.  out = {dx, dy, R2}.
 * ------------------------------------------------------------------------- */
void oracle_derive_f64(double xmin, double xmax, double ymin, double ymax,
                       uint32_t W, uint32_t H, double R, double out[3])
{
    out[0] = (xmax - xmin) / (double)W;
    out[1] = (ymax - ymin) / (double)H;
    out[2] = R * R;
}

/* fp32: bounds and R are rounded to float first (a C cast rounds to nearest).
 * out = {xmin_f, ymax_f, dx, dy, R2}. */
void oracle_derive_f32(double xmin, double xmax, double ymin, double ymax,
                       uint32_t W, uint32_t H, double R, float out[5])
{
    float xa = (float)xmin, xb = (float)xmax;
    float ya = (float)ymin, yb = (float)ymax;
    float Rf = (float)R;
    out[0] = xa;
    out[1] = yb;
    out[2] = (xb - xa) / (float)W;
    out[3] = (yb - ya) / (float)H;
    out[4] = Rf * Rf;
}

/* ---------------------------------------------------------------------------
 * Step a3: the Cx / Cy arrays.  Row 0 is ymax.
 * ------------------------------------------------------------------------- */
double oracle_cx_f64(double xmin, double dx, uint32_t j) { double t = (double)j * dx; return xmin + t; }
double oracle_cy_f64(double ymax, double dy, uint32_t i) { double t = (double)i * dy; return ymax - t; }
float  oracle_cx_f32(float xmin, float dx, uint32_t j)   { float t = (float)j * dx;  return xmin + t; }
float  oracle_cy_f32(float ymax, float dy, uint32_t i)   { float t = (float)i * dy;  return ymax - t; }

/* ---------------------------------------------------------------------------
 * Rows [row0, row1) of the W x H map, row-major, out[(i-row0)*W + j].
 * Follows the paper's serial structure: build Cx, Cy; loop rows; loop columns.
 * Returns 0, or -1 on an argument the oracle does not define.
 * ------------------------------------------------------------------------- */
int oracle_render_rows(double xmin, double xmax, double ymin, double ymax,
                       uint32_t W, uint32_t H, uint32_t iterMax, double R,
                       int dtype, uint32_t row0, uint32_t row1, uint32_t *out)
{
    if (W == 0 || H == 0 || iterMax == 0 || row0 > row1 || row1 > H || out == NULL)
        return -1;
    if (dtype == ORACLE_FP64 || dtype == ORACLE_FP64_FMA) {
        double k[3];
        oracle_derive_f64(xmin, xmax, ymin, ymax, W, H, R, k);
        for (uint32_t i = row0; i < row1; ++i) {
            double ci = oracle_cy_f64(ymax, k[1], i);
            for (uint32_t j = 0; j < W; ++j) {
                double cr = oracle_cx_f64(xmin, k[0], j);
                out[(size_t)(i - row0) * W + j] = dtype == ORACLE_FP64
                    ? oracle_escape_f64(cr, ci, iterMax, k[2])
                    : oracle_escape_f64fma(cr, ci, iterMax, k[2]);
            }
        }
        return 0;
    }
    if (dtype == ORACLE_FP32) {
        float k[5];
        oracle_derive_f32(xmin, xmax, ymin, ymax, W, H, R, k);
        for (uint32_t i = row0; i < row1; ++i) {
            float ci = oracle_cy_f32(k[1], k[3], i);
            for (uint32_t j = 0; j < W; ++j) {
                float cr = oracle_cx_f32(k[0], k[2], j);
                out[(size_t)(i - row0) * W + j] = oracle_escape_f32(cr, ci, iterMax, k[4]);
            }
        }
        return 0;
    }
    return -1;
}

/* Arbitrary pixels (ii[p], jj[p]), p < n: used to check sampled outputs of the
 * full-size configurations one by one. */
int oracle_render_pixels(double xmin, double xmax, double ymin, double ymax,
                         uint32_t W, uint32_t H, uint32_t iterMax, double R,
                         int dtype, const uint32_t *ii, const uint32_t *jj,
                         size_t n, uint32_t *out)
{
    if (W == 0 || H == 0 || iterMax == 0 || (n > 0 && (ii == NULL || jj == NULL || out == NULL)))
        return -1;
    for (size_t p = 0; p < n; ++p)
        if (ii[p] >= H || jj[p] >= W)
            return -1;
    if (dtype == ORACLE_FP64 || dtype == ORACLE_FP64_FMA) {
        double k[3];
        oracle_derive_f64(xmin, xmax, ymin, ymax, W, H, R, k);
        for (size_t p = 0; p < n; ++p) {
            double cr = oracle_cx_f64(xmin, k[0], jj[p]), ci = oracle_cy_f64(ymax, k[1], ii[p]);
            out[p] = dtype == ORACLE_FP64 ? oracle_escape_f64(cr, ci, iterMax, k[2])
                                          : oracle_escape_f64fma(cr, ci, iterMax, k[2]);
        }
        return 0;
    }
    if (dtype == ORACLE_FP32) {
        float k[5];
        oracle_derive_f32(xmin, xmax, ymin, ymax, W, H, R, k);
        for (size_t p = 0; p < n; ++p)
            out[p] = oracle_escape_f32(oracle_cx_f32(k[0], k[2], jj[p]),
                                       oracle_cy_f32(k[1], k[3], ii[p]), iterMax, k[4]);
        return 0;
    }
    return -1;
}
