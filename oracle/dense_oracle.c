/*
 * TEST INFRASTRUCTURE ONLY -- parity oracle, never part of the product path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.
 *
 * Exact dense restatement of the reference's slow oracle:
 *   - kernel value  = area( [x1 +- a1/2] x [x2 +- a3/2]
 *                           intersect {|y1+y2| <= a2/sqrt2, |y1-y2| <= a4/sqrt2} )
 *                     / (a1 a2 a3 a4)
 *     (reference: pkg/src/rubs/_exact.py:1-16 states the geometry; the
 *      reference integrates slice lengths, _exact.py:63-106.  Here the
 *      same area is obtained by an independent route: Sutherland-Hodgman
 *      clipping of the rectangle by the four diamond half-planes followed
 *      by the shoelace formula.)
 *   - dense filter  = out(n) = sum_m K_{a(n)}(n - m) cur(m), zero outside
 *     the image, the scale field floored at 0.05 and divided by sqrt(m)
 *     (reference: pkg/src/rubs/oracle.py:177-241, floor at :197-198).
 *   - iterated passes run on canvases extended by the per-pass support,
 *     the field edge-clamped (oracle.py:200-241).
 *
 * Entry points are plain C so tests can ctypes-load oracle/_build/liboracle.so.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdint.h>

#define SQRT2 1.4142135623730951

/* Area of the axis rectangle [rx0,rx1]x[ry0,ry1] clipped by
 * |y1+y2| <= hs and |y1-y2| <= hd. */
static double clipped_area(double rx0, double rx1, double ry0, double ry1,
                           double hs, double hd)
{
    double px[16], py[16], qx[16], qy[16];
    int n = 4;
    px[0] = rx0; py[0] = ry0;
    px[1] = rx1; py[1] = ry0;
    px[2] = rx1; py[2] = ry1;
    px[3] = rx0; py[3] = ry1;
    /* half-planes nx*x + ny*y <= c */
    const double hpn[4][2] = {{1.0, 1.0}, {-1.0, -1.0}, {1.0, -1.0}, {-1.0, 1.0}};
    const double hpc[4] = {hs, hs, hd, hd};
    for (int h = 0; h < 4 && n > 0; ++h) {
        int m = 0;
        for (int i = 0; i < n; ++i) {
            int j = (i + 1) % n;
            double dp = hpn[h][0] * px[i] + hpn[h][1] * py[i] - hpc[h];
            double dq = hpn[h][0] * px[j] + hpn[h][1] * py[j] - hpc[h];
            if (dp <= 0.0) { qx[m] = px[i]; qy[m] = py[i]; ++m; }
            if ((dp < 0.0 && dq > 0.0) || (dp > 0.0 && dq < 0.0)) {
                double t = dp / (dp - dq);
                qx[m] = px[i] + t * (px[j] - px[i]);
                qy[m] = py[i] + t * (py[j] - py[i]);
                ++m;
            }
        }
        n = m;
        memcpy(px, qx, sizeof(double) * (size_t)n);
        memcpy(py, qy, sizeof(double) * (size_t)n);
    }
    if (n < 3) return 0.0;
    /* shoelace relative to the first vertex for accuracy */
    double acc = 0.0;
    for (int i = 1; i + 1 < n; ++i) {
        double ax = px[i] - px[0], ay = py[i] - py[0];
        double bx = px[i + 1] - px[0], by = py[i + 1] - py[0];
        acc += ax * by - ay * bx;
    }
    return 0.5 * fabs(acc);
}

double rubs_oracle_kernel(const double *a, double x1, double x2)
{
    double hs = a[1] / SQRT2, hd = a[3] / SQRT2;
    double area = clipped_area(x1 - 0.5 * a[0], x1 + 0.5 * a[0],
                               x2 - 0.5 * a[2], x2 + 0.5 * a[2], hs, hd);
    return area / (a[0] * a[1] * a[2] * a[3]);
}

void rubs_oracle_kernel_many(const double *a, const double *x1, const double *x2,
                             int64_t n, double *out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = rubs_oracle_kernel(a, x1[i], x2[i]);
}

/* Per-pass prepared field: floored, divided by sqrt(m). */
typedef struct {
    const double *field; /* H*W*4 or 4 */
    int uniform;
    int H, W;
    double div;          /* sqrt(iterations) */
} field_t;

static void field_at(const field_t *F, int row, int col, double a[4])
{
    /* edge clamp (oracle.py:217-221 uses min/max on the original grid) */
    if (row < 0) row = 0;
    if (row > F->H - 1) row = F->H - 1;
    if (col < 0) col = 0;
    if (col > F->W - 1) col = F->W - 1;
    const double *src = F->uniform ? F->field : F->field + ((int64_t)row * F->W + col) * 4;
    for (int k = 0; k < 4; ++k) {
        double v = src[k] < 0.05 ? 0.05 : src[k];
        a[k] = v / F->div;
    }
}

static void support_radius(const double a[4], int *rx, int *ry)
{
    double diag = (a[1] + a[3]) / SQRT2;
    *rx = (int)ceil(0.5 * (a[0] + diag)) + 1;
    *ry = (int)ceil(0.5 * (a[2] + diag)) + 1;
}

/* Value of the pass-`p` signal at original-image pixel (row, col).
 * p == 0 is the zero-padded input image.  Recursive definition, used with
 * a per-call window cache for p >= 1 (see points API below). */
typedef struct {
    const double *f;
    int H, W;
    field_t F;
} ctx_t;

static double pass1_at(const ctx_t *C, int row, int col)
{
    double a[4];
    int rx, ry;
    field_at(&C->F, row, col, a);
    support_radius(a, &rx, &ry);
    int r0 = row - ry < 0 ? 0 : row - ry;
    int r1 = row + ry > C->H - 1 ? C->H - 1 : row + ry;
    int c0 = col - rx < 0 ? 0 : col - rx;
    int c1 = col + rx > C->W - 1 ? C->W - 1 : col + rx;
    double acc = 0.0;
    for (int r = r0; r <= r1; ++r)
        for (int c = c0; c <= c1; ++c) {
            double k = rubs_oracle_kernel(a, (double)(col - c), (double)(row - r));
            if (k != 0.0) acc += k * C->f[(int64_t)r * C->W + c];
        }
    return acc;
}

/* Global per-pass support radius (oracle.py:200-203). */
static void global_radius(const field_t *F, int *grx, int *gry)
{
    int mx = 0, my = 0;
    int n = F->uniform ? 1 : F->H * F->W;
    for (int i = 0; i < n; ++i) {
        double a[4];
        field_at(F, F->uniform ? 0 : i / F->W, F->uniform ? 0 : i % F->W, a);
        int rx, ry;
        support_radius(a, &rx, &ry);
        if (rx > mx) mx = rx;
        if (ry > my) my = ry;
    }
    *grx = mx;
    *gry = my;
}

/* Pass-p value at (row,col), recursion on windows.  For p >= 2 each
 * level materialises its window (cost ~ support^2 per level value). */
static double passp_at(const ctx_t *C, int p, int row, int col, int grx, int gry)
{
    if (p == 1) return pass1_at(C, row, col);
    /* pass p output at (row,col): sum over support of pass p-1 values.
     * Pass p-1 values exist on the canvas extended by (iterations - (p-1))
     * radii; beyond it they are zero.  We evaluate them directly. */
    double a[4];
    int rx, ry;
    field_at(&C->F, row, col, a);
    support_radius(a, &rx, &ry);
    double acc = 0.0;
    for (int r = row - ry; r <= row + ry; ++r)
        for (int c = col - rx; c <= col + rx; ++c) {
            double k = rubs_oracle_kernel(a, (double)(col - c), (double)(row - r));
            if (k == 0.0) continue;
            acc += k * passp_at(C, p - 1, r, c, grx, gry);
        }
    return acc;
}

/* Exact filter output at a list of pixels (pts = [row, col] pairs, int64).
 * iterations >= 1.  Cost per point ~ support^(2*iterations). */
int rubs_oracle_points(const double *f, int H, int W, const double *field, int uniform,
                       int iterations, const int64_t *pts, int64_t npts, double *out)
{
    if (iterations < 1) return 1;
    ctx_t C;
    C.f = f; C.H = H; C.W = W;
    C.F.field = field; C.F.uniform = uniform; C.F.H = H; C.F.W = W;
    C.F.div = sqrt((double)iterations);
    int grx = 0, gry = 0;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < npts; ++i) {
        int row = (int)pts[2 * i], col = (int)pts[2 * i + 1];
        out[i] = passp_at(&C, iterations, row, col, grx, gry);
    }
    return 0;
}

/* Full dense filter (small images): the reference's dense_convolve output.
 * For iterations > 1 intermediate passes are computed on canvases extended
 * by the global per-pass radius, exactly like oracle.py:205-241. */
int rubs_oracle_dense(const double *f, int H, int W, const double *field, int uniform,
                      int iterations, double *out)
{
    if (iterations < 1) return 1;
    field_t F;
    F.field = field; F.uniform = uniform; F.H = H; F.W = W;
    F.div = sqrt((double)iterations);
    int grx, gry;
    global_radius(&F, &grx, &gry);

    const double *cur = f;
    double *buf = NULL;
    int ch = H, cw = W, top = 0, left = 0;
    for (int p = 0; p < iterations; ++p) {
        int remain = iterations - 1 - p;
        int oh = H + 2 * gry * remain, ow = W + 2 * grx * remain;
        int otop = gry * remain, oleft = grx * remain;
        double *o = (remain == 0) ? out : (double *)malloc(sizeof(double) * (size_t)oh * ow);
        if (!o) return 2;
#pragma omp parallel for schedule(dynamic, 1)
        for (int i = 0; i < oh; ++i) {
            int yi = i - otop;
            for (int j = 0; j < ow; ++j) {
                int xi = j - oleft;
                double a[4];
                int rx, ry;
                field_at(&F, yi, xi, a);
                support_radius(a, &rx, &ry);
                int r0 = yi - ry + top, r1 = yi + ry + top;
                int c0 = xi - rx + left, c1 = xi + rx + left;
                if (r0 < 0) r0 = 0;
                if (r1 > ch - 1) r1 = ch - 1;
                if (c0 < 0) c0 = 0;
                if (c1 > cw - 1) c1 = cw - 1;
                double acc = 0.0;
                for (int r = r0; r <= r1; ++r)
                    for (int c = c0; c <= c1; ++c) {
                        double k = rubs_oracle_kernel(a, (double)(xi - (c - left)),
                                                      (double)(yi - (r - top)));
                        if (k != 0.0) acc += k * cur[(int64_t)r * cw + c];
                    }
                o[(int64_t)i * ow + j] = acc;
            }
        }
        if (buf) free(buf);
        buf = (remain == 0) ? NULL : o;
        cur = o;
        ch = oh; cw = ow; top = otop; left = oleft;
    }
    return 0;
}
