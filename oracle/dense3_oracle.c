/*
 * TEST INFRASTRUCTURE ONLY -- parity oracle, never part of the product path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.
 *
 * Exact dense filter with the three-direction (N=3) radially-uniform box
 * spline: directions u_k at (k-1) pi / 3, i.e. 0, 60 and 120 degrees
 * (reference: pkg/src/rubs/geometry.py:76-81 direction_vectors(3); the
 * kernel is the convolution of three centred unit-mass boxes of widths
 * a_k along u_k; covariance sum a_k^2/12 u_k u_k^T,
 * geometry.py:102-106).  The reference has no N=3 filter (SURVEY.md §0
 * fact 6); its only N=3 capability is the spectral sampler
 * oracle.synthesize_kernel (oracle.py:87-167), which pins this kernel in
 * tests/test_oracle_n3.py.
 *
 * Kernel value, by a route independent of the GPU's (which slices along
 * u1): box(u1) * box(u2) is the uniform density 1 / (a1 a2 sin 60) on the
 * parallelogram Q = {al u1 + be u2 : |al| <= a1/2, |be| <= a2/2}; sweeping
 * it along u3 gives
 *     beta(x) = |{ t in [-a3/2, a3/2] : x - t u3 in Q }| / (a1 a2 a3 sin 60).
 * With p(t) = x - t u3:  be(t) = 2 x2 / sqrt3 - t,  al(t) = x1 - x2 / sqrt3 + t.
 *
 * Dense filter: out(n) = sum_m beta_{a(n)}(n - m) cur(m), zero outside the
 * image; the scale field is floored at 0.05 and divided by sqrt(m); for
 * m > 1 passes the intermediate lives on canvases extended by the global
 * support radius with the field edge-clamped -- the semantics of the N=4
 * path (engine.py:292-323, oracle.py:200-241) carried over to N=3.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define SQRT3 1.7320508075688772
#define SIN60 0.8660254037844386

double rubs_oracle3_kernel(const double *a, double x1, double x2)
{
    const double al0 = x1 - x2 / SQRT3, be0 = 2.0 * x2 / SQRT3;
    double lo = -0.5 * a[2], hi = 0.5 * a[2];
    /* |al0 + t| <= a1/2 */
    double l = -0.5 * a[0] - al0, h = 0.5 * a[0] - al0;
    if (l > lo) lo = l;
    if (h < hi) hi = h;
    /* |be0 - t| <= a2/2 */
    l = be0 - 0.5 * a[1];
    h = be0 + 0.5 * a[1];
    if (l > lo) lo = l;
    if (h < hi) hi = h;
    if (hi <= lo) return 0.0;
    return (hi - lo) / (a[0] * a[1] * a[2] * SIN60);
}

void rubs_oracle3_kernel_many(const double *a, const double *x1, const double *x2, int64_t n,
                              double *out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = rubs_oracle3_kernel(a, x1[i], x2[i]);
}

typedef struct {
    const double *field; /* H*W*3 or 3 */
    int uniform;
    int H, W;
    double div;
} field3_t;

static void field3_at(const field3_t *F, int row, int col, double a[3])
{
    if (row < 0) row = 0;
    if (row > F->H - 1) row = F->H - 1;
    if (col < 0) col = 0;
    if (col > F->W - 1) col = F->W - 1;
    const double *src = F->uniform ? F->field : F->field + ((int64_t)row * F->W + col) * 3;
    for (int k = 0; k < 3; ++k) {
        double v = src[k] < 0.05 ? 0.05 : src[k];
        a[k] = v / F->div;
    }
}

/* support half-extents: x <= a1/2 + (a2 + a3)/4, |y| <= (a2 + a3) sqrt3 / 4 */
static void support3(const double a[3], int *rx, int *ry)
{
    *rx = (int)ceil(0.5 * a[0] + 0.25 * (a[1] + a[2])) + 1;
    *ry = (int)ceil(0.25 * SQRT3 * (a[1] + a[2])) + 1;
}

static void global3(const field3_t *F, int *grx, int *gry)
{
    int mx = 0, my = 0;
    int64_t n = F->uniform ? 1 : (int64_t)F->H * F->W;
    for (int64_t i = 0; i < n; ++i) {
        double a[3];
        field3_at(F, F->uniform ? 0 : (int)(i / F->W), F->uniform ? 0 : (int)(i % F->W), a);
        int rx, ry;
        support3(a, &rx, &ry);
        if (rx > mx) mx = rx;
        if (ry > my) my = ry;
    }
    *grx = mx;
    *gry = my;
}

static double point3(const double *cur, int ch, int cw, int top, int left, const double a[3],
                     int yi, int xi)
{
    int rx, ry;
    support3(a, &rx, &ry);
    int r0 = yi - ry + top, r1 = yi + ry + top;
    int c0 = xi - rx + left, c1 = xi + rx + left;
    if (r0 < 0) r0 = 0;
    if (r1 > ch - 1) r1 = ch - 1;
    if (c0 < 0) c0 = 0;
    if (c1 > cw - 1) c1 = cw - 1;
    double acc = 0.0;
    for (int r = r0; r <= r1; ++r)
        for (int c = c0; c <= c1; ++c) {
            double k = rubs_oracle3_kernel(a, (double)(xi - (c - left)), (double)(yi - (r - top)));
            if (k != 0.0) acc += k * cur[(int64_t)r * cw + c];
        }
    return acc;
}

/* Full dense N=3 filter. */
int rubs_oracle3_dense(const double *f, int H, int W, const double *field, int uniform,
                       int iterations, double *out)
{
    if (iterations < 1) return 1;
    field3_t F;
    F.field = field; F.uniform = uniform; F.H = H; F.W = W;
    F.div = sqrt((double)iterations);
    int grx, gry;
    global3(&F, &grx, &gry);
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
        for (int i = 0; i < oh; ++i)
            for (int j = 0; j < ow; ++j) {
                double a[3];
                field3_at(&F, i - otop, j - oleft, a);
                o[(int64_t)i * ow + j] = point3(cur, ch, cw, top, left, a, i - otop, j - oleft);
            }
        if (buf) free(buf);
        buf = (remain == 0) ? NULL : o;
        cur = o;
        ch = oh; cw = ow; top = otop; left = oleft;
    }
    return 0;
}

/* One pass at a list of pixels (pts = [row, col] pairs): large images,
 * sampled checks. */
int rubs_oracle3_points(const double *f, int H, int W, const double *field, int uniform,
                        const int64_t *pts, int64_t npts, double *out)
{
    field3_t F;
    F.field = field; F.uniform = uniform; F.H = H; F.W = W;
    F.div = 1.0;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < npts; ++i) {
        int row = (int)pts[2 * i], col = (int)pts[2 * i + 1];
        double a[3];
        field3_at(&F, row, col, a);
        out[i] = point3(f, H, W, 0, 0, a, row, col);
    }
    return 0;
}

/*
 * Lattice (O(1)) mode of the N=3 filter, by brute force -- the independent
 * route for this repo's interpolated three-direction algorithm (DESIGN.md
 * §9b; off-grid running sums need interpolation).
 *
 * The image f = sum_m f[m] delta(x - m) is moved onto the triangular lattice
 * p(al, ga) = h (al u1 + ga u3) = h (al - ga/2, ga sqrt3/2) (origin at pixel
 * (0, 0)) by the adjoint of piecewise-linear interpolation -- each pixel's
 * value is split over the three corners of its lattice triangle with its
 * barycentric weights (mass and first moment kept):
 *     f_hex[p] = sum_m f[m] hat((m - p) / h),
 *     hat(d) = max(0, 1 - max(|da|, |dg|, |da - dg|)),  d = da u1 + dg u3.
 * The lattice filter is then the EXACT N=3 kernel applied to that delta
 * train:  out(n) = sum_p f_hex[p] beta_a(n)(n - p).
 * Here both sums are taken literally (O(support) per pixel); the product
 * path gets the same numbers in O(1) per pixel from running sums along the
 * three lattice directions.
 */
static double splat3(const double *f, int H, int W, double h, double px, double py)
{
    const double gh = SIN60 * h;
    const int c0 = (int)floor(px), r0 = (int)floor(py);
    double acc = 0.0;
    for (int r = r0; r <= r0 + 1; ++r)
        for (int c = c0; c <= c0 + 1; ++c) {
            if (r < 0 || r >= H || c < 0 || c >= W) continue;
            const double dg = (r - py) / gh, da = (c - px) / h + 0.5 * dg;
            double m = fabs(da);
            if (fabs(dg) > m) m = fabs(dg);
            if (fabs(da - dg) > m) m = fabs(da - dg);
            if (m < 1.0) acc += f[(int64_t)r * W + c] * (1.0 - m);
        }
    return acc;
}

/* f_hex at lattice indices (al, ga), n of them. */
void rubs_oracle3_splat(const double *f, int H, int W, double h, const int64_t *al,
                        const int64_t *ga, int64_t n, double *out)
{
    for (int64_t i = 0; i < n; ++i)
        out[i] = splat3(f, H, W, h, h * ((double)al[i] - 0.5 * (double)ga[i]),
                        SIN60 * h * (double)ga[i]);
}

int rubs_oracle3_lattice_points(const double *f, int H, int W, const double *field, int uniform,
                                double h, const int64_t *pts, int64_t npts, double *out)
{
    if (!(h > 0.0) || h > 1.0) return 1;
    field3_t F;
    F.field = field; F.uniform = uniform; F.H = H; F.W = W;
    F.div = 1.0;
    const double gh = SIN60 * h;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < npts; ++i) {
        const int Y = (int)pts[2 * i], X = (int)pts[2 * i + 1];
        double a[3];
        field3_at(&F, Y, X, a);
        int rx, ry;
        support3(a, &rx, &ry);
        const int64_t g0 = (int64_t)ceil((Y - ry) / gh), g1 = (int64_t)floor((Y + ry) / gh);
        double acc = 0.0;
        for (int64_t g = g0; g <= g1; ++g) {
            const double py = gh * (double)g;
            const int64_t a0 = (int64_t)ceil((X - rx) / h + 0.5 * g);
            const int64_t a1 = (int64_t)floor((X + rx) / h + 0.5 * g);
            for (int64_t al = a0; al <= a1; ++al) {
                const double px = h * ((double)al - 0.5 * (double)g);
                const double w = rubs_oracle3_kernel(a, X - px, Y - py);
                if (w != 0.0) acc += w * splat3(f, H, W, h, px, py);
            }
        }
        out[i] = acc;
    }
    return 0;
}
