// rubs_device.cuh -- device-side building blocks of the B200 filter path.
//
// Everything here is fp64: the finite-difference stage recovers O(1) values
// from running sums of magnitude O(L^4) by cancellation (SURVEY.md §0 fact
// 10), so neither the plane nor the interpolation weights survive fp32.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rubs {

constexpr double kSqrt2 = 1.4142135623730951;
constexpr double kInvSqrt2 = 0.70710678118654752440;
constexpr double kScaleFloor = 0.05;             // engine.py:58
constexpr double kQuarter = 0.7853981633974483;  // 0.25 * math.pi, solver.py:310
constexpr double kPi = 3.141592653589793;
// 1.5 * 2^52: adding it with round-toward-minus-infinity floors any |y| < 2^51.
constexpr double kFloorMagic = 6755399441055744.0;

// field modes
constexpr int kModeField = 0;    // (FH, FW, 4) float64 array
constexpr int kModeUniform = 1;  // one (4,) vector
constexpr int kModeLut = 2;      // (size, elongation, orientation) float64 + LUT
constexpr int kModeLut32 = 3;    // same, float32 parameters

// status flags (bit set -> error class)
constexpr unsigned kFlagFieldNonFinite = 1u;  // engine.py:214-215 -> ValueError
constexpr unsigned kFlagParamInvalid = 2u;    // solver.py:298-303 -> ValueError
constexpr unsigned kFlagOutOfGrid = 4u;       // solver.py:304-307 -> OutOfGrid
constexpr unsigned kFlagRegionTooLarge = 8u;  // halo beyond the on-chip region capacity
// Not an error: some pixel's OWN minimal region already exceeds the float64
// precision budget w L4 (a "needle" kernel: three floored widths next to a
// long one), so its result may be accurate to ~1e-8 only.
// Reported through rubs_b200_precision_limited().
constexpr unsigned kFlagPrecisionLimited = 64u;

struct Status {
  unsigned int flags;
  unsigned int guard_hi;          // max over planes of the high word of |g| (IEEE)
  unsigned long long guard_bits;  // same for the global-canvas path, full bits
  int gm[4];                      // global margins left, right, below, above
  int ovf_count;                  // tiles deferred to the large-smem launch
  int pix_count;                  // pixels deferred to the per-pixel pass
  unsigned long long smax_bits;   // max LUT size parameter (bits of a positive double)
  int w2_count;                   // tiles listed for the primary kernel's stage 2
  int w2_next;                    // stage 2's take counter
};

// A tile deferred by the primary launch (its regions exceed the primary
// configuration's shared memory): tile index (32-pixel grid), the read
// margins (left, right, below, above) and max 1/(a1 a2 a3 a4) over the
// deferred cells, and which 8x8 cells are deferred -- the other cells of the
// tile were computed by the primary launch with their own (smaller,
// better-conditioned) regions and must not be overwritten.
struct OvfRec {
  int tile;
  int m[4];
  float w;
  unsigned mask;  // the tile's 8x8 cells (bit cy * 4 + cx) that need the overflow pass
};

// Where the per-pixel scale-vector comes from.
struct FieldSpec {
  int mode;
  const double *a;
  int64_t ld;  // mode 0 row stride in pixels
  double u[4];
  const void *ps, *pr, *pt;
  int pdt;  // 0 f32, 1 f64
  int64_t pld;
  const double *lut;  // (n_rho, n_phi, 4)
  const float *lut32;  // the same in float32 (planning bounds)
  int n_rho, n_phi;
  double rho_max, log_rho_max, inv_log_rho_max;
  double phi_scale;  // n_phi / (pi / 4)
  double lut_amax;   // largest component of any table entry (canvas bounds)
  double rho_lim;  // rho_max * (1 + 1e-12)
  int FH, FW;      // field grid, edge-clamped (np.pad mode="edge", engine.py:306-314)
  int fr_off;      // global row of the first row held in the arrays (row bands)
  double div;      // sqrt(iterations), engine.py:293
  int scaled;      // iterations > 1
};

// Input image of a pass: img[r, c] sits at lattice (col0 + c, row0 + r).
struct ImageSpec {
  const void *f;
  int dt;  // 0 f32, 1 f64
  int64_t ld;
  int h, w;
  int col0, row0;
};

// Output pixel domain of a pass: pixel (x, y) of the domain is lattice
// (pc_lo + x, pr_lo + y); result stored at out[y * ld_out + x].
struct DomainSpec {
  int pc_lo, pr_lo, pw, ph;
  double *out;
  int64_t ld_out;
};

template <int DT>
__device__ __forceinline__ double load_px(const void *p, int64_t i) {
  if constexpr (DT == 1)
    return __ldg(static_cast<const double *>(p) + i);
  else
    return static_cast<double>(__ldg(static_cast<const float *>(p) + i));
}

__device__ __forceinline__ double load_scalar(const void *p, int dt, int64_t i) {
  return dt ? __ldg(static_cast<const double *>(p) + i)
            : static_cast<double>(__ldg(static_cast<const float *>(p) + i));
}

__device__ __forceinline__ double dabs(double x) {  // bit op, keeps the fp64 pipe free
  return __hiloint2double(__double2hiint(x) & 0x7fffffff, __double2loint(x));
}

// numpy float floor-divide for the quarter index (solver.py:311):
// q = k with k * quarter <= theta < (k + 1) * quarter in exact arithmetic
// (npy_divmod semantics for theta >= 0), decided with exact FMA residuals.
__device__ __forceinline__ int quarter_index(double th) {
  double k = floor(th * (1.0 / kQuarter));
  if (fma(-k, kQuarter, th) < 0.0) k -= 1.0;
  else if (fma(-(k + 1.0), kQuarter, th) >= 0.0) k += 1.0;
  int q = (int)k;
  return q > 3 ? 3 : (q < 0 ? 0 : q);
}

// log(x) for finite x >= 1 (the LUT's log rho, solver.py:318): table +
// short series instead of the general libm routine (~20 instead of ~85
// instructions).  x = 2^e m, m in [1, 2); c = the centre of m's 1/128
// bucket, r = m/c - 1 (|r| <= 2^-8 + 2^-52), log m = log c + log1p(r) with
// log1p to degree 6 (truncation < 3e-18).  Error <= ~3e-16 absolute,
// the order of libm's.  g_logtab[i] = (1/c_i, log c_i), filled on the host.
__device__ double2 g_logtab[128];

__device__ __forceinline__ double log_ge1(double x) {
  const int hi = __double2hiint(x);
  const int e = (hi >> 20) - 1023;
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, __double2loint(x));
  const double2 t = g_logtab[(hi >> 13) & 127];
  const double r = __fma_rn(m, t.x, -1.0);
  double q = __fma_rn(r, -1.0 / 6.0, 0.2);
  q = __fma_rn(r, q, -0.25);
  q = __fma_rn(r, q, 1.0 / 3.0);
  q = __fma_rn(r, q, -0.5);
  const double l1p = __fma_rn(__dmul_rn(r, r), q, r);
  return __fma_rn((double)e, 0.6931471805599453, __dadd_rn(t.y, l1p));
}

// solver.lookup_many (solver.py:308-335) for one pixel; validation flags per
// solver.py:298-307.
__device__ __forceinline__ void lut_map(const FieldSpec &F, double s, double rho, double th,
                                        double a[4], unsigned &flags) {
  const bool s_ok = (s > 0.0) && (s < INFINITY);
  const bool r_ok = (rho >= 1.0) && (rho < INFINITY);
  const bool t_ok = (th >= 0.0) && (th < kPi);
  if (!(s_ok && r_ok && t_ok)) flags |= kFlagParamInvalid;
  if (rho > F.rho_lim) flags |= kFlagOutOfGrid;
  if (!s_ok) s = 1.0;
  if (!r_ok) rho = 1.0;
  if (!t_ok) th = 0.0;
  rho = fmin(rho, F.rho_max);
  const int q = quarter_index(th);
  const double phi = __dsub_rn(th, __dmul_rn((double)q, kQuarter));
  const int nr = F.n_rho, np_ = F.n_phi;
  // explicit roundings: identical bits wherever this is inlined
  double u = __dmul_rn(__dmul_rn(log_ge1(rho), F.inv_log_rho_max), (double)(nr - 1));
  // n_phi / quarter is a runtime division: hoisted to the host (F.phi_scale,
  // the same correctly rounded quotient)
  double v = __dsub_rn(__dmul_rn(phi, F.phi_scale), 0.5);
  u = fmin(fmax(u, 0.0), (double)(nr - 1));
  v = fmin(fmax(v, 0.0), (double)(np_ - 1));
  int i0 = min((int)u, nr - 2);
  int j0 = min((int)v, np_ - 2);
  const double fu = __dsub_rn(u, (double)i0), fv = __dsub_rn(v, (double)j0);
  const double gu = __dsub_rn(1.0, fu), gv = __dsub_rn(1.0, fv);
  const double w00 = __dmul_rn(gu, gv), w10 = __dmul_rn(fu, gv), w01 = __dmul_rn(gu, fv),
               w11 = __dmul_rn(fu, fv);
  // F.lut holds four copies of the table, copy q already rolled by q
  // quarter turns (solver.py:286, 332-334), so no per-pixel selects
  const double2 *e00 = reinterpret_cast<const double2 *>(
      F.lut + ((int64_t)q * nr * np_ + (int64_t)i0 * np_ + j0) * 4);
  const double2 *e01 = e00 + 2;
  const double2 *e10 = e00 + (int64_t)np_ * 2;
  const double2 *e11 = e10 + 2;
  const double ss = sqrt(s);
  {
    const double2 A = __ldg(e00), B = __ldg(e10), C = __ldg(e01), Dd = __ldg(e11);
    a[0] = __dmul_rn(__fma_rn(A.x, w00, __fma_rn(B.x, w10, __fma_rn(C.x, w01, __dmul_rn(Dd.x, w11)))), ss);
    a[1] = __dmul_rn(__fma_rn(A.y, w00, __fma_rn(B.y, w10, __fma_rn(C.y, w01, __dmul_rn(Dd.y, w11)))), ss);
  }
  {
    const double2 A = __ldg(e00 + 1), B = __ldg(e10 + 1), C = __ldg(e01 + 1), Dd = __ldg(e11 + 1);
    a[2] = __dmul_rn(__fma_rn(A.x, w00, __fma_rn(B.x, w10, __fma_rn(C.x, w01, __dmul_rn(Dd.x, w11)))), ss);
    a[3] = __dmul_rn(__fma_rn(A.y, w00, __fma_rn(B.y, w10, __fma_rn(C.y, w01, __dmul_rn(Dd.y, w11)))), ss);
  }
}

#ifndef RUBS_MARGIN_SLACK
#define RUBS_MARGIN_SLACK 0
#endif
// Planning bounds of one LUT-mapped pixel in float32 (the primary kernel's
// large-kernel tiles, which are deferred anyway: their exact mapping is
// done by the pass that computes them).  Validation flags and the quarter
// index exactly as lut_map; the log, blend and sqrt in float32 from the same
// table cells (the blend is continuous across cells, so an f32 cell index
// differing at a cell edge changes nothing).  Component error <= ~1e-6
// relative: the margins from an extent inflated by (1 + 2e-5) + 2e-3 and
// w x (1 + 1e-4) bound the exact ones (pixel_margins_fast, 1 / prod a).
__device__ __forceinline__ void lut_bounds_f32(const FieldSpec &F, double s, double rho, double th,
                                               int4 &m, float &w, unsigned &flags) {
  const bool s_ok = (s > 0.0) && (s < INFINITY);
  const bool r_ok = (rho >= 1.0) && (rho < INFINITY);
  const bool t_ok = (th >= 0.0) && (th < kPi);
  if (!(s_ok && r_ok && t_ok)) flags |= kFlagParamInvalid;
  if (rho > F.rho_lim) flags |= kFlagOutOfGrid;
  if (!s_ok) s = 1.0;
  if (!r_ok) rho = 1.0;
  if (!t_ok) th = 0.0;
  rho = fmin(rho, F.rho_max);
  const int q = quarter_index(th);
  const double phi = __dsub_rn(th, __dmul_rn((double)q, kQuarter));
  const int nr = F.n_rho, np_ = F.n_phi;
  float u = __logf((float)rho) * (float)F.inv_log_rho_max * (float)(nr - 1);
  float v = (float)phi * (float)F.phi_scale - 0.5f;
  u = fminf(fmaxf(u, 0.f), (float)(nr - 1));
  v = fminf(fmaxf(v, 0.f), (float)(np_ - 1));
  const int i0 = min((int)u, nr - 2), j0 = min((int)v, np_ - 2);
  const float fu = u - (float)i0, fv = v - (float)j0, gu = 1.f - fu, gv = 1.f - fv;
  const float w00 = gu * gv, w10 = fu * gv, w01 = gu * fv, w11 = fu * fv;
  const float4 *e00 = reinterpret_cast<const float4 *>(F.lut32) +
                      ((int64_t)q * nr * np_ + (int64_t)i0 * np_ + j0);
  const float4 *e10 = e00 + np_;
  const float ss = sqrtf((float)s);
  const float4 A = __ldg(e00), B = __ldg(e10), C = __ldg(e00 + 1), Dd = __ldg(e10 + 1);
  float a[4] = {(A.x * w00 + B.x * w10 + C.x * w01 + Dd.x * w11) * ss,
                (A.y * w00 + B.y * w10 + C.y * w01 + Dd.y * w11) * ss,
                (A.z * w00 + B.z * w10 + C.z * w01 + Dd.z * w11) * ss,
                (A.w * w00 + B.w * w10 + C.w * w01 + Dd.w * w11) * ss};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    a[k] = fmaxf(a[k], (float)kScaleFloor);
    if (F.scaled) a[k] = a[k] / (float)F.div;
  }
  const float d = (a[1] + a[3]) * 0.70710678f;
  const float hx = 0.5f * (a[0] + d) * (1.f + 2e-5f) + 2e-3f;
  const float hy = 0.5f * (a[2] + d) * (1.f + 2e-5f) + 2e-3f;
  const int fx = (int)floorf(hx), fy = (int)floorf(hy), k = RUBS_MARGIN_SLACK;
  m = make_int4(fx + 2 + k, fx + 1 + k, fy + 3 + k, fy + k);
  w = 1.0f / (a[0] * a[1] * a[2] * a[3]) * (1.f + 1e-4f);
}

template <int MODE>
__device__ __forceinline__ void field_raw(const FieldSpec &F, int fr, int fc, double a[4],
                                          unsigned &flags) {
  if constexpr (MODE == kModeField) {
    const double2 *p = reinterpret_cast<const double2 *>(F.a + ((int64_t)fr * F.ld + fc) * 4);
    const double2 lo = __ldg(p), hi = __ldg(p + 1);
    a[0] = lo.x; a[1] = lo.y; a[2] = hi.x; a[3] = hi.y;
    // NaN / inf <=> exponent all ones
    const bool bad = ((__double2hiint(a[0]) & 0x7ff00000) == 0x7ff00000) ||
                     ((__double2hiint(a[1]) & 0x7ff00000) == 0x7ff00000) ||
                     ((__double2hiint(a[2]) & 0x7ff00000) == 0x7ff00000) ||
                     ((__double2hiint(a[3]) & 0x7ff00000) == 0x7ff00000);
    if (bad) flags |= kFlagFieldNonFinite;
  } else if constexpr (MODE == kModeUniform) {
    a[0] = F.u[0]; a[1] = F.u[1]; a[2] = F.u[2]; a[3] = F.u[3];
  } else {
    constexpr int PDT = MODE == kModeLut ? 1 : 0;
    const int64_t i = (int64_t)fr * F.pld + fc;
    lut_map(F, load_px<PDT>(F.ps, i), load_px<PDT>(F.pr, i), load_px<PDT>(F.pt, i), a, flags);
  }
}

// Floored and pass-scaled scale-vector for lattice pixel (n1, n2):
// a <- max(a, 0.05) / sqrt(m)   (engine.py:292-293, floor first).
template <int MODE>
__device__ __forceinline__ void field_at(const FieldSpec &F, int n1, int n2, double a[4],
                                         unsigned &flags) {
  const int fc = min(max(n1, 0), F.FW - 1);
  const int fr = min(max(n2, 0), F.FH - 1) - F.fr_off;
  field_raw<MODE>(F, fr, fc, a, flags);
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = fmax(a[k], kScaleFloor);  // fmax(NaN, x) = x; NaN flagged
  if (F.scaled) {  // uniform branch: the divisions only for iterated passes
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = __ddiv_rn(a[k], F.div);
  }
}

// LUT modes with the three parameters already loaded (the primary kernel
// issues all of a thread's parameter loads up front): lut_map, floor, scale
// exactly as field_at.
__device__ __forceinline__ void field_from_params(const FieldSpec &F, double s, double r, double t,
                                                  double a[4], unsigned &flags) {
  lut_map(F, s, r, t, a, flags);
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = fmax(a[k], kScaleFloor);
  if (F.scaled) {
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = __ddiv_rn(a[k], F.div);
  }
}

// Runtime-mode dispatch (pre-pass kernels, not on the hot path).
__device__ __forceinline__ void field_at_rt(const FieldSpec &F, int n1, int n2, double a[4],
                                            unsigned &flags) {
  if (F.mode == kModeField) field_at<kModeField>(F, n1, n2, a, flags);
  else if (F.mode == kModeUniform) field_at<kModeUniform>(F, n1, n2, a, flags);
  else if (F.mode == kModeLut) field_at<kModeLut>(F, n1, n2, a, flags);
  else field_at<kModeLut32>(F, n1, n2, a, flags);
}

// Per-pixel read extents relative to the pixel, engine.py:219-229, 247-262:
// lo1 = tau1 - a1 - p2, hi1 = tau1 + p4, lo2 = tau2 - a3 - p2 - p4, hi2 = tau2,
// returned as the integer margins max(0, ceil(-lo)+2), max(0, ceil(hi)+2).
// Evaluated in the reference's operation order without FMA contraction, so
// the iterated-pass canvases match engine.py exactly.
__device__ __forceinline__ int4 pixel_margins(const double a[4]) {
  double p2 = __ddiv_rn(a[1], kSqrt2), p4 = __ddiv_rn(a[3], kSqrt2);
  double t1 = __dsub_rn(__dadd_rn(__dmul_rn(0.5, a[0]), __dmul_rn(0.5, __dsub_rn(p2, p4))), 0.5);
  double t2 = __dsub_rn(__dadd_rn(__dmul_rn(0.5, a[2]), __dmul_rn(0.5, __dadd_rn(p2, p4))), 1.5);
  int4 m;
  m.x = max(0, (int)ceil(-__dsub_rn(__dsub_rn(t1, a[0]), p2)) + 2);
  m.y = max(0, (int)ceil(__dadd_rn(t1, p4)) + 2);
  m.z = max(0, (int)ceil(-__dsub_rn(__dsub_rn(__dsub_rn(t2, a[2]), p2), p4)) + 2);
  m.w = max(0, (int)ceil(t2) + 2);
  return m;
}

// Tight read margins from the half-extents of the vertex cloud.  With
// t1, t2 of pixel_fd_t, vertex x - n1 lies in [-hx - 1/2, hx - 1/2] and
// y - n2 in [-hy - 3/2, hy - 3/2] (hx = (a1 + (a2 + a4)/sqrt2) / 2, hy the
// same with a3); the nearest lattice point is within 1/2 of a vertex and the
// ZP taps within 1 of it, so the taps span columns n1 - floor(hx) - 2 ..
// n1 + floor(hx) + 1 and rows n2 - floor(hy) - 3 .. n2 + floor(hy).  The
// 1e-6 covers the rounding of the vertex arithmetic.
#ifndef RUBS_MARGIN_SLACK
#define RUBS_MARGIN_SLACK 0
#endif
__device__ __forceinline__ int4 margins_from_extent(double hx, double hy) {
  const int fx = (int)floor(hx + 1e-6), fy = (int)floor(hy + 1e-6), k = RUBS_MARGIN_SLACK;
  return make_int4(fx + 2 + k, fx + 1 + k, fy + 3 + k, fy + k);
}

__device__ __forceinline__ int4 pixel_margins_fast(const double a[4]) {
  const double d = (a[1] + a[3]) * kInvSqrt2;
  return margins_from_extent(0.5 * (a[0] + d), 0.5 * (a[2] + d));
}

// Nearest lattice point m of x and residual d = m - x (zp.py:204-210).  The
// reference takes m = floor(x + 0.5); at exact half-integers rounding to
// nearest-even may pick the other neighbour (d = -1/2 instead of +1/2), which
// reads the same value of the C1 spline, so one rounding add suffices.
__device__ __forceinline__ void lattice_split(double x, int &m, double &d) {
  const double t = __dadd_rn(x, kFloorMagic);
  m = __double2loint(t);
  d = __dsub_rn(__dsub_rn(t, kFloorMagic), x);
}

}  // namespace rubs
