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
constexpr double kScaleFloor = 0.05;           // engine.py:58
constexpr double kQuarter = 0.7853981633974483;  // 0.25 * math.pi, solver.py:310
constexpr double kPi = 3.141592653589793;
// 1.5 * 2^52: adding it with round-toward-minus-infinity floors any |y| < 2^51.
constexpr double kFloorMagic = 6755399441055744.0;

// status flags (bit set -> error class)
constexpr unsigned kFlagFieldNonFinite = 1u;   // engine.py:214-215 -> ValueError
constexpr unsigned kFlagParamInvalid = 2u;     // solver.py:298-303 -> ValueError
constexpr unsigned kFlagOutOfGrid = 4u;        // solver.py:304-307 -> OutOfGrid
constexpr unsigned kFlagRegionTooLarge = 8u;   // halo beyond the on-chip region capacity

struct Status {
  unsigned int flags;
  unsigned int pad;
  unsigned long long guard_bits;  // max |plane| over all tiles, as IEEE bits
  int gm[4];                      // global margins left, right, below, above
};

// Where the per-pixel scale-vector comes from.
struct FieldSpec {
  int mode;  // 0: (FH, FW, 4) f64 field; 1: uniform; 2: (size, elong, orient) + LUT
  const double *a;
  int64_t ld;  // mode 0 row stride in pixels
  double u[4];
  const void *ps, *pr, *pt;
  int pdt;  // 0 f32, 1 f64
  int64_t pld;
  const double *lut;  // (n_rho, n_phi, 4)
  int n_rho, n_phi;
  double rho_max, log_rho_max;
  int FH, FW;  // field grid, edge-clamped (np.pad mode="edge", engine.py:306-314)
  double div;  // sqrt(iterations), engine.py:293
  int scaled;  // iterations > 1
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

__device__ __forceinline__ double load_scalar(const void *p, int dt, int64_t i) {
  return dt ? __ldg(static_cast<const double *>(p) + i)
            : static_cast<double>(__ldg(static_cast<const float *>(p) + i));
}

// numpy float floor-divide for b > 0 (npy_divmod): fmod, exact quotient,
// snap to the nearest integer.  Used for the quarter index, solver.py:311.
__device__ __forceinline__ double np_floordiv_pos(double a, double b) {
  double mod = fmod(a, b);
  double div = __ddiv_rn(__dsub_rn(a, mod), b);
  if (mod != 0.0 && ((b < 0.0) != (mod < 0.0))) div = __dsub_rn(div, 1.0);
  double fd;
  if (div != 0.0) {
    fd = floor(div);
    if (__dsub_rn(div, fd) > 0.5) fd = __dadd_rn(fd, 1.0);
  } else {
    fd = copysign(0.0, a / b);
  }
  return fd;
}

// solver.lookup_many (solver.py:308-335) for one pixel; validation flags per
// solver.py:298-307.  Arithmetic order follows numpy's evaluation order
// with FMA contraction disabled, so the result is the reference's bit for
// bit up to libm differences in log/sqrt.
__device__ __forceinline__ void lut_map(const FieldSpec &F, double s, double rho, double th,
                                        double a[4], unsigned &flags) {
  if (!(s > 0.0) || !isfinite(s)) flags |= kFlagParamInvalid;
  if (!(rho >= 1.0) || !isfinite(rho)) flags |= kFlagParamInvalid;
  if (!(th >= 0.0 && th < kPi)) flags |= kFlagParamInvalid;
  if (rho > __dmul_rn(F.rho_max, 1.0 + 1e-12)) flags |= kFlagOutOfGrid;
  // keep going with sane values so no NaN reaches the indexing below
  if (!(s > 0.0) || !isfinite(s)) s = 1.0;
  if (!(rho >= 1.0) || !isfinite(rho)) rho = 1.0;
  if (!(th >= 0.0 && th < kPi)) th = 0.0;
  rho = fmin(rho, F.rho_max);
  double qd = np_floordiv_pos(th, kQuarter);
  int q = (int)qd;
  if (q > 3) q = 3;
  double phi = __dsub_rn(th, __dmul_rn((double)q, kQuarter));
  const int nr = F.n_rho, np_ = F.n_phi;
  double u = __dmul_rn(__ddiv_rn(log(rho), F.log_rho_max), (double)(nr - 1));
  double v = __dsub_rn(__dmul_rn(__ddiv_rn(phi, kQuarter), (double)np_), 0.5);
  u = fmin(fmax(u, 0.0), (double)(nr - 1));
  v = fmin(fmax(v, 0.0), (double)(np_ - 1));
  int i0 = (int)u;
  if (i0 > nr - 2) i0 = nr - 2;
  int j0 = (int)v;
  if (j0 > np_ - 2) j0 = np_ - 2;
  double fu = __dsub_rn(u, (double)i0), fv = __dsub_rn(v, (double)j0);
  double gu = __dsub_rn(1.0, fu), gv = __dsub_rn(1.0, fv);
  const double *e00 = F.lut + ((int64_t)i0 * np_ + j0) * 4;
  const double *e10 = e00 + (int64_t)np_ * 4;
  const double *e01 = e00 + 4;
  const double *e11 = e10 + 4;
  double ss = sqrt(s);
  double mix[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double t = __dmul_rn(__dmul_rn(__ldg(e00 + k), gu), gv);
    t = __dadd_rn(t, __dmul_rn(__dmul_rn(__ldg(e10 + k), fu), gv));
    t = __dadd_rn(t, __dmul_rn(__dmul_rn(__ldg(e01 + k), gu), fv));
    t = __dadd_rn(t, __dmul_rn(__dmul_rn(__ldg(e11 + k), fu), fv));
    mix[k] = t;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = __dmul_rn(mix[(k - q + 4) & 3], ss);
}

// Raw (un-floored) scale-vector at field cell (fr, fc), already clamped.
__device__ __forceinline__ void field_raw(const FieldSpec &F, int fr, int fc, double a[4],
                                          unsigned &flags) {
  if (F.mode == 0) {
    const double2 *p = reinterpret_cast<const double2 *>(F.a + ((int64_t)fr * F.ld + fc) * 4);
    double2 lo = __ldg(p), hi = __ldg(p + 1);
    a[0] = lo.x; a[1] = lo.y; a[2] = hi.x; a[3] = hi.y;
    if (!(isfinite(a[0]) && isfinite(a[1]) && isfinite(a[2]) && isfinite(a[3])))
      flags |= kFlagFieldNonFinite;
  } else if (F.mode == 1) {
    a[0] = F.u[0]; a[1] = F.u[1]; a[2] = F.u[2]; a[3] = F.u[3];
  } else {
    int64_t i = (int64_t)fr * F.pld + fc;
    lut_map(F, load_scalar(F.ps, F.pdt, i), load_scalar(F.pr, F.pdt, i),
            load_scalar(F.pt, F.pdt, i), a, flags);
  }
}

// Floored and pass-scaled scale-vector for lattice pixel (n1, n2):
// a <- max(a, 0.05) / sqrt(m)   (engine.py:292-293, floor first).
__device__ __forceinline__ void field_at(const FieldSpec &F, int n1, int n2, double a[4],
                                         unsigned &flags) {
  int fc = min(max(n1, 0), F.FW - 1);
  int fr = min(max(n2, 0), F.FH - 1);
  field_raw(F, fr, fc, a, flags);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double v = fmax(a[k], kScaleFloor);
    if (!(a[k] == a[k])) v = kScaleFloor;  // NaN already flagged
    a[k] = F.scaled ? __ddiv_rn(v, F.div) : v;
  }
}

// Per-pixel read extents relative to the pixel, engine.py:219-229, 247-262:
// lo1 = tau1 - a1 - p2, hi1 = tau1 + p4, lo2 = tau2 - a3 - p2 - p4, hi2 = tau2.
// Returned as the integer margins max(0, ceil(-lo)+2), max(0, ceil(hi)+2).
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

// floor(x + 0.5) split: m (int) and residual d = m - x (zp.py:204-210).
__device__ __forceinline__ void lattice_split(double x, int &m, double &d) {
  double y = __dadd_rn(x, 0.5);
  double t = __dadd_rd(y, kFloorMagic);
  m = __double2loint(t);
  d = __dsub_rn(__dsub_rn(t, kFloorMagic), x);
}

// One ZP read F(x) * 8 at the vertex whose nearest lattice point is the
// plane element S[c] and residual (d1, d2).  The 4 x 7 quadratic table of
// zp.py (exact multiples of 1/8) folds into one canonical
// wedge: the partition q (zp.py:82-86) only decides which axis is "major"
// (q in {0,3}: x, else y) and the sign of the major residual; the seven
// taps are then centre, the two major neighbours N (-sign) / P (+sign),
// the two minor neighbours, and the two corners on the N side.
__device__ __forceinline__ double zp_read8(const double *__restrict__ S, int c, int pitch,
                                           double d1, double d2) {
  const bool gp = d1 >= -d2;  // d1 + d2 >= 0
  const bool gm = d1 >= d2;   // d1 - d2 >= 0
  const bool xmaj = (gp == gm);
  const int sA = xmaj ? (d1 >= 0.0 ? 1 : -1) : (d2 > 0.0 ? pitch : -pitch);
  const int sB = xmaj ? pitch : 1;
  const double u = xmaj ? fabs(d1) : fabs(d2);
  const double v = xmaj ? d2 : d1;
  const double g0 = S[c];
  const double N = S[c - sA];
  const double P = S[c + sA];
  const double Bm = S[c - sB];
  const double Bp = S[c + sB];
  const double Cm = S[c - sA - sB];
  const double Cp = S[c - sA + sB];
  const double sBv = Bm + Bp, dBv = Bm - Bp, sC = Cm + Cp, dC = Cm - Cp;
  const double A0 = fma(4.0, g0, N + P) + sBv;
  const double L1 = N - P;
  const double Caa2 = fma(2.0, P - g0, sC - sBv);
  const double Cab4 = dC - dBv;
  const double Cbb2 = fma(-2.0, g0 + N, sC + sBv);
  const double u2 = u + u, v2 = v + v;
  const double i1 = fma(u, Caa2, fma(2.0, L1, v2 * Cab4));
  const double i2 = fma(v, Cbb2, dBv + dBv);
  return fma(u2, i1, fma(v2, i2, A0));
}

}  // namespace rubs
