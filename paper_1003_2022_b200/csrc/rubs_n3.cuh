// rubs_n3.cuh -- definitions shared by the two N=3 translation units:
// the exact row-profile filter (rubs_n3.cu) and the O(1) lattice mode
// (rubs_n3_lattice.cu).  Directions u1 = (1, 0), u2 = (1/2, sqrt3/2),
// u3 = (-1/2, sqrt3/2) in (column, row) coordinates (the reference's
// direction_vectors(3), geometry.py:76-81).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "rubs_device.cuh"

namespace rubs3 {

using namespace rubs;

constexpr double kInvSqrt3 = 0.5773502691896258;
constexpr double kQuarterSqrt3 = 0.4330127018922193;  // sqrt3 / 4
constexpr double kRoundMagic = 6755399441055744.0;     // 1.5 * 2^52: round to nearest
constexpr unsigned kFlagInfeasible = 16u;              // a_k^2 < 0: covariance out of reach

// field modes
constexpr int kM3Field = 0;     // (FH, FW, 3) float64
constexpr int kM3Uniform = 1;   // one (3,) vector
constexpr int kM3Params = 2;    // (size, elongation, orientation) float64
constexpr int kM3Params32 = 3;  // same, float32

struct Field3 {
  int mode;
  const double *a;
  int64_t ld;  // field row stride in pixels
  double u[3];
  const void *ps, *pr, *pt;
  int64_t pld;
  int FH, FW;  // field grid (edge-clamped on iterated canvases)
  int fr_off;  // global row of the first row held in the arrays (row bands)
  double div;  // sqrt(iterations)
  int scaled;
};

struct Status3 {
  unsigned flags;
  int rx, ry;  // global support radii (iterations > 1)
};

// (size, elongation, orientation) -> N=3 scales: C = sum_k a_k^2/12 u_k u_k^T
// solved in closed form (u1 = (1,0), u2 = (1/2, sqrt3/2), u3 = (-1/2, sqrt3/2)):
//   p1 = C11 - C22/3,  p2,3 = 2/3 C22 +- 2/sqrt3 C12,  a_k = sqrt(12 p_k).
// Validation as solver.lookup_many (solver.py:298-303); p_k < -1e-12 size is
// beyond the N=3 elongation bound -> Infeasible.
__device__ __forceinline__ void params_to_scales3(double s, double rho, double th, double a[3],
                                                  unsigned &flags) {
  const bool s_ok = (s > 0.0) && (s < INFINITY);
  const bool r_ok = (rho >= 1.0) && (rho < INFINITY);
  const bool t_ok = (th >= 0.0) && (th < kPi);
  if (!(s_ok && r_ok && t_ok)) {
    flags |= kFlagParamInvalid;
    s = 1.0;
    rho = 1.0;
    th = 0.0;
  }
  double sn, cs;
  sincos(th, &sn, &cs);
  const double inv = 1.0 / (1.0 + rho);
  const double big = s * rho * inv, small = s * inv;
  const double c11 = big * cs * cs + small * sn * sn;
  const double c22 = big * sn * sn + small * cs * cs;
  const double c12 = (big - small) * cs * sn;
  double p[3];
  p[0] = c11 - c22 * (1.0 / 3.0);
  p[1] = c22 * (2.0 / 3.0) + c12 * (2.0 * kInvSqrt3);
  p[2] = c22 * (2.0 / 3.0) - c12 * (2.0 * kInvSqrt3);
  const double tol = -1e-12 * s;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (p[k] < tol) flags |= kFlagInfeasible;
    a[k] = sqrt(12.0 * fmax(p[k], 0.0));
  }
}

// Floored, pass-scaled scales of lattice pixel (gx, gy); field edge-clamped.
template <int MODE>
__device__ __forceinline__ void scales3_at(const Field3 &F, int gx, int gy, double a[3],
                                           unsigned &flags) {
  const int c = min(max(gx, 0), F.FW - 1), r = min(max(gy, 0), F.FH - 1) - F.fr_off;
  if constexpr (MODE == kM3Field) {
    const double *p = F.a + ((int64_t)r * F.ld + c) * 3;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      a[k] = __ldg(p + k);
      if ((__double2hiint(a[k]) & 0x7ff00000) == 0x7ff00000) flags |= kFlagFieldNonFinite;
    }
  } else if constexpr (MODE == kM3Uniform) {
    a[0] = F.u[0];
    a[1] = F.u[1];
    a[2] = F.u[2];
  } else {
    const int64_t i = (int64_t)r * F.pld + c;
    const int dt = MODE == kM3Params ? 1 : 0;
    params_to_scales3(load_scalar(F.ps, dt, i), load_scalar(F.pr, dt, i),
                      load_scalar(F.pt, dt, i), a, flags);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double v = fmax(a[k], kScaleFloor);  // engine.py:292 (NaN -> flagged above)
    a[k] = F.scaled ? v / F.div : v;     // engine.py:293
  }
}

}  // namespace rubs3
