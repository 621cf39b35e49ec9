// rubs_n3_lattice.cu -- the O(1)-per-pixel "lattice" mode of the
// three-direction (N=3) box-spline filter on sm_100a (BASELINE.json config 3:
// "N=3 radially-uniform directions (0,60,120 deg, off-grid, needs
// interpolation)").
//
// The paper's O(1) algorithm realises the box spline as
// running sums along its directions followed by a 2^N-vertex finite
// difference.  60 and 120 degrees are off the pixel lattice, so "one needs to
// interpolate the image for implementing the associated running-sums"
// (PAPER.md:285, 662).  Here the image is moved ONCE onto the triangular
// lattice that contains all three directions,
//     p(al, ga) = h (al u1 + ga u3) = h (al - ga/2, ga sqrt3/2),
// by the adjoint of piecewise-linear interpolation (each pixel's value split
// over the corners of its lattice triangle: mass and first moments kept),
//     f_hex[p] = sum_m f[m] hat((m - p) / h),
// and everything after that is exact:
//   G  = triple running sum of f_hex along (1,0), (0,1), (1,1) in (al, ga),
//        i.e. the lattice vectors h u1, h u3, h u2 = h (u1 + u3);
//   F(y) = (h / sin60) Lin[G](y - h u2)  -- the continuous triple integral of
//        the f_hex delta train (the unit three-direction box spline of this
//        lattice is its linear "hat" element, centred at h u2);
//   out(n) = 1/(a1 a2 a3) sum_{s in {+-1}^3} s1 s2 s3 F(n + sum_k s_k a_k u_k/2).
// So out(n) = sum_p f_hex[p] beta_a(n)(n - p): the EXACT N=3 kernel applied to
// the resampled image (oracle/dense3_oracle.c rubs_oracle3_lattice_points
// takes that sum literally).  Cost per pixel: 8 vertices x 3 taps, whatever
// the kernel size.
//
// Arithmetic.  f_hex is quantised to 62-bit integers (scale 2^S per block of
// rows, from the block's max |f|) and the running sums are EXACT int128: no
// cancellation in the sums, no precision budget on the region size, and the
// result is independent of summation order.  Per pixel, G is re-based by the
// exact affine function through its base lattice point (the finite
// difference annihilates affine functions), so the 24 taps that reach
// floating point are small second-order quantities; the vertex coordinates
// are small offsets from the pixel's base point.
//
// Layout.  Output rows are cut into blocks of bp rows; block b's region (its
// pixels' supports, margin 2) is an NG x NA (ga, al) parallelogram of int128
// in HBM, restarted (exact).  Four kernels per pass: splat + running sum
// along al (one CTA per region row), running sum along ga (thread per
// column), along the diagonal (thread per diagonal), and the per-pixel
// gather with the fused (size, elongation, orientation) mapping.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rubs_b200.h"
#include "rubs_device.cuh"
#include "rubs_internal.h"
#include "rubs_n3.cuh"

using namespace rubs;
using namespace rubs3;
using rubs_internal::set_error;

namespace {

#define LAT_CUDA_TRY(expr)                                                           \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return set_error(RUBS_ECUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
  } while (0)

typedef __int128 i128;

constexpr double kSin60 = 0.8660254037844386;
constexpr unsigned kFlagImageNonFinite = 32u;  // integer running sums: no NaN/Inf to carry
constexpr int kQBits = 59;                     // |f_hex| 2^S < 4 max|f| 2^(59 - e) < 2^62

struct LatStatus {
  unsigned flags;
  int rx, ry;  // support half-extents (pixels, +1), max over the field
};

// One pass: output rows [y0, y0 + ph) cut into nb blocks of bp rows; block
// b's region is NG lattice rows from ga = glo(b) by NA columns from
// al = alo(b).
struct LatGeom {
  double h, gh, inv_h, inv_gh;  // spacing along u1, row pitch h sin60, inverses
  int x_lo;                     // global column of the region's left margin
  int y0, ph;                   // first output row (global), output rows
  int bp, nb;                   // rows per block, blocks
  int NG, NA;                   // region rows / columns, the same for every block
  int RY;                       // row margin
};

__host__ __device__ __forceinline__ int blk_glo(const LatGeom &g, int b) {
  return (int)floor((double)(g.y0 + b * g.bp - g.RY) / g.gh) - 2;
}
__host__ __device__ __forceinline__ int blk_alo(const LatGeom &g, int glo) {
  return (int)floor((double)g.x_lo / g.h + 0.5 * (double)glo) - 2;
}

__device__ __forceinline__ i128 shfl_up128(i128 v, int o) {
  unsigned long long lo = (unsigned long long)v;
  long long hi = (long long)(v >> 64);
  lo = __shfl_up_sync(0xffffffffu, lo, o);
  hi = __shfl_up_sync(0xffffffffu, hi, o);
  return (i128)(((unsigned __int128)(unsigned long long)hi << 64) | lo);
}

__device__ __forceinline__ i128 ld128(const i128 *p) {
  const ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2 *>(p));
  return (i128)(((unsigned __int128)v.y << 64) | v.x);
}
__device__ __forceinline__ i128 ldg128(const i128 *p) {
  const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2 *>(p));
  return (i128)(((unsigned __int128)v.y << 64) | v.x);
}
__device__ __forceinline__ void st128(i128 *p, i128 v) {
  ulonglong2 w;
  w.x = (unsigned long long)v;
  w.y = (unsigned long long)((unsigned __int128)v >> 64);
  __stcg(reinterpret_cast<ulonglong2 *>(p), w);
}
__device__ __forceinline__ double i128_to_double(i128 v) {
  const long long hi = (long long)(v >> 64);
  const unsigned long long lo = (unsigned long long)v;
  return __fma_rn((double)hi, 18446744073709551616.0, (double)lo);
}

// ---------------------------------------------------------------------------
// field validation and support radii (as n3_margins_kernel, rubs_n3.cu)
template <int MODE>
__global__ void __launch_bounds__(256) lat_margins_kernel(Field3 F, LatStatus *st) {
  unsigned flags = 0;
  int rx = 0, ry = 0;
  const int64_t n = MODE == kM3Uniform ? 1 : (int64_t)F.FH * F.FW;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double a[3];
    scales3_at<MODE>(F, (int)(i % F.FW), (int)(i / F.FW) + F.fr_off, a, flags);
    rx = max(rx, (int)fmin(ceil(0.5 * a[0] + 0.25 * (a[1] + a[2])) + 1.0, 1.0e8));
    ry = max(ry, (int)fmin(ceil(kQuarterSqrt3 * (a[1] + a[2])) + 1.0, 1.0e8));
  }
  rx = __reduce_max_sync(0xffffffffu, rx);
  ry = __reduce_max_sync(0xffffffffu, ry);
  flags = __reduce_or_sync(0xffffffffu, flags);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&st->rx, rx);
    atomicMax(&st->ry, ry);
    if (flags) atomicOr(&st->flags, flags);
  }
}

// Parameter modes: support radii from a BOUND instead of mapping every pixel
// (the mapping kernel above cost 1.0 ms of config 3's 7.8 ms step; this one
// reads the size plane only).  With C = sum_k a_k^2 / 12 u_k u_k^T and trace
// s: a1^2 = 12 (C11 - C22/3) <= 12 s and a2^2 + a3^2 = 16 C22 <= 16 s, so
// a1 <= sqrt(12 s), a2 + a3 <= sqrt(32 s), for every elongation and
// orientation the mapping accepts (infeasible p_k are clamped to 0, invalid
// parameters replaced: params_to_scales3); each scale is then floored.  A
// wider region changes no sum (exact integers), only the area swept; the
// gather validates every pixel's parameters itself.
template <int DT>
__global__ void __launch_bounds__(256) lat_sizebound_kernel(Field3 F, LatStatus *st, int r_lo,
                                                            int r_hi) {
  double smax = 0.0;
  for (int r = r_lo + blockIdx.x; r < r_hi; r += gridDim.x) {
    const int64_t row = (int64_t)(r - F.fr_off) * F.pld;
    for (int c = threadIdx.x; c < F.FW; c += 256) {
      const double s = load_scalar(F.ps, DT, row + c);
      if (s > 0.0 && s < INFINITY) smax = fmax(smax, s);  // others: flagged by the gather, mapped as s = 1
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, o));
  if ((threadIdx.x & 31) == 0) {
    smax = fmax(smax, 1.0) * (1.0 + 1e-9);
    const double inv = F.scaled ? 1.0 / F.div : 1.0;
    const double a1 = (sqrt(12.0 * smax) + kScaleFloor) * inv;
    const double a23 = (sqrt(32.0 * smax) + 2.0 * kScaleFloor) * inv;
    // (sizes beyond any image are refused by the region check: keep the
    // conversion to int defined)
    atomicMax(&st->rx, (int)fmin(ceil(0.5 * a1 + 0.25 * a23) + 1.0, 1.0e8));
    atomicMax(&st->ry, (int)fmin(ceil(kQuarterSqrt3 * a23) + 1.0, 1.0e8));
  }
}

// max |f| of every canvas row (non-finite entries flagged)
template <int DT>
__global__ void __launch_bounds__(256) lat_rowmax_kernel(ImageSpec I, double *rowmax,
                                                         LatStatus *st, int r_lo, int r_hi) {
  __shared__ double wm[8];
  for (int r = r_lo + blockIdx.x; r < r_hi; r += gridDim.x) {
    double m = 0.0;
    bool bad = false;
    for (int c = threadIdx.x; c < I.w; c += blockDim.x) {
      const double v = load_px<DT>(I.f, (int64_t)r * I.ld + c);
      bad |= !isfinite(v);
      m = fmax(m, fabs(v));
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
      atomicOr(&st->flags, kFlagImageNonFinite);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, wm[w]);
      rowmax[r] = t;
    }
    __syncthreads();
  }
}

// quantisation exponent S of each block: 2^S max|f over the block's region
// rows| < 2^(kQBits + 1)
__global__ void __launch_bounds__(32) lat_scale_kernel(const double *rowmax, ImageSpec I,
                                                       LatGeom g, int *S, int b_first) {
  const int b = b_first + blockIdx.x;
  const int glo = blk_glo(g, b);
  const int r0 = max((int)floor(glo * g.gh) - 1 - I.row0, 0);
  const int r1 = min((int)ceil((glo + g.NG - 1) * g.gh) + 1 - I.row0, I.h - 1);
  double m = 0.0;
  for (int r = r0 + (int)threadIdx.x; r <= r1; r += 32) m = fmax(m, rowmax[r]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (threadIdx.x == 0) {
    // per block: {quantisation exponent, glo, alo} (the gather reads the
    // region origin from here instead of redoing the divisions per pixel)
    S[3 * b] = m > 0.0 ? min(max(kQBits - ilogb(m), -960), 960) : 0;
    S[3 * b + 1] = glo;
    S[3 * b + 2] = blk_alo(g, glo);
  }
}

// ---------------------------------------------------------------------------
// K1: splat onto lattice row ga of block b + running sum along al.
// One CTA (256 threads) per region row; each thread 4 consecutive entries of
// a 1024-entry chunk; chunks chained by a block-wide int128 scan.
template <int DT>
__global__ void __launch_bounds__(256) lat_splat_kernel(ImageSpec I, LatGeom g, int b0,
                                                        const int *S, i128 *G) {
  __shared__ i128 wsum[8];
  const int r = blockIdx.x, bl = blockIdx.y, b = b0 + bl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int glo = blk_glo(g, b), alo = blk_alo(g, glo);
  const int ga = glo + r;
  const double py = g.gh * (double)ga;
  const int pr0 = (int)floor(py);
  const int ir0 = pr0 - I.row0;
  const bool v0 = ir0 >= 0 && ir0 < I.h, v1 = ir0 + 1 >= 0 && ir0 + 1 < I.h;
  const double dg0 = ((double)pr0 - py) * g.inv_gh, dg1 = dg0 + g.inv_gh;  // in (-1, 1]
  const double scale = ldexp(1.0, S[3 * b]);
  i128 *row = G + ((int64_t)bl * g.NG + r) * g.NA;
  i128 carry = 0;
  for (int c0 = 0; c0 < g.NA; c0 += 1024) {
    const int e = c0 + 4 * (int)threadIdx.x;
    i128 p[4];
    i128 run = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      long long q = 0;
      if (e + i < g.NA) {
        const double px = g.h * ((double)(alo + e + i) - 0.5 * (double)ga);
        const int pc0 = (int)floor(px);
        const double fx = px - (double)pc0;
        const int ic = pc0 - I.col0;
        double acc = 0.0;
#pragma unroll
        for (int dc = 0; dc < 2; ++dc) {
          const int c = ic + dc;
          if (c < 0 || c >= I.w) continue;
          const double dx = ((double)dc - fx) * g.inv_h;
#pragma unroll
          for (int dr = 0; dr < 2; ++dr) {
            if (!(dr ? v1 : v0)) continue;
            const double dg = dr ? dg1 : dg0;
            const double da = dx + 0.5 * dg;
            const double m = fmax(fmax(fabs(da), fabs(dg)), fabs(da - dg));
            if (m < 1.0) acc += load_px<DT>(I.f, (int64_t)(ir0 + dr) * I.ld + c) * (1.0 - m);
          }
        }
        q = __double2ll_rn(acc * scale);
      }
      run += (i128)q;
      p[i] = run;
    }
    i128 t = run;  // warp-inclusive scan of the thread totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const i128 n = shfl_up128(t, o);
      if (lane >= o) t += n;
    }
    if (lane == 31) wsum[warp] = t;
    __syncthreads();
    i128 woff = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const i128 ws = wsum[w];
      if (w < warp) woff += ws;
      tot += ws;
    }
    const i128 base = carry + woff + (t - run);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (e + i < g.NA) st128(row + e + i, base + p[i]);
    carry += tot;
    __syncthreads();
  }
}

// Loads in flight per thread in the two line sums below: the grids are small
// (one thread per column / diagonal of a few blocks, ~8 warps per SM on
// config 3), so the memory-level parallelism has to come from each thread.
#ifndef RUBS_LAT_UNROLL
#define RUBS_LAT_UNROLL 32
#endif
constexpr int kLineUnroll = RUBS_LAT_UNROLL;

// K2: running sum along ga (thread per column).
__global__ void __launch_bounds__(128) lat_colsum_kernel(LatGeom g, i128 *G) {
  const int i = blockIdx.x * 128 + threadIdx.x;
  if (i >= g.NA) return;
  i128 *p = G + (int64_t)blockIdx.y * g.NG * g.NA + i;
  const int64_t ld = g.NA;
  i128 acc = 0;
  int r = 0;
  for (; r + kLineUnroll <= g.NG; r += kLineUnroll) {
    i128 v[kLineUnroll];
#pragma unroll
    for (int j = 0; j < kLineUnroll; ++j) v[j] = ld128(p + (r + j) * ld);
#pragma unroll
    for (int j = 0; j < kLineUnroll; ++j) {
      acc += v[j];
      st128(p + (r + j) * ld, acc);
    }
  }
  for (; r < g.NG; ++r) {
    acc += ld128(p + r * ld);
    st128(p + r * ld, acc);
  }
}

// K3: running sum along the diagonal (1, 1) (thread per diagonal d = al - ga).
__global__ void __launch_bounds__(128) lat_diagsum_kernel(LatGeom g, i128 *G) {
  const int t = blockIdx.x * 128 + threadIdx.x;
  const int d = t - (g.NG - 1);
  if (d >= g.NA) return;
  const int r0 = max(0, -d), r1 = min(g.NG - 1, g.NA - 1 - d);
  i128 *p = G + (int64_t)blockIdx.y * g.NG * g.NA + (int64_t)r0 * g.NA + (d + r0);
  const int64_t st = g.NA + 1;
  const int n = r1 - r0 + 1;
  i128 acc = 0;
  int r = 0;
  for (; r + kLineUnroll <= n; r += kLineUnroll) {
    i128 v[kLineUnroll];
#pragma unroll
    for (int j = 0; j < kLineUnroll; ++j) v[j] = ld128(p + (r + j) * st);
#pragma unroll
    for (int j = 0; j < kLineUnroll; ++j) {
      acc += v[j];
      st128(p + (r + j) * st, acc);
    }
  }
  for (; r < n; ++r) {
    acc += ld128(p + r * st);
    st128(p + r * st, acc);
  }
}

// K4: per pixel, 8 vertices x 3 taps of the block's running sums.
// y_lo / y_hi: output rows (relative to g.y0) of blocks [b0, b0 + nbw).
template <int MODE>
__global__ void __launch_bounds__(256) lat_gather_kernel(Field3 F, DomainSpec D, LatGeom g,
                                                         int b0, int y_lo, int y_hi,
                                                         const int *S, const i128 *G,
                                                         LatStatus *st) {
  const int x = blockIdx.x * 32 + threadIdx.x;
  const int y = y_lo + blockIdx.y * 8 + threadIdx.y;
  unsigned flags = 0;
  if (x < D.pw && y < y_hi) {
    const int X = D.pc_lo + x, Y = D.pr_lo + y;
    double a[3];
    scales3_at<MODE>(F, X, Y, a, flags);
    const int b = y / g.bp;
    const int glo = __ldg(S + 3 * b + 1), alo = __ldg(S + 3 * b + 2);
    const i128 *Gb = G + (int64_t)(b - b0) * g.NG * g.NA;
    // base: the pixel shifted by -h u2, in lattice coordinates (region-local)
    const double gy = (double)Y * g.inv_gh;
    const double gb = gy - 1.0, ab = (double)X * g.inv_h + 0.5 * gy - 1.0;
    const double gfl = floor(gb), afl = floor(ab);
    const double gf = gb - gfl, af = ab - afl;
    const int gi = (int)gfl - glo, ai = (int)afl - alo;
    const i128 *B = Gb + (int64_t)gi * g.NA + ai;
    const i128 B00 = ldg128(B);
    const i128 c1 = ldg128(B + 1) - B00, c2 = ldg128(B + g.NA) - B00;
    // Vertex offsets sum_k s_k a_k u_k / 2 in lattice units (al, ga):
    // (s1 k1 + s2 k2, s2 k2 + s3 k3) with k = a / (2 h)  [u1 = (1, 0),
    // u2 = (1, 1), u3 = (0, 1) in lattice coordinates].
    const double k1 = 0.5 * a[0] * g.inv_h, k2 = 0.5 * a[1] * g.inv_h, k3 = 0.5 * a[2] * g.inv_h;
    // Each vertex interpolates G linearly on its lattice triangle:
    //   lin = G00 + w1 (Gx - G00) + w2 (G11 - Gx).
    // G is re-based by the affine function B00 + c1 (al - ai) + c2 (ga - gi)
    // through the pixel's base point (the finite difference annihilates it),
    // in exact integers: the two first differences minus c1 / c2 per vertex,
    // and the G00 terms summed over the eight vertices BEFORE any rounding
    // (sum_v s_v (G00_v - B00 - c1 da_v - c2 dg_v): sum_v s_v = 0, one
    // multiplication per direction for the pixel).
    i128 sum0 = 0;
    int sda = 0, sdg = 0;
    double acc = 0.0;
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const bool n1 = v & 1, n2 = v & 2, n3 = v & 4;
      const bool neg = n1 ^ n2 ^ n3;
      const double oa = (n1 ? -k1 : k1) + (n2 ? -k2 : k2);
      const double og = (n2 ? -k2 : k2) + (n3 ? -k3 : k3);
      const double tg = gf + og, ta = af + oa;
      const double fgf = floor(tg), faf = floor(ta);
      const double wg = tg - fgf, wa = ta - faf;
      const int dg = (int)fgf, da = (int)faf;
      const i128 *T = B + (int64_t)dg * g.NA + da;
      const bool low = wa >= wg;  // lower triangle: via (al + 1, ga); upper: via (al, ga + 1)
      const i128 t00 = ldg128(T), t11 = ldg128(T + g.NA + 1);
      const i128 tx = ldg128(low ? T + 1 : T + g.NA);
      const i128 e1 = (tx - t00) - (low ? c1 : c2);
      const i128 e2 = (t11 - tx) - (low ? c2 : c1);
      const double w1 = low ? wa : wg, w2 = low ? wg : wa;
      const double part = fma(w1, i128_to_double(e1), w2 * i128_to_double(e2));
      if (neg) {
        acc -= part;
        sum0 -= t00;
        sda -= da;
        sdg -= dg;
      } else {
        acc += part;
        sum0 += t00;
        sda += da;
        sdg += dg;
      }
    }
    acc += i128_to_double(sum0 - c1 * (i128)sda - c2 * (i128)sdg);
    D.out[(int64_t)y * D.ld_out + x] =
        ldexp(acc * (g.h / (kSin60 * a[0] * a[1] * a[2])), -__ldg(S + 3 * b));
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(&st->flags, flags);
}

// ---------------------------------------------------------------------------
// host side

struct LatScratch {
  int device = -1;
  LatStatus *d_st = nullptr, *h_st = nullptr;
  i128 *G = nullptr;
  size_t gcap = 0;  // entries
  double *rowmax = nullptr;
  size_t rcap = 0;
  int *S = nullptr;
  size_t scap = 0;
  double *pass[2] = {nullptr, nullptr};
  size_t pcap[2] = {0, 0};
  void *stage[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t stcap[5] = {0, 0, 0, 0, 0};
  cudaStream_t up = nullptr, cmp = nullptr, down = nullptr;  // host-buffer pipeline
};
thread_local LatScratch tl_dev[rubs_internal::kMaxDevices];
thread_local int tl_cur = 0;
#define tl (tl_dev[tl_cur])

int lat_ensure() {
  int dev = 0;
  LAT_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= rubs_internal::kMaxDevices)
    return set_error(RUBS_ECUDA, "device index beyond the per-device state table");
  tl_cur = dev;
  if (tl.device != dev) {
    tl.device = dev;
    LAT_CUDA_TRY(cudaMalloc(&tl.d_st, sizeof(LatStatus)));
    LAT_CUDA_TRY(cudaMallocHost(&tl.h_st, sizeof(LatStatus)));
  }
  return RUBS_OK;
}

template <typename T>
int lat_grow(T *&p, size_t &cap, size_t n) {
  if (n > cap) {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    LAT_CUDA_TRY(cudaMalloc(&p, n * sizeof(T)));
    cap = n;
  }
  return RUBS_OK;
}

int lat_fetch(cudaStream_t s, LatStatus &out) {
  LAT_CUDA_TRY(cudaMemcpyAsync(tl.h_st, tl.d_st, sizeof(LatStatus), cudaMemcpyDeviceToHost, s));
  LAT_CUDA_TRY(cudaStreamSynchronize(s));
  out = *tl.h_st;
  rubs_internal::timer_collect();
  return RUBS_OK;
}

int lat_code(const LatStatus &st) {
  if (st.rx > (1 << 24) || st.ry > (1 << 24))
    return set_error(RUBS_EUNSUPPORTED, "kernel support beyond the lattice mode's range");
  if (st.flags & kFlagFieldNonFinite)
    return set_error(RUBS_EVALUE, "scale field entries must be finite");
  if (st.flags & kFlagParamInvalid)
    return set_error(RUBS_EVALUE,
                     "size must be positive and finite, elongation >= 1 and finite, "
                     "orientation in [0, pi)");
  if (st.flags & kFlagInfeasible)
    return set_error(RUBS_EINFEASIBLE,
                     "elongation beyond the three-direction bound at this orientation");
  if (st.flags & kFlagImageNonFinite)
    return set_error(RUBS_EVALUE, "image entries must be finite in the lattice mode");
  return RUBS_OK;
}

// Block geometry of one pass: bp minimises region entries per output row,
// (NG x NA) / bp, over multiples of 32.
LatGeom lat_geometry(const DomainSpec &D, int rx, int ry, double h, int bp_cap = INT_MAX) {
  LatGeom g{};
  g.h = h;
  g.gh = h * kSin60;
  g.inv_h = 1.0 / h;
  g.inv_gh = 1.0 / g.gh;
  const int RX = rx + 2;
  g.RY = ry + 2;
  g.x_lo = D.pc_lo - RX;
  g.y0 = D.pr_lo;
  g.ph = D.ph;
  auto dims = [&](int bp, int &NG, int &NA) {
    NG = (int)std::ceil((double)(bp - 1 + 2 * g.RY) / g.gh) + 6;
    NA = (int)std::ceil((double)(D.pw - 1 + 2 * RX) / h + 0.5 * NG) + 6;
  };
  // bp: region points per pass, NG x NA x blocks, is flat near its minimum;
  // among the sizes within 4 % of it the SMALLEST wins (more blocks = more
  // columns and diagonals for the line sums, which draw their parallelism
  // from them: config 3, 1024 against 2048 rows per block: -2 %)
  const int top = std::max(32, std::min(((D.ph + 31) / 32) * 32, bp_cap / 32 * 32));
  auto cost_of = [&](int bp) {
    int NG, NA;
    dims(bp, NG, NA);
    return (double)NG * NA * ((D.ph + bp - 1) / bp);
  };
  double best_cost = 1e300;
  for (int bp = 32; bp <= top; bp += 32) best_cost = std::min(best_cost, cost_of(bp));
  int best = top;
  for (int bp = 32; bp <= top; bp += 32)
    if (cost_of(bp) <= 1.04 * best_cost) {
      best = bp;
      break;
    }
  g.bp = best;
  g.nb = (D.ph + best - 1) / best;
  dims(best, g.NG, g.NA);
  return g;
}

size_t lat_budget_entries() {
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = (size_t)8 << 30;
  const size_t cap = std::max<size_t>((size_t)1 << 30, free_b / 2);
  return std::min<size_t>(cap, (size_t)16 << 30) / sizeof(i128);
}

template <int M>
void lat_launch_gather(const Field3 &F, const DomainSpec &D, const LatGeom &g, int b0, int ylo,
                       int yhi, cudaStream_t s) {
  dim3 grid((D.pw + 31) / 32, (yhi - ylo + 7) / 8);
  lat_gather_kernel<M><<<grid, dim3(32, 8), 0, s>>>(F, D, g, b0, ylo, yhi, tl.S, tl.G, tl.d_st);
}

// Blocks [b0, b0 + n) of a pass, their regions in tl.G: splat + three
// running sums + gather.
void lat_block_kernels(const ImageSpec &I, const Field3 &F, const DomainSpec &D, const LatGeom &g,
                       int b0, int n, cudaStream_t s) {
  if (I.dt)
    lat_splat_kernel<1><<<dim3(g.NG, n), 256, 0, s>>>(I, g, b0, tl.S, tl.G);
  else
    lat_splat_kernel<0><<<dim3(g.NG, n), 256, 0, s>>>(I, g, b0, tl.S, tl.G);
  lat_colsum_kernel<<<dim3((g.NA + 127) / 128, n), 128, 0, s>>>(g, tl.G);
  lat_diagsum_kernel<<<dim3((g.NA + g.NG - 1 + 127) / 128, n), 128, 0, s>>>(g, tl.G);
  const int ylo = b0 * g.bp, yhi = std::min(D.ph, (b0 + n) * g.bp);
  switch (F.mode) {
    case kM3Field: lat_launch_gather<kM3Field>(F, D, g, b0, ylo, yhi, s); break;
    case kM3Uniform: lat_launch_gather<kM3Uniform>(F, D, g, b0, ylo, yhi, s); break;
    case kM3Params: lat_launch_gather<kM3Params>(F, D, g, b0, ylo, yhi, s); break;
    default: lat_launch_gather<kM3Params32>(F, D, g, b0, ylo, yhi, s);
  }
}

int lat_pass(const ImageSpec &I, const Field3 &F, const DomainSpec &D, int rx, int ry, double h,
             cudaStream_t s) {
  static const int bp_cap = [] {
    const char *e = std::getenv("RUBS_B200_LAT_BP");
    const int v = e ? std::atoi(e) : 0;
    return v >= 32 ? v : INT_MAX;
  }();
  LatGeom g = lat_geometry(D, rx, ry, h, bp_cap);
  const size_t per_block = (size_t)g.NG * g.NA;
  if ((double)g.NG * g.NA * std::min(g.NG, g.NA) > 4.0e18 || g.NA > (1 << 30))
    return set_error(RUBS_EUNSUPPORTED, "lattice region beyond the exact int128 range");
  // cudaMemGetInfo costs milliseconds of host time: only when the scratch
  // must grow
  size_t cap = tl.gcap;
  if (per_block * g.nb > cap) cap = std::max(cap, lat_budget_entries());
  const int nbw = (int)std::max<size_t>(1, std::min<size_t>((size_t)g.nb, cap / per_block));
  int rc;
  if ((rc = lat_grow(tl.G, tl.gcap, per_block * nbw))) return rc;
  if ((rc = lat_grow(tl.rowmax, tl.rcap, (size_t)std::max(I.h, 1)))) return rc;
  if ((rc = lat_grow(tl.S, tl.scap, (size_t)3 * g.nb))) return rc;
  void *tok = rubs_internal::timed_begin(0, s);
  const int rm_blocks = std::max(1, std::min(I.h, 148 * 8));
  if (I.dt)
    lat_rowmax_kernel<1><<<rm_blocks, 256, 0, s>>>(I, tl.rowmax, tl.d_st, 0, I.h);
  else
    lat_rowmax_kernel<0><<<rm_blocks, 256, 0, s>>>(I, tl.rowmax, tl.d_st, 0, I.h);
  lat_scale_kernel<<<g.nb, 32, 0, s>>>(tl.rowmax, I, g, tl.S, 0);
  int launches = 2;
  for (int b0 = 0; b0 < g.nb; b0 += nbw) {
    lat_block_kernels(I, F, D, g, b0, std::min(nbw, g.nb - b0), s);
    launches += 4;
  }
  rubs_internal::timed_end(tok);
  rubs_internal::count_launches(launches);
  LAT_CUDA_TRY(cudaGetLastError());
  return RUBS_OK;
}

// filter_space_variant orchestration (engine.py:285-324) for the lattice
// mode: global support radii first (field validation, canvases of iterated
// passes), then each pass on its canvas.
int run_lattice(const ImageSpec &img, Field3 F, int iterations, double h, double *out,
                int64_t ld_out, cudaStream_t s) {
  if (img.h < 0 || img.w < 0) return set_error(RUBS_EVALUE, "image must be 2-D");
  if (iterations < 1) return set_error(RUBS_EVALUE, "iterations must be >= 1");
  if (!(h >= 0.125 && h <= 1.0))
    return set_error(RUBS_EVALUE, "lattice spacing must be in [0.125, 1]");
  int rc = lat_ensure();
  if (rc) return rc;
  if (img.h == 0 || img.w == 0) return RUBS_OK;
  F.FH = img.h;
  F.FW = img.w;
  F.div = std::sqrt((double)iterations);
  F.scaled = iterations > 1;
  LAT_CUDA_TRY(cudaMemsetAsync(tl.d_st, 0, sizeof(LatStatus), s));
  {
    const int blocks = F.mode == kM3Uniform ? 1 : 4 * 148;
    switch (F.mode) {
      case kM3Field: lat_margins_kernel<kM3Field><<<blocks, 256, 0, s>>>(F, tl.d_st); break;
      case kM3Uniform: lat_margins_kernel<kM3Uniform><<<blocks, 256, 0, s>>>(F, tl.d_st); break;
      case kM3Params: lat_sizebound_kernel<1><<<blocks, 256, 0, s>>>(F, tl.d_st, 0, F.FH); break;
      default: lat_sizebound_kernel<0><<<blocks, 256, 0, s>>>(F, tl.d_st, 0, F.FH);
    }
    rubs_internal::count_launches(1);
    LAT_CUDA_TRY(cudaGetLastError());
  }
  LatStatus st;
  if ((rc = lat_fetch(s, st))) return rc;
  if ((rc = lat_code(st))) return rc;
  const int rx = st.rx, ry = st.ry;
  ImageSpec cur = img;
  for (int p = 0; p < iterations; ++p) {
    const int remain = iterations - 1 - p;
    DomainSpec Dp;
    Dp.pc_lo = -remain * rx;
    Dp.pr_lo = -remain * ry;
    Dp.pw = img.w + 2 * remain * rx;
    Dp.ph = img.h + 2 * remain * ry;
    if (remain == 0) {
      Dp.out = out;
      Dp.ld_out = ld_out;
    } else {
      const int k = p & 1;
      if ((rc = lat_grow(tl.pass[k], tl.pcap[k], (size_t)Dp.pw * Dp.ph))) return rc;
      Dp.out = tl.pass[k];
      Dp.ld_out = Dp.pw;
    }
    if ((rc = lat_pass(cur, F, Dp, rx, ry, h, s))) return rc;
    cur = ImageSpec{Dp.out, 1, Dp.ld_out, Dp.ph, Dp.pw, Dp.pc_lo, Dp.pr_lo};
  }
  if ((rc = lat_fetch(s, st))) return rc;
  return lat_code(st);
}

int lat_check_image(int f_dtype, int64_t H, int64_t W) {
  if (f_dtype != RUBS_F32 && f_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (H < 0 || W < 0) return set_error(RUBS_EVALUE, "image must be 2-D");
  if (H > (1 << 30) || W > (1 << 30)) return set_error(RUBS_EUNSUPPORTED, "image too large");
  return RUBS_OK;
}

int lat_field_of(const double *field, int uniform, int64_t ld_field, Field3 &F) {
  F = Field3{};
  if (uniform) {
    F.mode = kM3Uniform;
    for (int k = 0; k < 3; ++k) {
      if (!std::isfinite(field[k]))
        return set_error(RUBS_EVALUE, "scale field entries must be finite");
      F.u[k] = field[k];
    }
  } else {
    F.mode = kM3Field;
    F.a = field;
    F.ld = ld_field;
  }
  return RUBS_OK;
}

Field3 lat_params_of(const void *size, const void *elong, const void *orient, int p_dtype,
                     int64_t ld_p) {
  Field3 F{};
  F.mode = p_dtype == RUBS_F64 ? kM3Params : kM3Params32;
  F.ps = size;
  F.pr = elong;
  F.pt = orient;
  F.pld = ld_p;
  return F;
}

int lat_stage(int k, size_t bytes, void **out) {
  if (bytes > tl.stcap[k]) {
    if (tl.stage[k]) cudaFree(tl.stage[k]);
    tl.stage[k] = nullptr;
    tl.stcap[k] = 0;
    LAT_CUDA_TRY(cudaMalloc(&tl.stage[k], bytes));
    tl.stcap[k] = bytes;
  }
  *out = tl.stage[k];
  return RUBS_OK;
}

// Host-buffer call, one pass, parameter modes, on three streams (uploads,
// kernels, downloads): the size plane goes up first (the support bound needs
// it: one small round trip while the image follows), then the image in row
// chunks, then each block's elongation / orientation rows; block b's
// kernels start when its image rows and parameters have landed, and its
// output rows travel back while block b + 1 is filtered.  The blocks are
// capped at 1/8 of the rows (the last block's kernels and download are the
// part that does not overlap).  Results equal the device-pointer entry's up
// to the quantisation exponents of the (smaller) blocks.
constexpr int kLatStreamRows = 2048;  // images with at least this many rows
constexpr int kLatChunkRows = 512;

int lat_stream_params_host(const void *f, int f_dtype, int64_t H, int64_t W, const void *size,
                           const void *elong, const void *orient, int p_dtype, double h,
                           double *out, void *df, void *dout, void *const dp[3]) {
  int rc;
  if (!tl.up) {
    LAT_CUDA_TRY(cudaStreamCreateWithFlags(&tl.up, cudaStreamNonBlocking));
    LAT_CUDA_TRY(cudaStreamCreateWithFlags(&tl.cmp, cudaStreamNonBlocking));
    LAT_CUDA_TRY(cudaStreamCreateWithFlags(&tl.down, cudaStreamNonBlocking));
  }
  const cudaStream_t up = tl.up, cmp = tl.cmp, down = tl.down;
  const size_t esz = f_dtype == RUBS_F64 ? 8 : 4, psz = p_dtype == RUBS_F64 ? 8 : 4;
  std::vector<cudaEvent_t> evs;
  auto fail = [&](int code) {
    cudaStreamSynchronize(up);
    cudaStreamSynchronize(cmp);
    cudaStreamSynchronize(down);
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    return code;
  };
  auto mark = [&](cudaStream_t st, cudaEvent_t &e) -> cudaError_t {
    cudaError_t err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (err != cudaSuccess) return err;
    evs.push_back(e);
    return cudaEventRecord(e, st);
  };
#define LAT_PIPE_TRY(expr)                                                                  \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess)                                                                  \
      return fail(set_error(RUBS_ECUDA, std::string(#expr ": ") + cudaGetErrorString(_e))); \
  } while (0)
  // uploads that need no geometry: the size plane, then the image in chunks
  cudaEvent_t e_size;
  LAT_PIPE_TRY(cudaMemcpyAsync(dp[0], size, (size_t)H * W * psz, cudaMemcpyHostToDevice, up));
  LAT_PIPE_TRY(mark(up, e_size));
  const int nchunk = (int)((H + kLatChunkRows - 1) / kLatChunkRows);
  std::vector<cudaEvent_t> e_img(nchunk);
  for (int c = 0; c < nchunk; ++c) {
    const int64_t r0 = (int64_t)c * kLatChunkRows, r1 = std::min<int64_t>(H, r0 + kLatChunkRows);
    LAT_PIPE_TRY(cudaMemcpyAsync(static_cast<char *>(df) + r0 * W * esz,
                                 static_cast<const char *>(f) + r0 * W * esz,
                                 (size_t)(r1 - r0) * W * esz, cudaMemcpyHostToDevice, up));
    LAT_PIPE_TRY(mark(up, e_img[c]));
  }
  // the support bound (one round trip on the kernel stream)
  Field3 F = lat_params_of(dp[0], dp[1], dp[2], p_dtype, W);
  F.FH = (int)H;
  F.FW = (int)W;
  F.div = 1.0;
  F.scaled = 0;
  LAT_PIPE_TRY(cudaStreamWaitEvent(cmp, e_size, 0));
  LAT_PIPE_TRY(cudaMemsetAsync(tl.d_st, 0, sizeof(LatStatus), cmp));
  if (p_dtype == RUBS_F64)
    lat_sizebound_kernel<1><<<4 * 148, 256, 0, cmp>>>(F, tl.d_st, 0, F.FH);
  else
    lat_sizebound_kernel<0><<<4 * 148, 256, 0, cmp>>>(F, tl.d_st, 0, F.FH);
  LatStatus st;
  if ((rc = lat_fetch(cmp, st))) return fail(rc);
  if (st.rx > (1 << 24) || st.ry > (1 << 24)) return fail(lat_code(st));
  DomainSpec D{0, 0, (int)W, (int)H, static_cast<double *>(dout), W};
  const LatGeom g = lat_geometry(D, st.rx, st.ry, h, std::max(64, (int)(H / 8)));
  const size_t per_block = (size_t)g.NG * g.NA;
  if ((double)g.NG * g.NA * std::min(g.NG, g.NA) > 4.0e18 || g.NA > (1 << 30))
    return fail(set_error(RUBS_EUNSUPPORTED, "lattice region beyond the exact int128 range"));
  if ((rc = lat_grow(tl.G, tl.gcap, per_block)) || (rc = lat_grow(tl.rowmax, tl.rcap, (size_t)H)) ||
      (rc = lat_grow(tl.S, tl.scap, (size_t)3 * g.nb)))
    return fail(rc);
  // each block's elongation / orientation rows, in block order
  std::vector<cudaEvent_t> e_par(g.nb), e_done(g.nb);
  for (int b = 0; b < g.nb; ++b) {
    const int64_t r0 = (int64_t)b * g.bp, r1 = std::min<int64_t>(H, r0 + g.bp);
    const void *src[2] = {elong, orient};
    for (int k = 0; k < 2; ++k)
      LAT_PIPE_TRY(cudaMemcpyAsync(static_cast<char *>(dp[1 + k]) + r0 * W * psz,
                                   static_cast<const char *>(src[k]) + r0 * W * psz,
                                   (size_t)(r1 - r0) * W * psz, cudaMemcpyHostToDevice, up));
    LAT_PIPE_TRY(mark(up, e_par[b]));
  }
  const ImageSpec I{df, f_dtype, W, (int)H, (int)W, 0, 0};
  int rm_done = 0, img_waited = -1, launches = 1;
  for (int b = 0; b < g.nb; ++b) {
    // image rows the block's region reaches
    const int glo = blk_glo(g, b);
    const int need = (int)std::min<int64_t>(H, (int64_t)std::ceil((glo + g.NG - 1) * g.gh) + 2);
    const int chunk = std::max(0, (need - 1) / kLatChunkRows);
    for (int c = img_waited + 1; c <= chunk; ++c) LAT_PIPE_TRY(cudaStreamWaitEvent(cmp, e_img[c], 0));
    img_waited = std::max(img_waited, chunk);
    LAT_PIPE_TRY(cudaStreamWaitEvent(cmp, e_par[b], 0));
    if (need > rm_done) {
      const int blocks = std::max(1, std::min(need - rm_done, 148 * 8));
      if (I.dt)
        lat_rowmax_kernel<1><<<blocks, 256, 0, cmp>>>(I, tl.rowmax, tl.d_st, rm_done, need);
      else
        lat_rowmax_kernel<0><<<blocks, 256, 0, cmp>>>(I, tl.rowmax, tl.d_st, rm_done, need);
      rm_done = need;
      ++launches;
    }
    lat_scale_kernel<<<1, 32, 0, cmp>>>(tl.rowmax, I, g, tl.S, b);
    lat_block_kernels(I, F, D, g, b, 1, cmp);
    launches += 5;
    LAT_PIPE_TRY(cudaGetLastError());
    LAT_PIPE_TRY(mark(cmp, e_done[b]));
    LAT_PIPE_TRY(cudaStreamWaitEvent(down, e_done[b], 0));
    const int64_t r0 = (int64_t)b * g.bp, r1 = std::min<int64_t>(H, r0 + g.bp);
    LAT_PIPE_TRY(cudaMemcpyAsync(out + r0 * W, static_cast<double *>(dout) + r0 * W,
                                 (size_t)(r1 - r0) * W * 8, cudaMemcpyDeviceToHost, down));
  }
  rubs_internal::count_launches(launches);
  LAT_PIPE_TRY(cudaStreamSynchronize(down));
  LAT_PIPE_TRY(cudaStreamSynchronize(up));
  if ((rc = lat_fetch(cmp, st))) return fail(rc);
  for (cudaEvent_t e : evs) cudaEventDestroy(e);
#undef LAT_PIPE_TRY
  return lat_code(st);
}

}  // namespace

extern "C" {

int rubs_b200_filter3_lattice(const void *f, int f_dtype, int64_t H, int64_t W, int64_t ld_f,
                              const double *field, int field_is_uniform, int64_t ld_field,
                              int iterations, double spacing, double *out, int64_t ld_out,
                              void *stream) {
  int rc;
  if ((rc = lat_check_image(f_dtype, H, W))) return rc;
  Field3 F;
  if ((rc = lat_field_of(field, field_is_uniform, ld_field, F))) return rc;
  ImageSpec I{f, f_dtype, ld_f, (int)H, (int)W, 0, 0};
  return run_lattice(I, F, iterations, spacing, out, ld_out, static_cast<cudaStream_t>(stream));
}

int rubs_b200_filter3_lattice_params(const void *f, int f_dtype, int64_t H, int64_t W,
                                     int64_t ld_f, const void *size, const void *elong,
                                     const void *orient, int p_dtype, int64_t ld_p,
                                     int iterations, double spacing, double *out,
                                     int64_t ld_out, void *stream) {
  int rc;
  if ((rc = lat_check_image(f_dtype, H, W))) return rc;
  if (p_dtype != RUBS_F32 && p_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  ImageSpec I{f, f_dtype, ld_f, (int)H, (int)W, 0, 0};
  return run_lattice(I, lat_params_of(size, elong, orient, p_dtype, ld_p), iterations, spacing,
                     out, ld_out, static_cast<cudaStream_t>(stream));
}

int rubs_b200_filter3_lattice_params_rows(const void *f, int f_dtype, int64_t f_row0,
                                          int64_t f_rows, int64_t W, int64_t ld_f,
                                          int64_t H_total, const void *size, const void *elong,
                                          const void *orient, int p_dtype, int64_t p_row0,
                                          int64_t ld_p, int64_t out_row0, int64_t out_rows,
                                          double spacing, double *out, int64_t ld_out,
                                          void *stream) {
  int rc;
  if ((rc = lat_check_image(f_dtype, H_total, W))) return rc;
  if (p_dtype != RUBS_F32 && p_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (!(spacing >= 0.125 && spacing <= 1.0))
    return set_error(RUBS_EVALUE, "lattice spacing must be in [0.125, 1]");
  if (out_row0 < 0 || out_rows < 0 || out_row0 + out_rows > H_total || p_row0 > out_row0 ||
      f_row0 < 0 || f_rows < 0 || f_row0 + f_rows > H_total)
    return set_error(RUBS_EVALUE, "row ranges out of the image");
  if ((rc = lat_ensure())) return rc;
  if (out_rows == 0 || W == 0) return RUBS_OK;
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  const ImageSpec I{f, f_dtype, ld_f, (int)f_rows, (int)W, 0, (int)f_row0};
  Field3 F = lat_params_of(size, elong, orient, p_dtype, ld_p);
  F.FH = (int)H_total;
  F.FW = (int)W;
  F.fr_off = (int)p_row0;
  F.div = 1.0;
  F.scaled = 0;
  LAT_CUDA_TRY(cudaMemsetAsync(tl.d_st, 0, sizeof(LatStatus), s));
  // the support bound from the band's own size rows (the rows it filters)
  if (p_dtype == RUBS_F64)
    lat_sizebound_kernel<1><<<4 * 148, 256, 0, s>>>(F, tl.d_st, (int)out_row0,
                                                    (int)(out_row0 + out_rows));
  else
    lat_sizebound_kernel<0><<<4 * 148, 256, 0, s>>>(F, tl.d_st, (int)out_row0,
                                                    (int)(out_row0 + out_rows));
  rubs_internal::count_launches(1);
  LAT_CUDA_TRY(cudaGetLastError());
  LatStatus st;
  if ((rc = lat_fetch(s, st))) return rc;
  if (st.rx > (1 << 24) || st.ry > (1 << 24)) return lat_code(st);
  const DomainSpec D{0, (int)out_row0, (int)W, (int)out_rows, out, ld_out};
  if ((rc = lat_pass(I, F, D, st.rx, st.ry, spacing, s))) return rc;
  if ((rc = lat_fetch(s, st))) return rc;
  return lat_code(st);
}

int rubs_b200_filter3_lattice_host(const void *f, int f_dtype, int64_t H, int64_t W,
                                   const double *field, int field_is_uniform, int iterations,
                                   double spacing, double *out) {
  int rc;
  if ((rc = lat_check_image(f_dtype, H, W))) return rc;
  if (iterations < 1) return set_error(RUBS_EVALUE, "iterations must be >= 1");
  Field3 F;
  if ((rc = lat_field_of(field, field_is_uniform, W, F))) return rc;
  if ((rc = lat_ensure())) return rc;
  if (H == 0 || W == 0) return RUBS_OK;
  const size_t n = (size_t)H * W, esz = f_dtype == RUBS_F64 ? 8 : 4;
  void *df, *dout, *dfl = nullptr;
  if ((rc = lat_stage(0, n * esz, &df)) || (rc = lat_stage(1, n * 8, &dout))) return rc;
  if (!field_is_uniform && (rc = lat_stage(2, n * 24, &dfl))) return rc;
  const cudaStream_t s = 0;
  LAT_CUDA_TRY(cudaMemcpyAsync(df, f, n * esz, cudaMemcpyHostToDevice, s));
  if (!field_is_uniform) {
    LAT_CUDA_TRY(cudaMemcpyAsync(dfl, field, n * 24, cudaMemcpyHostToDevice, s));
    F.a = static_cast<const double *>(dfl);
  }
  ImageSpec I{df, f_dtype, W, (int)H, (int)W, 0, 0};
  if ((rc = run_lattice(I, F, iterations, spacing, static_cast<double *>(dout), W, s))) return rc;
  LAT_CUDA_TRY(cudaMemcpyAsync(out, dout, n * 8, cudaMemcpyDeviceToHost, s));
  LAT_CUDA_TRY(cudaStreamSynchronize(s));
  return RUBS_OK;
}

int rubs_b200_filter3_lattice_params_host(const void *f, int f_dtype, int64_t H, int64_t W,
                                          const void *size, const void *elong,
                                          const void *orient, int p_dtype, int iterations,
                                          double spacing, double *out) {
  int rc;
  if ((rc = lat_check_image(f_dtype, H, W))) return rc;
  if (p_dtype != RUBS_F32 && p_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (iterations < 1) return set_error(RUBS_EVALUE, "iterations must be >= 1");
  if ((rc = lat_ensure())) return rc;
  if (H == 0 || W == 0) return RUBS_OK;
  const size_t n = (size_t)H * W, esz = f_dtype == RUBS_F64 ? 8 : 4,
               psz = p_dtype == RUBS_F64 ? 8 : 4;
  void *df, *dout, *dp[3];
  if ((rc = lat_stage(0, n * esz, &df)) || (rc = lat_stage(1, n * 8, &dout))) return rc;
  for (int k = 0; k < 3; ++k)
    if ((rc = lat_stage(2 + k, n * psz, &dp[k]))) return rc;
  if (iterations == 1 && H >= kLatStreamRows && !std::getenv("RUBS_B200_NO_STREAM"))
    return lat_stream_params_host(f, f_dtype, H, W, size, elong, orient, p_dtype, spacing, out, df,
                                  dout, dp);
  const cudaStream_t s = 0;
  const void *src[3] = {size, elong, orient};
  LAT_CUDA_TRY(cudaMemcpyAsync(df, f, n * esz, cudaMemcpyHostToDevice, s));
  for (int k = 0; k < 3; ++k)
    LAT_CUDA_TRY(cudaMemcpyAsync(dp[k], src[k], n * psz, cudaMemcpyHostToDevice, s));
  ImageSpec I{df, f_dtype, W, (int)H, (int)W, 0, 0};
  if ((rc = run_lattice(I, lat_params_of(dp[0], dp[1], dp[2], p_dtype, W), iterations, spacing,
                        static_cast<double *>(dout), W, s)))
    return rc;
  LAT_CUDA_TRY(cudaMemcpyAsync(out, dout, n * 8, cudaMemcpyDeviceToHost, s));
  LAT_CUDA_TRY(cudaStreamSynchronize(s));
  return RUBS_OK;
}

}  // extern "C"
