// rubs_n3.cu -- the three-direction (N=3) radially-uniform box-spline filter
// on sm_100a: directions at 0, 60 and 120 degrees (BASELINE.json config 3;
// the reference's direction_vectors(3), geometry.py:76-81, covariance
// sum a_k^2/12 u_k u_k^T, geometry.py:102-106).
//
// The reference has no N=3 filter: the paper's O(1)
// algorithm needs running sums along the box directions on the pixel
// lattice, and 60/120 degrees are not lattice directions (PAPER.md:285,
// 662).  Any interpolation there changes the kernel.  This path is EXACT
// instead: only the on-lattice direction u1 = (1, 0) is
// pre-integrated, and the rest of the kernel is taken row by row.
//
// Slicing the kernel at height y: box(u2) * box(u3) is uniform on a
// parallelogram whose horizontal chord is [L(y), U(y)],
//   L(y) = max(-a2/2 - y/sqrt3, y/sqrt3 - a3/2),
//   U(y) = min( a2/2 - y/sqrt3, y/sqrt3 + a3/2),
// so beta(x, y) = K |[x - a1/2, x + a1/2] n [L(y), U(y)]|, K = 2/(sqrt3 a1 a2 a3),
// a trapezoid in x = four ramps.  With the row's double running sum
// S_j(t) = sum_m f[j, m] max(t - m, 0) -- piecewise linear between integers,
// so linear interpolation of its integer samples is exact --
//   out(n) = K sum_d [S(n1+h-L) - S(n1+h-U) - S(n1-h-L) + S(n1-h-U)],  j = n2 - d.
// Cost per pixel is O(kernel height), four interpolated reads per row.
//
// Layout: one 32x32 output tile per CTA (256 threads, 2 CTAs per SM).  The
// tile's region -- the columns its pixels read, rows streamed in chunks --
// holds per entry k the pair (S[k] + C[k]/2, C[k]) (C = inclusive running
// sum), restarted at the region's left edge: a restart adds a linear
// function of t to S, which the four-ramp difference cancels exactly.  A
// read at real t is then one LDS.128 and one FMA: S(t) = M[k] + phi C[k]
// with k = round(t - 1/2), phi = t - 1/2 - k.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <string>

#include "../../include/rubs_b200.h"
#include "rubs_device.cuh"
#include "rubs_internal.h"
#include "rubs_n3.cuh"

using namespace rubs;
using rubs_internal::set_error;
using namespace rubs3;

namespace {

#define RUBS3_CUDA_TRY(expr)                                                         \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return set_error(RUBS_ECUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
  } while (0)

// tile geometry (dev A/B builds override with -D)
#ifndef RUBS3_TH
#define RUBS3_TH 64
#endif
#ifndef RUBS3_NT
#define RUBS3_NT 256
#endif
#ifndef RUBS3_SMEM_KB
#define RUBS3_SMEM_KB 110
#endif
constexpr int kTW = 32, kTH = RUBS3_TH, kNT = RUBS3_NT, kWarps = kNT / 32, kPx = kTH / kWarps;
constexpr int kMinBlocks = (RUBS3_SMEM_KB <= 110) ? 2 : 1;
constexpr int kSmem3 = RUBS3_SMEM_KB * 1024;

__device__ __forceinline__ double2 lds128(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// S at entry coordinate t' + 1/2 of the row at shared address `row`.
__device__ __forceinline__ double s_read(uint32_t row, double tp) {
  const double r = __dadd_rn(tp, kRoundMagic);
  const int k = __double2loint(r);
  const double phi = __dsub_rn(tp, __dsub_rn(r, kRoundMagic));
  const double2 e = lds128(row + 16u * (uint32_t)k);
  return __fma_rn(phi, e.y, e.x);
}

// Region rows: Wr entries of 16 bytes (Wr a multiple of 4).  The raw image
// values of a row are staged packed at the END of the row's own area
// (float64: byte 8 Wr + 8 e; float32: 12 Wr + 4 e), then scanned into the
// (S + C/2, C) pairs from the front: a pass writes entries below e0 + 128,
// i.e. bytes below 16 (e0 + 128), while its unread raw values sit at or
// above (8|12) Wr + (8|4)(e0 + 128) -- never clobbered while Wr >= e0 + 128.
template <int DT>
__host__ __device__ __forceinline__ uint32_t raw_offset(int Wr) {
  return (DT == 1 ? 8u : 12u) * (uint32_t)Wr;
}

// One raw value into the staging area (zero outside the image and for the
// guard entry): cp.async, so a chunk's loads are all in flight at once.
template <int DT>
__device__ __forceinline__ void fill_raw(uint32_t dst, const ImageSpec &I, int ir, int ic,
                                         bool valid) {
  if constexpr (DT == 1) {
    const double *src = static_cast<const double *>(I.f) + (valid ? (int64_t)ir * I.ld + ic : 0);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
                 "r"(valid ? 8 : 0)
                 : "memory");
  } else {
    const float *src = static_cast<const float *>(I.f) + (valid ? (int64_t)ir * I.ld + ic : 0);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src),
                 "r"(valid ? 4 : 0)
                 : "memory");
  }
}

__device__ __forceinline__ float4 lds128f(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

__device__ __forceinline__ void sts128(uint32_t addr, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(x), "d"(y) : "memory");
}

// One row of the region: raw values -> pairs (S + C/2, C).  Each lane owns
// 4 consecutive entries of a 128-entry pass; the lane blocks are chained by
// a warp scan of the affine maps (C, S) -> (C + F, S + n C + G) (F = block
// sum of f, G = block sum of its local running sums, n = length).  Shared
// accesses are rotated per lane so that every quarter-warp touches 8
// distinct 16-byte bank groups (no conflicts).
template <int DT>
__device__ __forceinline__ void scan_row(uint32_t rowS, int Wr, int lane) {
  const uint32_t rawS = rowS + raw_offset<DT>(Wr);
  double Cp = 0.0, Sp = 0.0;
  for (int e0 = 0; e0 < Wr; e0 += 128) {
    const int eb = e0 + 4 * lane;
    const bool in = eb < Wr;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    if (in) {
      if constexpr (DT == 1) {
        const uint32_t p = rawS + 8u * (uint32_t)eb;
        const bool sw = (lane >> 2) & 1;
        const double2 q0 = lds128(p + (sw ? 16u : 0u)), q1 = lds128(p + (sw ? 0u : 16u));
        v[0] = sw ? q1.x : q0.x;
        v[1] = sw ? q1.y : q0.y;
        v[2] = sw ? q0.x : q1.x;
        v[3] = sw ? q0.y : q1.y;
      } else {
        const float4 q = lds128f(rawS + 4u * (uint32_t)eb);
        v[0] = q.x;
        v[1] = q.y;
        v[2] = q.z;
        v[3] = q.w;
      }
    }
    double c[4], sl[4];
    double acc = 0.0, sacc = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      sl[i] = sacc;  // exclusive prefix of the local running sums
      acc += v[i];
      c[i] = acc;
      sacc += acc;
    }
    double F = acc, G = sacc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double Fa = __shfl_up_sync(0xffffffffu, F, o);
      const double Ga = __shfl_up_sync(0xffffffffu, G, o);
      if (lane >= o) {
        G = __fma_rn((double)(4 * o), Fa, G + Ga);
        F += Fa;
      }
    }
    double Fe = __shfl_up_sync(0xffffffffu, F, 1), Ge = __shfl_up_sync(0xffffffffu, G, 1);
    if (lane == 0) Fe = Ge = 0.0;
    const double Cin = Cp + Fe;
    const double Sin = __fma_rn((double)(4 * lane), Cp, Sp) + Ge;
    double M[4], Cv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      Cv[i] = Cin + c[i];
      M[i] = __fma_rn(0.5, Cv[i], __fma_rn((double)i, Cin, Sin) + sl[i]);
    }
    if (in) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = ((lane >> 1) + i) & 3;
        const double m = r == 0 ? M[0] : r == 1 ? M[1] : r == 2 ? M[2] : M[3];
        const double cc = r == 0 ? Cv[0] : r == 1 ? Cv[1] : r == 2 ? Cv[2] : Cv[3];
        sts128(rowS + 16u * (uint32_t)(eb + r), m, cc);
      }
    }
    const double F31 = __shfl_sync(0xffffffffu, F, 31), G31 = __shfl_sync(0xffffffffu, G, 31);
    Sp = __fma_rn(128.0, Cp, Sp) + G31;
    Cp += F31;
  }
}

// Rows [j0, j0 + n) of one pixel with the chord edges moving linearly:
// per row t1, t3 (= x -/+ h - L) move by -sL, t2, t4 (= x -/+ h - U) by -sU.
__device__ __forceinline__ double gather_seg(uint32_t row, uint32_t rstep, int n, double t1,
                                             double t2, double t3, double t4, double sL,
                                             double sU) {
  double s = 0.0;
#pragma unroll 2
  for (int r = 0; r < n; ++r, row += rstep) {
    const double e1 = s_read(row, t1), e2 = s_read(row, t2);
    const double e3 = s_read(row, t3), e4 = s_read(row, t4);
    s += (e1 - e2) - (e3 - e4);
    t1 -= sL;
    t3 -= sL;
    t2 -= sU;
    t4 -= sU;
  }
  return s;
}

// Pixel (x1, x3 = entry offsets, half widths ha, hb, lattice row Y) over the
// rows [ja, jb] of the chunk starting at row cr0.  The chord edges are
//   L = max(-ha - yd, yd - hb),  U = min(ha - yd, yd + hb),  yd = (Y - j)/sqrt3,
// piecewise linear in j with breaks at yd = +-|hb - ha|/2: three segments
// (A: yd >= |dl|, B: between, C: yd <= -|dl|), each initialised exactly and
// then stepped by +-1/sqrt3 per row.
__device__ __forceinline__ double gather_pixel(uint32_t Es, int Wr, int cr0, int ja, int jb,
                                               int Y, double x1, double x3, double ha,
                                               double hb) {
  const double dl = 0.5 * (hb - ha);
  const double w = fabs(dl) * 1.7320508075688772;
  const int jA = (int)floor(Y - w), jB = (int)ceil(Y + w) - 1;
  const uint32_t rstep = 16u * (uint32_t)Wr;
  double s = 0.0;
  // jB = jA - 1 when hb == ha (no middle segment): keep the bounds monotone
  const int sA = min(jb, jA) + 1;
  const int segs[4] = {ja, sA, max(sA, min(jb, jB) + 1), jb + 1};
  const double c = kInvSqrt3;
  const double sLs[3] = {-c, dl > 0.0 ? c : -c, c};
  const double sUs[3] = {c, dl > 0.0 ? c : -c, -c};
#pragma unroll
  for (int g = 0; g < 3; ++g) {
    const int j0 = max(segs[g], ja), j1 = segs[g + 1];
    if (j1 <= j0) continue;
    const double yd = (double)(Y - j0) * c;
    const double L = fmax(-ha - yd, yd - hb);
    const double U = fmax(fmin(ha - yd, yd + hb), L);
    s += gather_seg(Es + (uint32_t)(j0 - cr0) * rstep, rstep, j1 - j0, x1 - L, x1 - U, x3 - L,
                    x3 - U, sLs[g], sUs[g]);
  }
  return s;
}

// Per-pixel state kept in shared memory (h = a1/2, ha = a2/2, hb = a3/2),
// so that registers go to loads in flight in the gather loop.
constexpr int kStateBytes = 3 * 8 * kTW * kTH;

template <int MODE, int DT>
__global__ void __launch_bounds__(kNT, kMinBlocks)
    n3_tile_kernel(ImageSpec I, Field3 F, DomainSpec D, Status3 *st) {
  extern __shared__ __align__(16) double SM[];
  double *Ph = SM, *Pa = SM + kTW * kTH, *Pb = SM + 2 * kTW * kTH;
  __shared__ int s_ext[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tx0 = blockIdx.x * kTW, ty0 = blockIdx.y * kTH;
  if (threadIdx.x == 0) {
    s_ext[0] = INT_MAX;
    s_ext[1] = INT_MIN;
    s_ext[2] = INT_MAX;
    s_ext[3] = INT_MIN;
  }
  __syncthreads();

  // --- per-pixel scales and the tile's region extent
  unsigned flags = 0;
  int cmin = INT_MAX, cmax = INT_MIN, rmin = INT_MAX, rmax = INT_MIN;
  const int X = D.pc_lo + tx0 + lane;
  const bool colok = tx0 + lane < D.pw;
#pragma unroll
  for (int i = 0; i < kPx; ++i) {
    const int py = ty0 + warp + kWarps * i;
    const int Y = D.pr_lo + py;
    double a[3] = {-2.0, -2.0, -2.0};  // dead pixel: empty row range
    if (colok && py < D.ph) {
      scales3_at<MODE>(F, X, Y, a, flags);
      const double hx = 0.5 * a[0] + 0.25 * (a[1] + a[2]);
      const double hy = kQuarterSqrt3 * (a[1] + a[2]);
      cmin = min(cmin, (int)floor(X - hx));
      cmax = max(cmax, (int)floor(X + hx));
      rmin = min(rmin, (int)ceil(Y - hy));
      rmax = max(rmax, (int)floor(Y + hy));
    }
    const int q = i * kNT + threadIdx.x;
    Ph[q] = 0.5 * a[0];
    Pa[q] = 0.5 * a[1];
    Pb[q] = 0.5 * a[2];
  }
  cmin = __reduce_min_sync(0xffffffffu, cmin);
  cmax = __reduce_max_sync(0xffffffffu, cmax);
  rmin = __reduce_min_sync(0xffffffffu, rmin);
  rmax = __reduce_max_sync(0xffffffffu, rmax);
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (lane == 0) {
    atomicMin(&s_ext[0], cmin);
    atomicMax(&s_ext[1], cmax);
    atomicMin(&s_ext[2], rmin);
    atomicMax(&s_ext[3], rmax);
    if (flags) atomicOr(&st->flags, flags);
  }
  __syncthreads();
  const int c0 = s_ext[0], c1 = s_ext[1], r0 = s_ext[2], r1 = s_ext[3];
  if (c0 > c1) return;  // no live pixel
  const int Wr = (c1 - c0 + 5) & ~3;  // entries k = c0 - 1 .. c1, padded to a multiple of 4
  const int Rc = min(r1 - r0 + 1, (int)((kSmem3 - kStateBytes) / (16 * Wr)));
  if (Rc < 1) {
    if (threadIdx.x == 0) atomicOr(&st->flags, kFlagRegionTooLarge);
    return;
  }
  // entry coordinates: x's entry is X - c0 + 1, and reads take t - 1/2
  const double xe = (double)(X - c0) + 0.5;
  double acc[kPx];
#pragma unroll
  for (int i = 0; i < kPx; ++i) acc[i] = 0.0;

  const uint32_t Es = (uint32_t)__cvta_generic_to_shared(SM) + kStateBytes;
  for (int cr0 = r0; cr0 <= r1; cr0 += Rc) {
    const int nrows = min(Rc, r1 - cr0 + 1);
    __syncthreads();  // previous chunk's reads are done
    // --- the warp's rows of the chunk: raw values (all of its loads in
    // flight together), then the running sums
    for (int rr = warp; rr < nrows; rr += kWarps) {
      const int ir = cr0 + rr - I.row0;
      const bool rin = ir >= 0 && ir < I.h;
      const uint32_t rb = Es + 16u * (uint32_t)(rr * Wr) + raw_offset<DT>(Wr);
      for (int e = lane; e < Wr; e += 32) {
        const int ic = c0 - 1 + e - I.col0;
        fill_raw<DT>(rb + (DT == 1 ? 8u : 4u) * (uint32_t)e, I, ir, ic,
                     rin && e >= 1 && ic >= 0 && ic < I.w);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    for (int rr = warp; rr < nrows; rr += kWarps)
      scan_row<DT>(Es + 16u * (uint32_t)(rr * Wr), Wr, lane);
    __syncthreads();
    // --- rows of the chunk into every pixel's sum
    const int cr1 = cr0 + nrows - 1;
#pragma unroll 1
    for (int i = 0; i < kPx; ++i) {
      const int q = i * kNT + threadIdx.x;
      const double h = Ph[q], ha = Pa[q], hb = Pb[q];
      const int Y = D.pr_lo + ty0 + warp + kWarps * i;
      const double hy = kQuarterSqrt3 * (2.0 * ha + 2.0 * hb);  // == phase A's bound
      const int ja = max((int)ceil(Y - hy), cr0), jb = min((int)floor(Y + hy), cr1);
      if (ja <= jb) acc[i] += gather_pixel(Es, Wr, cr0, ja, jb, Y, xe + h, xe - h, ha, hb);
    }
  }
#pragma unroll
  for (int i = 0; i < kPx; ++i) {
    const int py = ty0 + warp + kWarps * i;
    const int q = i * kNT + threadIdx.x;
    if (colok && py < D.ph)
      D.out[(int64_t)py * D.ld_out + tx0 + lane] =
          (0.25 * kInvSqrt3 / (Ph[q] * Pa[q] * Pb[q])) * acc[i];
  }
}

// Global support radii of the (floored, scaled) field: canvases of iterated
// passes (the N=3 counterpart of engine.py:295 + oracle.py:200-203).
template <int MODE>
__global__ void __launch_bounds__(256) n3_margins_kernel(Field3 F, Status3 *st) {
  unsigned flags = 0;
  int rx = 0, ry = 0;
  const int64_t n = MODE == kM3Uniform ? 1 : (int64_t)F.FH * F.FW;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double a[3];
    scales3_at<MODE>(F, (int)(i % F.FW), (int)(i / F.FW), a, flags);
    rx = max(rx, (int)ceil(0.5 * a[0] + 0.25 * (a[1] + a[2])) + 1);
    ry = max(ry, (int)ceil(kQuarterSqrt3 * (a[1] + a[2])) + 1);
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

// Standalone mapping (size, elongation, orientation) -> (n, 3) scales.
template <int DT>
__global__ void scales3_kernel(const void *ps, const void *pr, const void *pt, int64_t n,
                               double *out, Status3 *st) {
  unsigned flags = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double a[3];
    params_to_scales3(load_scalar(ps, DT, i), load_scalar(pr, DT, i), load_scalar(pt, DT, i), a,
                      flags);
    out[3 * i] = a[0];
    out[3 * i + 1] = a[1];
    out[3 * i + 2] = a[2];
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(&st->flags, flags);
}

// ---------------------------------------------------------------------------
// host side

struct Scratch3 {
  int device = -1;
  Status3 *d_st = nullptr;
  Status3 *h_st = nullptr;  // pinned
  double *d_pass[2] = {nullptr, nullptr};
  size_t pass_cap[2] = {0, 0};
  bool attr = false;
};
thread_local Scratch3 t3_dev[rubs_internal::kMaxDevices];
thread_local int t3_cur = 0;  // set by ensure3() / stage3()
#define t3 (t3_dev[t3_cur])

template <int M, int T>
int set_attr() {
  RUBS3_CUDA_TRY(cudaFuncSetAttribute(n3_tile_kernel<M, T>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem3));
  return RUBS_OK;
}

int ensure3() {
  int dev = 0;
  RUBS3_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= rubs_internal::kMaxDevices)
    return set_error(RUBS_ECUDA, "device index beyond the per-device state table");
  t3_cur = dev;
  if (t3.device != dev) {  // first call on this device
    t3.device = dev;
    RUBS3_CUDA_TRY(cudaMalloc(&t3.d_st, sizeof(Status3)));
    RUBS3_CUDA_TRY(cudaMallocHost(&t3.h_st, sizeof(Status3)));
  }
  if (!t3.attr) {
    int rc;
    if ((rc = set_attr<kM3Field, 0>()) || (rc = set_attr<kM3Field, 1>()) ||
        (rc = set_attr<kM3Uniform, 0>()) || (rc = set_attr<kM3Uniform, 1>()) ||
        (rc = set_attr<kM3Params, 0>()) || (rc = set_attr<kM3Params, 1>()) ||
        (rc = set_attr<kM3Params32, 0>()) || (rc = set_attr<kM3Params32, 1>()))
      return rc;
    t3.attr = true;
  }
  return RUBS_OK;
}

int fetch3(cudaStream_t s, Status3 &out) {
  RUBS3_CUDA_TRY(cudaMemcpyAsync(t3.h_st, t3.d_st, sizeof(Status3), cudaMemcpyDeviceToHost, s));
  RUBS3_CUDA_TRY(cudaStreamSynchronize(s));
  out = *t3.h_st;
  rubs_internal::timer_collect();
  return RUBS_OK;
}

int code3(const Status3 &st) {
  if (st.flags & kFlagFieldNonFinite)
    return set_error(RUBS_EVALUE, "scale field entries must be finite");
  if (st.flags & kFlagParamInvalid)
    return set_error(RUBS_EVALUE,
                     "size must be positive and finite, elongation >= 1 and finite, "
                     "orientation in [0, pi)");
  if (st.flags & kFlagInfeasible)
    return set_error(RUBS_EINFEASIBLE,
                     "elongation beyond the three-direction bound at this orientation");
  if (st.flags & kFlagRegionTooLarge)
    return set_error(RUBS_EUNSUPPORTED,
                     "kernel support exceeds the on-chip region capacity of this build");
  return RUBS_OK;
}

template <int M, int T>
void launch3(const ImageSpec &I, const Field3 &F, const DomainSpec &D, cudaStream_t s) {
  dim3 grid((D.pw + kTW - 1) / kTW, (D.ph + kTH - 1) / kTH);
  n3_tile_kernel<M, T><<<grid, kNT, kSmem3, s>>>(I, F, D, t3.d_st);
}

int launch_pass3(const ImageSpec &I, const Field3 &F, const DomainSpec &D, cudaStream_t s) {
  void *tok = rubs_internal::timed_begin(0, s);
  const int t = I.dt;
  switch (F.mode) {
    case kM3Field: t ? launch3<kM3Field, 1>(I, F, D, s) : launch3<kM3Field, 0>(I, F, D, s); break;
    case kM3Uniform:
      t ? launch3<kM3Uniform, 1>(I, F, D, s) : launch3<kM3Uniform, 0>(I, F, D, s);
      break;
    case kM3Params: t ? launch3<kM3Params, 1>(I, F, D, s) : launch3<kM3Params, 0>(I, F, D, s); break;
    default: t ? launch3<kM3Params32, 1>(I, F, D, s) : launch3<kM3Params32, 0>(I, F, D, s);
  }
  rubs_internal::timed_end(tok);
  rubs_internal::count_launches(1);
  RUBS3_CUDA_TRY(cudaGetLastError());
  return RUBS_OK;
}

int ensure_pass3(int k, size_t n) {
  if (n > t3.pass_cap[k]) {
    if (t3.d_pass[k]) cudaFree(t3.d_pass[k]);
    t3.d_pass[k] = nullptr;
    t3.pass_cap[k] = 0;
    RUBS3_CUDA_TRY(cudaMalloc(&t3.d_pass[k], n * sizeof(double)));
    t3.pass_cap[k] = n;
  }
  return RUBS_OK;
}

// filter_space_variant orchestration (engine.py:285-324) for N=3.
int run3(const ImageSpec &img, Field3 F, int iterations, double *out, int64_t ld_out,
         cudaStream_t s) {
  if (img.h < 0 || img.w < 0) return set_error(RUBS_EVALUE, "image must be 2-D");
  if (iterations < 1) return set_error(RUBS_EVALUE, "iterations must be >= 1");
  int rc = ensure3();
  if (rc) return rc;
  if (img.h == 0 || img.w == 0) return RUBS_OK;
  F.FH = img.h;
  F.FW = img.w;
  F.div = std::sqrt((double)iterations);
  F.scaled = iterations > 1;
  RUBS3_CUDA_TRY(cudaMemsetAsync(t3.d_st, 0, sizeof(Status3), s));
  Status3 st;
  if (iterations == 1) {
    DomainSpec D{0, 0, img.w, img.h, out, ld_out};
    if ((rc = launch_pass3(img, F, D, s))) return rc;
    if ((rc = fetch3(s, st))) return rc;
    return code3(st);
  }
  {
    const int blocks = F.mode == kM3Uniform ? 1 : 4 * 148;
    switch (F.mode) {
      case kM3Field: n3_margins_kernel<kM3Field><<<blocks, 256, 0, s>>>(F, t3.d_st); break;
      case kM3Uniform: n3_margins_kernel<kM3Uniform><<<blocks, 256, 0, s>>>(F, t3.d_st); break;
      case kM3Params: n3_margins_kernel<kM3Params><<<blocks, 256, 0, s>>>(F, t3.d_st); break;
      default: n3_margins_kernel<kM3Params32><<<blocks, 256, 0, s>>>(F, t3.d_st);
    }
    rubs_internal::count_launches(1);
    RUBS3_CUDA_TRY(cudaGetLastError());
  }
  if ((rc = fetch3(s, st))) return rc;
  if ((rc = code3(st))) return rc;
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
      if ((rc = ensure_pass3(k, (size_t)Dp.pw * Dp.ph))) return rc;
      Dp.out = t3.d_pass[k];
      Dp.ld_out = Dp.pw;
    }
    if ((rc = launch_pass3(cur, F, Dp, s))) return rc;
    cur = ImageSpec{Dp.out, 1, Dp.ld_out, Dp.ph, Dp.pw, Dp.pc_lo, Dp.pr_lo};
  }
  if ((rc = fetch3(s, st))) return rc;
  return code3(st);
}

int check_image(int f_dtype, int64_t H, int64_t W) {
  if (f_dtype != RUBS_F32 && f_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (H < 0 || W < 0) return set_error(RUBS_EVALUE, "image must be 2-D");
  if (H > (1 << 30) || W > (1 << 30)) return set_error(RUBS_EUNSUPPORTED, "image too large");
  return RUBS_OK;
}

int field3_of(const double *field, int uniform, int64_t ld_field, Field3 &F) {
  F = Field3{};
  if (uniform) {
    F.mode = kM3Uniform;
    for (int k = 0; k < 3; ++k) {
      if (!std::isfinite(field[k])) return set_error(RUBS_EVALUE, "scale field entries must be finite");
      F.u[k] = field[k];
    }
  } else {
    F.mode = kM3Field;
    F.a = field;
    F.ld = ld_field;
  }
  return RUBS_OK;
}

Field3 params3_of(const void *size, const void *elong, const void *orient, int p_dtype,
                  int64_t ld_p) {
  Field3 F{};
  F.mode = p_dtype == RUBS_F64 ? kM3Params : kM3Params32;
  F.ps = size;
  F.pr = elong;
  F.pt = orient;
  F.pld = ld_p;
  return F;
}

// Host-buffer calls: device staging buffers (kept across calls) and, for
// one pass, a pipeline over bands of output rows on three streams -- the
// image goes up whole (a band's rows read the image beyond the band), then
// each band's per-pixel inputs; a band's tiles launch once its inputs have
// landed and its rows go back while later bands are still in flight (the
// N=4 path's scheme, rubs_b200.cu run_streamed).
struct Stage3 {
  int device = -1;
  void *buf[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t cap[5] = {0, 0, 0, 0, 0};
  cudaStream_t h2d = nullptr, cmp = nullptr, d2h = nullptr;
  cudaEvent_t ev[32];
};
thread_local Stage3 t_st3_dev[rubs_internal::kMaxDevices];
#define t_st3 (t_st3_dev[t3_cur])

int stage3(int k, size_t bytes, void **out) {
  int dev = 0;
  RUBS3_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= rubs_internal::kMaxDevices)
    return set_error(RUBS_ECUDA, "device index beyond the per-device state table");
  t3_cur = dev;
  if (t_st3.device != dev) {  // first call on this device
    t_st3.device = dev;
    RUBS3_CUDA_TRY(cudaStreamCreateWithFlags(&t_st3.h2d, cudaStreamNonBlocking));
    RUBS3_CUDA_TRY(cudaStreamCreateWithFlags(&t_st3.cmp, cudaStreamNonBlocking));
    RUBS3_CUDA_TRY(cudaStreamCreateWithFlags(&t_st3.d2h, cudaStreamNonBlocking));
    for (auto &e : t_st3.ev) RUBS3_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if (bytes > t_st3.cap[k]) {
    if (t_st3.buf[k]) cudaFree(t_st3.buf[k]);
    t_st3.buf[k] = nullptr;
    t_st3.cap[k] = 0;
    RUBS3_CUDA_TRY(cudaMalloc(&t_st3.buf[k], bytes));
    t_st3.cap[k] = bytes;
  }
  *out = t_st3.buf[k];
  return RUBS_OK;
}

struct Plane3 {
  const void *host;
  void *dev;
  size_t row_bytes;
};

// One pass from host buffers: image f_host (already described by I, whose
// .f is the device copy), per-pixel planes (uploaded by row band), result
// into out_host.
int run3_streamed(ImageSpec I, Field3 F, const void *f_host, const Plane3 *planes, int np,
                  double *dout, double *out_host) {
  int rc = ensure3();
  if (rc) return rc;
  const int H = I.h, W = I.w;
  F.FH = H;
  F.FW = W;
  F.div = 1.0;
  F.scaled = 0;
  const cudaStream_t h2d = t_st3.h2d, cmp = t_st3.cmp, d2h = t_st3.d2h;
  const int ty = (H + kTH - 1) / kTH;
  const int nb = std::max(1, std::min(8, ty));
  const int per = (ty + nb - 1) / nb;
  RUBS3_CUDA_TRY(cudaMemsetAsync(t3.d_st, 0, sizeof(Status3), cmp));
  RUBS3_CUDA_TRY(cudaMemcpyAsync(const_cast<void *>(I.f), f_host,
                                 (size_t)H * W * (I.dt ? 8 : 4), cudaMemcpyHostToDevice, h2d));
  int bands = 0;
  for (int b = 0; b < nb; ++b, ++bands) {
    const int r0 = b * per * kTH, r1 = std::min(H, (b + 1) * per * kTH);
    if (r0 >= r1) break;
    for (int k = 0; k < np; ++k)
      RUBS3_CUDA_TRY(cudaMemcpyAsync(static_cast<char *>(planes[k].dev) + r0 * planes[k].row_bytes,
                                     static_cast<const char *>(planes[k].host) + r0 * planes[k].row_bytes,
                                     (size_t)(r1 - r0) * planes[k].row_bytes, cudaMemcpyHostToDevice,
                                     h2d));
    RUBS3_CUDA_TRY(cudaEventRecord(t_st3.ev[2 * b], h2d));
    RUBS3_CUDA_TRY(cudaStreamWaitEvent(cmp, t_st3.ev[2 * b], 0));
    DomainSpec D{0, r0, W, r1 - r0, dout + (size_t)r0 * W, W};
    if ((rc = launch_pass3(I, F, D, cmp))) return rc;
    RUBS3_CUDA_TRY(cudaEventRecord(t_st3.ev[2 * b + 1], cmp));
  }
  // returns last: a copy into pageable memory blocks the host until it ran
  for (int b = 0; b < bands; ++b) {
    const int r0 = b * per * kTH, r1 = std::min(H, (b + 1) * per * kTH);
    RUBS3_CUDA_TRY(cudaStreamWaitEvent(d2h, t_st3.ev[2 * b + 1], 0));
    RUBS3_CUDA_TRY(cudaMemcpyAsync(out_host + (size_t)r0 * W, dout + (size_t)r0 * W,
                                   (size_t)(r1 - r0) * W * 8, cudaMemcpyDeviceToHost, d2h));
  }
  RUBS3_CUDA_TRY(cudaStreamSynchronize(d2h));
  Status3 st;
  if ((rc = fetch3(cmp, st))) return rc;
  return code3(st);
}

}  // namespace

extern "C" {

int rubs_b200_filter3(const void *f, int f_dtype, int64_t H, int64_t W, int64_t ld_f,
                      const double *field, int field_is_uniform, int64_t ld_field, int iterations,
                      double *out, int64_t ld_out, void *stream) {
  int rc;
  if ((rc = check_image(f_dtype, H, W))) return rc;
  Field3 F;
  if ((rc = field3_of(field, field_is_uniform, ld_field, F))) return rc;
  ImageSpec I{f, f_dtype, ld_f, (int)H, (int)W, 0, 0};
  return run3(I, F, iterations, out, ld_out, static_cast<cudaStream_t>(stream));
}

int rubs_b200_filter3_params(const void *f, int f_dtype, int64_t H, int64_t W, int64_t ld_f,
                             const void *size, const void *elong, const void *orient, int p_dtype,
                             int64_t ld_p, int iterations, double *out, int64_t ld_out,
                             void *stream) {
  int rc;
  if ((rc = check_image(f_dtype, H, W))) return rc;
  if (p_dtype != RUBS_F32 && p_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  ImageSpec I{f, f_dtype, ld_f, (int)H, (int)W, 0, 0};
  return run3(I, params3_of(size, elong, orient, p_dtype, ld_p), iterations, out, ld_out,
              static_cast<cudaStream_t>(stream));
}

int rubs_b200_filter3_host(const void *f, int f_dtype, int64_t H, int64_t W, const double *field,
                           int field_is_uniform, int iterations, double *out) {
  int rc;
  if ((rc = check_image(f_dtype, H, W))) return rc;
  if (iterations < 1) return set_error(RUBS_EVALUE, "iterations must be >= 1");
  Field3 F;
  if ((rc = field3_of(field, field_is_uniform, W, F))) return rc;
  if (H == 0 || W == 0) return RUBS_OK;
  const size_t n = (size_t)H * W, esz = f_dtype == RUBS_F64 ? 8 : 4;
  void *df, *dout, *dfl = nullptr;
  if ((rc = stage3(0, n * esz, &df)) || (rc = stage3(1, n * 8, &dout))) return rc;
  if (!field_is_uniform && (rc = stage3(2, n * 24, &dfl))) return rc;
  ImageSpec I{df, f_dtype, W, (int)H, (int)W, 0, 0};
  if (iterations == 1) {
    if (!field_is_uniform) F.a = static_cast<const double *>(dfl);
    Plane3 pl{field, dfl, (size_t)W * 24};
    return run3_streamed(I, F, f, &pl, field_is_uniform ? 0 : 1, static_cast<double *>(dout), out);
  }
  const cudaStream_t s = t_st3.cmp;
  RUBS3_CUDA_TRY(cudaMemcpyAsync(df, f, n * esz, cudaMemcpyHostToDevice, s));
  if (!field_is_uniform) {
    RUBS3_CUDA_TRY(cudaMemcpyAsync(dfl, field, n * 24, cudaMemcpyHostToDevice, s));
    F.a = static_cast<const double *>(dfl);
  }
  if ((rc = run3(I, F, iterations, static_cast<double *>(dout), W, s))) return rc;
  RUBS3_CUDA_TRY(cudaMemcpyAsync(out, dout, n * 8, cudaMemcpyDeviceToHost, s));
  RUBS3_CUDA_TRY(cudaStreamSynchronize(s));
  return RUBS_OK;
}

int rubs_b200_filter3_params_host(const void *f, int f_dtype, int64_t H, int64_t W,
                                  const void *size, const void *elong, const void *orient,
                                  int p_dtype, int iterations, double *out) {
  int rc;
  if ((rc = check_image(f_dtype, H, W))) return rc;
  if (p_dtype != RUBS_F32 && p_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (iterations < 1) return set_error(RUBS_EVALUE, "iterations must be >= 1");
  if (H == 0 || W == 0) return RUBS_OK;
  const size_t n = (size_t)H * W, esz = f_dtype == RUBS_F64 ? 8 : 4,
               psz = p_dtype == RUBS_F64 ? 8 : 4;
  void *df, *dout, *dp[3];
  if ((rc = stage3(0, n * esz, &df)) || (rc = stage3(1, n * 8, &dout))) return rc;
  for (int k = 0; k < 3; ++k)
    if ((rc = stage3(2 + k, n * psz, &dp[k]))) return rc;
  ImageSpec I{df, f_dtype, W, (int)H, (int)W, 0, 0};
  Field3 F = params3_of(dp[0], dp[1], dp[2], p_dtype, W);
  const void *src[3] = {size, elong, orient};
  if (iterations == 1) {
    Plane3 pl[3];
    for (int k = 0; k < 3; ++k) pl[k] = Plane3{src[k], dp[k], (size_t)W * psz};
    return run3_streamed(I, F, f, pl, 3, static_cast<double *>(dout), out);
  }
  const cudaStream_t s = t_st3.cmp;
  RUBS3_CUDA_TRY(cudaMemcpyAsync(df, f, n * esz, cudaMemcpyHostToDevice, s));
  for (int k = 0; k < 3; ++k)
    RUBS3_CUDA_TRY(cudaMemcpyAsync(dp[k], src[k], n * psz, cudaMemcpyHostToDevice, s));
  if ((rc = run3(I, F, iterations, static_cast<double *>(dout), W, s))) return rc;
  RUBS3_CUDA_TRY(cudaMemcpyAsync(out, dout, n * 8, cudaMemcpyDeviceToHost, s));
  RUBS3_CUDA_TRY(cudaStreamSynchronize(s));
  return RUBS_OK;
}

int rubs_b200_read_margins3_params(const void *size, const void *elong, const void *orient,
                                   int p_dtype, int64_t rows, int64_t W, int64_t ld_p,
                                   int *out2, void *stream) {
  if (p_dtype != RUBS_F32 && p_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (rows < 0 || W < 0) return set_error(RUBS_EVALUE, "negative size");
  int rc = ensure3();
  if (rc) return rc;
  out2[0] = out2[1] = 0;
  if (rows == 0 || W == 0) return RUBS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Field3 F = params3_of(size, elong, orient, p_dtype, ld_p);
  F.FH = (int)rows;
  F.FW = (int)W;
  F.div = 1.0;
  RUBS3_CUDA_TRY(cudaMemsetAsync(t3.d_st, 0, sizeof(Status3), s));
  if (p_dtype == RUBS_F64)
    n3_margins_kernel<kM3Params><<<4 * 148, 256, 0, s>>>(F, t3.d_st);
  else
    n3_margins_kernel<kM3Params32><<<4 * 148, 256, 0, s>>>(F, t3.d_st);
  rubs_internal::count_launches(1);
  RUBS3_CUDA_TRY(cudaGetLastError());
  Status3 st;
  if ((rc = fetch3(s, st))) return rc;
  out2[0] = st.rx;
  out2[1] = st.ry;
  return code3(st);
}

int rubs_b200_filter3_params_rows(const void *f, int f_dtype, int64_t f_row0, int64_t f_rows,
                                  int64_t W, int64_t ld_f, int64_t H_total, const void *size,
                                  const void *elong, const void *orient, int p_dtype,
                                  int64_t p_row0, int64_t ld_p, int64_t out_row0,
                                  int64_t out_rows, double *out, int64_t ld_out, void *stream) {
  int rc;
  if ((rc = check_image(f_dtype, H_total, W))) return rc;
  if (p_dtype != RUBS_F32 && p_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (out_row0 < 0 || out_rows < 0 || out_row0 + out_rows > H_total || p_row0 > out_row0 ||
      f_row0 < 0 || f_rows < 0 || f_row0 + f_rows > H_total)
    return set_error(RUBS_EVALUE, "row ranges out of the image");
  if ((rc = ensure3())) return rc;
  if (out_rows == 0 || W == 0) return RUBS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ImageSpec I{f, f_dtype, ld_f, (int)f_rows, (int)W, 0, (int)f_row0};
  Field3 F = params3_of(size, elong, orient, p_dtype, ld_p);
  F.FH = (int)H_total;
  F.FW = (int)W;
  F.fr_off = (int)p_row0;
  F.div = 1.0;
  RUBS3_CUDA_TRY(cudaMemsetAsync(t3.d_st, 0, sizeof(Status3), s));
  DomainSpec D{0, (int)out_row0, (int)W, (int)out_rows, out, ld_out};
  if ((rc = launch_pass3(I, F, D, s))) return rc;
  Status3 st;
  if ((rc = fetch3(s, st))) return rc;
  return code3(st);
}

int rubs_b200_scales3(const void *size, const void *elong, const void *orient, int p_dtype,
                      int64_t n, double *out, void *stream) {
  if (p_dtype != RUBS_F32 && p_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (n < 0) return set_error(RUBS_EVALUE, "negative count");
  int rc = ensure3();
  if (rc) return rc;
  if (n == 0) return RUBS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  RUBS3_CUDA_TRY(cudaMemsetAsync(t3.d_st, 0, sizeof(Status3), s));
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 8 * 148);
  if (p_dtype == RUBS_F64)
    scales3_kernel<1><<<blocks, 256, 0, s>>>(size, elong, orient, n, out, t3.d_st);
  else
    scales3_kernel<0><<<blocks, 256, 0, s>>>(size, elong, orient, n, out, t3.d_st);
  rubs_internal::count_launches(1);
  RUBS3_CUDA_TRY(cudaGetLastError());
  Status3 st;
  if ((rc = fetch3(s, st))) return rc;
  return code3(st);
}

}  // extern "C"
