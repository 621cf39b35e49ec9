// rubs_b200.cu -- B200 (sm_100a) kernels and the C ABI (include/rubs_b200.h)
// for the reference's hot path, engine.filter_space_variant
// (pkg/src/rubs/engine.py:265-324).
//
// Design (DESIGN.md has the full story):
//   * The output domain is cut into 32x32 tiles (16x16 cells for the margin
//     pre-pass).  Every tile pre-integrates ITS OWN region -- the tile grown
//     by the read margins of its own pixels -- in shared memory, with the
//     running sums restarted at the region edge.  This is exact: the filter
//     is linear and zero-padded, so cropping f to the region changes nothing
//     for the tile's pixels, and restarting a sweep on a rectangle only adds
//     ridge functions (constant along one of the four box directions) that
//     the 16-vertex finite difference annihilates.  No canvas widening
//     (engine.py:177) is needed and the sums stay O(region^4) instead of
//     O(image^4), which is what keeps every config inside 1e-9.
//   * The four sweeps (engine.py:186-193) run in shared memory, one thread
//     per row / diagonal / column / anti-diagonal.
//   * Each pixel then takes its 16-vertex finite difference (engine.py:232-244)
//     reading the region through the 7-tap ZP interpolant (zp.py:186-228) in
//     one canonical-wedge form (rubs_device.cuh: zp_read8).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rubs_b200.h"
#include "rubs_device.cuh"

using namespace rubs;

namespace {

constexpr int kTile = 32;        // output tile edge
constexpr int kCell = 16;        // margin cell edge
constexpr int kThreads = 512;    // tile kernel CTA size
constexpr int kSmemBytes = 225 * 1024;  // dynamic shared memory per tile CTA (+ static <= 227 KiB)
constexpr int kRegionCap = kSmemBytes / 8;  // doubles

thread_local std::string t_last_error;
thread_local int64_t t_launches = 0;

// optional per-kernel event timing (bench.py roofline)
struct KTimer {
  bool on = false;
  double ms[2] = {0.0, 0.0};
  int64_t n[2] = {0, 0};
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  std::vector<cudaEvent_t> pool;
};
thread_local KTimer t_timer;

cudaEvent_t timer_event() {
  if (!t_timer.pool.empty()) {
    cudaEvent_t e = t_timer.pool.back();
    t_timer.pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Bracket one launch: returns the start event (or null when off).
struct TimedLaunch {
  int kind;
  cudaEvent_t a = nullptr;
  cudaStream_t s;
  TimedLaunch(int k, cudaStream_t st) : kind(k), s(st) {
    if (t_timer.on) {
      a = timer_event();
      cudaEventRecord(a, s);
    }
  }
  ~TimedLaunch() {
    if (a) {
      cudaEvent_t b = timer_event();
      cudaEventRecord(b, s);
      t_timer.pending.push_back({kind, {a, b}});
    }
  }
};

// Called after the stream was synchronised.
void timer_collect() {
  for (auto &p : t_timer.pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.second.first, p.second.second) == cudaSuccess) {
      t_timer.ms[p.first] += ms;
      t_timer.n[p.first] += 1;
    }
    t_timer.pool.push_back(p.second.first);
    t_timer.pool.push_back(p.second.second);
  }
  t_timer.pending.clear();
}

int set_error(int code, const std::string &msg) {
  t_last_error = msg;
  return code;
}

#define RUBS_CUDA_TRY(expr)                                                          \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return set_error(RUBS_ECUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
  } while (0)

// ---------------------------------------------------------------------------
// Kernels

// Pass-domain cell margins.  One CTA per 16x16 cell: every pixel fetches its
// scale-vector (field, uniform or LUT-mapped), the CTA reduces the four
// integer read margins.  With `global_out` it also folds them into the
// status word (the reference's whole-field _read_margins, engine.py:247-262).
__global__ void __launch_bounds__(256) cell_margins_kernel(FieldSpec F, DomainSpec D,
                                                           int cells_x, int4 *cells,
                                                           Status *st, int global_out) {
  const int cx = blockIdx.x % cells_x, cy = blockIdx.x / cells_x;
  const int x = cx * kCell + (threadIdx.x & 15), y = cy * kCell + (threadIdx.x >> 4);
  unsigned flags = 0;
  int4 m = make_int4(0, 0, 0, 0);
  if (x < D.pw && y < D.ph) {
    double a[4];
    field_at(F, D.pc_lo + x, D.pr_lo + y, a, flags);
    m = pixel_margins(a);
  }
  // warp reduce
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m.x = max(m.x, __shfl_xor_sync(0xffffffffu, m.x, o));
    m.y = max(m.y, __shfl_xor_sync(0xffffffffu, m.y, o));
    m.z = max(m.z, __shfl_xor_sync(0xffffffffu, m.z, o));
    m.w = max(m.w, __shfl_xor_sync(0xffffffffu, m.w, o));
    flags |= __shfl_xor_sync(0xffffffffu, flags, o);
  }
  __shared__ int4 red[8];
  __shared__ unsigned redf[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[warp] = m;
    redf[warp] = flags;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int4 r = red[0];
    unsigned f = redf[0];
    for (int w = 1; w < 8; ++w) {
      r.x = max(r.x, red[w].x);
      r.y = max(r.y, red[w].y);
      r.z = max(r.z, red[w].z);
      r.w = max(r.w, red[w].w);
      f |= redf[w];
    }
    cells[blockIdx.x] = r;
    if (f) atomicOr(&st->flags, f);
    if (global_out) {
      atomicMax(&st->gm[0], r.x);
      atomicMax(&st->gm[1], r.y);
      atomicMax(&st->gm[2], r.z);
      atomicMax(&st->gm[3], r.w);
    }
  }
}

// Load the image over region lattice [rc0, rc0+RW) x [rr0, rr0+RH) into
// shared memory as fp64, zero outside the image (zero padding, engine.py:155).
__device__ __forceinline__ void load_region(double *S, int P, const ImageSpec &I, int rc0,
                                            int rr0, int RW, int RH) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int r = warp; r < RH; r += nw) {
    const int ir = rr0 + r - I.row0;
    double *row = S + r * P;
    const bool rin = (ir >= 0 && ir < I.h);
    for (int c = lane; c < RW; c += 32) {
      const int ic = rc0 + c - I.col0;
      double v = 0.0;
      if (rin && ic >= 0 && ic < I.w) v = load_scalar(I.f, I.dt, (int64_t)ir * I.ld + ic);
      row[c] = v;
    }
  }
}

// The four running-sum sweeps of engine.py:186-193 on the region, with the
// sums started at the region edge.  Returns (via gmax) max |plane|.
__device__ __forceinline__ void region_sweeps(double *S, int P, int RW, int RH, double &gmax) {
  const int tid = threadIdx.x, nt = blockDim.x;
  // RS1: cumulative sum along +x, then x sqrt2
  for (int r = tid; r < RH; r += nt) {
    double *p = S + r * P;
    double s = 0.0;
    for (int c = 0; c < RW; ++c) {
      s += p[c];
      p[c] = s * kSqrt2;
    }
  }
  __syncthreads();
  // RS2: g[r][c] += g[r-1][c-1] (lines c - r = const)
  for (int L = tid; L < RH + RW - 1; L += nt) {
    const int k = L - (RH - 1);
    const int r0 = k < 0 ? -k : 0, c0 = k < 0 ? 0 : k;
    const int len = min(RH - r0, RW - c0);
    double *p = S + r0 * P + c0;
    double s = 0.0;
    for (int j = 0; j < len; ++j) {
      s += *p;
      *p = s;
      p += P + 1;
    }
  }
  __syncthreads();
  // RS3: cumulative sum along +y, then x sqrt2
  for (int c = tid; c < RW; c += nt) {
    double *p = S + c;
    double s = 0.0;
    for (int r = 0; r < RH; ++r) {
      s += *p;
      *p = s * kSqrt2;
      p += P;
    }
  }
  __syncthreads();
  // RS4: g[r][c] += g[r-1][c+1] (lines c + r = const)
  double gm = 0.0;
  for (int k = tid; k < RH + RW - 1; k += nt) {
    const int r0 = max(0, k - (RW - 1)), c0 = k - r0;
    const int len = min(RH - r0, c0 + 1);
    double *p = S + r0 * P + c0;
    double s = 0.0;
    for (int j = 0; j < len; ++j) {
      s += *p;
      *p = s;
      gm = fmax(gm, fabs(s));
      p += P - 1;
    }
  }
  gmax = fmax(gmax, gm);
  __syncthreads();
}

// Filter one pixel from the region plane (engine.py:219-244).
//   n1, n2: lattice coordinates of the pixel; off0 = rr0 * P + rc0.
__device__ __forceinline__ double pixel_fd(const double *__restrict__ S, int P, int off0,
                                           int n1, int n2, const double a[4]) {
  const double a1 = a[0], a2 = a[1], a3 = a[2], a4 = a[3];
  const double p2 = a2 * kInvSqrt2, p4 = a4 * kInvSqrt2;
  const double t1 = 0.5 * a1 + 0.5 * (p2 - p4) - 0.5;
  const double t2 = 0.5 * a3 + 0.5 * (p2 + p4) - 1.5;
  const double w = 0.125 / (a1 * a2 * a3 * a4);
  const double xb = (double)n1 + t1, yb = (double)n2 + t2;
  // distinct vertex abscissae: index q1 | q2 << 1 | q4 << 2
  // x = xb - (q1 a1 + q2 p2 - q4 p4)     (engine.py:240)
  // distinct ordinates:       index q2 | q3 << 1 | q4 << 2
  // y = yb - (q2 p2 + q3 a3 + q4 p4)     (engine.py:241)
  const double ox[8] = {0.0, a1, p2, a1 + p2, -p4, a1 - p4, p2 - p4, (a1 + p2) - p4};
  const double oy[8] = {0.0, p2, a3, p2 + a3, p4, p2 + p4, a3 + p4, (p2 + a3) + p4};
  int mx[8], my[8];
  double dx[8], dy[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    lattice_split(xb - ox[k], mx[k], dx[k]);
    lattice_split(yb - oy[k], my[k], dy[k]);
    my[k] = my[k] * P - off0;
  }
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int q1 = i & 1, q2 = (i >> 1) & 1, q3 = (i >> 2) & 1, q4 = (i >> 3) & 1;
    const int ix = q1 | (q2 << 1) | (q4 << 2);
    const int iy = q2 | (q3 << 1) | (q4 << 2);
    const double v = zp_read8(S, my[iy] + mx[ix], P, dx[ix], dy[iy]);
    if (__popc(i) & 1)
      acc -= v;
    else
      acc += v;
  }
  return acc * w;
}

// One CTA per 32x32 output tile.  If the tile's region does not fit in
// shared memory the tile is processed as its four 16x16 cells.
__global__ void __launch_bounds__(kThreads, 1)
    tile_filter_kernel(ImageSpec I, FieldSpec F, DomainSpec D, const int4 *__restrict__ cells,
                       int cells_x, int tiles_x, int region_cap, Status *st) {
  extern __shared__ double S[];
  __shared__ int s_sub[4][8];
  __shared__ int s_nsub;
  const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  const int x0 = tx * kTile, y0 = ty * kTile;
  if (threadIdx.x == 0) {
    const int tw = min(kTile, D.pw - x0), th = min(kTile, D.ph - y0);
    int4 cm[4];
    int present[4];
    for (int k = 0; k < 4; ++k) {
      const int ccx = tx * 2 + (k & 1), ccy = ty * 2 + (k >> 1);
      present[k] = (ccx * kCell < D.pw) && (ccy * kCell < D.ph);
      cm[k] = present[k] ? cells[ccy * cells_x + ccx] : make_int4(0, 0, 0, 0);
    }
    int4 u = cm[0];
    for (int k = 1; k < 4; ++k)
      if (present[k]) {
        u.x = max(u.x, cm[k].x);
        u.y = max(u.y, cm[k].y);
        u.z = max(u.z, cm[k].z);
        u.w = max(u.w, cm[k].w);
      }
    const int RW = tw + u.x + u.y, RH = th + u.z + u.w;
    const int P = RW | 1;
    if (P * RH <= region_cap) {
      s_nsub = 1;
      int *d = s_sub[0];
      d[0] = x0; d[1] = y0; d[2] = tw; d[3] = th;
      d[4] = u.x; d[5] = u.z; d[6] = RW; d[7] = RH;
    } else {
      int n = 0;
      for (int k = 0; k < 4; ++k) {
        if (!present[k]) continue;
        const int sx = x0 + (k & 1) * kCell, sy = y0 + (k >> 1) * kCell;
        const int sw = min(kCell, D.pw - sx), sh = min(kCell, D.ph - sy);
        int *d = s_sub[n++];
        d[0] = sx; d[1] = sy; d[2] = sw; d[3] = sh;
        d[4] = cm[k].x; d[5] = cm[k].z;
        d[6] = sw + cm[k].x + cm[k].y;
        d[7] = sh + cm[k].z + cm[k].w;
      }
      s_nsub = n;
    }
  }
  __syncthreads();
  const int nsub = s_nsub;
  double gmax = 0.0;
  unsigned flags = 0;
  for (int sI = 0; sI < nsub; ++sI) {
    const int sx = s_sub[sI][0], sy = s_sub[sI][1], sw = s_sub[sI][2], sh = s_sub[sI][3];
    const int left = s_sub[sI][4], below = s_sub[sI][5], RW = s_sub[sI][6], RH = s_sub[sI][7];
    const int P = RW | 1;
    if (P * RH > region_cap) {
      if (threadIdx.x == 0) atomicOr(&st->flags, kFlagRegionTooLarge);
      continue;
    }
    // region lattice origin
    const int rc0 = D.pc_lo + sx - left, rr0 = D.pr_lo + sy - below;
    load_region(S, P, I, rc0, rr0, RW, RH);
    __syncthreads();
    region_sweeps(S, P, RW, RH, gmax);
    const int off0 = rr0 * P + rc0;
    const int npx = sw * sh;
    for (int p = threadIdx.x; p < npx; p += blockDim.x) {
      const int px = sx + p % sw, py = sy + p / sw;
      const int n1 = D.pc_lo + px, n2 = D.pr_lo + py;
      double a[4];
      field_at(F, n1, n2, a, flags);
      D.out[(int64_t)py * D.ld_out + px] = pixel_fd(S, P, off0, n1, n2, a);
    }
    __syncthreads();
  }
  // fold guard magnitude (non-negative doubles order like their bit patterns)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
  if ((threadIdx.x & 31) == 0 && gmax > 0.0)
    atomicMax(&st->guard_bits, (unsigned long long)__double_as_longlong(gmax));
  if (flags) atomicOr(&st->flags, flags);
}

// ---- standalone lookup (solver.lookup_many) ------------------------------
__global__ void lookup_kernel(FieldSpec F, int64_t n, double *out, Status *st) {
  unsigned flags = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double a[4];
    lut_map(F, load_scalar(F.ps, F.pdt, i), load_scalar(F.pr, F.pdt, i),
            load_scalar(F.pt, F.pdt, i), a, flags);
    double2 *o = reinterpret_cast<double2 *>(out + i * 4);
    o[0] = make_double2(a[0], a[1]);
    o[1] = make_double2(a[2], a[3]);
  }
  if (flags) atomicOr(&st->flags, flags);
}

// ---- global pre-integration (engine.preintegrate API parity) -------------
__global__ void canvas_fill_kernel(ImageSpec I, double *plane, int64_t ld, int64_t rows,
                                   int64_t cols, int64_t c_lo, int64_t r_lo) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * cols;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, c = e - r * cols;
    const int64_t ir = r_lo + r - I.row0, ic = c_lo + c - I.col0;
    double v = 0.0;
    if (ir >= 0 && ir < I.h && ic >= 0 && ic < I.w) v = load_scalar(I.f, I.dt, ir * I.ld + ic);
    plane[r * ld + c] = v;
  }
}

// RS1 on global rows (one warp per row, shuffle scan over 32-wide chunks).
__global__ void canvas_rs1_kernel(double *g, int64_t ld, int64_t rows, int64_t cols) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (row >= rows) return;
  double *p = g + row * ld;
  double carry = 0.0;
  for (int64_t c0 = 0; c0 < cols; c0 += 32) {
    const int64_t c = c0 + lane;
    double v = c < cols ? p[c] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    v += carry;
    if (c < cols) p[c] = v * kSqrt2;
    carry = __shfl_sync(0xffffffffu, v, 31);
  }
}

// RS2 / RS3 / RS4 on global memory: one thread per line, coalesced across
// neighbouring lines.  dir: 2 = (+1,+1), 3 = (0,+1), 4 = (-1,+1).
__global__ void canvas_line_kernel(double *g, int64_t ld, int64_t rows, int64_t cols, int dir,
                                   unsigned long long *gbits) {
  const int64_t L = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double gm = 0.0;
  if (dir == 3) {
    if (L < cols) {
      double *p = g + L;
      double s = 0.0;
      for (int64_t r = 0; r < rows; ++r, p += ld) {
        s += *p;
        *p = s * kSqrt2;
      }
    }
  } else if (dir == 2) {
    if (L < rows + cols - 1) {
      const int64_t k = L - (rows - 1);
      const int64_t r0 = k < 0 ? -k : 0, c0 = k < 0 ? 0 : k;
      const int64_t len = min(rows - r0, cols - c0);
      double *p = g + r0 * ld + c0;
      double s = 0.0;
      for (int64_t j = 0; j < len; ++j, p += ld + 1) {
        s += *p;
        *p = s;
      }
    }
  } else {
    if (L < rows + cols - 1) {
      const int64_t r0 = max((int64_t)0, L - (cols - 1)), c0 = L - r0;
      const int64_t len = min(rows - r0, c0 + 1);
      double *p = g + r0 * ld + c0;
      double s = 0.0;
      for (int64_t j = 0; j < len; ++j, p += ld - 1) {
        s += *p;
        *p = s;
        gm = fmax(gm, fabs(s));
      }
    }
  }
  if (dir == 4) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gm = fmax(gm, __shfl_xor_sync(0xffffffffu, gm, o));
    if ((threadIdx.x & 31) == 0 && gm > 0.0)
      atomicMax(gbits, (unsigned long long)__double_as_longlong(gm));
  }
}

// ---- point interpolation (zp.interpolate API parity) ---------------------
__global__ void interpolate_kernel(const double *__restrict__ plane, int64_t rows, int64_t cols,
                                   int64_t ld, int64_t col0, int64_t row0,
                                   const double *__restrict__ x1, const double *__restrict__ x2,
                                   int64_t n, double *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = x1[i], y = x2[i];
    const double fx = floor(__dadd_rn(x, 0.5)), fy = floor(__dadd_rn(y, 0.5));
    const double d1 = __dsub_rn(fx, x), d2 = __dsub_rn(fy, y);
    const int64_t cb = (int64_t)fx - col0, rb = (int64_t)fy - row0;
    const bool gp = d1 >= -d2, gmn = d1 >= d2;
    const bool xmaj = (gp == gmn);
    // canonical wedge offsets (dx, dy) for the taps N, P, Bm, Bp, Cm, Cp
    int ax, ay, bx, by;
    if (xmaj) {
      ax = d1 >= 0.0 ? 1 : -1; ay = 0; bx = 0; by = 1;
    } else {
      ax = 0; ay = d2 > 0.0 ? 1 : -1; bx = 1; by = 0;
    }
    auto tap = [&](int dx, int dy) {
      int64_t cc = min(max(cb + dx, (int64_t)0), cols - 1);
      int64_t rr = min(max(rb + dy, (int64_t)0), rows - 1);
      return plane[rr * ld + cc];
    };
    const double u = xmaj ? fabs(d1) : fabs(d2);
    const double v = xmaj ? d2 : d1;
    const double g0 = tap(0, 0), N = tap(-ax, -ay), P = tap(ax, ay);
    const double Bm = tap(-bx, -by), Bp = tap(bx, by);
    const double Cm = tap(-ax - bx, -ay - by), Cp = tap(-ax + bx, -ay + by);
    const double sBv = Bm + Bp, dBv = Bm - Bp, sC = Cm + Cp, dC = Cm - Cp;
    const double A0 = fma(4.0, g0, N + P) + sBv;
    const double L1 = N - P;
    const double Caa2 = fma(2.0, P - g0, sC - sBv);
    const double Cab4 = dC - dBv;
    const double Cbb2 = fma(-2.0, g0 + N, sC + sBv);
    const double u2 = u + u, v2 = v + v;
    const double i1 = fma(u, Caa2, fma(2.0, L1, v2 * Cab4));
    const double i2 = fma(v, Cbb2, dBv + dBv);
    out[i] = 0.125 * fma(u2, i1, fma(v2, i2, A0));
  }
}

// ---------------------------------------------------------------------------
// Host side

struct Scratch {
  int device = -1;
  Status *d_status = nullptr;
  Status *h_status = nullptr;  // pinned
  int4 *d_cells = nullptr;
  size_t cells_cap = 0;
  double *d_pass[2] = {nullptr, nullptr};
  size_t pass_cap[2] = {0, 0};
  bool attr_set = false;
};
thread_local Scratch t_scr;

int ensure_scratch() {
  int dev = 0;
  RUBS_CUDA_TRY(cudaGetDevice(&dev));
  if (t_scr.device != dev) {
    t_scr = Scratch();
    t_scr.device = dev;
    RUBS_CUDA_TRY(cudaMalloc(&t_scr.d_status, sizeof(Status)));
    RUBS_CUDA_TRY(cudaMallocHost(&t_scr.h_status, sizeof(Status)));
  }
  if (!t_scr.attr_set) {
    RUBS_CUDA_TRY(cudaFuncSetAttribute(tile_filter_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    t_scr.attr_set = true;
  }
  return RUBS_OK;
}

int ensure_cells(size_t n) {
  if (n > t_scr.cells_cap) {
    if (t_scr.d_cells) cudaFree(t_scr.d_cells);
    t_scr.d_cells = nullptr;
    RUBS_CUDA_TRY(cudaMalloc(&t_scr.d_cells, n * sizeof(int4)));
    t_scr.cells_cap = n;
  }
  return RUBS_OK;
}

int ensure_pass(int k, size_t n) {
  if (n > t_scr.pass_cap[k]) {
    if (t_scr.d_pass[k]) cudaFree(t_scr.d_pass[k]);
    t_scr.d_pass[k] = nullptr;
    RUBS_CUDA_TRY(cudaMalloc(&t_scr.d_pass[k], n * sizeof(double)));
    t_scr.pass_cap[k] = n;
  }
  return RUBS_OK;
}

int status_to_code(const Status &s) {
  if (s.flags & kFlagFieldNonFinite)
    return set_error(RUBS_EVALUE, "scale field entries must be finite");
  if (s.flags & kFlagParamInvalid)
    return set_error(RUBS_EVALUE,
                     "size must be positive and finite, elongation >= 1 and finite, "
                     "orientation in [0, pi)");
  if (s.flags & kFlagOutOfGrid) return set_error(RUBS_EOUTOFGRID, "elongation beyond table maximum");
  if (s.flags & kFlagRegionTooLarge)
    return set_error(RUBS_EUNSUPPORTED,
                     "kernel support exceeds the on-chip region capacity of this build");
  double g;
  unsigned long long b = s.guard_bits;
  std::memcpy(&g, &b, sizeof(g));
  if (g >= 9007199254740992.0) {
    char buf[160];
    std::snprintf(buf, sizeof(buf),
                  "running sums reached %.3e, beyond the 2^53 precision guard; "
                  "split the image or reduce its dynamic range",
                  g);
    return set_error(RUBS_EOVERFLOW, buf);
  }
  return RUBS_OK;
}

int fetch_status(cudaStream_t s, Status &out) {
  RUBS_CUDA_TRY(cudaMemcpyAsync(t_scr.h_status, t_scr.d_status, sizeof(Status),
                                cudaMemcpyDeviceToHost, s));
  RUBS_CUDA_TRY(cudaStreamSynchronize(s));
  out = *t_scr.h_status;
  timer_collect();
  return RUBS_OK;
}

int launch_cells(const FieldSpec &F, const DomainSpec &D, int global_out, cudaStream_t s,
                 int &cells_x) {
  cells_x = (D.pw + kCell - 1) / kCell;
  const int cells_y = (D.ph + kCell - 1) / kCell;
  int rc = ensure_cells((size_t)cells_x * cells_y);
  if (rc) return rc;
  {
    TimedLaunch tl(1, s);
    cell_margins_kernel<<<cells_x * cells_y, 256, 0, s>>>(F, D, cells_x, t_scr.d_cells,
                                                          t_scr.d_status, global_out);
  }
  ++t_launches;
  RUBS_CUDA_TRY(cudaGetLastError());
  return RUBS_OK;
}

int launch_pass(const ImageSpec &I, const FieldSpec &F, const DomainSpec &D, int cells_x,
                cudaStream_t s) {
  const int tiles_x = (D.pw + kTile - 1) / kTile, tiles_y = (D.ph + kTile - 1) / kTile;
  {
    TimedLaunch tl(0, s);
    tile_filter_kernel<<<tiles_x * tiles_y, kThreads, kSmemBytes, s>>>(
        I, F, D, t_scr.d_cells, cells_x, tiles_x, kRegionCap, t_scr.d_status);
  }
  ++t_launches;
  RUBS_CUDA_TRY(cudaGetLastError());
  return RUBS_OK;
}

// engine.filter_space_variant orchestration (engine.py:285-324) on device.
int run_filter(const ImageSpec &img, FieldSpec F, int iterations, double *out, int64_t ld_out,
               cudaStream_t s) {
  if (img.h < 0 || img.w < 0) return set_error(RUBS_EVALUE, "image must be 2-D");
  if (iterations < 1) return set_error(RUBS_EVALUE, "iterations must be >= 1");
  int rc = ensure_scratch();
  if (rc) return rc;
  if (img.h == 0 || img.w == 0) return RUBS_OK;
  F.FH = img.h;
  F.FW = img.w;
  F.div = std::sqrt((double)iterations);
  F.scaled = iterations > 1;
  RUBS_CUDA_TRY(cudaMemsetAsync(t_scr.d_status, 0, sizeof(Status), s));
  DomainSpec D{0, 0, img.w, img.h, out, ld_out};
  int cells_x = 0;
  if (iterations == 1) {
    if ((rc = launch_cells(F, D, 0, s, cells_x))) return rc;
    if ((rc = launch_pass(img, F, D, cells_x, s))) return rc;
  } else {
    // whole-field margins (engine.py:295) decide the pass canvases
    if ((rc = launch_cells(F, D, 1, s, cells_x))) return rc;
    Status st;
    if ((rc = fetch_status(s, st))) return rc;
    if ((rc = status_to_code(st))) return rc;
    const int left = st.gm[0], right = st.gm[1], below = st.gm[2], above = st.gm[3];
    ImageSpec cur = img;
    for (int p = 0; p < iterations; ++p) {
      const int remain = iterations - 1 - p;
      DomainSpec Dp;
      Dp.pc_lo = -remain * left;
      Dp.pr_lo = -remain * below;
      Dp.pw = img.w + remain * (left + right);
      Dp.ph = img.h + remain * (below + above);
      if (remain == 0) {
        Dp.out = out;
        Dp.ld_out = ld_out;
      } else {
        const int k = p & 1;
        if ((rc = ensure_pass(k, (size_t)Dp.pw * Dp.ph))) return rc;
        Dp.out = t_scr.d_pass[k];
        Dp.ld_out = Dp.pw;
      }
      if ((rc = launch_cells(F, Dp, 0, s, cells_x))) return rc;
      if ((rc = launch_pass(cur, F, Dp, cells_x, s))) return rc;
      cur = ImageSpec{Dp.out, 1, Dp.ld_out, Dp.ph, Dp.pw, Dp.pc_lo, Dp.pr_lo};
    }
  }
  Status st;
  if ((rc = fetch_status(s, st))) return rc;
  return status_to_code(st);
}

// Host-buffer staging for the _host entry points (copies inside the call).
struct HostStage {
  void *buf[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t cap[5] = {0, 0, 0, 0, 0};
  cudaStream_t stream = nullptr;
  int device = -1;
};
thread_local HostStage t_stage;

int stage_buf(int k, size_t bytes, void **out) {
  if (bytes > t_stage.cap[k]) {
    if (t_stage.buf[k]) cudaFree(t_stage.buf[k]);
    t_stage.buf[k] = nullptr;
    RUBS_CUDA_TRY(cudaMalloc(&t_stage.buf[k], bytes));
    t_stage.cap[k] = bytes;
  }
  *out = t_stage.buf[k];
  return RUBS_OK;
}

int stage_stream(cudaStream_t *s) {
  int dev = 0;
  RUBS_CUDA_TRY(cudaGetDevice(&dev));
  if (t_stage.device != dev || !t_stage.stream) {
    t_stage = HostStage();
    t_stage.device = dev;
    RUBS_CUDA_TRY(cudaStreamCreateWithFlags(&t_stage.stream, cudaStreamNonBlocking));
  }
  *s = t_stage.stream;
  return RUBS_OK;
}

}  // namespace

struct rubs_lut {
  double *entries = nullptr;
  int n_rho = 0, n_phi = 0;
  double rho_max = 0.0;
};

namespace {
FieldSpec lut_field(const rubs_lut *lut, const void *size, const void *elong, const void *orient,
                    int p_dtype, int64_t ld_p) {
  FieldSpec F{};
  F.mode = 2;
  F.ps = size;
  F.pr = elong;
  F.pt = orient;
  F.pdt = p_dtype;
  F.pld = ld_p;
  F.lut = lut->entries;
  F.n_rho = lut->n_rho;
  F.n_phi = lut->n_phi;
  F.rho_max = lut->rho_max;
  F.log_rho_max = std::log(lut->rho_max);
  return F;
}
}  // namespace

extern "C" {

const char *rubs_b200_version(void) { return "rubs_b200 0.1.0 (sm_100a)"; }

void rubs_b200_set_profiling(int enable) { t_timer.on = enable != 0; }

void rubs_b200_kernel_time(int kind, double *total_ms, int64_t *launches) {
  double ms = 0.0;
  int64_t n = 0;
  for (int k = 0; k < 2; ++k)
    if (kind == k || kind == 2) {
      ms += t_timer.ms[k];
      n += t_timer.n[k];
    }
  if (total_ms) *total_ms = ms;
  if (launches) *launches = n;
}

void rubs_b200_reset_kernel_time(void) {
  t_timer.ms[0] = t_timer.ms[1] = 0.0;
  t_timer.n[0] = t_timer.n[1] = 0;
}
const char *rubs_b200_last_error(void) { return t_last_error.c_str(); }
int64_t rubs_b200_launch_count(void) { return t_launches; }
void rubs_b200_reset_launch_count(void) { t_launches = 0; }

int rubs_b200_filter(const void *f, int f_dtype, int64_t H, int64_t W, int64_t ld_f,
                     const double *field, int field_is_uniform, int64_t ld_field, int iterations,
                     double *out, int64_t ld_out, void *stream) {
  if (f_dtype != RUBS_F32 && f_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (H > (1 << 30) || W > (1 << 30)) return set_error(RUBS_EUNSUPPORTED, "image too large");
  ImageSpec I{f, f_dtype, ld_f, (int)H, (int)W, 0, 0};
  FieldSpec F{};
  if (field_is_uniform) {
    F.mode = 1;
    for (int k = 0; k < 4; ++k) {
      F.u[k] = field[k];
      if (!std::isfinite(field[k])) return set_error(RUBS_EVALUE, "scale field entries must be finite");
    }
  } else {
    F.mode = 0;
    F.a = field;
    F.ld = ld_field;
  }
  return run_filter(I, F, iterations, out, ld_out, static_cast<cudaStream_t>(stream));
}

int rubs_b200_filter_host(const void *f, int f_dtype, int64_t H, int64_t W, const double *field,
                          int field_is_uniform, int iterations, double *out) {
  cudaStream_t s;
  int rc = stage_stream(&s);
  if (rc) return rc;
  const size_t esz = f_dtype == RUBS_F64 ? 8 : 4;
  const size_t npx = (size_t)H * W;
  void *df, *dfield = nullptr, *dout;
  if ((rc = stage_buf(0, npx * esz, &df))) return rc;
  if ((rc = stage_buf(2, npx * 8, &dout))) return rc;
  RUBS_CUDA_TRY(cudaMemcpyAsync(df, f, npx * esz, cudaMemcpyHostToDevice, s));
  if (!field_is_uniform) {
    if ((rc = stage_buf(1, npx * 32, &dfield))) return rc;
    RUBS_CUDA_TRY(cudaMemcpyAsync(dfield, field, npx * 32, cudaMemcpyHostToDevice, s));
  }
  rc = rubs_b200_filter(df, f_dtype, H, W, W, field_is_uniform ? field : (const double *)dfield,
                        field_is_uniform, W, iterations, (double *)dout, W, s);
  if (rc) return rc;
  RUBS_CUDA_TRY(cudaMemcpyAsync(out, dout, npx * 8, cudaMemcpyDeviceToHost, s));
  RUBS_CUDA_TRY(cudaStreamSynchronize(s));
  return RUBS_OK;
}

int rubs_b200_lut_create(const double *rho_grid, const double *phi_grid, const double *entries,
                         int n_rho, int n_phi, rubs_lut **out) {
  if (n_rho < 2 || n_phi < 2) return set_error(RUBS_EVALUE, "grid needs at least 2 points per axis");
  (void)phi_grid;
  rubs_lut *L = new rubs_lut();
  L->n_rho = n_rho;
  L->n_phi = n_phi;
  L->rho_max = rho_grid[n_rho - 1];
  size_t bytes = (size_t)n_rho * n_phi * 4 * sizeof(double);
  cudaError_t e = cudaMalloc(&L->entries, bytes);
  if (e == cudaSuccess) e = cudaMemcpy(L->entries, entries, bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (L->entries) cudaFree(L->entries);
    delete L;
    return set_error(RUBS_ECUDA, std::string("lut upload: ") + cudaGetErrorString(e));
  }
  *out = L;
  return RUBS_OK;
}

void rubs_b200_lut_destroy(rubs_lut *lut) {
  if (!lut) return;
  if (lut->entries) cudaFree(lut->entries);
  delete lut;
}

int rubs_b200_lookup(const rubs_lut *lut, const void *size, const void *elong, const void *orient,
                     int p_dtype, int64_t n, double *out, void *stream) {
  int rc = ensure_scratch();
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n <= 0) return RUBS_OK;
  FieldSpec F = lut_field(lut, size, elong, orient, p_dtype, 0);
  RUBS_CUDA_TRY(cudaMemsetAsync(t_scr.d_status, 0, sizeof(Status), s));
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  lookup_kernel<<<blocks, 256, 0, s>>>(F, n, out, t_scr.d_status);
  ++t_launches;
  RUBS_CUDA_TRY(cudaGetLastError());
  Status st;
  if ((rc = fetch_status(s, st))) return rc;
  return status_to_code(st);
}

int rubs_b200_filter_params(const void *f, int f_dtype, int64_t H, int64_t W, int64_t ld_f,
                            const void *size, const void *elong, const void *orient, int p_dtype,
                            int64_t ld_p, const rubs_lut *lut, int iterations, double *out,
                            int64_t ld_out, void *stream) {
  if (f_dtype != RUBS_F32 && f_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (p_dtype != RUBS_F32 && p_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (!lut) return set_error(RUBS_EVALUE, "lut is NULL");
  ImageSpec I{f, f_dtype, ld_f, (int)H, (int)W, 0, 0};
  FieldSpec F = lut_field(lut, size, elong, orient, p_dtype, ld_p);
  return run_filter(I, F, iterations, out, ld_out, static_cast<cudaStream_t>(stream));
}

int rubs_b200_filter_params_host(const void *f, int f_dtype, int64_t H, int64_t W,
                                 const void *size, const void *elong, const void *orient,
                                 int p_dtype, const rubs_lut *lut, int iterations, double *out) {
  cudaStream_t s;
  int rc = stage_stream(&s);
  if (rc) return rc;
  const size_t esz = f_dtype == RUBS_F64 ? 8 : 4, psz = p_dtype == RUBS_F64 ? 8 : 4;
  const size_t npx = (size_t)H * W;
  void *df, *dp, *dout;
  if ((rc = stage_buf(0, npx * esz, &df))) return rc;
  if ((rc = stage_buf(1, npx * psz * 3, &dp))) return rc;
  if ((rc = stage_buf(2, npx * 8, &dout))) return rc;
  char *pb = static_cast<char *>(dp);
  RUBS_CUDA_TRY(cudaMemcpyAsync(df, f, npx * esz, cudaMemcpyHostToDevice, s));
  RUBS_CUDA_TRY(cudaMemcpyAsync(pb, size, npx * psz, cudaMemcpyHostToDevice, s));
  RUBS_CUDA_TRY(cudaMemcpyAsync(pb + npx * psz, elong, npx * psz, cudaMemcpyHostToDevice, s));
  RUBS_CUDA_TRY(cudaMemcpyAsync(pb + 2 * npx * psz, orient, npx * psz, cudaMemcpyHostToDevice, s));
  rc = rubs_b200_filter_params(df, f_dtype, H, W, W, pb, pb + npx * psz, pb + 2 * npx * psz,
                               p_dtype, W, lut, iterations, (double *)dout, W, s);
  if (rc) return rc;
  RUBS_CUDA_TRY(cudaMemcpyAsync(out, dout, npx * 8, cudaMemcpyDeviceToHost, s));
  RUBS_CUDA_TRY(cudaStreamSynchronize(s));
  return RUBS_OK;
}

int rubs_b200_preintegrate_shape(int64_t h, int64_t w, int64_t col0, int64_t row0,
                                 int64_t need_c0, int64_t need_c1, int64_t need_r0,
                                 int64_t need_r1, int64_t *rows, int64_t *cols, int64_t *c_lo,
                                 int64_t *r_lo) {
  // engine.py:174-177
  const int64_t cl = std::min(need_c0, col0);
  const int64_t rl = std::min(need_r0, row0 - 1);
  const int64_t rh = std::max(need_r1, row0 + h - 1);
  const int64_t ch = std::max(need_c1, col0 + w - 1) + (rh - row0) + 1;
  *rows = rh - rl + 1;
  *cols = ch - cl + 1;
  *c_lo = cl;
  *r_lo = rl;
  return RUBS_OK;
}

int rubs_b200_preintegrate(const void *f, int f_dtype, int64_t h, int64_t w, int64_t ld_f,
                           int64_t col0, int64_t row0, int64_t need_c0, int64_t need_c1,
                           int64_t need_r0, int64_t need_r1, double *plane, int64_t ld_plane,
                           void *stream) {
  int rc = ensure_scratch();
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int64_t rows, cols, c_lo, r_lo;
  rubs_b200_preintegrate_shape(h, w, col0, row0, need_c0, need_c1, need_r0, need_r1, &rows, &cols,
                               &c_lo, &r_lo);
  ImageSpec I{f, f_dtype, ld_f, (int)h, (int)w, (int)col0, (int)row0};
  RUBS_CUDA_TRY(cudaMemsetAsync(t_scr.d_status, 0, sizeof(Status), s));
  canvas_fill_kernel<<<148 * 8, 256, 0, s>>>(I, plane, ld_plane, rows, cols, c_lo, r_lo);
  ++t_launches;
  // sweeps only touch rows at and above the image (engine.py:182-184)
  const int64_t skip = row0 - r_lo;
  double *g = plane + skip * ld_plane;
  const int64_t grows = rows - skip;
  if (grows > 0) {
    canvas_rs1_kernel<<<(int)((grows * 32 + 255) / 256), 256, 0, s>>>(g, ld_plane, grows, cols);
    const int64_t nl = grows + cols - 1;
    canvas_line_kernel<<<(int)((nl + 255) / 256), 256, 0, s>>>(g, ld_plane, grows, cols, 2,
                                                               &t_scr.d_status->guard_bits);
    canvas_line_kernel<<<(int)((cols + 255) / 256), 256, 0, s>>>(g, ld_plane, grows, cols, 3,
                                                                 &t_scr.d_status->guard_bits);
    canvas_line_kernel<<<(int)((nl + 255) / 256), 256, 0, s>>>(g, ld_plane, grows, cols, 4,
                                                               &t_scr.d_status->guard_bits);
    t_launches += 4;
  }
  RUBS_CUDA_TRY(cudaGetLastError());
  Status st;
  if ((rc = fetch_status(s, st))) return rc;
  return status_to_code(st);
}

int rubs_b200_interpolate(const double *plane, int64_t rows, int64_t cols, int64_t ld_plane,
                          int64_t col0, int64_t row0, const double *x1, const double *x2, int64_t n,
                          double *out, void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n <= 0) return RUBS_OK;
  if (rows <= 0 || cols <= 0) return set_error(RUBS_EVALUE, "empty plane");
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  interpolate_kernel<<<blocks, 256, 0, s>>>(plane, rows, cols, ld_plane, col0, row0, x1, x2, n, out);
  ++t_launches;
  RUBS_CUDA_TRY(cudaGetLastError());
  RUBS_CUDA_TRY(cudaStreamSynchronize(s));
  return RUBS_OK;
}

}  // extern "C"
