// rubs_b200.cu -- B200 (sm_100a) kernels and the C ABI (include/rubs_b200.h)
// for the reference's hot path, engine.filter_space_variant
// (pkg/src/rubs/engine.py:265-324).
//
// Design (DESIGN.md has the full story):
//   * The output domain is cut into 64x32 tiles (wide_filter_kernel, two CTAs
//     per SM).  Every tile pre-integrates ITS OWN region -- the tile grown by
//     the read margins of its own pixels -- in shared memory (TMA loads), with
//     the running sums restarted at the region edge.  This is exact: the
//     filter is linear and zero-padded, so cropping f to the region changes
//     nothing for the tile's pixels, and restarting a sweep on a rectangle
//     only adds ridge functions (constant along one of the four box
//     directions) that the 16-vertex finite difference annihilates.  No
//     canvas widening (engine.py:177) is needed and the sums stay
//     O(region^4) instead of O(image^4), which is what keeps every config
//     inside 1e-9.  A tile whose region is too large or too ill-conditioned
//     is split into smaller units, down to 8x8 cells.
//   * The four sweeps (engine.py:186-193) run in shared memory, one thread
//     per row / diagonal / column / anti-diagonal.
//   * Each pixel then takes its 16-vertex finite difference (engine.py:232-244)
//     reading the region through the 7-tap ZP interpolant (zp.py:186-228) in
//     one canonical-wedge form (zp_read8).
//   * Cells whose regions exceed the shared memory are deferred: planned on
//     the device (plan_* kernels) into the 225 KB shared-memory overflow pass
//     or into power-of-two blocks whose regions live in global scratch
//     (big_fill_rs1 / big_rs234 or the line sweeps / big_gather); pixels
//     whose own precision budget fails go to a per-pixel pass.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <string>
#include <vector>

#include "../../include/rubs_b200.h"
#include "rubs_device.cuh"
#include "rubs_internal.h"

using namespace rubs;

namespace {

constexpr int kTile = 32;        // output tile edge
constexpr int kThreadsSmall = 256;  // primary launch: 2 CTAs per SM
constexpr int kThreadsLarge = 512;  // overflow launch: 1 CTA per SM
constexpr int kSmemSmall = 112 * 1024;  // dynamic shared memory, primary CTA
constexpr int kSmemLarge = 225 * 1024;  // overflow CTA (+ static <= 227 KiB)

thread_local std::string t_last_error;
thread_local int t_precision_limited = 0;  // since the last rubs_b200_precision_limited()
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
  // a bracket whose end event has not completed yet (one still open around
  // the read that triggered this collection closes later) stays pending
  size_t keep = 0;
  for (auto &p : t_timer.pending) {
    if (cudaEventQuery(p.second.second) == cudaErrorNotReady) {
      t_timer.pending[keep++] = p;
      continue;
    }
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.second.first, p.second.second) == cudaSuccess) {
      t_timer.ms[p.first] += ms;
      t_timer.n[p.first] += 1;
    }
    t_timer.pool.push_back(p.second.first);
    t_timer.pool.push_back(p.second.second);
  }
  t_timer.pending.resize(keep);
  (void)cudaGetLastError();  // cudaErrorNotReady is not sticky, but leave no trace
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

// Largest LUT size parameter over the field grid (positive finite values;
// anything else is left to the passes' validation).  Bounds the iterated
// canvases in LUT modes without mapping every pixel (see run_filter).
__global__ void __launch_bounds__(256) size_max_kernel(FieldSpec F, Status *st) {
  double m = 0.0;
  const int64_t n = (int64_t)F.FH * F.FW;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F.FW, c = i - r * F.FW;
    const double v = load_scalar(F.ps, F.pdt, r * F.pld + c);
    if (v > m && v < INFINITY) m = v;
  }
  unsigned long long b = (unsigned long long)__double_as_longlong(m);
  b = max(b, __shfl_xor_sync(0xffffffffu, b, 16));
  b = max(b, __shfl_xor_sync(0xffffffffu, b, 8));
  b = max(b, __shfl_xor_sync(0xffffffffu, b, 4));
  b = max(b, __shfl_xor_sync(0xffffffffu, b, 2));
  b = max(b, __shfl_xor_sync(0xffffffffu, b, 1));
  if ((threadIdx.x & 31) == 0) atomicMax(&st->smax_bits, b);
}

// Whole-field margins (the reference's _read_margins, engine.py:247-262),
// needed before launch only when iterations > 1 (they size the extended
// pass canvases).  One CTA per 16x16 cell, exact reference arithmetic.
__global__ void __launch_bounds__(256) global_margins_kernel(FieldSpec F, DomainSpec D,
                                                             int cells_x, Status *st) {
  const int cx = blockIdx.x % cells_x, cy = blockIdx.x / cells_x;
  const int x = cx * 16 + (threadIdx.x & 15), y = cy * 16 + (threadIdx.x >> 4);
  unsigned flags = 0;
  int4 m = make_int4(0, 0, 0, 0);
  if (x < D.pw && y < D.ph) {
    double a[4];
    field_at_rt(F, D.pc_lo + x, D.pr_lo + y, a, flags);
    m = pixel_margins(a);
  }
  m.x = __reduce_max_sync(0xffffffffu, m.x);
  m.y = __reduce_max_sync(0xffffffffu, m.y);
  m.z = __reduce_max_sync(0xffffffffu, m.z);
  m.w = __reduce_max_sync(0xffffffffu, m.w);
  flags = __reduce_or_sync(0xffffffffu, flags);
  if ((threadIdx.x & 31) == 0) {
    if (flags) atomicOr(&st->flags, flags);
    atomicMax(&st->gm[0], m.x);
    atomicMax(&st->gm[1], m.y);
    atomicMax(&st->gm[2], m.z);
    atomicMax(&st->gm[3], m.w);
  }
}

// Load the image over region lattice [rc0, rc0+RW) x [rr0, rr0+RH) into
// shared memory as fp64, zero outside the image (zero padding, engine.py:155).
// float64 images: asynchronous global->shared copies (cp.async, LDGSTS) of
// the in-image part of each row, plain zero stores outside, so every element
// of the region is in flight at once.  float32 images: eight loads in flight
// per thread, widened to fp64 on the way.

// Synchronise the NT threads of a group: the whole CTA (BAR 0), one warp
// (BAR -1) or a named barrier shared by a subset of warps.
template <int NT, int BAR>
__device__ __forceinline__ void group_sync() {
  if constexpr (BAR == 0)
    __syncthreads();
  else if constexpr (BAR < 0)
    __syncwarp();  // a one-warp group
  else
    asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
}

// Region row pitch (doubles): >= RW and = 4 (mod 16).  With the 4x8-pixel
// warp shape of the gather, the rows a half-warp reads are about one pitch
// apart, i.e. 4 bank pairs apart, so its 16 near-consecutive taps spread over
// all 16 bank pairs.  All sweeps are conflict-free for any pitch.
__host__ __device__ __forceinline__ int region_pitch(int RW) { return RW + ((20 - (RW & 15)) & 15); }
// Shared-memory footprint (doubles) of an RW x RH region: rows rounded up to
// the 8-row TMA box.
__host__ __device__ __forceinline__ int region_elems(int RW, int RH) {
  return region_pitch(RW) * ((RH + 7) & ~7);
}
// float64 regions start on an even image column (a TMA box's first column
// must be 16-byte aligned): grow the region one column to the left when
// needed.  Exact -- any region containing the read support is (see top).
template <int DT>
__device__ __forceinline__ void align_region(const ImageSpec &I, int x_lattice, int &left,
                                             int &RW) {
  if (DT == 1 && ((x_lattice - left - I.col0) & 1)) {
    ++left;
    ++RW;
  }
}

// Tensor-memory-accelerator (TMA) region loads for float64 images: one 2-D
// tensor map per region pitch P = 20 + 16 k (box P columns x 8 rows, so a
// box lands with exactly the region's row pitch); out-of-image elements are
// zero-filled by the TMA unit itself.  A region takes ceil(RH / 8) box copies
// issued by one thread, completing on an mbarrier.  Columns [RW, P) and rows
// [RH, ceil8(RH)) receive real image data the sweeps never read.
constexpr int kTmaP0 = 20, kTmaMaps = 15;  // P = 20 .. 244
struct TmaMaps {
  CUtensorMap m[kTmaMaps];
  unsigned valid;  // bit k: map k usable
};

__device__ __forceinline__ void mbar_init(uint32_t mbar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "RUBS_MBAR_WAIT%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
      " @!p bra RUBS_MBAR_WAIT%=;\n}" ::"r"(mbar),
      "r"(phase)
      : "memory");
}

template <int DT, int NT, int BAR>
__device__ __forceinline__ void load_region(double *S, int P, const ImageSpec &I, int rc0,
                                            int rr0, int RW, int RH, int tid,
                                            const TmaMaps *tm, uint32_t mbar, uint32_t &phase) {
  constexpr int nw = NT >> 5;
  const int warp = tid >> 5, lane = tid & 31;
  const int ic0 = rc0 - I.col0, ir0 = rr0 - I.row0;
  if constexpr (DT == 1) {
    const int k = (P - kTmaP0) >> 4;
    // (the box's first column must be 16-byte aligned: align_region makes
    // ic0 even; anything else takes the copy loop below)
    if (tm != nullptr && k < kTmaMaps && ((tm->valid >> k) & 1u) && (ic0 & 1) == 0) {
      // order this group's earlier generic accesses of the buffer before the
      // async-proxy writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      group_sync<NT, BAR>();
      if (tid == 0) {
        const int nbox = (RH + 7) >> 3;
        const uint32_t bytes = (uint32_t)nbox * 64u * (uint32_t)P;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar),
                     "r"(bytes)
                     : "memory");
        const uint32_t sb = (uint32_t)__cvta_generic_to_shared(S);
        const uint64_t map = reinterpret_cast<uint64_t>(&tm->m[k]);
        for (int b = 0; b < nbox; ++b)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3}], [%4];" ::"r"(sb + (uint32_t)b * 64u * (uint32_t)P),
              "l"(map), "r"(ic0), "r"(ir0 + 8 * b), "r"(mbar)
              : "memory");
      }
      mbar_wait(mbar, phase);
      phase ^= 1u;
      return;
    }
  }
  // region columns [cl, ch) lie inside the image
  const int cl = min(RW, max(0, -ic0)), ch = max(cl, min(RW, I.w - ic0));
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(S);
  if (DT == 1 && cl == 0 && ch == RW && ir0 >= 0 && ir0 + RH <= I.h) {
    // interior region: one flat loop over all elements, pointers advanced
    // incrementally (NT elements per step, row carry when c wraps)
    const int n = RW * RH;
    int r = tid / RW, c = tid - r * RW;
    const int sr = NT / RW, sc = NT - sr * RW;
    const double *src = static_cast<const double *>(I.f) + (int64_t)(ir0 + r) * I.ld + ic0 + c;
    uint32_t dst = sb + (uint32_t)(r * P + c) * 8u;
    const int64_t sstep = (int64_t)sr * I.ld + sc, scarry = I.ld - RW;
    const uint32_t dstep = (uint32_t)(sr * P + sc) * 8u, dcarry = (uint32_t)(P - RW) * 8u;
    for (int e = tid; e < n; e += NT) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
      src += sstep;
      dst += dstep;
      c += sc;
      if (c >= RW) {
        c -= RW;
        src += scarry;
        dst += dcarry;
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }
  for (int r = warp; r < RH; r += nw) {
    const int ir = ir0 + r;
    const uint32_t drow = sb + (uint32_t)(r * P) * 8u;
    const bool rin = ir >= 0 && ir < I.h;
    const int c0 = rin ? cl : RW, c1 = rin ? ch : RW;
    // zero fill outside the image
    for (int c = lane; c < c0; c += 32)
      asm volatile("st.shared.f64 [%0], %1;" ::"r"(drow + c * 8u), "d"(0.0) : "memory");
    for (int c = c1 + lane; c < RW; c += 32)
      asm volatile("st.shared.f64 [%0], %1;" ::"r"(drow + c * 8u), "d"(0.0) : "memory");
    if (c0 < c1) {
      if constexpr (DT == 1) {
        const double *src = static_cast<const double *>(I.f) + (int64_t)ir * I.ld + ic0 + c0 + lane;
        uint32_t d = drow + (uint32_t)(c0 + lane) * 8u;
        for (int c = c0 + lane; c < c1; c += 32, src += 32, d += 256u)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
      } else {
        const float *src = static_cast<const float *>(I.f) + (int64_t)ir * I.ld + ic0 + c0 + lane;
        double *dst = S + r * P + c0 + lane;
        int c = c0 + lane;
        for (; c + 96 < c1; c += 128, src += 128, dst += 128) {
          const float v0 = __ldg(src), v1 = __ldg(src + 32), v2 = __ldg(src + 64), v3 = __ldg(src + 96);
          dst[0] = v0; dst[32] = v1; dst[64] = v2; dst[96] = v3;
        }
        for (; c < c1; c += 32, src += 32, dst += 32) *dst = __ldg(src);
      }
    }
  }
  if constexpr (DT == 1) asm volatile("cp.async.wait_all;" ::: "memory");
}

// The four running sums of engine.py:186-193 on the region, started at the
// region edge.  The two x sqrt(2) scalings are folded into the output weight
// (the pipeline is linear), so the plane here is g / 2.  RS2 and RS4 run
// row-synchronously inside a warp (lane = line) so every shared access of a
// warp hits consecutive addresses.  Tracks max high word of |plane| for the
// 2^53 guard.
template <int NT, int BAR>
__device__ __forceinline__ void region_sweeps(double *S, int P, int RW, int RH, unsigned &ghi,
                                              int tid) {
  constexpr int nt = NT, nw = NT >> 5;
  const int warp = tid >> 5, lane = tid & 31;
  // RS1: along +x, one thread per row.  Thread r runs s_r = (P-1) r mod 16
  // steps late, so at every step the 16 rows of a half-warp touch bank pair
  // (r + step) mod 16 -- conflict-free for any pitch.
  for (int r = tid; r < RH; r += nt) {
    const int sk = ((P - 1) * r) & 15;
    double *p = S + r * P - sk;  // p[j] = column j - sk
    const unsigned span = (unsigned)RW;
    double s = 0.0;
    for (int j = 0; j < RW + 15; j += 4) {
      double v[4];
      bool ok[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ok[u] = (unsigned)(j + u - sk) < span;
        v[u] = ok[u] ? p[j + u] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s += v[u];
        if (ok[u]) p[j + u] = s;
      }
    }
  }
  group_sync<NT, BAR>();
  // RS2: g[r][c] += g[r-1][c-1]; lines k = c - r in [-(RH-1), RW-1].
  // Lane = line, all lanes of a warp on the same row: consecutive columns;
  // lane k is active on rows [ta, tb] of its line.
  const int nlines = RH + RW - 1;
  for (int lb = warp * 32; lb < nlines; lb += nw * 32) {
    const int kb = lb - (RH - 1), k = kb + lane;
    const int t0 = max(0, -(kb + 31)), t1 = min(RH - 1, RW - 1 - kb);
    const int ta = max(t0, -k), tb = min(t1, RW - 1 - k);
    const unsigned span = (unsigned)(tb - ta);
    const bool any = tb >= ta;
    double *p = S + t0 * (P + 1) + k;
    const int st = P + 1;
    double s = 0.0;
    for (int t = t0; t <= t1; t += 4, p += 4 * st) {
      double v[4];
      bool ok[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ok[u] = any && (unsigned)(t + u - ta) <= span;
        v[u] = ok[u] ? p[u * st] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s += v[u];
        if (ok[u]) p[u * st] = s;
      }
    }
  }
  group_sync<NT, BAR>();
  // RS3: along +y (one thread per column)
  for (int c = tid; c < RW; c += nt) {
    double *p = S + c;
    double s = 0.0;
    int r = 0;
    for (; r + 4 <= RH; r += 4) {
      const double v0 = p[0], v1 = p[P], v2 = p[2 * P], v3 = p[3 * P];
      s += v0; p[0] = s;
      s += v1; p[P] = s;
      s += v2; p[2 * P] = s;
      s += v3; p[3 * P] = s;
      p += 4 * P;
    }
    for (; r < RH; ++r, p += P) {
      s += *p;
      *p = s;
    }
  }
  group_sync<NT, BAR>();
  // RS4: g[r][c] += g[r-1][c+1]; lines k = c + r in [0, RH+RW-2], lane =
  // line, all lanes of a warp on the same row.
  unsigned gh = 0;
  for (int kb = warp * 32; kb < nlines; kb += nw * 32) {
    const int k = kb + lane;
    const int t0 = max(0, kb - (RW - 1)), t1 = min(RH - 1, kb + 31);
    const int ta = max(t0, k - (RW - 1)), tb = min(t1, k);
    const unsigned span = (unsigned)(tb - ta);
    const bool any = tb >= ta;
    const int st = P - 1;
    double *p = S + t0 * st + k;
    double s = 0.0;
    for (int t = t0; t <= t1; t += 4, p += 4 * st) {
      double v[4];
      bool ok[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ok[u] = any && (unsigned)(t + u - ta) <= span;
        v[u] = ok[u] ? p[u * st] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s += v[u];
        if (ok[u]) {
          p[u * st] = s;
          gh = max(gh, (unsigned)__double2hiint(s) & 0x7fffffffu);
        }
      }
    }
  }
  ghi = max(ghi, gh);
  group_sync<NT, BAR>();
}

// Per-pixel finite difference (engine.py:219-244) over the region plane,
// 16 vertices x 7 ZP taps.  Sb = shared byte address of region element
// (0, 0) shifted so that (m2 * P + m1) * 8 is the element at lattice
// (m1, m2):  Sb = base - (rr0 * P + rc0) * 8.
//
// The 4 x 7 quadratic table of zp.py (exact multiples of 1/8)
// folds into one canonical wedge: partition q (zp.py:82-86) only decides
// which axis is "major" (q in {0, 3}: x) and the sign of the major residual,
// which is +1 exactly when d1 + d2 >= 0 in both cases.  The seven taps are
// the centre, the two major neighbours N (-sign) and P (+sign), the two
// minor neighbours Bm/Bp and the two corners on the N side Cm/Cp.
// 2 x by an exponent increment on the integer pipe (exact for the normal
// values met here; 0 becomes 2^-1022, i.e. stays negligible).
__device__ __forceinline__ double dtwice(double x) {
  return __hiloint2double(__double2hiint(x) + (1 << 20), __double2loint(x));
}

__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ double ld64(uint32_t a) { return lds64(a); }
__device__ __forceinline__ double ld64(const char *p) {
  return __ldg(reinterpret_cast<const double *>(p));
}

// One ZP read (x 8) at the vertex whose nearest lattice element is at byte
// address c (shared: 32-bit address; global: pointer), residual (d1, d2),
// row pitch P8 bytes.
template <class A, class S>
__device__ __forceinline__ double zp_read8(A c, S P8, double d1, double d2) {
  const bool gp = d1 >= -d2;  // d1 + d2 >= 0
  const bool gm = d1 >= d2;   // d1 - d2 >= 0
  const bool xmaj = (gp == gm);
  S sA = xmaj ? (S)8 : P8;
  sA = gp ? sA : -sA;
  const S sB = xmaj ? P8 : (S)8;
  const double u = dabs(xmaj ? d1 : d2);
  const double v = xmaj ? d2 : d1;
  const double g0 = ld64(c);
  const double N = ld64(c - sA);
  const double Pp = ld64(c + sA);
  const double Bm = ld64(c - sB);
  const double Bp = ld64(c + sB);
  const double Cm = ld64(c - sA - sB);
  const double Cp = ld64(c - sA + sB);
  const double sBv = Bm + Bp, dBv = Bm - Bp, sC = Cm + Cp, dC = Cm - Cp;
  const double A0 = fma(4.0, g0, N + Pp) + sBv;
  const double L1 = N - Pp;
  const double Caa2 = fma(2.0, Pp - g0, sC - sBv);
  const double Cab4 = dC - dBv;
  const double Cbb2 = fma(-2.0, g0 + N, sC + sBv);
  const double V = dtwice(v);
  const double i1 = fma(u, Caa2, fma(V, Cab4, dtwice(L1)));
  const double i2 = fma(v, Cbb2, dtwice(dBv));
  return fma(dtwice(u), i1, fma(V, i2, A0));
}

// Per-pixel finite difference (engine.py:219-244) over a region plane,
// 16 vertices x 7 ZP taps.  (n1, n2) = the pixel's lattice position relative
// to the region origin; Sb = byte address of region element (0, 0), so
// Sb + m2 * P8 + m1 * 8 is the element at local lattice (m1, m2).
//
// The 4 x 7 quadratic table of zp.py (exact multiples of 1/8)
// folds into one canonical wedge: partition q (zp.py:82-86) only decides
// which axis is "major" (q in {0, 3}: x) and the sign of the major residual,
// which is +1 exactly when d1 + d2 >= 0 in both cases.  The seven taps are
// the centre, the two major neighbours N (-sign) and P (+sign), the two
// minor neighbours Bm/Bp and the two corners on the N side Cm/Cp.
template <class A, class S>
__device__ __forceinline__ double pixel_fd_t(A Sb, S P8, int n1, int n2, const double a[4]) {
  const double a1 = a[0], a2 = a[1], a3 = a[2], a4 = a[3];
  const double p2 = a2 * kInvSqrt2, p4 = a4 * kInvSqrt2;
  const double t1 = 0.5 * a1 + 0.5 * (p2 - p4) - 0.5;
  const double t2 = 0.5 * a3 + 0.5 * (p2 + p4) - 1.5;
  // 1/8 of the ZP table and the factor 2 folded out of the sweeps
  const double w = 0.25 / (a1 * a2 * a3 * a4);
  const double xb = (double)n1 + t1, yb = (double)n2 + t2;
  double acc = 0.0;
  // vertex i = q1 | q2 << 1 | q3 << 2 | q4 << 4; sign (-1)^popcount
  //   x = xb - (q1 a1 + q2 p2 - q4 p4)   (engine.py:240)
  //   y = yb - (q2 p2 + q3 a3 + q4 p4)   (engine.py:241)
#pragma unroll
  for (int q4 = 0; q4 < 2; ++q4) {
    const double ox[4] = {q4 ? -p4 : 0.0, q4 ? a1 - p4 : a1, q4 ? p2 - p4 : p2,
                          q4 ? (a1 + p2) - p4 : a1 + p2};  // index q1 | q2 << 1
    const double oy[4] = {q4 ? p4 : 0.0, q4 ? p2 + p4 : p2, q4 ? a3 + p4 : a3,
                          q4 ? (p2 + a3) + p4 : p2 + a3};  // index q2 | q3 << 1
    S cx[4];
    A cy[4];
    double dx[4], dy[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int m;
      lattice_split(xb - ox[k], m, dx[k]);
      cx[k] = (S)m * 8;
      lattice_split(yb - oy[k], m, dy[k]);
      cy[k] = Sb + (S)m * P8;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int q1 = j & 1, q2 = (j >> 1) & 1, q3 = (j >> 2) & 1;
      const int ix = q1 | (q2 << 1), iy = q2 | (q3 << 1);
      const double F8 = zp_read8<A, S>(cy[iy] + cx[ix], P8, dx[ix], dy[iy]);
      if ((q1 + q2 + q3 + q4) & 1)
        acc -= F8;
      else
        acc += F8;
    }
  }
  return acc * w;
}

__device__ __forceinline__ double pixel_fd(uint32_t Sb, int P, int n1, int n2, const double a[4]) {
  return pixel_fd_t<uint32_t, int>(Sb, P * 8, n1, n2, a);
}

// Several planes in shared memory, PSTRIDE bytes apart, filtered with the
// same per-pixel kernel (the adaptive_smooth pipeline's channels): the
// vertex geometry, lattice splits and ZP partition choice are computed once
// and each plane is read at the same seven taps.  Per plane the arithmetic
// is that of zp_read8 / pixel_fd_t.
template <int NCH, int PSTRIDE>
__device__ __forceinline__ void zp_read8_n(uint32_t c, int P8, double d1, double d2,
                                           double F8[NCH]) {
  const bool gp = d1 >= -d2;
  const bool gm = d1 >= d2;
  const bool xmaj = (gp == gm);
  int sA = xmaj ? 8 : P8;
  sA = gp ? sA : -sA;
  const int sB = xmaj ? P8 : 8;
  const double u = dabs(xmaj ? d1 : d2);
  const double v = xmaj ? d2 : d1;
  const double V = dtwice(v), U2 = dtwice(u);
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) {
    const uint32_t b = c + (uint32_t)(ch * PSTRIDE);
    const double g0 = lds64(b);
    const double N = lds64(b - sA);
    const double Pp = lds64(b + sA);
    const double Bm = lds64(b - sB);
    const double Bp = lds64(b + sB);
    const double Cm = lds64(b - sA - sB);
    const double Cp = lds64(b - sA + sB);
    const double sBv = Bm + Bp, dBv = Bm - Bp, sC = Cm + Cp, dC = Cm - Cp;
    const double A0 = fma(4.0, g0, N + Pp) + sBv;
    const double L1 = N - Pp;
    const double Caa2 = fma(2.0, Pp - g0, sC - sBv);
    const double Cab4 = dC - dBv;
    const double Cbb2 = fma(-2.0, g0 + N, sC + sBv);
    const double i1 = fma(u, Caa2, fma(V, Cab4, dtwice(L1)));
    const double i2 = fma(v, Cbb2, dtwice(dBv));
    F8[ch] = fma(U2, i1, fma(V, i2, A0));
  }
}

template <int NCH, int PSTRIDE>
__device__ __forceinline__ void pixel_fd_n(uint32_t Sb, int P8, int n1, int n2, const double a[4],
                                           double out[NCH]) {
  const double a1 = a[0], a2 = a[1], a3 = a[2], a4 = a[3];
  const double p2 = a2 * kInvSqrt2, p4 = a4 * kInvSqrt2;
  const double t1 = 0.5 * a1 + 0.5 * (p2 - p4) - 0.5;
  const double t2 = 0.5 * a3 + 0.5 * (p2 + p4) - 1.5;
  const double w = 0.25 / (a1 * a2 * a3 * a4);
  const double xb = (double)n1 + t1, yb = (double)n2 + t2;
  double acc[NCH];
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) acc[ch] = 0.0;
#pragma unroll 1
  for (int q4 = 0; q4 < 2; ++q4) {
    const double ox[4] = {q4 ? -p4 : 0.0, q4 ? a1 - p4 : a1, q4 ? p2 - p4 : p2,
                          q4 ? (a1 + p2) - p4 : a1 + p2};
    const double oy[4] = {q4 ? p4 : 0.0, q4 ? p2 + p4 : p2, q4 ? a3 + p4 : a3,
                          q4 ? (p2 + a3) + p4 : p2 + a3};
    int cx[4];
    uint32_t cy[4];
    double dx[4], dy[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int m;
      lattice_split(xb - ox[k], m, dx[k]);
      cx[k] = m * 8;
      lattice_split(yb - oy[k], m, dy[k]);
      cy[k] = Sb + (uint32_t)(m * P8);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int q1 = j & 1, q2 = (j >> 1) & 1, q3 = (j >> 2) & 1;
      const int ix = q1 | (q2 << 1), iy = q2 | (q3 << 1);
      double F8[NCH];
      zp_read8_n<NCH, PSTRIDE>(cy[iy] + cx[ix], P8, dx[ix], dy[iy], F8);
      const bool neg = (q1 + q2 + q3 + q4) & 1;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) acc[ch] = neg ? acc[ch] - F8[ch] : acc[ch] + F8[ch];
    }
  }
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) out[ch] = acc[ch] * w;
}

// Region planning.  A unit is a rectangle of output pixels with its own
// region (the rectangle grown by the maximum read margins of its pixels).
// Precision model (measured): the error of a pixel is about
//   kappa * eps * w * L4,  w = 1 / (a1 a2 a3 a4),  L4 = RW RH min(RW,RH)^2 / 4,
// -- the finite difference cancels running sums of size ~L4 down to O(1)
// with weight w.  kappa is ~0.04 for round kernels but reaches ~0.5 for
// kernels with one floored direction (adaptive_smooth's small kernels:
// a = (1.5, 1.9, 0.3, 0.05) gave 7e-10 at w L4 = 1.1e7), so the budget is
// w L4 <= 5e5, i.e. <= ~3e-11 for round and <= ~1e-10 for skewed kernels.
// Well-conditioned pixels (w small) tolerate big regions; pixels with
// floored widths (w large) need small ones, so a unit whose budget is
// exceeded is cut in halves / quadrants down to 8x8 cells.  Regions that do
// not fit shared memory are cut the same way; 8x8 cells that still do not
// fit send the tile to the overflow launch.  (Config 2 never splits for
// precision: its smallest kernels have w ~ 0.1.)
#ifndef RUBS_PREC_BUDGET
#define RUBS_PREC_BUDGET 5e5f
#endif
constexpr float kPrecisionBudget = RUBS_PREC_BUDGET;  // w * L4 (see above)
// w * L4 from which a pixel that cannot get a smaller region is reported as
// precision-limited: 0.5 * 2^-53 * 2e7 ~ 1e-9
constexpr float kPrecisionWarn = 2.0e7f;

// Per-pixel precision fallback.  The overflow passes share one region among
// many pixels; a pixel whose weight w = 1/(a1 a2 a3 a4) is large (a small,
// partly floored kernel) next to huge kernels would exceed the precision
// budget w L4 in that region.  Such pixels are listed and computed one per
// warp, each with the region of its own taps (pixel_kernel).
constexpr int kPixSlab = 3072;  // doubles of shared memory per warp (24 KB)
// initial deferred-pixel list entries (grown on demand); the environment
// variable RUBS_B200_PIX_LIST_INIT overrides it (tests of the regrow path)
size_t pix_list_init() {
  static const size_t v = [] {
    const char *e = std::getenv("RUBS_B200_PIX_LIST_INIT");
    const long long n = e ? std::atoll(e) : 0;
    return n > 0 ? (size_t)n : (size_t)1 << 22;
  }();
  return v;
}

__device__ __forceinline__ bool defer_pixel(const double a[4], float l4, int x, int y, int2 *pix,
                                            int pix_cap, Status *st) {
  const float w = 1.0f / (float)(a[0] * a[1] * a[2] * a[3]);
  if (pix == nullptr || !(w * l4 > kPrecisionBudget)) return false;
  // only if the pixel's own region fits a warp's slab (large w goes with a
  // small kernel; a pixel that is neither stays in the shared region)
  const int4 m = pixel_margins_fast(a);
  if (region_pitch(1 + m.x + m.y) * (1 + m.z + m.w) > kPixSlab) {
    // neither: the pixel stays in the shared region.  If even its OWN
    // minimal region predicts an error near 1e-9 (kappa eps w L4 with the
    // worst kappa met, 0.5) it is a needle kernel, limited in any region:
    // the call reports it (rubs_b200_precision_limited)
    const float rw = (float)(1 + m.x + m.y), rh = (float)(1 + m.z + m.w), mn = fminf(rw, rh);
    if (w * 0.25f * rw * rh * mn * mn > kPrecisionWarn) atomicOr(&st->flags, kFlagPrecisionLimited);
    return false;
  }
  // beyond the list's capacity the pixel is only counted: the host grows
  // the list to the count and runs the deferred-tile passes again
  const int i = atomicAdd(&st->pix_count, 1);
  if (i < pix_cap) pix[i] = make_int2(x, y);
  return true;
}


struct PlanCtx {
  int m[16][4];     // per 8x8 cell: left, right, below, above
  float w[16];      // per 8x8 cell: max 1/(a1 a2 a3 a4)
};

__device__ __forceinline__ bool plan_unit(const PlanCtx &pc, const DomainSpec &D, int x0, int y0,
                                          int cx0, int cy0, int ncell, int region_cap,
                                          int *d, bool &fits) {
  // cells [cx0, cx0+ncell) x [cy0, cy0+ncell) of the tile (8x8 each)
  const int sx = x0 + cx0 * 8, sy = y0 + cy0 * 8;
  if (sx >= D.pw || sy >= D.ph) return false;
  int u[4] = {0, 0, 0, 0};
  float wm = 0.f;
  for (int cy = cy0; cy < cy0 + ncell; ++cy)
    for (int cx = cx0; cx < cx0 + ncell; ++cx) {
      const int c = cy * 4 + cx;
      for (int j = 0; j < 4; ++j) u[j] = max(u[j], pc.m[c][j]);
      wm = fmaxf(wm, pc.w[c]);
    }
  const int sw = min(8 * ncell, D.pw - sx), sh = min(8 * ncell, D.ph - sy);
  const int RW = sw + u[0] + u[1], RH = sh + u[2] + u[3];
  // (+1: the region may grow a column to start on an even image column)
  const float mn = (float)min(RW + 1, RH);
  const float l4 = 0.25f * (float)(RW + 1) * (float)RH * mn * mn;
  d[0] = sx; d[1] = sy; d[2] = sw; d[3] = sh; d[4] = u[0]; d[5] = u[2]; d[6] = RW; d[7] = RH;
  fits = region_elems(RW + 1, RH) <= region_cap;
  return fits && wm * l4 <= kPrecisionBudget;
}

// One 32x32 output tile of the pass domain, processed by one CTA of NT
// threads (1024 / NT pixels per thread):
//   A. every thread maps its pixels' scale-vectors (field / uniform / LUT,
//      engine.py:291-293 + solver.py:289-335) once and keeps them in
//      registers; the CTA reduces read margins and weights per 8x8 cell;
//   B. each unit's region is loaded into shared memory and pre-integrated;
//   C. every pixel of the unit takes its finite difference from the region.
template <int MODE, int DT, int NT>
__device__ __forceinline__ void process_tile(const ImageSpec &I, const FieldSpec &F,
                                             const DomainSpec &D, int tile, unsigned cmask,
                                             int tiles_x, int region_cap, int *ovf_list,
                                             Status *st, double *S, unsigned &ghi,
                                             unsigned &flags, const TmaMaps *tm, uint32_t mbar,
                                             uint32_t &phase, int2 *pix = nullptr,
                                             int pix_cap = 0) {
  constexpr int PPT = 1024 / NT;   // pixels per thread
  constexpr int NW = NT / 32;      // warps
  __shared__ PlanCtx s_pc;
  __shared__ int s_plan[16][8];
  __shared__ int s_nsub;
  const int tid = threadIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int x0 = tx * kTile, y0 = ty * kTile;
  const int lane = tid & 31, warp = tid >> 5;
  // pixel k of this thread: 4x8-pixel block b = warp + NW k of the tile
  // (8 blocks across, 4 down); lane = column (l & 3) and row (l >> 2).
  // With the region pitch = 4 (mod 16) a half-warp's 4 rows x 4 columns of
  // near-consecutive taps land in distinct bank pairs (64-bit shared loads
  // are served per half-warp): 1.66x ideal wavefronts, 2.05x for 32x1.
  auto px_of = [&](int k, int &x, int &y) {
    const int b = warp + NW * k;
    x = x0 + 4 * (b & 7) + (lane & 3);
    y = y0 + 8 * (b >> 3) + (lane >> 2);
  };
  if (tid < 80) {
    if (tid < 64) s_pc.m[tid >> 2][tid & 3] = 0;
    else s_pc.w[tid - 64] = 0.f;
  }
  __syncthreads();

  // ---- A: scale-vectors (independent per pixel: all in flight), then the
  //         per-8x8-cell maxima of the margins and of w (one cell per warp
  //         and k: a full-warp reduction)
  double av[PPT][4];
  bool valid[PPT];
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    int x, y;
    px_of(k, x, y);
    valid[k] = (x < D.pw) && (y < D.ph);
    field_at<MODE>(F, D.pc_lo + min(x, D.pw - 1), D.pr_lo + min(y, D.ph - 1), av[k], flags);
  }
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    int4 m = make_int4(0, 0, 0, 0);
    float w = 0.f;
    if (valid[k]) {
      m = pixel_margins_fast(av[k]);
      w = 1.0f / (float)(av[k][0] * av[k][1] * av[k][2] * av[k][3]);
    }
    m.x = __reduce_max_sync(0xffffffffu, m.x);
    m.y = __reduce_max_sync(0xffffffffu, m.y);
    m.z = __reduce_max_sync(0xffffffffu, m.z);
    m.w = __reduce_max_sync(0xffffffffu, m.w);
    const int wi = __reduce_max_sync(0xffffffffu, __float_as_int(w));  // w >= 0
    const int b = warp + NW * k;
    const int c = (b >> 3) * 4 + ((b & 7) >> 1);
    if (lane == 0 && ((cmask >> c) & 1u)) {  // cells outside the mask are not computed
      atomicMax(&s_pc.m[c][0], m.x);
      atomicMax(&s_pc.m[c][1], m.y);
      atomicMax(&s_pc.m[c][2], m.z);
      atomicMax(&s_pc.m[c][3], m.w);
      atomicMax(reinterpret_cast<int *>(&s_pc.w[c]), wi);
    }
  }
  __syncthreads();
  if (tid == 0) {
    int n = 0;
    bool fits;
    bool ok = true;
    if (!plan_unit(s_pc, D, x0, y0, 0, 0, 4, region_cap, s_plan[n], fits)) {
      for (int q = 0; q < 4 && ok; ++q) {
        const int qx = (q & 1) * 2, qy = (q >> 1) * 2;
        if (plan_unit(s_pc, D, x0, y0, qx, qy, 2, region_cap, s_plan[n], fits)) {
          ++n;
          continue;
        }
        if (x0 + qx * 8 >= D.pw || y0 + qy * 8 >= D.ph) continue;
        for (int c = 0; c < 4; ++c) {
          const bool good = plan_unit(s_pc, D, x0, y0, qx + (c & 1), qy + (c >> 1), 1, region_cap,
                                      s_plan[n], fits);
          if (x0 + (qx + (c & 1)) * 8 >= D.pw || y0 + (qy + (c >> 1)) * 8 >= D.ph) continue;
          (void)good;
          if (!fits) ok = false;  // even an 8x8 region does not fit
          ++n;
        }
      }
    } else {
      n = 1;
    }
    if (!ok) {
      if (ovf_list) {
        OvfRec r;
        r.tile = tile;
        r.mask = cmask;
        r.m[0] = r.m[1] = r.m[2] = r.m[3] = 0;
        r.w = 0.f;
        for (int c = 0; c < 16; ++c) {
          for (int j = 0; j < 4; ++j) r.m[j] = max(r.m[j], s_pc.m[c][j]);
          r.w = fmaxf(r.w, s_pc.w[c]);
        }
        reinterpret_cast<OvfRec *>(ovf_list)[atomicAdd(&st->ovf_count, 1)] = r;
      } else {
        atomicOr(&st->flags, kFlagRegionTooLarge);
      }
      n = 0;
    }
    s_nsub = n;
  }
  __syncthreads();

  const int nsub = s_nsub;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(S);
  for (int si = 0; si < nsub; ++si) {
    const int sx = s_plan[si][0], sy = s_plan[si][1], sw = s_plan[si][2], sh = s_plan[si][3];
    const int below = s_plan[si][5], RH = s_plan[si][7];
    int left = s_plan[si][4], RW = s_plan[si][6];
    align_region<DT>(I, D.pc_lo + sx, left, RW);
    const int P = region_pitch(RW);
    const float mnu = (float)min(RW, RH);
    const float l4u = 0.25f * (float)RW * (float)RH * mnu * mnu;  // precision model
    // ---- B: region load + running sums
    const int rc0 = D.pc_lo + sx - left, rr0 = D.pr_lo + sy - below;
    load_region<DT, NT, 0>(S, P, I, rc0, rr0, RW, RH, tid, tm, mbar, phase);
    __syncthreads();
    region_sweeps<NT, 0>(S, P, RW, RH, ghi, tid);
    // ---- C: finite differences
    // positions relative to the region origin: small coordinates keep the
    // vertex residuals exact to ~1e-14 (thin kernels difference vertices
    // 0.05 apart; global coordinates up to 32768 would cost ~1e-12 each)
    const uint32_t Sb = sbase;
#pragma unroll 1
    for (int k = 0; k < PPT; ++k) {
      int x, y;
      px_of(k, x, y);
      const int cb = warp + NW * k, cc = (cb >> 3) * 4 + ((cb & 7) >> 1);
      if (valid[k] && ((cmask >> cc) & 1u) && x >= sx && x < sx + sw && y >= sy && y < sy + sh) {
        const int n1 = D.pc_lo + x, n2 = D.pr_lo + y;
        double ak[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          ak[j] = av[0][j];
#pragma unroll
          for (int kk = 1; kk < PPT; ++kk) ak[j] = (k == kk) ? av[kk][j] : ak[j];
        }
        if (defer_pixel(ak, l4u, x, y, pix, pix_cap, st)) continue;
        D.out[(int64_t)y * D.ld_out + x] = pixel_fd(Sb, P, n1 - rc0, n2 - rr0, ak);
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void flush_status(Status *st, unsigned ghi, unsigned flags) {
  ghi = __reduce_max_sync(0xffffffffu, ghi);
  flags = __reduce_or_sync(0xffffffffu, flags);
  if ((threadIdx.x & 31) == 0) {
    if (ghi) atomicMax(&st->guard_hi, ghi);
    if (flags) atomicOr(&st->flags, flags);
  }
}

// Primary launch: one tile per CTA, two CTAs per SM (half the shared
// memory each) so one CTA's load / sweeps overlap the other's gather.
template <int MODE, int DT>
__global__ void __launch_bounds__(kThreadsSmall, 2)
    tile_filter_kernel(ImageSpec I, FieldSpec F, DomainSpec D, int tiles_x, int region_cap,
                       int *ovf_list, Status *st, const __grid_constant__ TmaMaps tm) {
  extern __shared__ __align__(128) double S[];
  __shared__ uint64_t s_mbar;
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&s_mbar);
  if (threadIdx.x == 0) mbar_init(mbar);
  __syncthreads();
  unsigned ghi = 0, flags = 0;
  uint32_t phase = 0;
  process_tile<MODE, DT, kThreadsSmall>(I, F, D, blockIdx.x, 0xffffu, tiles_x, region_cap,
                                        ovf_list, st, S, ghi, flags, &tm, mbar, phase);
  flush_status(st, ghi, flags);
}

// Overflow launch: persistent CTAs with the whole shared memory for the
// tiles whose quadrant regions did not fit the primary configuration.
template <int MODE, int DT>
__global__ void __launch_bounds__(kThreadsLarge, 1)
    tile_overflow_kernel(ImageSpec I, FieldSpec F, DomainSpec D, int tiles_x, int region_cap,
                         const int2 *list, int n, Status *st, int2 *pix, int pix_cap,
                         const __grid_constant__ TmaMaps tm) {
  extern __shared__ __align__(128) double S[];
  __shared__ uint64_t s_mbar;
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&s_mbar);
  if (threadIdx.x == 0) mbar_init(mbar);
  __syncthreads();
  unsigned ghi = 0, flags = 0;
  uint32_t phase = 0;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int2 e = list[i];  // (tile, mask of its deferred 8x8 cells)
    process_tile<MODE, DT, kThreadsLarge>(I, F, D, e.x, (unsigned)e.y, tiles_x, region_cap,
                                          nullptr, st, S, ghi, flags, &tm, mbar, phase, pix,
                                          pix_cap);
  }
  flush_status(st, ghi, flags);
}

// ---------------------------------------------------------------------------
// Primary launch: 64 x 32-pixel tiles, two CTAs of 256 threads per SM.
//
// A wide tile halves the halo overhead of a 32 x 32 one at config-2 margins
// (region elements per pixel ~8.3 -> ~5.6).  To keep registers free for the
// gather, the exact scale-vectors are NOT held across the tile: planning
// uses cheap float32 bounds (read margins, and 1/(a1 a2 a3 a4) from a
// per-LUT-cell table), and each pixel's exact scale-vector is computed in
// the gather loop, one 4 x 8 block ahead, so its global loads overlap the
// previous block's finite differences.
#ifndef RUBS_DEV_SKIP_SWEEPS
#define RUBS_DEV_SKIP_SWEEPS 0  // dev timing experiments only
#endif
#ifndef RUBS_DEV_SKIP_GATHER
#define RUBS_DEV_SKIP_GATHER 0
#endif
constexpr int kWideW = 64, kWideH = 32;
// LUT modes: tiles whose smallest size parameter is at least this are
// planned from float32 bounds (see wide_filter_kernel, phase A)
#ifndef RUBS_BOUND_TILE_SIZE
#define RUBS_BOUND_TILE_SIZE 1500.0f
#endif
constexpr float kBoundTileSize = RUBS_BOUND_TILE_SIZE;
// primary kernel stage 2: tiles whose split units would hold more than this
// many region elements per output pixel (and that fit whole in the 224 KB
// one-CTA-per-SM configuration) are filtered whole by a second launch
#ifndef RUBS_W2_ELEMS
#define RUBS_W2_ELEMS 24.0f
#endif
// (RUBS_B200_W2_ELEMS overrides at run time: A/B runs)
float w2_elems() {
  static const float v = [] {
    const char *e = std::getenv("RUBS_B200_W2_ELEMS");
    return e ? (float)std::atof(e) : RUBS_W2_ELEMS;
  }();
  return v;
}
// CTAs per SM of a wide-kernel launch: 2 (110 KB regions, 384 threads) by
// default; 3 (72 KB, 256 threads) for the two-channel LUT launch of the
// adaptive_smooth pipeline, where it measured faster (1.22 -> 0.95 ms).
constexpr int kSlotsPerSm = 3;  // parked scale-vector slots per SM (any CT)
template <int CT>
__host__ __device__ constexpr int wide_smem() { return (CT == 3 ? 72 : CT == 1 ? 224 : 110) * 1024; }
constexpr int kSmemWide = wide_smem<2>();
constexpr int kMaxSmId = 256;          // bound of %smid (scale-vector slots)
#ifndef RUBS_WIDE_THREADS
#define RUBS_WIDE_THREADS 384
#endif
constexpr int kThreadsWide = RUBS_WIDE_THREADS;  // 2 CTAs per SM
template <int CT>
__host__ __device__ constexpr int wide_threads() { return CT == 3 ? 256 : CT == 1 ? 512 : kThreadsWide; }

// Planning bounds of one pixel: read margins (left, right, below, above)
// covering its taps, and an upper bound of w = 1 / (a1 a2 a3 a4).
// Read margins and w = 1 / (a1 a2 a3 a4) of one pixel whose scale-vector
// comes from a field or a uniform vector (LUT modes compute the exact
// mapping in phase A and park it instead).
template <int MODE>
__device__ __forceinline__ void pixel_bound(const FieldSpec &F, int n1, int n2, int4 &m,
                                            float &w) {
  double a[4];
  unsigned fl = 0;
  field_at<MODE>(F, n1, n2, a, fl);
  m = pixel_margins_fast(a);
  w = 1.0f / (float)(a[0] * a[1] * a[2] * a[3]);
}

// Channels of a multi-channel launch: images (same geometry and dtype as
// the ImageSpec) and outputs (same row stride as the DomainSpec).
struct MultiChan {
  const void *f[3];
  double *out[3];
};
template <int NCH>
struct TmaMapsN {
  TmaMaps m[NCH];
};
// shared memory per channel region (doubles, 128-byte multiple)
template <int NCH, int CT = 2>
__host__ __device__ constexpr int wide_cap() {
  return (wide_smem<CT>() / 8 / NCH) & ~15;
}

// Take the next listed stage-2 tile, or -1.  A take past the end is undone,
// so the counter never overshoots: the streamed path launches stage 2 once
// per band, and a later launch must still find the tiles listed after an
// earlier one ran dry.
__device__ __forceinline__ int w2_take(Status *st, const int *w2_list) {
  const int k = atomicAdd(&st->w2_next, 1);
  if (k < *(volatile int *)&st->w2_count) return w2_list[k];
  atomicSub(&st->w2_next, 1);
  return -1;
}

template <int MODE, int DT, int NT, int NCH, int CT = 2>
__global__ void __launch_bounds__(NT, CT)
    wide_filter_kernel(ImageSpec I, FieldSpec F, DomainSpec D, int tiles_x, int tiles_x32,
                       int region_cap, int *ovf_list, Status *st, double *aslots,
                       unsigned *slotmask, int tile_base, MultiChan mc,
                       const __grid_constant__ TmaMapsN<NCH> tm, int *w2_list, int w2_mode,
                       float w2_elems_px) {
  constexpr int CAP = wide_cap<NCH, CT>();
  constexpr int NW = NT / 32;
  constexpr int NCX = kWideW / 8, NCY = kWideH / 8;  // 8 x 4 cells of 8 x 8
  extern __shared__ __align__(128) double S[];
  __shared__ uint64_t s_mbar;
  __shared__ int s_cm[NCX * NCY][4];
  __shared__ float s_cw[NCX * NCY];
  __shared__ int s_unit[NCX * NCY][8];
  __shared__ int s_nu;
  __shared__ int s_slot;
  __shared__ float s_smin;  // smallest size parameter of the tile (LUT modes)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&s_mbar);
  // LUT modes: the exact scale-vectors of the tile are computed once (phase
  // A) and parked in an L2-resident slot of this SM (two CTAs per SM: two
  // slots, claimed with an atomic bit) until the gather reads them back
  constexpr bool kPark = MODE >= kModeLut;
  // stage 2 (CT == 1) takes its first listed tile before any set-up: with
  // an empty list (the common case on small-kernel fields) every CTA exits
  // at once
  constexpr bool kList = CT == 1;
  __shared__ int s_tile;
  if constexpr (kList) {
    if (tid == 0) s_tile = w2_take(st, w2_list);
    __syncthreads();
    if (s_tile < 0) return;
  }
  unsigned smid = 0;
  if (tid == 0) {
    mbar_init(mbar);
    if (kPark) {
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      int slot = -1;
      while (slot < 0) {
        for (int b = 0; b < CT && slot < 0; ++b)
          if (!(atomicOr(&slotmask[smid], 1u << b) & (1u << b))) slot = (int)smid * kSlotsPerSm + b;
      }
      s_slot = slot;
    }
  }
  unsigned ghi = 0, flags = 0;
  uint32_t phase = 0;
  // w2_mode 0: one tile per CTA (tile_base + blockIdx.x); tiles whose split
  //   units would be costly but whose whole region fits the one-CTA-per-SM
  //   configuration are appended to w2_list (st->w2_count) instead
  // w2_mode 1: persistent CTAs of that configuration take the listed tiles
  //   (st->w2_next); w2_mode 2: one tile per CTA, no list (multi-channel,
  //   streamed bands)
  // (the one-CTA-per-SM configuration, CT == 1, is stage 2 and loops; the
  // others take one tile, so the loop below runs once and compiles away)
  for (int it = 0;; ++it) {
  if (tid == 0) {
    int t = -1;
    if constexpr (kList) {
      if (it == 0) {
        t = s_tile;  // taken above
      } else {
        t = w2_take(st, w2_list);
      }
    } else {
      t = tile_base + blockIdx.x;
    }
    s_tile = t;
  }
  if (tid < 4 * NCX * NCY) (&s_cm[0][0])[tid] = 0;
  if (tid < NCX * NCY) s_cw[tid] = 0.f;
  if (tid == 0) s_smin = INFINITY;
  __syncthreads();
  const int tile = s_tile;
  if (tile < 0) break;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int x0 = tx * kWideW, y0 = ty * kWideH;

  double *const apark =
      kPark ? aslots + (size_t)s_slot * (kWideW * kWideH * 4) : nullptr;
  bool bound_tile = false;  // planned from float32 bounds (phase A)
  // ---- A: read margins and weights of the 2048 pixels; thread = one
  //         column, rows (tid >> 6) + 4 k; 8-lane groups share an 8 x 8 cell
  {
    constexpr int RS = NT / kWideW;  // rows per sweep of the CTA over the tile
    const int px = tid & 63, py = tid / kWideW;  // py is warp-uniform
    int cur = -1;
    int4 acc = make_int4(0, 0, 0, 0);
    float wacc = 0.f;
    // reduce (m, w) over the 8 lanes of each 8 x 8 cell, merge into the cell
    auto flush = [&](int r) {
      int wi = __float_as_int(wacc);  // w >= 0: int order = float order
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        acc.x = max(acc.x, __shfl_xor_sync(0xffffffffu, acc.x, o));
        acc.y = max(acc.y, __shfl_xor_sync(0xffffffffu, acc.y, o));
        acc.z = max(acc.z, __shfl_xor_sync(0xffffffffu, acc.z, o));
        acc.w = max(acc.w, __shfl_xor_sync(0xffffffffu, acc.w, o));
        wi = max(wi, __shfl_xor_sync(0xffffffffu, wi, o));
      }
      if ((lane & 7) == 0) {
        const int c = r * NCX + (px >> 3);
        atomicMax(&s_cm[c][0], acc.x);
        atomicMax(&s_cm[c][1], acc.y);
        atomicMax(&s_cm[c][2], acc.z);
        atomicMax(&s_cm[c][3], acc.w);
        atomicMax(reinterpret_cast<int *>(&s_cw[c]), wi);
      }
      acc = make_int4(0, 0, 0, 0);
      wacc = 0.f;
    };
    constexpr int NK = (kWideH + RS - 1) / RS;
    // LUT modes: all of this thread's parameter loads in flight at once
    using PT = typename std::conditional<MODE == kModeLut, double, float>::type;
    PT pre[kPark ? NK : 1][3];
    if constexpr (kPark) {
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        const int ty_ = py + RS * k;
        const int fc = min(max(D.pc_lo + x0 + px, 0), F.FW - 1);
        const int fr = min(max(D.pr_lo + y0 + min(ty_, kWideH - 1), 0), F.FH - 1) - F.fr_off;
        const int64_t i = (int64_t)fr * F.pld + fc;
        pre[k][0] = __ldg(static_cast<const PT *>(F.ps) + i);
        pre[k][1] = __ldg(static_cast<const PT *>(F.pr) + i);
        pre[k][2] = __ldg(static_cast<const PT *>(F.pt) + i);
      }
    }
    // LUT modes: a tile whose sizes are all large (>= kBoundTileSize) is
    // planned from float32 bounds of its pixels' mapping (lut_bounds_f32)
    // instead of the exact fp64 mapping: such tiles are deferred (config 5:
    // nearly all), and the pass that computes a pixel maps it exactly itself,
    // so the exact mapping is done once.  A unit of such a tile that does fit
    // maps its pixels exactly in the gather (fetch below).
    if constexpr (kPark) {
      float smin = INFINITY;
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        const int ty_ = py + RS * k;
        if (ty_ < kWideH && x0 + px < D.pw && y0 + ty_ < D.ph)
          smin = fminf(smin, fabsf((float)pre[k][0]));
      }
      smin = fminf(smin, __shfl_xor_sync(0xffffffffu, smin, 16));
      smin = fminf(smin, __shfl_xor_sync(0xffffffffu, smin, 8));
      smin = fminf(smin, __shfl_xor_sync(0xffffffffu, smin, 4));
      smin = fminf(smin, __shfl_xor_sync(0xffffffffu, smin, 2));
      smin = fminf(smin, __shfl_xor_sync(0xffffffffu, smin, 1));
      if (lane == 0) atomicMin(reinterpret_cast<int *>(&s_smin), __float_as_int(smin));
      __syncthreads();
    }
    bound_tile = kPark && __int_as_float(*reinterpret_cast<volatile int *>(&s_smin)) >= kBoundTileSize;
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      const int ty_ = py + RS * k;  // tile row (warp-uniform)
      if (ty_ < kWideH) {
        if ((ty_ >> 3) != cur) {
          if (cur >= 0) flush(cur);
          cur = ty_ >> 3;
        }
        const int x = x0 + px, y = y0 + ty_;
        if (x < D.pw && y < D.ph) {
          int4 m;
          float w;
          if constexpr (kPark) {
            if (bound_tile) {
              lut_bounds_f32(F, (double)pre[k][0], (double)pre[k][1], (double)pre[k][2], m, w, flags);
            } else {
              double a[4];
              field_from_params(F, (double)pre[k][0], (double)pre[k][1], (double)pre[k][2], a, flags);
              m = pixel_margins_fast(a);
              w = 1.0f / (float)(a[0] * a[1] * a[2] * a[3]);
              double2 *dst = reinterpret_cast<double2 *>(apark + (ty_ * kWideW + px) * 4);
              dst[0] = make_double2(a[0], a[1]);
              dst[1] = make_double2(a[2], a[3]);
            }
          } else {
            pixel_bound<MODE>(F, D.pc_lo + x, D.pr_lo + y, m, w);
          }
          acc.x = max(acc.x, m.x);
          acc.y = max(acc.y, m.y);
          acc.z = max(acc.z, m.z);
          acc.w = max(acc.w, m.w);
          wacc = fmaxf(wacc, w);
        }
      }
    }
    if (cur >= 0) flush(cur);
  }
  __syncthreads();

  // ---- plan: the whole tile if its region fits and meets the precision
  //      budget, else split the longer side recursively down to 8 x 8
  //      cells; a cell that still fails sends its 32 x 32 half of the tile
  //      (a tile of the overflow launches' 32-pixel grid) to the overflow pass.
  //      The split rule depends only on a node's shape, so the tree is
  //      fixed: 8x4 -> 4x4 -> 2x4 -> 2x2 -> 1x2 -> 1x1 cells.  Warp 0 plans
  //      it with one lane per cell: node aggregates by butterfly max over
  //      the lanes of each level's node, and a node becomes a unit iff it
  //      fits and no ancestor does (exactly the depth-first split's units;
  //      only their order differs, which no result depends on).  The
  //      single-thread tree walk this replaces was ~6 % of the kernel's
  //      stall samples on large kernels (config 3n4), every other warp
  //      waiting at the barrier.
  static_assert(NCX == 8 && NCY == 4, "one lane per cell, fixed split tree");
  if (warp == 0) {
    constexpr int kLv = 6;  // leaf (1x1) first
    constexpr int kLw[kLv] = {1, 1, 2, 2, 4, 8}, kLh[kLv] = {1, 2, 2, 4, 4, 4};
    constexpr int kXor[kLv] = {0, 8, 1, 16, 2, 4};  // lane = cy * 8 + cx
    const int cx = lane & 7, cy = lane >> 3;
    // a node's fit test (as the tree walk did it): region within the
    // buffer and the precision budget met
    auto node = [&](int L, const int *u, float wm, int *d) -> bool {
      const int cx0 = cx & ~(kLw[L] - 1), cy0 = cy & ~(kLh[L] - 1);
      const int sx = x0 + 8 * cx0, sy = y0 + 8 * cy0;
      if (sx >= D.pw || sy >= D.ph) return false;
      const int sw = min(8 * kLw[L], D.pw - sx), sh = min(8 * kLh[L], D.ph - sy);
      const int RW = sw + u[0] + u[1], RH = sh + u[2] + u[3];
      const float mn = (float)min(RW + 1, RH);
      const float l4 = 0.25f * (float)(RW + 1) * (float)RH * mn * mn;
      d[0] = sx; d[1] = sy; d[2] = sw; d[3] = sh; d[4] = u[0]; d[5] = u[2]; d[6] = RW; d[7] = RH;
      return region_elems(RW + 1, RH) <= region_cap && wm * l4 <= kPrecisionBudget;
    };
    int u[4], d[8];
    float wm;
    bool full2 = false;  // the whole tile fits the stage-2 configuration
    unsigned fitm = 0;  // bit L: this lane's level-L node fits
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      // pass 0 finds the levels that fit; pass 1 rebuilds the aggregates of
      // the topmost fitting level (all lanes take part in the shuffles)
      const int top = fitm ? 31 - __clz(fitm) : -1;
      for (int j = 0; j < 4; ++j) u[j] = s_cm[lane][j];
      wm = s_cw[lane];
#pragma unroll
      for (int L = 0; L < kLv; ++L) {
        if (L > 0) {
          for (int j = 0; j < 4; ++j) u[j] = max(u[j], __shfl_xor_sync(0xffffffffu, u[j], kXor[L]));
          wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, kXor[L]));
        }
        if (pass == 0) {
          int dd[8];
          if (node(L, u, wm, dd)) fitm |= 1u << L;
          if (L == kLv - 1) {
            // the whole tile in the one-CTA-per-SM configuration (stage 2)
            const float mn2 = (float)min(dd[6] + 1, dd[7]);
            const float l42 = 0.25f * (float)(dd[6] + 1) * (float)dd[7] * mn2 * mn2;
            full2 = dd[2] > 0 && region_elems(dd[6] + 1, dd[7]) <= wide_cap<1, 1>() &&
                    wm * l42 <= kPrecisionBudget;
          }
        } else if (L == top) {
          node(L, u, wm, d);
        }
      }
    }
    const int top = fitm ? 31 - __clz(fitm) : -1;
    // the unit is written by its node's first lane
    bool writer =
        top >= 0 && cx == (cx & ~(kLw[top] - 1)) && cy == (cy & ~(kLh[top] - 1));
    if (!kList && w2_mode == 0) {
      // stage 2: a tile that the split units would cost more than
      // w2_elems_px region elements per pixel (or that defers cells) but
      // that fits whole in the 224 KB configuration goes to the list
      const bool in_t = x0 + 8 * cx < D.pw && y0 + 8 * cy < D.ph;
      const int re = writer ? region_elems(d[6] + 1, d[7]) : 0;
      const int px = writer ? d[2] * d[3] : 0;
      const int re_sum = __reduce_add_sync(0xffffffffu, re);
      const int px_sum = __reduce_add_sync(0xffffffffu, px);
      const bool any_ovf = __any_sync(0xffffffffu, in_t && top < 0);
      const bool whole = __all_sync(0xffffffffu, !in_t || top == kLv - 1);
      const bool to2 = __shfl_sync(0xffffffffu, (int)full2, 0) && !whole &&
                       (any_ovf || (float)re_sum > w2_elems_px * (float)px_sum);
      if (to2) {
        if (lane == 0) {
          w2_list[atomicAdd(&st->w2_count, 1)] = tile;
          s_nu = 0;
        }
        writer = false;
        fitm = 0;
      }
      if (to2) goto plan_done;
    }
    {
    const unsigned wb = __ballot_sync(0xffffffffu, writer);
    if (writer) {
      int *dst = s_unit[__popc(wb & ((1u << lane) - 1u))];
      for (int j = 0; j < 8; ++j) dst[j] = d[j];
    }
    // a cell no node fits goes to the overflow pass; the rest of the tile
    // keeps its (smaller, better-conditioned) units
    const bool in = x0 + 8 * cx < D.pw && y0 + 8 * cy < D.ph;
    const bool dfr = in && top < 0;
    const unsigned ovf_cells = __ballot_sync(0xffffffffu, dfr);
    if (ovf_cells) {
      // one record per 32 x 32 half with deferred cells (the overflow passes
      // work on the 32-pixel grid), margins and w over those cells: a max
      // over the lanes (cells) of each half, lane 0 / lane 4 write half 0 / 1
      // (one atomic per tile; the serial per-cell loop of lane 0 held the
      // other warps at the barrier)
      int rm[4];
      float rw = 0.f;
      for (int j = 0; j < 4; ++j) rm[j] = dfr ? s_cm[lane][j] : 0;
      if (dfr) rw = s_cw[lane];
#pragma unroll
      for (int o : {1, 2, 8, 16}) {  // lanes of one half: cx bits 0-1, cy bits 3-4
        for (int j = 0; j < 4; ++j) rm[j] = max(rm[j], __shfl_xor_sync(0xffffffffu, rm[j], o));
        rw = fmaxf(rw, __shfl_xor_sync(0xffffffffu, rw, o));
      }
      auto half_mask = [&](int h) {
        unsigned m = 0;
        for (int ccy = 0; ccy < NCY; ++ccy) m |= ((ovf_cells >> (ccy * NCX + 4 * h)) & 0xFu) << (4 * ccy);
        return m;
      };
      const unsigned m0 = half_mask(0), m1 = half_mask(1);
      int base = 0;
      if (lane == 0) base = atomicAdd(&st->ovf_count, (m0 != 0) + (m1 != 0));
      base = __shfl_sync(0xffffffffu, base, 0);
      if ((lane == 0 && m0) || (lane == 4 && m1)) {
        const int h = lane >> 2;
        OvfRec r;
        r.tile = ty * tiles_x32 + 2 * tx + h;
        for (int j = 0; j < 4; ++j) r.m[j] = rm[j];
        r.w = rw;
        r.mask = h ? m1 : m0;
        reinterpret_cast<OvfRec *>(ovf_list)[base + (h && m0 ? 1 : 0)] = r;
      }
    }
    if (lane == 0) s_nu = __popc(wb);
    }
  plan_done:;
  }
  __syncthreads();

  const int nu = s_nu;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(S);
  for (int ui = 0; ui < nu; ++ui) {
    const int sx = s_unit[ui][0], sy = s_unit[ui][1], sw = s_unit[ui][2], sh = s_unit[ui][3];
    const int below = s_unit[ui][5], RH = s_unit[ui][7];
    int left = s_unit[ui][4], RW = s_unit[ui][6];
    align_region<DT>(I, D.pc_lo + sx, left, RW);
    const int P = region_pitch(RW);
    // ---- B: region load (TMA for float64) + running sums
    const int rc0 = D.pc_lo + sx - left, rr0 = D.pr_lo + sy - below;
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
      ImageSpec Ic = I;
      Ic.f = mc.f[ch];
      load_region<DT, NT, 0>(S + ch * CAP, P, Ic, rc0, rr0, RW, RH, tid, &tm.m[ch], mbar, phase);
    }
    __syncthreads();
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch)
      if (!RUBS_DEV_SKIP_SWEEPS) region_sweeps<NT, 0>(S + ch * CAP, P, RW, RH, ghi, tid);
    // ---- C: 4 x 8-pixel blocks of the unit, warp-strided; the exact
    //         scale-vector of the next block is fetched before this one's
    //         finite differences
    const uint32_t Sb = sbase;  // local coordinates (see process_tile)
    const int nbx = (sw + 3) >> 2, nblk = nbx * ((sh + 7) >> 3);
    // block b = by * nbx + bx, walked in steps of NW without a division:
    // (cbx, cby) is the current block, (nbx_, nby_) the next one
    auto block_xy = [&](int bx, int by, int &x, int &y) {
      x = sx + 4 * bx + (lane & 3);
      y = sy + 8 * by + (lane >> 2);
    };
    auto advance = [&](int &bx, int &by) {
      bx += NW;
      while (bx >= nbx) {
        bx -= nbx;
        ++by;
      }
    };
    auto fetch = [&](int x, int y, double a[4]) {
      x = min(x, sx + sw - 1);
      y = min(y, sy + sh - 1);
      if constexpr (kPark) {
        if (bound_tile) {
          field_at<MODE>(F, D.pc_lo + x, D.pr_lo + y, a, flags);  // exact mapping, once
        } else {
          const double2 *p =
              reinterpret_cast<const double2 *>(apark + ((y - y0) * kWideW + (x - x0)) * 4);
          const double2 lo = p[0], hi = p[1];
          a[0] = lo.x; a[1] = lo.y; a[2] = hi.x; a[3] = hi.y;
        }
      } else {
        field_at<MODE>(F, D.pc_lo + x, D.pr_lo + y, a, flags);
      }
    };
    int b = warp;
    int cbx = warp, cby = 0;
    while (cbx >= nbx) {
      cbx -= nbx;
      ++cby;
    }
    double an[4] = {1.0, 1.0, 1.0, 1.0};
    if (b < nblk) {
      int x, y;
      block_xy(cbx, cby, x, y);
      fetch(x, y, an);
    }
#pragma unroll 1
    for (; b < nblk; b += NW) {
      double ac[4] = {an[0], an[1], an[2], an[3]};
      int x, y;
      block_xy(cbx, cby, x, y);
      advance(cbx, cby);
      if (b + NW < nblk) {
        int xn, yn;
        block_xy(cbx, cby, xn, yn);
        fetch(xn, yn, an);
      }
      if (x < sx + sw && y < sy + sh) {
        if constexpr (NCH == 1) {
          D.out[(int64_t)y * D.ld_out + x] =
              RUBS_DEV_SKIP_GATHER ? ac[0]
                                   : pixel_fd(Sb, P, D.pc_lo + x - rc0, D.pr_lo + y - rr0, ac);
        } else {
          double o[NCH];
          pixel_fd_n<NCH, CAP * 8>(Sb, P * 8, D.pc_lo + x - rc0, D.pr_lo + y - rr0, ac, o);
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) mc.out[ch][(int64_t)y * D.ld_out + x] = o[ch];
        }
      }
    }
    __syncthreads();
  }
  if constexpr (!kList) break;
  __syncthreads();  // shared tile state and the region buffer free for the next tile
  }  // tile loop
  if (kPark && tid == 0) atomicAnd(&slotmask[smid], ~(1u << (s_slot % kSlotsPerSm)));
  flush_status(st, ghi, flags);
}

// ---------------------------------------------------------------------------
// Large-halo path: regions in global memory (configs 3 and 5).
//
// Tiles whose 8x8 regions exceed even the 225 KB configuration are grouped
// on the host into square blocks of S = 2^k >= 2 h pixels (h = the tile's
// largest margin; S shrunk further if the w * L4 precision budget demands).
// Each block's region -- its member tiles' bounding box grown by their
// maximum margins -- is pre-integrated in a global scratch buffer by three
// grid-wide kernels (fill + RS1 as one warp scan per row; RS2 / RS3 / RS4
// one lane per line, a warp walking 32 neighbouring lines row by row so
// every access is coalesced), then gathered by a tile kernel that reads the
// taps through L1/L2.  Member tiles are gathered in block-raster order, so
// neighbouring CTAs share the rows their vertices touch in L2.

constexpr int kPixSmem = 8 * kPixSlab * 8;  // 8 warps per CTA
// Doubles of big-block scratch per batch (16 GB of the 180 GB HBM).
// L2-sized batches (8M doubles) were measured 2x slower on config 5: the
// region sweeps draw their parallelism from the number of regions in a
// batch (2^29 -> 2^31 doubles: config 5 180 -> 173 ms).
#ifndef RUBS_BIG_BATCH
#define RUBS_BIG_BATCH (1ll << 31)
#endif
constexpr int64_t kBigBatch = RUBS_BIG_BATCH;
constexpr int64_t kBigMinBatch = 1ll << 24;  // smallest budget tried after allocation failures
// fewer than SMs / kRsFewDiv regions in a batch: segmented line sweeps
// (flat-cost table: 4 regions 3.8 -> 1.6 -> 0.72 ms with segments; 64
// regions keep the fused sweep; below one region per SM measured slower)
constexpr int kRsFewDiv = 8;

template <int MODE, int DT>
__global__ void __launch_bounds__(256) pixel_kernel(ImageSpec I, FieldSpec F, DomainSpec D,
                                                    const int2 *pix, int n, Status *st) {
  extern __shared__ __align__(16) double Sw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double *S = Sw + warp * kPixSlab;
  unsigned flags = 0, ghi = 0;
  for (int i = blockIdx.x * 8 + warp; i < n; i += gridDim.x * 8) {
    const int2 p = pix[i];
    const int n1 = D.pc_lo + p.x, n2 = D.pr_lo + p.y;
    double a[4];
    field_at<MODE>(F, n1, n2, a, flags);
    const int4 m = pixel_margins_fast(a);
    const int RW = 1 + m.x + m.y, RH = 1 + m.z + m.w;
    const int P = region_pitch(RW);
    if (P * RH > kPixSlab) {  // a large kernel never has a large w
      if (lane == 0) atomicOr(&st->flags, kFlagRegionTooLarge);
      continue;
    }
    {
      const float mn = (float)min(RW, RH);
      const float l4own = 0.25f * (float)RW * (float)RH * mn * mn;
      if (l4own / (float)(a[0] * a[1] * a[2] * a[3]) > kPrecisionWarn) flags |= kFlagPrecisionLimited;
    }
    const int rc0 = n1 - m.x, rr0 = n2 - m.z;
    // region load (zero outside the image), then the four running sums
    for (int e = lane; e < RW * RH; e += 32) {
      const int r = e / RW, c = e - r * RW;
      const int ir = rr0 + r - I.row0, ic = rc0 + c - I.col0;
      S[r * P + c] = (ir >= 0 && ir < I.h && ic >= 0 && ic < I.w)
                         ? load_px<DT>(I.f, (int64_t)ir * I.ld + ic) : 0.0;
    }
    __syncwarp();
    region_sweeps<32, -1>(S, P, RW, RH, ghi, lane);
    if (lane == 0) {
      const uint32_t Sb = (uint32_t)__cvta_generic_to_shared(S);
      D.out[(int64_t)p.y * D.ld_out + p.x] = pixel_fd(Sb, P, n1 - rc0, n2 - rr0, a);
    }
    __syncwarp();
  }
  flush_status(st, ghi, flags);
}

struct BigRegion {
  int64_t off;       // element offset of region element (0, 0) in scratch
  int rc0, rr0;      // lattice of region element (0, 0)
  int RW, RH, P;
  float l4;          // RW RH min(RW, RH)^2 / 4 (precision model)
};
struct BigTile {
  int tile, region;
  unsigned mask;  // 8x8 cells of the tile to compute
};

template <int DT>
__global__ void __launch_bounds__(256) big_fill_rs1_kernel(ImageSpec I, const BigRegion *R,
                                                           double *scratch) {
  const BigRegion g = R[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  if (row >= g.RH) return;
  double *dst = scratch + g.off + (int64_t)row * g.P;
  const int ir = g.rr0 + row - I.row0;
  const bool rin = ir >= 0 && ir < I.h;
  const int64_t gi = (int64_t)ir * I.ld;
  double carry = 0.0;
  // four chunks of 32 columns per step: their loads are in flight together
  // (one chunk at a time left the warp waiting on each load's latency)
  for (int c0 = 0; c0 < g.RW; c0 += 128) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + 32 * u + lane;
      const int ic = g.rc0 + c - I.col0;
      v[u] = (rin && c < g.RW && ic >= 0 && ic < I.w) ? load_px<DT>(I.f, gi + ic) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, v[u], o);
        if (lane >= o) v[u] += t;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + 32 * u + lane;
      v[u] += carry;
      if (c < g.RW) dst[c] = v[u];
      carry = __shfl_sync(0xffffffffu, v[u], 31);
    }
  }
}

// dir 2: g[r][c] += g[r-1][c-1];  3: g[r][c] += g[r-1][c];  4: g[r][c] += g[r-1][c+1]
// Segmented line sweep for batches of few, large regions (the flat-cost
// table's single 2048^2 image at s >= 1024: four regions of ~1600^2).  The
// sequential sweep above walks every line with one lane, a dependent chain of
// RH loads and stores through L2 (latency-bound: ~0.3 ms per direction at
// RH = 1600).  Here the rows are cut into segments of kLineSeg: phase 0 sums
// each line's part of each segment (lane = line: a warp's 32 neighbouring
// lines touch consecutive addresses row by row), phase 1
// turns each line's segment sums into exclusive carries, phase 2 re-walks
// each segment from its carry.  tot holds nseg x nlines partial sums per region
// (region r at tot + r * tot_stride).  The additions per element differ from
// the sequential sweep only in where the running sum is restarted.
constexpr int kLineSeg = 32;
template <int DIR, int PHASE>
__global__ void __launch_bounds__(256) big_line_seg_kernel(const BigRegion *R, double *scratch,
                                                           double *tot, int64_t tot_stride,
                                                           Status *st) {
  const BigRegion g = R[blockIdx.z];
  const int lane = threadIdx.x & 31;
  const int nlines = DIR == 3 ? g.RW : g.RH + g.RW - 1;
  const int nseg = (g.RH + kLineSeg - 1) / kLineSeg;
  double *T = tot + blockIdx.z * tot_stride;  // [seg][line]
  if (PHASE == 1) {
    const int L = blockIdx.x * 256 + threadIdx.x;
    if (blockIdx.y != 0 || L >= nlines) return;
    // eight segment sums loaded before the carries are stored back (a load
    // cannot move above a store through the same pointer: one at a time was
    // a chain of nseg L2 round trips, ~30 us per direction at 50 segments)
    double c = 0.0;
    double *Tl = T + L;
    for (int k = 0; k < nseg; k += 8) {
      double t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) t[u] = k + u < nseg ? Tl[(int64_t)(k + u) * nlines] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (k + u < nseg) Tl[(int64_t)(k + u) * nlines] = c;
        c += t[u];
      }
    }
    return;
  }
  const int seg = blockIdx.y;
  if (seg >= nseg) return;
  const int lb = (blockIdx.x * 256 + threadIdx.x) & ~31;  // first line of this warp
  if (lb >= nlines) return;
  double *base = scratch + g.off;
  const int L = lb + lane;
  // the warp's row range within the segment (as big_line_kernel)
  int ta, tb;
  if (DIR == 2) {
    const int kb = lb - (g.RH - 1);
    ta = max(0, -(kb + 31));
    tb = min(g.RH - 1, g.RW - 1 - kb);
  } else if (DIR == 3) {
    ta = 0;
    tb = g.RH - 1;
  } else {
    ta = max(0, lb - (g.RW - 1));
    tb = min(g.RH - 1, lb + 31);
  }
  ta = max(ta, seg * kLineSeg);
  tb = min(tb, seg * kLineSeg + kLineSeg - 1);
  const int k2 = L - (g.RH - 1);
  double s = PHASE == 2 && L < nlines ? T[(int64_t)seg * nlines + L] : 0.0;
  unsigned gh = 0;
  for (int t = ta; t <= tb; t += 4) {
    double v[4];
    int64_t idx[4];
    bool ok[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int tt = t + u;
      const int c = DIR == 2 ? tt + k2 : (DIR == 3 ? L : L - tt);
      ok[u] = tt <= tb && c >= 0 && c < g.RW && L < nlines;
      idx[u] = (int64_t)tt * g.P + c;
      v[u] = ok[u] ? base[idx[u]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (ok[u]) {
        s += v[u];
        if (PHASE == 2) {
          base[idx[u]] = s;
          if (DIR == 4) gh = max(gh, (unsigned)__double2hiint(s) & 0x7fffffffu);
        }
      }
    }
  }
  if (PHASE == 0) {
    if (L < nlines) T[(int64_t)seg * nlines + L] = s;
  } else if (DIR == 4) {
    gh = __reduce_max_sync(0xffffffffu, gh);
    if (lane == 0 && gh) atomicMax(&st->guard_hi, gh);
  }
}

// RS2, RS3 and RS4 of a region in ONE top-down pass (one CTA per region).
// Row r of each sweep needs only row r of the previous sweep and row r - 1
// of its own, so three previous-row vectors carry the state (double-
// buffered in shared memory, one barrier per row); every element is read
// once (RS1, from big_fill_rs1_kernel) and written once (final).  The three
// separate line sweeps read and wrote the region three times.  Same adds in
// the same order per element as the line sweeps.
constexpr int kRsThreads = 512, kRsCols = 9;  // regions up to 4608 columns
// The sweep is latency-bound (one barrier per row); narrower batches run
// more resident CTAs per SM (NT threads x NC columns, MINB CTAs per SM):
// RS3's previous row is the thread's own column (registers), only RS2 / RS4
// read neighbours through shared memory (4 vectors instead of 6).
constexpr int rs_smem(int rw) { return 4 * (rw + 2) * 8; }
template <int NT, int NC, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    big_rs234_kernel(const BigRegion *R, double *scratch, Status *st) {
  extern __shared__ double prow[];
  const BigRegion g = R[blockIdx.x];
  const int W2 = g.RW + 2;  // entry c + 1 holds column c; 0 and RW + 1 stay zero
  double *A = prow, *B = prow + 2 * W2;  // [RS2 | RS4] of row r - 1, of row r
  for (int i = threadIdx.x; i < 4 * W2; i += NT) prow[i] = 0.0;
  double *base = scratch + g.off;
  // RS1 rows are prefetched two rows ahead (one row of lead did not cover
  // the load latency: the per-row time is a barrier plus a few shared ops)
  double na[NC], nb[NC], a3[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int c = threadIdx.x + k * NT;
    na[k] = (c < g.RW && g.RH > 0) ? base[c] : 0.0;
    nb[k] = (c < g.RW && g.RH > 1) ? base[g.P + c] : 0.0;
    a3[k] = 0.0;
  }
  __syncthreads();
  unsigned gh = 0;
  auto row_step = [&](int r, double (&buf)[NC]) {
    double *row = base + (int64_t)r * g.P;
    double cur[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      cur[k] = buf[k];
      const int c = threadIdx.x + k * NT;
      buf[k] = (c < g.RW && r + 2 < g.RH) ? row[2 * (int64_t)g.P + c] : 0.0;  // row r + 2
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = threadIdx.x + k * NT;
      if (c < g.RW) {
        const double v2 = cur[k] + A[c];           // RS2: + row r-1 at c-1
        const double v3 = v2 + a3[k];              // RS3: + row r-1 at c
        const double v4 = v3 + A[W2 + c + 2];      // RS4: + row r-1 at c+1
        B[c + 1] = v2;
        a3[k] = v3;
        B[W2 + c + 1] = v4;
        row[c] = v4;
        gh = max(gh, (unsigned)__double2hiint(v4) & 0x7fffffffu);
      }
    }
    __syncthreads();
    double *t = A;
    A = B;
    B = t;
  };
  for (int r = 0; r < g.RH; r += 2) {
    row_step(r, na);
    if (r + 1 < g.RH) row_step(r + 1, nb);
  }
  gh = __reduce_max_sync(0xffffffffu, gh);
  if ((threadIdx.x & 31) == 0 && gh) atomicMax(&st->guard_hi, gh);
}

#ifndef RUBS_BG_MINB
#define RUBS_BG_MINB 4  // 64 registers, 4 CTAs per SM: more loads in flight (config 5: -15 %)
#endif
template <int MODE>
// Tiles are taken from an atomic counter in slot order (block raster): the
// resident CTAs stay on a compact run of tiles, so the region rows their
// vertices read stay in L2 (static striding let CTAs drift apart).
__global__ void __launch_bounds__(256, RUBS_BG_MINB) big_gather_kernel(FieldSpec F, DomainSpec D, int tiles_x,
                                                         const BigTile *tl, int nt,
                                                         const BigRegion *R, const double *scratch,
                                                         Status *st, int2 *pix, int pix_cap,
                                                         int *next) {
  __shared__ int s_next;
  unsigned flags = 0;
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  for (int i = blockIdx.x;;) {
    if (next != nullptr) {
      if (threadIdx.x == 0) s_next = atomicAdd(next, 1);
      __syncthreads();
      i = s_next;
      __syncthreads();
    }
    if (i >= nt) break;
    const BigTile bt = tl[i];
    if (next == nullptr) i += gridDim.x;
    if (bt.tile < 0) continue;  // a gap of the block's tile raster
    const BigRegion g = R[bt.region];
    const int x0 = (bt.tile % tiles_x) * kTile, y0 = (bt.tile / tiles_x) * kTile;
    const char *Sb = reinterpret_cast<const char *>(scratch + g.off);  // local coordinates
    const int P8 = g.P * 8;  // 32-bit offsets: a region row is < 2^31 bytes (fewer live registers)
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
      const int x = x0 + lx, y = y0 + ly + 8 * k;
      const int c = (ly + 8 * k) / 8 * 4 + lx / 8;
      if (x < D.pw && y < D.ph && ((bt.mask >> c) & 1u)) {
        const int n1 = D.pc_lo + x, n2 = D.pr_lo + y;
        double a[4];
        field_at<MODE>(F, n1, n2, a, flags);
        // a small kernel sharing a tile with huge ones: its own region is
        // small, the block's is not -- deferred to the per-pixel pass
        if (defer_pixel(a, g.l4, x, y, pix, pix_cap, st)) continue;
        D.out[(int64_t)y * D.ld_out + x] =
            pixel_fd_t<const char *, int>(Sb, P8, n1 - g.rc0, n2 - g.rr0, a);
      }
    }
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (lx == 0 && flags) atomicOr(&st->flags, flags);
}

// fp64 FMA peak probe (rubs_b200_dfma_peak): 8 independent DFMA chains per
// thread hide the pipe latency; the result is stored so nothing is elided.
__global__ void __launch_bounds__(256) dfma_probe_kernel(double *out, int iters) {
  double x[8];
  const double a = 1.0 + 1e-12 * threadIdx.x, b = 1e-9;
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = 1.0 + k * 1e-3 + blockIdx.x * 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = s;
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
  int sms = 148;
  int *d_ovf = nullptr;  // OvfRec records
  size_t ovf_cap = 0;
  int2 *d_list = nullptr;  // (tile, cell mask) of the shared-memory overflow pass
  int2 *d_pix = nullptr;   // pixels deferred to the per-pixel pass
  size_t pix_cap = 0;
  size_t list_cap = 0;
  double *d_big = nullptr;
  size_t big_cap = 0;
  int64_t big_budget = 0;  // batch budget the scratch was sized for (0: none yet)
  BigRegion *d_regs = nullptr;
  size_t regs_cap = 0;
  BigTile *d_btiles = nullptr;
  size_t btiles_cap = 0;
  Status *d_status = nullptr;
  Status *h_status = nullptr;  // pinned
  double *d_pass[2] = {nullptr, nullptr};
  size_t pass_cap[2] = {0, 0};
  double *d_aslot = nullptr;     // wide kernel: per-(SM, slot) scale-vectors
  unsigned *d_slotmask = nullptr;
  int *d_next = nullptr;  // tile counter of the large-halo gather
  int *d_w2 = nullptr;    // primary kernel stage-2 tile list
  size_t w2_cap = 0;
  // status epochs: every entry (ensure_scratch) bumps `epoch`; a clearing
  // fetch records it, so "cleared by the previous entry, nothing in
  // between" is clean_epoch + 1 == epoch
  uint64_t epoch = 0, clean_epoch = ~0ull;
  double *d_seg = nullptr;  // segment sums of the segmented line sweeps
  size_t seg_cap = 0;
  char *h_stage = nullptr;  // pinned staging of small transfers (small_copy)
  size_t h_stage_cap = 0;
  bool attr_set = false;
};
thread_local Scratch t_scr_dev[rubs_internal::kMaxDevices];
thread_local int t_dev = 0;  // set by ensure_scratch(), which every entry calls first
#define t_scr (t_scr_dev[t_dev])

int ensure_scratch() {
  int dev = 0;
  RUBS_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= rubs_internal::kMaxDevices)
    return set_error(RUBS_ECUDA, "device index beyond the per-device state table");
  t_dev = dev;
  ++t_scr.epoch;
  if (t_scr.device != dev) {  // first call on this device
    t_scr.device = dev;
    RUBS_CUDA_TRY(cudaMalloc(&t_scr.d_status, sizeof(Status)));
    RUBS_CUDA_TRY(cudaMallocHost(&t_scr.h_status, sizeof(Status)));
    RUBS_CUDA_TRY(cudaDeviceGetAttribute(&t_scr.sms, cudaDevAttrMultiProcessorCount, dev));
    RUBS_CUDA_TRY(cudaMalloc(&t_scr.d_aslot, (size_t)kMaxSmId * kSlotsPerSm * kWideW * kWideH * 4 *
                                                 sizeof(double)));
    RUBS_CUDA_TRY(cudaMalloc(&t_scr.d_slotmask, kMaxSmId * sizeof(unsigned)));
    RUBS_CUDA_TRY(cudaMalloc(&t_scr.d_next, sizeof(int)));
    RUBS_CUDA_TRY(cudaMemset(t_scr.d_slotmask, 0, kMaxSmId * sizeof(unsigned)));
    {  // log table of log_ge1 (rubs_device.cuh)
      double2 tab[128];
      for (int i = 0; i < 128; ++i) {
        const double c = 1.0 + (i + 0.5) / 128.0;
        tab[i] = make_double2(1.0 / c, std::log(c));
      }
      RUBS_CUDA_TRY(cudaMemcpyToSymbol(g_logtab, tab, sizeof tab));
    }
  }
  if (!t_scr.attr_set) {
#define RUBS_SET_SMEM(M, T)                                                          \
  RUBS_CUDA_TRY(cudaFuncSetAttribute(tile_filter_kernel<M, T>,                       \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                     kSmemSmall));                                  \
  RUBS_CUDA_TRY(cudaFuncSetAttribute(tile_overflow_kernel<M, T>,                     \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                     kSmemLarge));                                  \
  RUBS_CUDA_TRY(cudaFuncSetAttribute(wide_filter_kernel<M, T, kThreadsWide, 1>,                       \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                     kSmemWide));                                   \
  RUBS_CUDA_TRY(cudaFuncSetAttribute(pixel_kernel<M, T>,                             \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                     kPixSmem))
    RUBS_SET_SMEM(kModeField, 0);
    RUBS_SET_SMEM(kModeField, 1);
    RUBS_SET_SMEM(kModeUniform, 0);
    RUBS_SET_SMEM(kModeUniform, 1);
    RUBS_SET_SMEM(kModeLut, 0);
    RUBS_SET_SMEM(kModeLut, 1);
    RUBS_SET_SMEM(kModeLut32, 0);
    RUBS_SET_SMEM(kModeLut32, 1);
#undef RUBS_SET_SMEM
    // multi-channel instantiations (adaptive_smooth pipeline)
#define RUBS_SET_CT1(M, T)                                                                  \
  RUBS_CUDA_TRY(cudaFuncSetAttribute(wide_filter_kernel<M, T, wide_threads<1>(), 1, 1>,      \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, wide_smem<1>()))
    RUBS_SET_CT1(kModeField, 0);
    RUBS_SET_CT1(kModeField, 1);
    RUBS_SET_CT1(kModeUniform, 0);
    RUBS_SET_CT1(kModeUniform, 1);
    RUBS_SET_CT1(kModeLut, 0);
    RUBS_SET_CT1(kModeLut, 1);
    RUBS_SET_CT1(kModeLut32, 0);
    RUBS_SET_CT1(kModeLut32, 1);
#undef RUBS_SET_CT1
    RUBS_CUDA_TRY(cudaFuncSetAttribute(wide_filter_kernel<kModeUniform, 1, kThreadsWide, 3>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWide));
    RUBS_CUDA_TRY(cudaFuncSetAttribute(wide_filter_kernel<kModeLut, 1, wide_threads<3>(), 2, 3>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, wide_smem<3>()));
    RUBS_CUDA_TRY(cudaFuncSetAttribute(wide_filter_kernel<kModeLut, 0, wide_threads<3>(), 2, 3>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, wide_smem<3>()));
    RUBS_CUDA_TRY(cudaFuncSetAttribute(big_rs234_kernel<128, 9, 4>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, rs_smem(128 * 9)));
    RUBS_CUDA_TRY(cudaFuncSetAttribute(big_rs234_kernel<256, 6, 3>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, rs_smem(256 * 6)));
    RUBS_CUDA_TRY(cudaFuncSetAttribute(big_rs234_kernel<256, 9, 2>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, rs_smem(256 * 9)));
    RUBS_CUDA_TRY(cudaFuncSetAttribute(big_rs234_kernel<384, 7, 2>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, rs_smem(384 * 7)));
    RUBS_CUDA_TRY(cudaFuncSetAttribute(big_rs234_kernel<512, 9, 1>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, rs_smem(512 * 9)));
    t_scr.attr_set = true;
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
  if (s.flags & kFlagPrecisionLimited) t_precision_limited = 1;
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
  // tile planes hold g / 2 (the two sqrt(2) factors are folded into the
  // output weight): the reference's |g| >= 2^53 is |g/2| >= 2^52, i.e. a
  // high word >= 0x43300000.  The global canvas (rubs_b200_preintegrate)
  // stores g itself and reports its full bits.
  double g;
  unsigned long long b = s.guard_bits;
  std::memcpy(&g, &b, sizeof(g));
  const unsigned long long hb = (unsigned long long)s.guard_hi << 32;
  double gt;
  std::memcpy(&gt, &hb, sizeof(gt));
  gt *= 2.0;
  if (gt > g) g = gt;
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

// Small transfers (status words, plan records) move through SM loads and
// stores of mapped pinned memory, not the copy engines: in a pipelined
// host-buffer call the copy engines are busy with image bands, and a small
// cudaMemcpyAsync queued behind them waited for whole bands (config 3n4's
// band pipeline: ~2 ms per band of planning stall).  Sizes are multiples of
// 4 bytes; pinned host memory is device-accessible under UVA.
__global__ void word_copy_kernel(const unsigned *src, unsigned *dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
int small_copy(void *dst, const void *src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return RUBS_OK;
  const size_t n = bytes / 4;
  const int blocks = (int)std::min<size_t>((n + 255) / 256, 1024);
  word_copy_kernel<<<blocks, 256, 0, s>>>(static_cast<const unsigned *>(src),
                                          static_cast<unsigned *>(dst), n);
  ++t_launches;
  RUBS_CUDA_TRY(cudaGetLastError());
  return RUBS_OK;
}
// Pinned staging for the small transfers of one planning round: `bytes`
// more at *off (grown only with the stream idle: callers sync first).
int host_stage(size_t bytes, size_t &off, char **out, cudaStream_t s) {
  const size_t need = off + ((bytes + 15) & ~(size_t)15);
  if (need > t_scr.h_stage_cap) {
    RUBS_CUDA_TRY(cudaStreamSynchronize(s));
    if (t_scr.h_stage) cudaFreeHost(t_scr.h_stage);
    t_scr.h_stage = nullptr;
    t_scr.h_stage_cap = 0;
    const size_t cap = std::max<size_t>(need * 2, 1 << 20);
    RUBS_CUDA_TRY(cudaMallocHost(&t_scr.h_stage, cap));
    t_scr.h_stage_cap = cap;
    off = 0;  // earlier stagings of this round have been consumed (synced)
  }
  *out = t_scr.h_stage + off;
  off += (bytes + 15) & ~(size_t)15;
  return RUBS_OK;
}

int fetch_status(cudaStream_t s, Status &out) {
  int rc = small_copy(t_scr.h_status, t_scr.d_status, sizeof(Status), s);
  if (rc) return rc;
  RUBS_CUDA_TRY(cudaStreamSynchronize(s));
  out = *t_scr.h_status;
  timer_collect();
  return RUBS_OK;
}

// Copy the status to the host AND zero it on the device (one kernel): the
// next one-pass call then skips its status memset (one stream operation
// fewer between consecutive filters).
__global__ void status_publish_kernel(unsigned *d, unsigned *h) {
  const int i = threadIdx.x;
  if (i < (int)(sizeof(Status) / 4)) {
    h[i] = d[i];
    d[i] = 0u;
  }
}
int fetch_status_clear(cudaStream_t s, Status &out) {
  status_publish_kernel<<<1, 32, 0, s>>>(reinterpret_cast<unsigned *>(t_scr.d_status),
                                         reinterpret_cast<unsigned *>(t_scr.h_status));
  ++t_launches;
  RUBS_CUDA_TRY(cudaGetLastError());
  RUBS_CUDA_TRY(cudaStreamSynchronize(s));
  out = *t_scr.h_status;
  t_scr.clean_epoch = t_scr.epoch;
  timer_collect();
  return RUBS_OK;
}

int launch_global_margins(const FieldSpec &F, const DomainSpec &D, cudaStream_t s) {
  const int cells_x = (D.pw + 15) / 16, cells_y = (D.ph + 15) / 16;
  {
    TimedLaunch tl(1, s);
    global_margins_kernel<<<cells_x * cells_y, 256, 0, s>>>(F, D, cells_x, t_scr.d_status);
  }
  ++t_launches;
  RUBS_CUDA_TRY(cudaGetLastError());
  return RUBS_OK;
}

// Tensor maps of a float64 image for the TMA region loads (cached per image
// geometry: encoding is a host-side call, ~1 us each).
struct TmaCache {
  const void *f = nullptr;
  int64_t ld = 0;
  int h = 0, w = 0, dt = -1;
  TmaMaps maps{};
};
constexpr int kTmaCacheSlots = 8;  // multi-channel launches use several images
thread_local TmaCache t_tma[kTmaCacheSlots];
thread_local int t_tma_next = 0;

const TmaMaps &tma_maps(const ImageSpec &I) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  for (TmaCache &e : t_tma)
    if (e.f == I.f && e.ld == I.ld && e.h == I.h && e.w == I.w && e.dt == I.dt) return e.maps;
  TmaCache &c = t_tma[t_tma_next];
  t_tma_next = (t_tma_next + 1) % kTmaCacheSlots;
  c.f = I.f; c.ld = I.ld; c.h = I.h; c.w = I.w; c.dt = I.dt;
  c.maps.valid = 0;
  if (std::getenv("RUBS_B200_NO_TMA")) return c.maps;
  const bool ok = encode != nullptr && I.dt == 1 && I.w > 0 && I.h > 0 &&
                  (reinterpret_cast<uintptr_t>(I.f) & 15) == 0 && ((I.ld * 8) & 15) == 0;
  if (!ok) return c.maps;
  for (int k = 0; k < kTmaMaps; ++k) {
    const cuuint64_t dims[2] = {(cuuint64_t)I.w, (cuuint64_t)I.h};
    const cuuint64_t strides[1] = {(cuuint64_t)I.ld * 8};
    const cuuint32_t box[2] = {(cuuint32_t)(kTmaP0 + 16 * k), 8};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r =
        encode(&c.maps.m[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void *>(I.f), dims,
               strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS) c.maps.valid |= 1u << k;
  }
  return c.maps;
}

int kernel_choice() {
  static int choice = -1;
  if (choice < 0) {
    const char *e = std::getenv("RUBS_B200_KERNEL");
    choice = (e && std::strcmp(e, "tile") == 0) ? 1 : 2;
  }
  return choice;
}

// Wide-kernel tiles of rows [wy0, wy1) of the 64 x 32 grid over domain D.
template <int M, int T, int NCH = 1, int CT = 2>
void launch_wide_rows(const ImageSpec &I, const FieldSpec &F, const DomainSpec &D, int wy0,
                      int wy1, cudaStream_t s, const MultiChan *mcp = nullptr, int w2_mode = 2) {
  const int tiles_x = (D.pw + kTile - 1) / kTile;
  const int wx = (D.pw + kWideW - 1) / kWideW;
  if (wy1 <= wy0) return;
  MultiChan mc{};
  TmaMapsN<NCH> tm;
  if (mcp) {
    mc = *mcp;
  } else {
    mc.f[0] = I.f;
    mc.out[0] = D.out;
  }
  for (int ch = 0; ch < NCH; ++ch) {
    ImageSpec Ic = I;
    Ic.f = mc.f[ch];
    tm.m[ch] = tma_maps(Ic);
  }
  const int grid = w2_mode == 1 ? t_scr.sms : wx * (wy1 - wy0);
  wide_filter_kernel<M, T, wide_threads<CT>(), NCH, CT>
      <<<grid, wide_threads<CT>(), wide_smem<CT>(), s>>>(
      I, F, D, wx, tiles_x, wide_cap<NCH, CT>(), t_scr.d_ovf, t_scr.d_status, t_scr.d_aslot,
      t_scr.d_slotmask, wy0 * wx, mc, tm, t_scr.d_w2, w2_mode, w2_elems());
}

void launch_wide_rows_rt(const ImageSpec &I, const FieldSpec &F, const DomainSpec &D, int wy0,
                         int wy1, cudaStream_t s, int w2_mode = 2) {
  const int m = F.mode, t = I.dt;
  if (m == kModeField) {
    if (t) launch_wide_rows<kModeField, 1>(I, F, D, wy0, wy1, s, nullptr, w2_mode);
    else launch_wide_rows<kModeField, 0>(I, F, D, wy0, wy1, s, nullptr, w2_mode);
  } else if (m == kModeUniform) {
    if (t) launch_wide_rows<kModeUniform, 1>(I, F, D, wy0, wy1, s, nullptr, w2_mode);
    else launch_wide_rows<kModeUniform, 0>(I, F, D, wy0, wy1, s, nullptr, w2_mode);
  } else if (m == kModeLut) {
    if (t) launch_wide_rows<kModeLut, 1>(I, F, D, wy0, wy1, s, nullptr, w2_mode);
    else launch_wide_rows<kModeLut, 0>(I, F, D, wy0, wy1, s, nullptr, w2_mode);
  } else {
    if (t) launch_wide_rows<kModeLut32, 1>(I, F, D, wy0, wy1, s, nullptr, w2_mode);
    else launch_wide_rows<kModeLut32, 0>(I, F, D, wy0, wy1, s, nullptr, w2_mode);
  }
}

// Stage 2 of the primary kernel: persistent one-CTA-per-SM launch over the
// tiles stage 1 listed (exits at once when the list is empty).
void launch_wide_stage2_rt(const ImageSpec &I, const FieldSpec &F, const DomainSpec &D,
                           cudaStream_t s) {
  const int m = F.mode, t = I.dt;
  const int wy = (D.ph + kWideH - 1) / kWideH;
  if (m == kModeField) {
    if (t) launch_wide_rows<kModeField, 1, 1, 1>(I, F, D, 0, wy, s, nullptr, 1);
    else launch_wide_rows<kModeField, 0, 1, 1>(I, F, D, 0, wy, s, nullptr, 1);
  } else if (m == kModeUniform) {
    if (t) launch_wide_rows<kModeUniform, 1, 1, 1>(I, F, D, 0, wy, s, nullptr, 1);
    else launch_wide_rows<kModeUniform, 0, 1, 1>(I, F, D, 0, wy, s, nullptr, 1);
  } else if (m == kModeLut) {
    if (t) launch_wide_rows<kModeLut, 1, 1, 1>(I, F, D, 0, wy, s, nullptr, 1);
    else launch_wide_rows<kModeLut, 0, 1, 1>(I, F, D, 0, wy, s, nullptr, 1);
  } else {
    if (t) launch_wide_rows<kModeLut32, 1, 1, 1>(I, F, D, 0, wy, s, nullptr, 1);
    else launch_wide_rows<kModeLut32, 0, 1, 1>(I, F, D, 0, wy, s, nullptr, 1);
  }
}


// Stage 2 of the primary kernel on (RUBS_B200_NO_STAGE2 turns it off: A/B)
bool use_stage2() {
  static const bool v = std::getenv("RUBS_B200_NO_STAGE2") == nullptr;
  return v;
}

template <int M, int T>
void launch_tiles(const ImageSpec &I, const FieldSpec &F, const DomainSpec &D, cudaStream_t s) {
  const int tiles_x = (D.pw + kTile - 1) / kTile, tiles_y = (D.ph + kTile - 1) / kTile;
  const int ntiles = tiles_x * tiles_y;
  // ovf_count is zero here: every caller clears the status before its first
  // pass and finish_pass clears the count after the deferred tiles
  if (kernel_choice() == 2) {
    const int mode = use_stage2() ? 0 : 2;
    // the stage-2 list and its take counter start empty for every pass
    if (mode == 0) cudaMemsetAsync(&t_scr.d_status->w2_count, 0, 2 * sizeof(int), s);
    launch_wide_rows<M, T>(I, F, D, 0, (D.ph + kWideH - 1) / kWideH, s, nullptr, mode);
    if (mode == 0) launch_wide_stage2_rt(I, F, D, s);
  }
  else
    tile_filter_kernel<M, T><<<ntiles, kThreadsSmall, kSmemSmall, s>>>(
        I, F, D, tiles_x, kSmemSmall / 8, t_scr.d_ovf, t_scr.d_status, tma_maps(I));
}

template <class V>
int upload(std::vector<V> &h, V *&d, size_t &cap, cudaStream_t s, size_t &stage_off) {
  if (h.size() > cap) {
    if (d) cudaFree(d);
    d = nullptr;
    RUBS_CUDA_TRY(cudaMalloc(&d, h.size() * sizeof(V)));
    cap = h.size();
  }
  if (!h.empty()) {
    char *st = nullptr;
    int rc = host_stage(h.size() * sizeof(V), stage_off, &st, s);
    if (rc) return rc;
    std::memcpy(st, h.data(), h.size() * sizeof(V));
    return small_copy(d, st, h.size() * sizeof(V), s);
  }
  return RUBS_OK;
}

// Tiles deferred by the primary launch: those whose 8x8 regions fit the
// 225 KB configuration go to the shared-memory overflow kernel, the rest to
// the global-memory block path (see big_* kernels).
// dev: RUBS_B200_HOST_TIMING=1 prints the host planning phases
struct HostClock {
  bool on = std::getenv("RUBS_B200_HOST_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void lap(const char *what) {
    if (!on) return;
    auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[host] %-22s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

// ---- planning of the deferred tiles, on the device ----------------------
// The primary launch appends one OvfRec per deferred 32-pixel tile.  Each
// record either goes to the shared-memory overflow pass, or to a block of
// side S = 2^k >= 2h (shrunk for the precision budget) whose region lives
// in global scratch.  Blocks are cells of a per-S grid; the records are
// classified and the cells aggregated by kernels (one thread per record /
// cell), so only the few used cells travel to the host, which orders them,
// cuts the scratch batches and uploads the regions.  (A host-side sort and
// merge of ~1M records cost ~60 ms on config 5 with the GPU idle.)
constexpr int kPlanLevels = 9;  // block sides 32 << lv, lv = 0..8 (32 .. 8192)
struct PlanGrid {
  int gx[kPlanLevels], gy[kPlanLevels], base[kPlanLevels + 1];
};
struct CellAgg {
  int x0, y0, x1, y1;  // member tiles' bounding box (domain pixels)
  int r[4];            // region: union of the member tiles' read extents (x0, x1, y0, y1)
  int count;
};

#ifndef RUBS_BIG_SK
#define RUBS_BIG_SK 2
#endif
// 0: shared-memory overflow pass; else the block side S.
#ifndef RUBS_BIG_K
#define RUBS_BIG_K 3.0
#endif
// sk: S >= sk * h (a region of side S + 2h holds (1 + 2h / S)^2 elements
// per output pixel: 4 at sk = 2, 2.25 at sk = 4), capped so the region's
// width stays within the fused sweep's limit (big_rs234_kernel).
__host__ __device__ inline int plan_side(const OvfRec &r, int tw, int th, int sk) {
  const int h = max(max(r.m[0], r.m[1]), max(r.m[2], r.m[3]));
  int S = 64;
  while (S < sk * h && S < 8192) S *= 2;
  while (S > 64 && S >= 2 * h && S + r.m[0] + r.m[1] > kRsThreads * kRsCols) S /= 2;
  while (S > kTile) {
    const double RW = S + r.m[0] + r.m[1], RH = S + r.m[2] + r.m[3];
    const double mn = RW < RH ? RW : RH;
    if ((double)r.w * 0.25 * RW * RH * mn * mn <= (double)kPrecisionBudget) break;
    S /= 2;
  }
  if (region_elems(min(8, tw) + r.m[0] + r.m[1] + 1, min(8, th) + r.m[2] + r.m[3]) <=
      kSmemLarge / 8) {
    // both paths can take the tile: region elements per tile pixel, the
    // global-scratch ones weighted by RUBS_BIG_K (a shared-memory region of
    // the 32 x 32 tile grows as (32 + 2h)^2, a block region as (S + 2h)^2)
    const double mx = r.m[0] + r.m[1], my = r.m[2] + r.m[3];
    const double smem = (kTile + mx) * (kTile + my) / (double)(kTile * kTile);
    const double big = RUBS_BIG_K * (S + mx) * (S + my) / ((double)S * S);
    if (S <= kTile || smem <= big) return 0;
  }
  return S;
}

__global__ void plan_init_kernel(CellAgg *c, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    c[i] = CellAgg{INT_MAX, INT_MAX, 0, 0, {INT_MAX, INT_MIN, INT_MAX, INT_MIN}, 0};
}

// counters: [0] records for the shared-memory pass, [1] used cells
__global__ void plan_classify_kernel(const OvfRec *rec, int n, PlanGrid G, int tiles_x, int pw,
                                     int ph, CellAgg *cells, int *rec_cell, int2 *smem_list,
                                     int *counters, int sk) {
  const int lane = threadIdx.x & 31;
  // grid-stride loop in whole warps (the warp-aggregated atomics below need
  // every lane; lanes past n carry no record)
  const int n32 = (n + 31) & ~31;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n32; i += gridDim.x * blockDim.x) {
    int cell = -1;
    int b[8] = {INT_MAX, INT_MAX, INT_MIN, INT_MIN, INT_MAX, INT_MIN, INT_MAX, INT_MIN};
    if (i < n) {
      const OvfRec r = rec[i];
      const int x0 = (r.tile % tiles_x) * kTile, y0 = (r.tile / tiles_x) * kTile;
      const int tw = min(kTile, pw - x0), th = min(kTile, ph - y0);
      const int S = plan_side(r, tw, th, sk);
      if (S == 0) {
        smem_list[atomicAdd(&counters[0], 1)] = make_int2(r.tile, (int)r.mask);
        rec_cell[i] = -1;
      } else {
        const int lv = __ffs(S) - 6;  // S = 32 << lv
        cell = G.base[lv] + (x0 / S) * G.gy[lv] + (y0 / S);
        rec_cell[i] = cell;
        // member box; region = bounding box of the members' own read
        // extents (not the member box grown by the largest margin: on
        // smoothly varying fields the margins differ across a block)
        b[0] = x0; b[1] = y0; b[2] = x0 + tw; b[3] = y0 + th;
        b[4] = x0 - r.m[0]; b[5] = x0 + tw + r.m[1]; b[6] = y0 - r.m[2]; b[7] = y0 + th + r.m[3];
      }
    }
    // warp aggregation: neighbouring records mostly share a cell (few large
    // blocks: thousands of records on a handful of cells serialised on the
    // cells' atomics)
    const unsigned peers = __match_any_sync(0xffffffffu, cell);
    const int leader = __ffs(peers) - 1;
    // (each group of peers reduces over its own mask; the groups are disjoint)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const bool mn = k == 0 || k == 1 || k == 4 || k == 6;
      b[k] = mn ? __reduce_min_sync(peers, b[k]) : __reduce_max_sync(peers, b[k]);
    }
    if (cell >= 0 && lane == leader) {
      CellAgg *c = cells + cell;
      atomicMin(&c->x0, b[0]);
      atomicMin(&c->y0, b[1]);
      atomicMax(&c->x1, b[2]);
      atomicMax(&c->y1, b[3]);
      atomicMin(&c->r[0], b[4]);
      atomicMax(&c->r[1], b[5]);
      atomicMin(&c->r[2], b[6]);
      atomicMax(&c->r[3], b[7]);
      atomicAdd(&c->count, __popc(peers));
    }
  }
}

__global__ void plan_compact_kernel(const CellAgg *cells, int n, int *used, CellAgg *agg,
                                    int *counters) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (cells[i].count > 0) {
      const int k = atomicAdd(&counters[1], 1);
      used[k] = i;
      agg[k] = cells[i];
    }
}

// per cell: region index relative to its batch, first tile slot
// per used cell: (batch-relative region, first slot, tile x0, tile y0, row
// width in tiles); the block's tiles take slots in raster order of its tile
// bounding box (gaps stay tile = -1), so the gather walks each block row by
// row, neighbouring CTAs sharing the region rows in L2
struct CellMap {
  int region, slot0, tx0, ty0, bw;
};
__global__ void plan_map_kernel(const int *cells, const CellMap *cm, int n, CellMap *cell_map) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    cell_map[cells[i]] = cm[i];
}

__global__ void plan_assign_kernel(const OvfRec *rec, int n, const int *rec_cell,
                                   const CellMap *cell_map, int tiles_x, BigTile *out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int cell = rec_cell[i];
    if (cell < 0) continue;
    const CellMap m = cell_map[cell];
    const OvfRec r = rec[i];
    const int tx = r.tile % tiles_x, ty = r.tile / tiles_x;
    out[m.slot0 + (ty - m.ty0) * m.bw + (tx - m.tx0)] = BigTile{r.tile, m.region, r.mask};
  }
}

struct PlanScratch {
  size_t ncell_cap = 0, nrec_cap = 0;
  CellAgg *cells = nullptr, *agg = nullptr;
  int *used = nullptr, *rec_cell = nullptr, *counters = nullptr;
  CellMap *cell_map = nullptr;
  int *h_counters = nullptr;  // pinned
  CellMap *d_cm = nullptr;
  int *d_cm_cell = nullptr;
  size_t cm_cap = 0, cmc_cap = 0;
};
thread_local PlanScratch t_plan_dev[rubs_internal::kMaxDevices];
#define t_plan (t_plan_dev[t_dev])

int plan_buffers(size_t ncell, size_t nrec) {
  if (!t_plan.h_counters) RUBS_CUDA_TRY(cudaMallocHost(&t_plan.h_counters, 2 * sizeof(int)));
  if (!t_plan.counters) RUBS_CUDA_TRY(cudaMalloc(&t_plan.counters, 2 * sizeof(int)));
  if (ncell > t_plan.ncell_cap) {
    for (void *p : {(void *)t_plan.cells, (void *)t_plan.agg, (void *)t_plan.used,
                    (void *)t_plan.cell_map})
      if (p) cudaFree(p);
    t_plan.cells = t_plan.agg = nullptr;
    t_plan.used = nullptr;
    t_plan.cell_map = nullptr;
    t_plan.ncell_cap = 0;
    RUBS_CUDA_TRY(cudaMalloc(&t_plan.cells, ncell * sizeof(CellAgg)));
    RUBS_CUDA_TRY(cudaMalloc(&t_plan.agg, ncell * sizeof(CellAgg)));
    RUBS_CUDA_TRY(cudaMalloc(&t_plan.used, ncell * sizeof(int)));
    RUBS_CUDA_TRY(cudaMalloc(&t_plan.cell_map, ncell * sizeof(CellMap)));
    t_plan.ncell_cap = ncell;
  }
  if (nrec > t_plan.nrec_cap) {
    if (t_plan.rec_cell) cudaFree(t_plan.rec_cell);
    t_plan.rec_cell = nullptr;
    t_plan.nrec_cap = 0;
    RUBS_CUDA_TRY(cudaMalloc(&t_plan.rec_cell, nrec * sizeof(int)));
    t_plan.nrec_cap = nrec;
  }
  return RUBS_OK;
}

// Block side factor sk of plan_side (RUBS_B200_BIG_SK overrides, A/B runs).
int big_side_factor() {
  static const int v = [] {
    const char *e = std::getenv("RUBS_B200_BIG_SK");
    const int k = e ? std::atoi(e) : 0;
    return k >= 2 && k <= 16 ? k : RUBS_BIG_SK;
  }();
  return v;
}

template <int M, int T>
int handle_overflow_tiles(const ImageSpec &I, const FieldSpec &F, const DomainSpec &D, int n_ovf,
                    cudaStream_t s) {
  HostClock hc;
  const int tiles_x = (D.pw + kTile - 1) / kTile;
  PlanGrid G;
  G.base[0] = 0;
  for (int lv = 0; lv < kPlanLevels; ++lv) {
    const int S = kTile << lv;
    G.gx[lv] = (D.pw + S - 1) / S;
    G.gy[lv] = (D.ph + S - 1) / S;
    G.base[lv + 1] = G.base[lv] + G.gx[lv] * G.gy[lv];
  }
  const int ncell = G.base[kPlanLevels];
  int rc;
  if ((rc = plan_buffers(ncell, n_ovf))) return rc;
  // shared-memory overflow list: at most one entry per record
  if ((size_t)n_ovf > t_scr.list_cap) {
    if (t_scr.d_list) cudaFree(t_scr.d_list);
    t_scr.d_list = nullptr;
    t_scr.list_cap = 0;
    RUBS_CUDA_TRY(cudaMalloc(&t_scr.d_list, (size_t)n_ovf * sizeof(int2)));
    t_scr.list_cap = n_ovf;
  }
  const OvfRec *rec = reinterpret_cast<const OvfRec *>(t_scr.d_ovf);
  const int gb = std::min((ncell + 255) / 256, 4 * t_scr.sms);
  const int rb = std::min((n_ovf + 255) / 256, 4 * t_scr.sms);
  RUBS_CUDA_TRY(cudaMemsetAsync(t_plan.counters, 0, 2 * sizeof(int), s));
  plan_init_kernel<<<gb, 256, 0, s>>>(t_plan.cells, ncell);
  plan_classify_kernel<<<rb, 256, 0, s>>>(rec, n_ovf, G, tiles_x, D.pw, D.ph, t_plan.cells,
                                          t_plan.rec_cell, t_scr.d_list, t_plan.counters,
                                          big_side_factor());
  plan_compact_kernel<<<gb, 256, 0, s>>>(t_plan.cells, ncell, t_plan.used, t_plan.agg,
                                         t_plan.counters);
  t_launches += 3;
  RUBS_CUDA_TRY(cudaGetLastError());
  if ((rc = small_copy(t_plan.h_counters, t_plan.counters, 2 * sizeof(int), s))) return rc;
  size_t stage_off = 0;  // pinned staging of this planning round (small_copy)
  // The first kPlanSpec used cells travel with the counters (speculatively:
  // their number is not known yet); a call with few blocks -- one image at a
  // large uniform scale: four -- then needs no second round trip.
  constexpr int kPlanSpec = 128;
  const int n_spec = std::min(ncell, kPlanSpec);
  char *hu0 = nullptr, *ha0 = nullptr;
  if ((rc = host_stage(n_spec * sizeof(int), stage_off, &hu0, s))) return rc;
  if ((rc = host_stage(n_spec * sizeof(CellAgg), stage_off, &ha0, s))) return rc;
  if ((rc = small_copy(hu0, t_plan.used, n_spec * sizeof(int), s))) return rc;
  if ((rc = small_copy(ha0, t_plan.agg, n_spec * sizeof(CellAgg), s))) return rc;
  RUBS_CUDA_TRY(cudaStreamSynchronize(s));
  const int n_smem = t_plan.h_counters[0], n_used = t_plan.h_counters[1];
  std::vector<int> used(n_used);
  std::vector<CellAgg> agg(n_used);
  if (n_used > 0 && n_used <= n_spec) {
    std::memcpy(used.data(), hu0, n_used * sizeof(int));
    std::memcpy(agg.data(), ha0, n_used * sizeof(CellAgg));
  } else if (n_used > 0) {
    char *hu = nullptr, *ha = nullptr;
    stage_off = 0;
    if ((rc = host_stage(n_used * sizeof(int), stage_off, &hu, s))) return rc;
    if ((rc = host_stage(n_used * sizeof(CellAgg), stage_off, &ha, s))) return rc;
    if ((rc = small_copy(hu, t_plan.used, n_used * sizeof(int), s))) return rc;
    if ((rc = small_copy(ha, t_plan.agg, n_used * sizeof(CellAgg), s))) return rc;
    RUBS_CUDA_TRY(cudaStreamSynchronize(s));
    std::memcpy(used.data(), hu, n_used * sizeof(int));
    std::memcpy(agg.data(), ha, n_used * sizeof(CellAgg));
  }
  stage_off = 0;  // the stream is idle: the staging is free again
  hc.lap("device plan");
  if (hc.on) std::fprintf(stderr, "[host] %d records: %d shared-memory tiles, %d blocks\n", n_ovf, n_smem, n_used);
  // per-pixel fallback list: grown on demand (handle_overflow), starting
  // at min(the deferred tiles' pixels, 4M entries = 32 MB)
  {
    const size_t want = std::min<size_t>((size_t)n_ovf * kTile * kTile, pix_list_init());
    if (want > t_scr.pix_cap) {
      if (t_scr.d_pix) cudaFree(t_scr.d_pix);
      t_scr.d_pix = nullptr;
      t_scr.pix_cap = 0;
      RUBS_CUDA_TRY(cudaMalloc(&t_scr.d_pix, want * sizeof(int2)));
      t_scr.pix_cap = want;
    }
  }
  const int pix_cap = (int)t_scr.pix_cap;
  RUBS_CUDA_TRY(cudaMemsetAsync(&t_scr.d_status->pix_count, 0, sizeof(int), s));
  if (n_smem > 0) {
    // tile order (the classify kernel appended them in arbitrary order):
    // neighbouring persistent-CTA tiles then share their region rows in L2
    char *hl = nullptr;
    if ((rc = host_stage(n_smem * sizeof(int2), stage_off, &hl, s))) return rc;
    if ((rc = small_copy(hl, t_scr.d_list, n_smem * sizeof(int2), s))) return rc;
    RUBS_CUDA_TRY(cudaStreamSynchronize(s));
    int2 *sl = reinterpret_cast<int2 *>(hl);
    std::sort(sl, sl + n_smem, [](const int2 &a, const int2 &b) { return a.x < b.x; });
    if ((rc = small_copy(t_scr.d_list, hl, n_smem * sizeof(int2), s))) return rc;
    tile_overflow_kernel<M, T><<<std::min(n_smem, t_scr.sms), kThreadsLarge,
                                 kSmemLarge, s>>>(I, F, D, tiles_x, kSmemLarge / 8, t_scr.d_list,
                                                  n_smem, t_scr.d_status,
                                                  t_scr.d_pix, pix_cap, tma_maps(I));
    ++t_launches;
    RUBS_CUDA_TRY(cudaGetLastError());
  }
  if (n_used == 0) return RUBS_OK;
  // blocks in cell order = (S, x0 / S, y0 / S): deterministic
  std::vector<int> order(n_used);
  for (int i = 0; i < n_used; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return used[a] < used[b]; });
  // Batches of blocks under a scratch budget.  A batch's kernels follow the
  // previous batch's in stream order, so the scratch is reused without a
  // host sync; region / tile lists of all batches are uploaded once.
  // When the scratch has to grow, the budget is capped at half the free
  // device memory (the scratch is kept for later calls; the cap is
  // remembered, so steady-state calls skip cudaMemGetInfo, which measured
  // 1-13 ms of host time with the GPU idle) and quartered on an allocation
  // failure.
  int64_t budget = t_scr.big_budget > 0 ? t_scr.big_budget : kBigBatch;
  bool capped = false;
  // All regions of a batch share one row pitch Pg (the batch's widest
  // region, rounded up to 4 doubles), stacked by rows: the batch's scratch
  // is one 2-D tensor of pitch Pg (a TMA-windowed gather over it was
  // measured slower than the L1 gather: DESIGN.md §7).
  struct Batch {
    int r0, r1, t0, t1;
    int64_t used;  // Pg * rows
    int maxRH, maxL, maxRW;
    int rows, Pg;
  };
  static const int pitch_align = [] {
    const char *e = std::getenv("RUBS_B200_BIG_PITCH");
    const int k = e ? std::atoi(e) : 0;
    return k >= 1 && k <= 64 ? k : 16;
  }();
  const int pitch_mask = pitch_align - 1;
  auto pitch_of = [pitch_mask](int rw) { return (rw + pitch_mask) & ~pitch_mask; };
  std::vector<BigRegion> regs;
  std::vector<CellMap> cm;
  std::vector<int> cm_cell;
  std::vector<Batch> batches;
  int ntl = 0;
  Batch cur{0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  int64_t max_used = 0;
 replan:
  regs.clear();
  cm.clear();
  cm_cell.clear();
  batches.clear();
  ntl = 0;
  cur = Batch{0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  max_used = 0;
  auto close_batch = [&]() {
    cur.r1 = (int)regs.size();
    cur.t1 = ntl;
    if (cur.r1 > cur.r0) {
      cur.Pg = pitch_of(cur.maxRW);
      cur.used = (int64_t)cur.Pg * cur.rows;
      for (int r = cur.r0; r < cur.r1; ++r) {
        regs[r].P = cur.Pg;
        regs[r].off *= cur.Pg;  // held the row offset
      }
      batches.push_back(cur);
      max_used = std::max(max_used, cur.used);
    }
    cur = Batch{(int)regs.size(), 0, ntl, 0, 0, 0, 0, 0, 0, 0};
  };
  for (int k : order) {
    const CellAgg &b = agg[k];
    BigRegion g;
    g.RW = b.r[1] - b.r[0];
    g.RH = b.r[3] - b.r[2];
    g.P = g.RW;
    g.rc0 = D.pc_lo + b.r[0];
    g.rr0 = D.pr_lo + b.r[2];
    {
      const double mn = std::min(g.RW, g.RH);
      g.l4 = (float)(0.25 * g.RW * (double)g.RH * mn * mn);
    }
    if (cur.rows > 0 &&
        (int64_t)pitch_of(std::max(cur.maxRW, g.RW)) * (cur.rows + g.RH) > budget)
      close_batch();
    g.off = cur.rows;  // row offset; element offset once the batch pitch is known
    cur.rows += g.RH;
    cur.maxRH = std::max(cur.maxRH, g.RH);
    cur.maxL = std::max(cur.maxL, g.RH + g.RW - 1);
    cur.maxRW = std::max(cur.maxRW, g.RW);
    const int tx0 = b.x0 / kTile, ty0 = b.y0 / kTile;
    const int bw = (b.x1 + kTile - 1) / kTile - tx0, bh = (b.y1 + kTile - 1) / kTile - ty0;
    cm.push_back(CellMap{(int)regs.size() - cur.r0, ntl, tx0, ty0, bw});
    cm_cell.push_back(used[k]);
    ntl += bw * bh;
    regs.push_back(g);
  }
  close_batch();
  hc.lap("regions");
  if (max_used > (int64_t)t_scr.big_cap && !capped) {
    capped = true;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
      const int64_t cap = (int64_t)((free_b + t_scr.big_cap * sizeof(double)) / 2 / sizeof(double));
      if (cap < budget) {
        budget = std::max<int64_t>(cap, kBigMinBatch);
        goto replan;
      }
    }
  }
  if (max_used > (int64_t)t_scr.big_cap) {
    if (t_scr.d_big) cudaFree(t_scr.d_big);
    t_scr.d_big = nullptr;
    t_scr.big_cap = 0;
    const cudaError_t e = cudaMalloc(&t_scr.d_big, (size_t)max_used * sizeof(double));
    if (e == cudaErrorMemoryAllocation && budget > 4 * (int64_t)kBigMinBatch) {
      (void)cudaGetLastError();  // clear, plan smaller batches
      budget /= 4;
      goto replan;
    }
    RUBS_CUDA_TRY(e);
    t_scr.big_cap = (size_t)max_used;
    t_scr.big_budget = budget;
  }
  hc.lap("scratch");
  if ((rc = upload(regs, t_scr.d_regs, t_scr.regs_cap, s, stage_off))) return rc;
  if ((rc = upload(cm, t_plan.d_cm, t_plan.cm_cap, s, stage_off))) return rc;
  if ((rc = upload(cm_cell, t_plan.d_cm_cell, t_plan.cmc_cap, s, stage_off))) return rc;
  if ((size_t)ntl > t_scr.btiles_cap) {
    if (t_scr.d_btiles) cudaFree(t_scr.d_btiles);
    t_scr.d_btiles = nullptr;
    t_scr.btiles_cap = 0;
    RUBS_CUDA_TRY(cudaMalloc(&t_scr.d_btiles, (size_t)ntl * sizeof(BigTile)));
    t_scr.btiles_cap = ntl;
  }
  RUBS_CUDA_TRY(cudaMemsetAsync(t_scr.d_btiles, 0xff, (size_t)ntl * sizeof(BigTile), s));  // tile -1
  plan_map_kernel<<<std::min((n_used + 255) / 256, t_scr.sms), 256, 0, s>>>(
      t_plan.d_cm_cell, t_plan.d_cm, n_used, t_plan.cell_map);
  plan_assign_kernel<<<rb, 256, 0, s>>>(rec, n_ovf, t_plan.rec_cell, t_plan.cell_map, tiles_x,
                                        t_scr.d_btiles);
  t_launches += 2;
  RUBS_CUDA_TRY(cudaGetLastError());
  hc.lap("regions + upload");
  if (hc.on) {
    int64_t area = 0;
    for (const BigRegion &g : regs) area += (int64_t)g.RW * g.RH;
    std::fprintf(stderr, "[host] %zu regions, %zu batches, region area %.3g elements\n", regs.size(),
                 batches.size(), (double)area);
    for (const Batch &bt : batches)
      std::fprintf(stderr, "[host]   batch: %d regions, %d tile slots, max %d x %d, %.3g doubles\n",
                   bt.r1 - bt.r0, bt.t1 - bt.t0, bt.maxRW, bt.maxRH, (double)bt.used);
  }
  for (const Batch &bt : batches) {
    const int nreg = bt.r1 - bt.r0, ntl = bt.t1 - bt.t0;
    const BigRegion *R = t_scr.d_regs + bt.r0;
    big_fill_rs1_kernel<T><<<dim3((bt.maxRH + 7) / 8, nreg), 256, 0, s>>>(I, R, t_scr.d_big);
    // the fused sweep runs one CTA per region: with few regions in the batch
    // the three line sweeps (parallel over every line of every region) win
    if (bt.maxRW <= kRsThreads * kRsCols && nreg * kRsFewDiv >= t_scr.sms &&
        !std::getenv("RUBS_B200_LINE_SWEEPS")) {
      const int rw = bt.maxRW, sm = rs_smem(rw);
      if (rw <= 128 * 9)
        big_rs234_kernel<128, 9, 4><<<nreg, 128, sm, s>>>(R, t_scr.d_big, t_scr.d_status);
      else if (rw <= 256 * 6)
        big_rs234_kernel<256, 6, 3><<<nreg, 256, sm, s>>>(R, t_scr.d_big, t_scr.d_status);
      else if (rw <= 256 * 9)
        big_rs234_kernel<256, 9, 2><<<nreg, 256, sm, s>>>(R, t_scr.d_big, t_scr.d_status);
      else if (rw <= 384 * 7)
        big_rs234_kernel<384, 7, 2><<<nreg, 384, sm, s>>>(R, t_scr.d_big, t_scr.d_status);
      else
        big_rs234_kernel<512, 9, 1><<<nreg, 512, sm, s>>>(R, t_scr.d_big, t_scr.d_status);
      t_launches -= 2;
    } else {
      // few regions: segmented line sweeps (parallel along the lines too)
      const int nseg = (bt.maxRH + kLineSeg - 1) / kLineSeg;
      const int64_t stride = (int64_t)nseg * bt.maxL;
      if ((size_t)(stride * nreg) > t_scr.seg_cap) {
        if (t_scr.d_seg) cudaFree(t_scr.d_seg);
        t_scr.d_seg = nullptr;
        t_scr.seg_cap = 0;
        RUBS_CUDA_TRY(cudaMalloc(&t_scr.d_seg, (size_t)stride * nreg * sizeof(double)));
        t_scr.seg_cap = (size_t)stride * nreg;
      }
      const dim3 g0((bt.maxL + 255) / 256, nseg, nreg), g1((bt.maxL + 255) / 256, 1, nreg);
#define RUBS_SEG_SWEEP(DIRV)                                                                      \
  big_line_seg_kernel<DIRV, 0><<<g0, 256, 0, s>>>(R, t_scr.d_big, t_scr.d_seg, stride, t_scr.d_status); \
  big_line_seg_kernel<DIRV, 1><<<g1, 256, 0, s>>>(R, t_scr.d_big, t_scr.d_seg, stride, t_scr.d_status); \
  big_line_seg_kernel<DIRV, 2><<<g0, 256, 0, s>>>(R, t_scr.d_big, t_scr.d_seg, stride, t_scr.d_status)
      RUBS_SEG_SWEEP(2);
      RUBS_SEG_SWEEP(3);
      RUBS_SEG_SWEEP(4);
#undef RUBS_SEG_SWEEP
      t_launches += 6;
    }
    int *next = nullptr;
    if (!std::getenv("RUBS_B200_GATHER_STATIC")) {
      next = t_scr.d_next;
      RUBS_CUDA_TRY(cudaMemsetAsync(next, 0, sizeof(int), s));
    }
    big_gather_kernel<M><<<std::min(ntl, t_scr.sms * 8), 256, 0, s>>>(
        F, D, tiles_x, t_scr.d_btiles + bt.t0, ntl, R, t_scr.d_big, t_scr.d_status, t_scr.d_pix,
        pix_cap, next);
    t_launches += 5;
    RUBS_CUDA_TRY(cudaGetLastError());
  }
  return RUBS_OK;
}

// The deferred tiles, then the pixels they deferred in turn (per-pixel pass).
// `merged` (the one-pass path, whose status reads clear the device words):
// the read of the deferred-pixel count is a clearing read of the whole
// status, so a call that defers no pixels -- the usual case -- has its final
// status here and the caller needs no further round trip; every later read
// is merged in.
template <int M, int T>
int handle_overflow(const ImageSpec &I, const FieldSpec &F, const DomainSpec &D, int n_ovf,
                    cudaStream_t s, Status *merged) {
  int rc = handle_overflow_tiles<M, T>(I, F, D, n_ovf, s);
  if (rc) return rc;
  HostClock hc;
  int cnt = 0;
  auto merge = [&](const Status &s2) {
    merged->flags |= s2.flags;
    merged->guard_hi = std::max(merged->guard_hi, s2.guard_hi);
    merged->guard_bits = std::max(merged->guard_bits, s2.guard_bits);
  };
  if (merged) {
    Status s2;
    if ((rc = fetch_status_clear(s, s2))) return rc;
    merge(s2);
    cnt = s2.pix_count;
  } else {
    if ((rc = small_copy(&t_scr.h_status->pix_count, &t_scr.d_status->pix_count, sizeof(int), s)))
      return rc;
    RUBS_CUDA_TRY(cudaStreamSynchronize(s));
    cnt = t_scr.h_status->pix_count;
  }
  hc.lap("overflow kernels (sync)");
  if ((size_t)cnt > t_scr.pix_cap) {
    // more precision-deferred pixels than the list holds (rare: fields with
    // many small kernels inside huge-kernel blocks): grow the list to the
    // count and run the deferred-tile passes again (same outputs, the
    // skipped pixels now listed)
    cudaFree(t_scr.d_pix);
    t_scr.d_pix = nullptr;
    t_scr.pix_cap = 0;
    RUBS_CUDA_TRY(cudaMalloc(&t_scr.d_pix, (size_t)cnt * sizeof(int2)));
    t_scr.pix_cap = (size_t)cnt;
    if ((rc = handle_overflow_tiles<M, T>(I, F, D, n_ovf, s))) return rc;
    if (merged) {
      Status s2;
      if ((rc = fetch_status_clear(s, s2))) return rc;
      merge(s2);
      cnt = s2.pix_count;
    } else {
      if ((rc = small_copy(&t_scr.h_status->pix_count, &t_scr.d_status->pix_count, sizeof(int), s)))
        return rc;
      RUBS_CUDA_TRY(cudaStreamSynchronize(s));
      cnt = t_scr.h_status->pix_count;
    }
  }
  cnt = std::min<int64_t>(cnt, (int64_t)t_scr.pix_cap);
  if (cnt > 0) {
    pixel_kernel<M, T><<<std::min((cnt + 7) / 8, t_scr.sms * 4), 256, kPixSmem, s>>>(
        I, F, D, t_scr.d_pix, cnt, t_scr.d_status);
    ++t_launches;
    RUBS_CUDA_TRY(cudaGetLastError());
    if (merged) {
      Status s2;
      if ((rc = fetch_status_clear(s, s2))) return rc;
      merge(s2);
    }
  }
  return RUBS_OK;
}

template <int M, int T>
int overflow_dispatch(const ImageSpec &I, const FieldSpec &F, const DomainSpec &D, int n,
                      cudaStream_t s, Status *merged) {
  return handle_overflow<M, T>(I, F, D, n, s, merged);
}

int run_overflow(const ImageSpec &I, const FieldSpec &F, const DomainSpec &D, int n,
                 cudaStream_t s, Status *merged = nullptr) {
  const int m = F.mode, t = I.dt;
  if (m == kModeField) return t ? overflow_dispatch<kModeField, 1>(I, F, D, n, s, merged)
                                : overflow_dispatch<kModeField, 0>(I, F, D, n, s, merged);
  if (m == kModeUniform) return t ? overflow_dispatch<kModeUniform, 1>(I, F, D, n, s, merged)
                                  : overflow_dispatch<kModeUniform, 0>(I, F, D, n, s, merged);
  if (m == kModeLut) return t ? overflow_dispatch<kModeLut, 1>(I, F, D, n, s, merged)
                              : overflow_dispatch<kModeLut, 0>(I, F, D, n, s, merged);
  return t ? overflow_dispatch<kModeLut32, 1>(I, F, D, n, s, merged)
           : overflow_dispatch<kModeLut32, 0>(I, F, D, n, s, merged);
}

// Overflow-record capacity for a pass over D: at most one record per tile
// of the 32-pixel grid.
int ensure_ovf(const DomainSpec &D) {
  const size_t ntiles = (size_t)((D.pw + kTile - 1) / kTile) * ((D.ph + kTile - 1) / kTile);
  if (4 * ntiles > t_scr.ovf_cap) {
    if (t_scr.d_ovf) cudaFree(t_scr.d_ovf);
    t_scr.d_ovf = nullptr;
    RUBS_CUDA_TRY(cudaMalloc(&t_scr.d_ovf, 4 * ntiles * sizeof(OvfRec)));
    t_scr.ovf_cap = 4 * ntiles;
  }
  // stage-2 list: at most one entry per wide tile
  const size_t nwide = (size_t)((D.pw + kWideW - 1) / kWideW) * ((D.ph + kWideH - 1) / kWideH);
  if (nwide > t_scr.w2_cap) {
    if (t_scr.d_w2) cudaFree(t_scr.d_w2);
    t_scr.d_w2 = nullptr;
    RUBS_CUDA_TRY(cudaMalloc(&t_scr.d_w2, nwide * sizeof(int)));
    t_scr.w2_cap = nwide;
  }
  return RUBS_OK;
}

int launch_pass(const ImageSpec &I, const FieldSpec &F, const DomainSpec &D, cudaStream_t s) {
  {
    TimedLaunch tl(0, s);
    const int m = F.mode, t = I.dt;
    int rc = ensure_ovf(D);
    if (rc) return rc;
    if (m == kModeField) {
      if (t) launch_tiles<kModeField, 1>(I, F, D, s); else launch_tiles<kModeField, 0>(I, F, D, s);
    } else if (m == kModeUniform) {
      if (t) launch_tiles<kModeUniform, 1>(I, F, D, s); else launch_tiles<kModeUniform, 0>(I, F, D, s);
    } else if (m == kModeLut) {
      if (t) launch_tiles<kModeLut, 1>(I, F, D, s); else launch_tiles<kModeLut, 0>(I, F, D, s);
    } else {
      if (t) launch_tiles<kModeLut32, 1>(I, F, D, s); else launch_tiles<kModeLut32, 0>(I, F, D, s);
    }
  }
  ++t_launches;
  RUBS_CUDA_TRY(cudaGetLastError());
  return RUBS_OK;
}

// Complete a pass: status fetch (one sync), then the deferred tiles if the
// primary launch recorded any.
int finish_pass(const ImageSpec &I, const FieldSpec &F, const DomainSpec &D, cudaStream_t s,
                Status &st, bool clear = false) {
  int rc;
  if ((rc = clear ? fetch_status_clear(s, st) : fetch_status(s, st))) return rc;
  if (st.ovf_count > 0 && !(st.flags & (kFlagFieldNonFinite | kFlagParamInvalid))) {
    {
      // the deferred-tile passes are part of the pass's filter work (kind 0)
      TimedLaunch tl(0, s);
      if ((rc = run_overflow(I, F, D, st.ovf_count, s, clear ? &st : nullptr))) return rc;
    }
    if (clear) {
      // the status was cleared by the first read; the deferred passes' words
      // were merged into st by their own (clearing) reads
      st.ovf_count = 0;
    } else {
      RUBS_CUDA_TRY(cudaMemsetAsync(&t_scr.d_status->ovf_count, 0, sizeof(int), s));
      if ((rc = fetch_status(s, st))) return rc;
    }
  }
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
  // the one-pass path clears the status as it reads it: the memset is
  // needed only when the last fetch did not clear (or a call was cut short)
  if (!(iterations == 1 && t_scr.clean_epoch + 1 == t_scr.epoch))
    RUBS_CUDA_TRY(cudaMemsetAsync(t_scr.d_status, 0, sizeof(Status), s));
  DomainSpec D{0, 0, img.w, img.h, out, ld_out};
  if (iterations == 1) {
    // one launch: every tile computes its own scale-vectors and margins
    if ((rc = launch_pass(img, F, D, s))) return rc;
    Status st;
    if ((rc = finish_pass(img, F, D, s, st, /*clear=*/true))) return rc;
    return status_to_code(st);
  } else {
    // whole-field margins (engine.py:295) decide the pass canvases.  In LUT
    // modes a bound replaces them: every mapped component is a convex blend
    // of table entries times sqrt(size) <= amax sqrt(max size), and the
    // margins grow with each component.  A larger pass canvas changes
    // nothing: the final pass only reads the previous pass within its own
    // margins (the passes' results differ from exact-canvas ones only by
    // rounding).  Mapping every pixel for exact margins cost ~1/4 of a
    // two-pass config-4 step.
    int left, right, below, above;
    bool bounded = false;
    if (F.mode >= kModeLut && F.lut_amax > 0.0) {
      size_max_kernel<<<4 * t_scr.sms, 256, 0, s>>>(F, t_scr.d_status);
      ++t_launches;
      RUBS_CUDA_TRY(cudaGetLastError());
      Status st;
      if ((rc = fetch_status(s, st))) return rc;
      double smax;
      std::memcpy(&smax, &st.smax_bits, sizeof(smax));
      if (smax > 0.0 && std::isfinite(smax)) {
        const double A = std::max(F.lut_amax * std::sqrt(smax), kScaleFloor) / F.div;
        const double p = A / kSqrt2;
        const double hx = 0.5 * A + p + 0.5;  // >= -(t1 - a1 - p2) and >= t1 + p4 (+1)
        const double hy = 0.5 * A + p + 1.5;  // >= -(t2 - a3 - p2 - p4) and >= t2 (+3)
        left = right = (int)std::ceil(hx) + 3;
        below = above = (int)std::ceil(hy) + 3;
        bounded = true;
      }
    }
    if (!bounded) {
      RUBS_CUDA_TRY(cudaMemsetAsync(t_scr.d_status, 0, sizeof(Status), s));
      if ((rc = launch_global_margins(F, D, s))) return rc;
      Status st;
      if ((rc = fetch_status(s, st))) return rc;
      if ((rc = status_to_code(st))) return rc;
      left = st.gm[0];
      right = st.gm[1];
      below = st.gm[2];
      above = st.gm[3];
    }
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
      if ((rc = launch_pass(cur, F, Dp, s))) return rc;
      Status stp;
      if ((rc = finish_pass(cur, F, Dp, s, stp))) return rc;
      if ((rc = status_to_code(stp))) return rc;
      cur = ImageSpec{Dp.out, 1, Dp.ld_out, Dp.ph, Dp.pw, Dp.pc_lo, Dp.pr_lo};
    }
  }
  Status st;
  if ((rc = fetch_status(s, st))) return rc;
  return status_to_code(st);
}

// One pass over output rows [out_row0, out_row0 + out_rows) of an image
// whose rows [I.row0, I.row0 + I.h) are given (row bands);
// field / parameter arrays hold global rows from F.fr_off on.
// One pass over an H x W image for several channels that share the field
// (the adaptive_smooth pipeline): one multi-channel launch, then the
// deferred tiles of every channel through the single-channel overflow path.
// Supported: uniform field with 3 float64 channels, LUT field (float64
// params) with 2 channels; anything else runs channel by channel.
int run_multi(const ImageSpec &I, const MultiChan &mc, int nch, FieldSpec F, int64_t ld_out,
              cudaStream_t s) {
  int rc = ensure_scratch();
  if (rc) return rc;
  if (I.h == 0 || I.w == 0) return RUBS_OK;
  F.FH = I.h;
  F.FW = I.w;
  F.div = 1.0;
  F.scaled = 0;
  DomainSpec D{0, 0, I.w, I.h, mc.out[0], ld_out};
  const bool fused = kernel_choice() == 2 &&
                     ((F.mode == kModeUniform && I.dt == 1 && nch == 3) ||
                      (F.mode == kModeLut && nch == 2));
  if (!fused) {
    for (int ch = 0; ch < nch; ++ch) {
      ImageSpec Ic = I;
      Ic.f = mc.f[ch];
      if ((rc = run_filter(Ic, F, 1, mc.out[ch], ld_out, s))) return rc;
    }
    return RUBS_OK;
  }
  if ((rc = ensure_ovf(D))) return rc;
  RUBS_CUDA_TRY(cudaMemsetAsync(t_scr.d_status, 0, sizeof(Status), s));
  const int wy = (I.h + kWideH - 1) / kWideH;
  {
    TimedLaunch tl(0, s);
    if (F.mode == kModeUniform)
      launch_wide_rows<kModeUniform, 1, 3>(I, F, D, 0, wy, s, &mc);
    else if (I.dt == 1)
      launch_wide_rows<kModeLut, 1, 2, 3>(I, F, D, 0, wy, s, &mc);
    else
      launch_wide_rows<kModeLut, 0, 2, 3>(I, F, D, 0, wy, s, &mc);
  }
  ++t_launches;
  RUBS_CUDA_TRY(cudaGetLastError());
  Status st;
  if ((rc = fetch_status(s, st))) return rc;
  if (st.ovf_count > 0 && !(st.flags & (kFlagFieldNonFinite | kFlagParamInvalid))) {
    for (int ch = 0; ch < nch; ++ch) {
      ImageSpec Ic = I;
      Ic.f = mc.f[ch];
      DomainSpec Dc = D;
      Dc.out = mc.out[ch];
      if ((rc = run_overflow(Ic, F, Dc, st.ovf_count, s))) return rc;
    }
    RUBS_CUDA_TRY(cudaMemsetAsync(&t_scr.d_status->ovf_count, 0, sizeof(int), s));
    if ((rc = fetch_status(s, st))) return rc;
  }
  return status_to_code(st);
}

int run_band(const ImageSpec &I, FieldSpec F, int64_t H_total, int64_t out_row0,
             int64_t out_rows, double *out, int64_t ld_out, cudaStream_t s) {
  int rc = ensure_scratch();
  if (rc) return rc;
  if (out_rows <= 0 || I.w == 0) return RUBS_OK;
  if (out_row0 < 0 || out_row0 + out_rows > H_total)
    return set_error(RUBS_EVALUE, "output rows outside the image");
  F.FH = (int)H_total;
  F.FW = I.w;
  F.div = 1.0;
  F.scaled = 0;
  RUBS_CUDA_TRY(cudaMemsetAsync(t_scr.d_status, 0, sizeof(Status), s));
  DomainSpec D{0, (int)out_row0, I.w, (int)out_rows, out, ld_out};
  if ((rc = launch_pass(I, F, D, s))) return rc;
  Status st;
  if ((rc = finish_pass(I, F, D, s, st))) return rc;
  return status_to_code(st);
}

// Host-buffer staging for the _host entry points (copies inside the call).
struct HostStage {
  void *buf[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t cap[5] = {0, 0, 0, 0, 0};
  cudaStream_t stream = nullptr;
  int device = -1;
};
thread_local HostStage t_stage_dev[rubs_internal::kMaxDevices];
#define t_stage (t_stage_dev[t_dev])

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
  int rc = ensure_scratch();  // selects the device's slot
  if (rc) return rc;
  if (!t_stage.stream) {
    t_stage.device = t_dev;
    RUBS_CUDA_TRY(cudaStreamCreateWithFlags(&t_stage.stream, cudaStreamNonBlocking));
  }
  *s = t_stage.stream;
  return RUBS_OK;
}

// Host-buffer calls, one pass: a pipeline over bands of output rows.  The
// image goes up whole, then each band's per-pixel inputs; a band's tiles
// launch as soon as its inputs have landed and its output rows go back
// while later bands are still in flight -- both copy engines and the SMs
// busy at once.  (The image must be complete first: a band's regions read
// rows beyond it by the read margins.)
struct HostPlane {
  const void *host;
  void *dev;
  size_t row_bytes;
};

struct StreamSet {
  int device = -1;
  cudaStream_t h2d = nullptr, cmp = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> ev;
};
thread_local StreamSet t_ss_dev[rubs_internal::kMaxDevices];
#define t_ss (t_ss_dev[t_dev])

int stream_set(size_t nev) {
  int rc = ensure_scratch();  // selects the device's slot
  if (rc) return rc;
  if (t_ss.device != t_dev) {
    t_ss.device = t_dev;
    RUBS_CUDA_TRY(cudaStreamCreateWithFlags(&t_ss.h2d, cudaStreamNonBlocking));
    RUBS_CUDA_TRY(cudaStreamCreateWithFlags(&t_ss.cmp, cudaStreamNonBlocking));
    RUBS_CUDA_TRY(cudaStreamCreateWithFlags(&t_ss.d2h, cudaStreamNonBlocking));
  }
  while (t_ss.ev.size() < nev) {
    cudaEvent_t e;
    RUBS_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    t_ss.ev.push_back(e);
  }
  return RUBS_OK;
}

int run_streamed(const ImageSpec &I, FieldSpec F, const void *f_host,
                 const std::vector<HostPlane> &planes, double *dout, double *out_host) {
  int rc = ensure_scratch();
  if (rc) return rc;
  const int H = I.h, W = I.w;
  F.FH = H;
  F.FW = W;
  F.div = 1.0;
  F.scaled = 0;
  const int wy = (H + kWideH - 1) / kWideH;
  // 8 bands: measured best on config 2 (4-8 equal, 16 -3 %, 32 -30 %: a
  // band's launch must still fill the GPU)
  const int nb = std::max(1, std::min(8, wy / 2));
  const int per = (wy + nb - 1) / nb;  // wide-tile rows per band
  if ((rc = stream_set(2 * (size_t)nb))) return rc;
  const cudaStream_t h2d = t_ss.h2d, cmp = t_ss.cmp, d2h = t_ss.d2h;
  DomainSpec D{0, 0, W, H, dout, W};
  if ((rc = ensure_ovf(D))) return rc;
  RUBS_CUDA_TRY(cudaMemsetAsync(t_scr.d_status, 0, sizeof(Status), cmp));
  const size_t esz = I.dt ? 8 : 4;
  RUBS_CUDA_TRY(cudaMemcpyAsync(const_cast<void *>(I.f), f_host, (size_t)H * W * esz,
                                cudaMemcpyHostToDevice, h2d));
  for (int b = 0; b < nb; ++b) {
    const int t0 = b * per, t1 = std::min(wy, (b + 1) * per);
    if (t0 >= t1) break;
    const int r0 = t0 * kWideH, r1 = std::min(H, t1 * kWideH);
    for (const HostPlane &pl : planes)
      RUBS_CUDA_TRY(cudaMemcpyAsync(static_cast<char *>(pl.dev) + r0 * pl.row_bytes,
                                    static_cast<const char *>(pl.host) + r0 * pl.row_bytes,
                                    (size_t)(r1 - r0) * pl.row_bytes, cudaMemcpyHostToDevice, h2d));
    RUBS_CUDA_TRY(cudaEventRecord(t_ss.ev[2 * b], h2d));
    RUBS_CUDA_TRY(cudaStreamWaitEvent(cmp, t_ss.ev[2 * b], 0));
    launch_wide_rows_rt(I, F, D, t0, t1, cmp, use_stage2() ? 0 : 2);
    ++t_launches;
    if (use_stage2()) {
      // stage 2 per band: the tiles listed so far are done before this
      // band's rows go back (each listed tile is taken by exactly one
      // stage-2 launch: the same outputs as the device path's single one)
      launch_wide_stage2_rt(I, F, D, cmp);
      ++t_launches;
    }
    RUBS_CUDA_TRY(cudaGetLastError());
    RUBS_CUDA_TRY(cudaEventRecord(t_ss.ev[2 * b + 1], cmp));
  }
  // the returns are enqueued last: a copy into pageable host memory blocks
  // the host until it has run, so every upload and launch is queued first
  for (int b = 0; b < nb; ++b) {
    const int t0 = b * per, t1 = std::min(wy, (b + 1) * per);
    if (t0 >= t1) break;
    const int r0 = t0 * kWideH, r1 = std::min(H, t1 * kWideH);
    RUBS_CUDA_TRY(cudaStreamWaitEvent(d2h, t_ss.ev[2 * b + 1], 0));
    RUBS_CUDA_TRY(cudaMemcpyAsync(out_host + (size_t)r0 * W, dout + (size_t)r0 * W,
                                  (size_t)(r1 - r0) * W * 8, cudaMemcpyDeviceToHost, d2h));
  }
  RUBS_CUDA_TRY(cudaStreamSynchronize(d2h));
  Status st;
  if ((rc = fetch_status(cmp, st))) return rc;
  const bool bad = st.flags & (kFlagFieldNonFinite | kFlagParamInvalid);
  if (st.ovf_count > 0 && !bad) {
    // deferred tiles: computed now; rows written after their band's return
    // go back once more
    if ((rc = run_overflow(I, F, D, st.ovf_count, cmp))) return rc;
    RUBS_CUDA_TRY(cudaMemsetAsync(&t_scr.d_status->ovf_count, 0, sizeof(int), cmp));
    if ((rc = fetch_status(cmp, st))) return rc;
    RUBS_CUDA_TRY(cudaMemcpyAsync(out_host, dout, (size_t)H * W * 8, cudaMemcpyDeviceToHost, cmp));
    RUBS_CUDA_TRY(cudaStreamSynchronize(cmp));
  }
  return status_to_code(st);
}

// Host-buffer calls on large images (H >= kBandStreamRows): the image is
// filtered band by band COMPLETELY -- each band of output rows through the
// whole path, deferred tiles and large-halo blocks included (run_band, the
// row-band entry of the multi-GPU split) -- so a band's rows go back while
// later bands are still uploading or computing.  (run_streamed defers every
// deferred tile to the end of the call: on config 5, where almost all tiles
// are deferred, that serialised ~110 ms of compute behind all the copies and
// returned the result twice.)  The image goes up in chunks first, then each
// band's parameters; band b waits for the image chunks its halo reaches
// (the LUT bound amax * sqrt(max size of the band), as sharding.py's
// halo_bound_params).  Band edges sit on the 32-row tile grid.
constexpr int64_t kBandStreamRows = 8192;
int run_streamed_bands(const ImageSpec &I, FieldSpec F, const void *f_host,
                       const std::vector<HostPlane> &planes, double *dout, double *out_host) {
  int rc = ensure_scratch();
  if (rc) return rc;
  const int H = I.h, W = I.w;
  constexpr int kChunks = 16;
  const int nb = 8;
  const int per = ((H + nb - 1) / nb + kTile - 1) / kTile * kTile;  // rows per band (tile grid)
  const int cper = (H + kChunks - 1) / kChunks;                     // rows per image chunk
  if ((rc = stream_set((size_t)kChunks + 2 * nb))) return rc;
  const cudaStream_t h2d = t_ss.h2d, cmp = t_ss.cmp, d2h = t_ss.d2h;
  const size_t esz = I.dt ? 8 : 4;
  for (int c = 0; c < kChunks; ++c) {
    const int r0 = c * cper, r1 = std::min(H, r0 + cper);
    if (r0 >= r1) break;
    RUBS_CUDA_TRY(cudaMemcpyAsync(static_cast<char *>(const_cast<void *>(I.f)) + (size_t)r0 * W * esz,
                                  static_cast<const char *>(f_host) + (size_t)r0 * W * esz,
                                  (size_t)(r1 - r0) * W * esz, cudaMemcpyHostToDevice, h2d));
    RUBS_CUDA_TRY(cudaEventRecord(t_ss.ev[c], h2d));
  }
  for (int b = 0; b < nb; ++b) {
    const int r0 = b * per, r1 = std::min(H, r0 + per);
    if (r0 >= r1) break;
    for (const HostPlane &pl : planes)
      RUBS_CUDA_TRY(cudaMemcpyAsync(static_cast<char *>(pl.dev) + r0 * pl.row_bytes,
                                    static_cast<const char *>(pl.host) + r0 * pl.row_bytes,
                                    (size_t)(r1 - r0) * pl.row_bytes, cudaMemcpyHostToDevice, h2d));
    RUBS_CUDA_TRY(cudaEventRecord(t_ss.ev[kChunks + 2 * b], h2d));
  }
  const size_t psz = F.pdt ? 8 : 4;
  for (int b = 0; b < nb; ++b) {
    const int r0 = b * per, r1 = std::min(H, r0 + per);
    if (r0 >= r1) break;
    RUBS_CUDA_TRY(cudaStreamWaitEvent(cmp, t_ss.ev[kChunks + 2 * b], 0));
    // the band's halo: largest size of its parameter rows (one reduction)
    FieldSpec Fb = F;
    Fb.ps = static_cast<const char *>(F.ps) + (size_t)r0 * F.pld * psz;
    Fb.FH = r1 - r0;
    Fb.FW = W;
    RUBS_CUDA_TRY(cudaMemsetAsync(t_scr.d_status, 0, sizeof(Status), cmp));
    size_max_kernel<<<4 * t_scr.sms, 256, 0, cmp>>>(Fb, t_scr.d_status);
    ++t_launches;
    Status st;
    if ((rc = fetch_status(cmp, st))) return rc;
    double smax = 0.0;
    std::memcpy(&smax, &st.smax_bits, sizeof(smax));
    const double A = std::max(F.lut_amax * std::sqrt(std::max(smax, 0.0)), 0.05);
    const int halo = (int)std::ceil(0.5 * A + A / std::sqrt(2.0) + 1.5) + 4;
    const int need_hi = std::min(H, r1 + halo);
    const int last_chunk = std::min(kChunks - 1, (need_hi - 1) / cper);
    RUBS_CUDA_TRY(cudaStreamWaitEvent(cmp, t_ss.ev[last_chunk], 0));
    if ((rc = run_band(I, F, H, r0, r1 - r0, dout + (size_t)r0 * W, W, cmp))) return rc;
    RUBS_CUDA_TRY(cudaEventRecord(t_ss.ev[kChunks + 2 * b + 1], cmp));
    RUBS_CUDA_TRY(cudaStreamWaitEvent(d2h, t_ss.ev[kChunks + 2 * b + 1], 0));
    RUBS_CUDA_TRY(cudaMemcpyAsync(out_host + (size_t)r0 * W, dout + (size_t)r0 * W,
                                  (size_t)(r1 - r0) * W * 8, cudaMemcpyDeviceToHost, d2h));
  }
  RUBS_CUDA_TRY(cudaStreamSynchronize(d2h));
  return RUBS_OK;
}

// The streamed path serves one-pass calls on the default (wide) kernel.
bool streamable(int iterations, int64_t H, int64_t W) {
  return iterations == 1 && kernel_choice() == 2 && H >= 2 * kWideH && W > 0 &&
         !std::getenv("RUBS_B200_NO_STREAM");
}

}  // namespace

struct rubs_lut {
  double *entries = nullptr;
  float *entries32 = nullptr;  // the same rolled copies in float32
  int n_rho = 0, n_phi = 0;
  double rho_max = 0.0;
  double amax = 0.0;  // largest component of any entry
};

namespace {
FieldSpec lut_field(const rubs_lut *lut, const void *size, const void *elong, const void *orient,
                    int p_dtype, int64_t ld_p) {
  FieldSpec F{};
  F.mode = p_dtype == RUBS_F64 ? kModeLut : kModeLut32;
  F.ps = size;
  F.pr = elong;
  F.pt = orient;
  F.pdt = p_dtype;
  F.pld = ld_p;
  F.lut = lut->entries;
  F.lut32 = lut->entries32;
  F.n_rho = lut->n_rho;
  F.n_phi = lut->n_phi;
  F.rho_max = lut->rho_max;
  F.log_rho_max = std::log(lut->rho_max);
  F.inv_log_rho_max = 1.0 / F.log_rho_max;
  F.phi_scale = (double)lut->n_phi / kQuarter;
  F.rho_lim = lut->rho_max * (1.0 + 1e-12);
  F.lut_amax = lut->amax;
  return F;
}
}  // namespace

extern "C" {

const char *rubs_b200_version(void) { return "rubs_b200 0.1.0 (sm_100a)"; }

int rubs_b200_dfma_peak(double *tflops, double *ms) {
  int rc = ensure_scratch();
  if (rc) return rc;
  constexpr int kIters = 4096;
  double *d = nullptr;
  const int blocks = t_scr.sms * 8, threads = 256;
  RUBS_CUDA_TRY(cudaMalloc(&d, (size_t)blocks * threads * sizeof(double)));
  cudaEvent_t e0, e1;
  RUBS_CUDA_TRY(cudaEventCreate(&e0));
  RUBS_CUDA_TRY(cudaEventCreate(&e1));
  dfma_probe_kernel<<<blocks, threads>>>(d, kIters);  // warm-up (clocks up)
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    RUBS_CUDA_TRY(cudaEventRecord(e0));
    dfma_probe_kernel<<<blocks, threads>>>(d, kIters);
    RUBS_CUDA_TRY(cudaEventRecord(e1));
    RUBS_CUDA_TRY(cudaEventSynchronize(e1));
    float t = 0.f;
    RUBS_CUDA_TRY(cudaEventElapsedTime(&t, e0, e1));
    best = std::min(best, t);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  const double fmas = (double)blocks * threads * 8.0 * kIters;
  if (ms) *ms = best;
  if (tflops) *tflops = 2.0 * fmas / (best * 1e-3) / 1e12;
  return RUBS_OK;
}

void rubs_b200_set_profiling(int enable) { t_timer.on = enable != 0; }

void rubs_b200_kernel_time(int kind, double *total_ms, int64_t *launches) {
  timer_collect();  // brackets closed after the call's last status read
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

int rubs_b200_precision_limited(void) {
  const int v = t_precision_limited;
  t_precision_limited = 0;
  return v;
}

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
  if (f_dtype != RUBS_F32 && f_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (streamable(iterations, H, W)) {
    ImageSpec I{df, f_dtype, W, (int)H, (int)W, 0, 0};
    FieldSpec F{};
    std::vector<HostPlane> planes;
    if (H > (1 << 30) || W > (1 << 30)) return set_error(RUBS_EUNSUPPORTED, "image too large");
    if (field_is_uniform) {
      F.mode = kModeUniform;
      for (int k = 0; k < 4; ++k) {
        F.u[k] = field[k];
        if (!std::isfinite(field[k])) return set_error(RUBS_EVALUE, "scale field entries must be finite");
      }
    } else {
      if ((rc = stage_buf(1, npx * 32, &dfield))) return rc;
      F.mode = kModeField;
      F.a = static_cast<const double *>(dfield);
      F.ld = W;
      planes.push_back({field, dfield, (size_t)W * 32});
    }
    return run_streamed(I, F, f, planes, (double *)dout, out);
  }
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
  for (size_t e = 0; e < (size_t)n_rho * n_phi * 4; ++e) L->amax = std::max(L->amax, entries[e]);
  // four copies, copy q rolled by q quarter turns: out[k] = mix[(k - q) mod 4]
  const size_t per = (size_t)n_rho * n_phi * 4;
  std::vector<double> rolled(4 * per);
  for (int q = 0; q < 4; ++q)
    for (size_t e = 0; e < (size_t)n_rho * n_phi; ++e)
      for (int k = 0; k < 4; ++k) rolled[q * per + e * 4 + k] = entries[e * 4 + ((k - q + 4) & 3)];
  size_t bytes = rolled.size() * sizeof(double);
  // float32 copy of the rolled table: the planning bounds (lut_bounds_f32)
  std::vector<float> rolled32(rolled.begin(), rolled.end());
  cudaError_t e = cudaMalloc(&L->entries, bytes);
  if (e == cudaSuccess) e = cudaMemcpy(L->entries, rolled.data(), bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&L->entries32, rolled32.size() * sizeof(float));
  if (e == cudaSuccess)
    e = cudaMemcpy(L->entries32, rolled32.data(), rolled32.size() * sizeof(float), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (L->entries) cudaFree(L->entries);
    if (L->entries32) cudaFree(L->entries32);
    delete L;
    return set_error(RUBS_ECUDA, std::string("lut upload: ") + cudaGetErrorString(e));
  }
  *out = L;
  return RUBS_OK;
}

void rubs_b200_lut_destroy(rubs_lut *lut) {
  if (!lut) return;
  if (lut->entries) cudaFree(lut->entries);
  if (lut->entries32) cudaFree(lut->entries32);
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
  if (f_dtype != RUBS_F32 && f_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (p_dtype != RUBS_F32 && p_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (!lut) return set_error(RUBS_EVALUE, "lut is NULL");
  if (streamable(iterations, H, W)) {
    ImageSpec I{df, f_dtype, W, (int)H, (int)W, 0, 0};
    FieldSpec F = lut_field(lut, pb, pb + npx * psz, pb + 2 * npx * psz, p_dtype, W);
    const size_t rb = (size_t)W * psz;
    std::vector<HostPlane> planes = {{size, pb, rb}, {elong, pb + npx * psz, rb},
                                     {orient, pb + 2 * npx * psz, rb}};
    if (H >= kBandStreamRows && !std::getenv("RUBS_B200_NO_BAND_STREAM"))
      return run_streamed_bands(I, F, f, planes, (double *)dout, out);
    return run_streamed(I, F, f, planes, (double *)dout, out);
  }
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

int rubs_b200_filter_params_batch_host(int n, const void *const *f, int f_dtype, int64_t H,
                                       int64_t W, const void *const *size,
                                       const void *const *elong, const void *const *orient,
                                       int p_dtype, const rubs_lut *lut, int iterations,
                                       double *const *out, int *failed) {
  if (failed) *failed = -1;
  if (n < 0) return set_error(RUBS_EVALUE, "negative batch size");
  if (f_dtype != RUBS_F32 && f_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (p_dtype != RUBS_F32 && p_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (!lut) return set_error(RUBS_EVALUE, "lut is NULL");
  if (iterations < 1) return set_error(RUBS_EVALUE, "iterations must be >= 1");
  if (H < 0 || W < 0) return set_error(RUBS_EVALUE, "image must be 2-D");
  if (n == 0 || H == 0 || W == 0) return RUBS_OK;
  int rc = stream_set(6);  // ev: [0, 2) inputs landed, [2, 4) filtered, [4, 6) returned
  if (rc) return rc;
  const cudaStream_t h2d = t_ss.h2d, cmp = t_ss.cmp, d2h = t_ss.d2h;
  const size_t esz = f_dtype == RUBS_F64 ? 8 : 4, psz = p_dtype == RUBS_F64 ? 8 : 4;
  const size_t npx = (size_t)H * W;
  // two slots of device inputs / outputs (stage buffers 0-2 and 3-4 + pass)
  void *df[2], *dp[2], *dout[2];
  if ((rc = stage_buf(0, npx * esz, &df[0]))) return rc;
  if ((rc = stage_buf(1, npx * psz * 3, &dp[0]))) return rc;
  if ((rc = stage_buf(2, npx * 8, &dout[0]))) return rc;
  if ((rc = stage_buf(3, npx * esz + npx * psz * 3, &df[1]))) return rc;
  dp[1] = static_cast<char *>(df[1]) + npx * esz;
  if ((rc = stage_buf(4, npx * 8, &dout[1]))) return rc;
  auto upload = [&](int i) -> int {
    const int k = i & 1;
    char *pb = static_cast<char *>(dp[k]);
    if (i >= 2) RUBS_CUDA_TRY(cudaStreamWaitEvent(h2d, t_ss.ev[2 + k], 0));  // slot's inputs consumed
    RUBS_CUDA_TRY(cudaMemcpyAsync(df[k], f[i], npx * esz, cudaMemcpyHostToDevice, h2d));
    RUBS_CUDA_TRY(cudaMemcpyAsync(pb, size[i], npx * psz, cudaMemcpyHostToDevice, h2d));
    RUBS_CUDA_TRY(cudaMemcpyAsync(pb + npx * psz, elong[i], npx * psz, cudaMemcpyHostToDevice, h2d));
    RUBS_CUDA_TRY(cudaMemcpyAsync(pb + 2 * npx * psz, orient[i], npx * psz, cudaMemcpyHostToDevice, h2d));
    RUBS_CUDA_TRY(cudaEventRecord(t_ss.ev[k], h2d));
    return RUBS_OK;
  };
  if ((rc = upload(0))) return rc;
  for (int i = 0; i < n; ++i) {
    const int k = i & 1;
    // the next image's inputs go up while this one is filtered
    if (i + 1 < n && (rc = upload(i + 1))) return rc;
    RUBS_CUDA_TRY(cudaStreamWaitEvent(cmp, t_ss.ev[k], 0));
    if (i >= 2) RUBS_CUDA_TRY(cudaStreamWaitEvent(cmp, t_ss.ev[4 + k], 0));  // slot's result returned
    char *pb = static_cast<char *>(dp[k]);
    rc = rubs_b200_filter_params(df[k], f_dtype, H, W, W, pb, pb + npx * psz, pb + 2 * npx * psz,
                                 p_dtype, W, lut, iterations, static_cast<double *>(dout[k]), W, cmp);
    if (rc) {
      if (failed) *failed = i;
      cudaStreamSynchronize(h2d);
      cudaStreamSynchronize(d2h);
      return rc;
    }
    RUBS_CUDA_TRY(cudaEventRecord(t_ss.ev[2 + k], cmp));
    RUBS_CUDA_TRY(cudaStreamWaitEvent(d2h, t_ss.ev[2 + k], 0));
    RUBS_CUDA_TRY(cudaMemcpyAsync(out[i], dout[k], npx * 8, cudaMemcpyDeviceToHost, d2h));
    RUBS_CUDA_TRY(cudaEventRecord(t_ss.ev[4 + k], d2h));
  }
  RUBS_CUDA_TRY(cudaStreamSynchronize(d2h));
  return RUBS_OK;
}

int rubs_b200_filter_rows(const void *f, int f_dtype, int64_t f_row0, int64_t f_rows, int64_t W,
                          int64_t ld_f, int64_t H_total, const double *field, int64_t field_row0,
                          int64_t ld_field, int64_t out_row0, int64_t out_rows, double *out,
                          int64_t ld_out, void *stream) {
  if (f_dtype != RUBS_F32 && f_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  ImageSpec I{f, f_dtype, ld_f, (int)f_rows, (int)W, 0, (int)f_row0};
  FieldSpec F{};
  F.mode = kModeField;
  F.a = field;
  F.ld = ld_field;
  F.fr_off = (int)field_row0;
  return run_band(I, F, H_total, out_row0, out_rows, out, ld_out, static_cast<cudaStream_t>(stream));
}

int rubs_b200_filter_params_rows(const void *f, int f_dtype, int64_t f_row0, int64_t f_rows,
                                 int64_t W, int64_t ld_f, int64_t H_total, const void *size,
                                 const void *elong, const void *orient, int p_dtype,
                                 int64_t p_row0, int64_t ld_p, const rubs_lut *lut,
                                 int64_t out_row0, int64_t out_rows, double *out, int64_t ld_out,
                                 void *stream) {
  if (f_dtype != RUBS_F32 && f_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (p_dtype != RUBS_F32 && p_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (!lut) return set_error(RUBS_EVALUE, "lut is NULL");
  ImageSpec I{f, f_dtype, ld_f, (int)f_rows, (int)W, 0, (int)f_row0};
  FieldSpec F = lut_field(lut, size, elong, orient, p_dtype, ld_p);
  F.fr_off = (int)p_row0;
  return run_band(I, F, H_total, out_row0, out_rows, out, ld_out, static_cast<cudaStream_t>(stream));
}

// _read_margins (engine.py:247-262) over rows [row0, row0 + rows) of a field
// or parameter set: out4 = (left, right, below, above), reference arithmetic.
static int read_margins(FieldSpec F, int64_t rows, int64_t W, int64_t H_total, int64_t row0,
                        int iterations, int *out4, cudaStream_t s) {
  int rc = ensure_scratch();
  if (rc) return rc;
  if (iterations < 1) return set_error(RUBS_EVALUE, "iterations must be >= 1");
  F.FH = (int)H_total;
  F.FW = (int)W;
  F.fr_off = (int)row0;
  F.div = std::sqrt((double)iterations);
  F.scaled = iterations > 1;
  RUBS_CUDA_TRY(cudaMemsetAsync(t_scr.d_status, 0, sizeof(Status), s));
  DomainSpec D{0, (int)row0, (int)W, (int)rows, nullptr, 0};
  if (rows > 0 && W > 0 && (rc = launch_global_margins(F, D, s))) return rc;
  Status st;
  if ((rc = fetch_status(s, st))) return rc;
  for (int k = 0; k < 4; ++k) out4[k] = st.gm[k];
  return status_to_code(st);
}

int rubs_b200_read_margins(const double *field, int field_is_uniform, int64_t rows, int64_t W,
                           int64_t ld_field, int64_t H_total, int64_t row0, int iterations,
                           int *out4, void *stream) {
  FieldSpec F{};
  if (field_is_uniform) {
    F.mode = kModeUniform;
    for (int k = 0; k < 4; ++k) F.u[k] = field[k];
  } else {
    F.mode = kModeField;
    F.a = field;
    F.ld = ld_field;
  }
  return read_margins(F, rows, W, H_total, row0, iterations, out4, static_cast<cudaStream_t>(stream));
}

int rubs_b200_read_margins_params(const void *size, const void *elong, const void *orient,
                                  int p_dtype, int64_t rows, int64_t W, int64_t ld_p,
                                  int64_t H_total, int64_t row0, const rubs_lut *lut,
                                  int iterations, int *out4, void *stream) {
  if (!lut) return set_error(RUBS_EVALUE, "lut is NULL");
  FieldSpec F = lut_field(lut, size, elong, orient, p_dtype, ld_p);
  return read_margins(F, rows, W, H_total, row0, iterations, out4, static_cast<cudaStream_t>(stream));
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

namespace rubs_internal {
int set_error(int code, const std::string &msg) { return ::set_error(code, msg); }
void count_launches(int n) { t_launches += n; }
void *timed_begin(int kind, void *stream) {
  return new TimedLaunch(kind, static_cast<cudaStream_t>(stream));
}
void timed_end(void *token) { delete static_cast<TimedLaunch *>(token); }
void timer_collect() { ::timer_collect(); }
double lut_rho_max(const rubs_lut *lut) { return lut->rho_max; }

int filter_uniform_multi(const double *const *f, int nch, int64_t H, int64_t W, int64_t ld,
                         const double a[4], double *const *out, int64_t ld_out, void *stream) {
  if (nch < 1 || nch > 3) return ::set_error(RUBS_EVALUE, "1 to 3 channels");
  ImageSpec I{f[0], 1, ld, (int)H, (int)W, 0, 0};
  FieldSpec F{};
  F.mode = kModeUniform;
  for (int k = 0; k < 4; ++k) {
    F.u[k] = a[k];
    if (!std::isfinite(a[k])) return ::set_error(RUBS_EVALUE, "scale field entries must be finite");
  }
  MultiChan mc{};
  for (int ch = 0; ch < nch; ++ch) {
    mc.f[ch] = f[ch];
    mc.out[ch] = out[ch];
  }
  return run_multi(I, mc, nch, F, ld_out, static_cast<cudaStream_t>(stream));
}

int filter_params_multi(const void *const *f, int f_dtype, int nch, int64_t H, int64_t W,
                        int64_t ld, const void *size, const void *elong, const void *orient,
                        int p_dtype, int64_t ld_p, const rubs_lut *lut, double *const *out,
                        int64_t ld_out, void *stream) {
  if (nch < 1 || nch > 3) return ::set_error(RUBS_EVALUE, "1 to 3 channels");
  if (f_dtype != RUBS_F32 && f_dtype != RUBS_F64) return ::set_error(RUBS_EVALUE, "bad dtype");
  if (p_dtype != RUBS_F32 && p_dtype != RUBS_F64) return ::set_error(RUBS_EVALUE, "bad dtype");
  if (!lut) return ::set_error(RUBS_EVALUE, "lut is NULL");
  ImageSpec I{f[0], f_dtype, ld, (int)H, (int)W, 0, 0};
  FieldSpec F = lut_field(lut, size, elong, orient, p_dtype, ld_p);
  MultiChan mc{};
  for (int ch = 0; ch < nch; ++ch) {
    mc.f[ch] = f[ch];
    mc.out[ch] = out[ch];
  }
  return run_multi(I, mc, nch, F, ld_out, static_cast<cudaStream_t>(stream));
}
}  // namespace rubs_internal
