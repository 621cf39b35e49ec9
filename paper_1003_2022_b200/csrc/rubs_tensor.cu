// rubs_tensor.cu -- the reference's own caller of the hot path, on the B200:
// the structure-tensor / adaptive smoothing pipeline of
// pkg/src/rubs/tensor.py.
//
//   structure_tensor        gradient kernel (reflect padding, central
//                           differences) + three isotropic filter passes
//                           through rubs_b200_filter (tensor.py:52-75)
//   anisotropy_from_tensor  5th / 95th percentiles of the trace by an
//                           exact radix select on the device, then one
//                           elementwise kernel (tensor.py:90-171)
//   adaptive_smooth         the above, the fused LUT filter on the image
//                           and on a flat image, and the gain correction
//                           (tensor.py:174-224)
//
// Everything runs on the caller's stream through the C ABI; the filter
// passes are the hot path itself.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rubs_b200.h"
#include "rubs_internal.h"

using rubs_internal::set_error;

namespace {

#define RT_CUDA_TRY(expr)                                                            \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return set_error(RUBS_ECUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
  } while (0)

constexpr double kPi = 3.141592653589793;
constexpr double kEigRel = 1e-8, kEigAbs = 1e-12;  // tensor.py:29-30
constexpr double kScaleFloor = 0.05;               // engine.py:58

// Grow-only device scratch of this host thread.
struct TScratch {
  int device = -1;
  void *buf[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t cap[6] = {0, 0, 0, 0, 0, 0};
  unsigned *d_hist = nullptr;      // 4 x 256 radix-select histograms
  unsigned *h_hist = nullptr;      // pinned
};
thread_local TScratch t_ts_dev[rubs_internal::kMaxDevices];
thread_local int t_ts_cur = 0;  // set by tbuf()
#define t_ts (t_ts_dev[t_ts_cur])

int tbuf(int k, size_t bytes, void **out) {
  int dev = 0;
  RT_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= rubs_internal::kMaxDevices)
    return set_error(RUBS_ECUDA, "device index beyond the per-device state table");
  t_ts_cur = dev;
  t_ts.device = dev;
  if (bytes > t_ts.cap[k]) {
    if (t_ts.buf[k]) cudaFree(t_ts.buf[k]);
    t_ts.buf[k] = nullptr;
    RT_CUDA_TRY(cudaMalloc(&t_ts.buf[k], bytes));
    t_ts.cap[k] = bytes;
  }
  *out = t_ts.buf[k];
  return RUBS_OK;
}

// ---------------------------------------------------------------------------
// structure tensor: gradients on the reflect-padded image (np.pad
// mode="reflect": index -1 -> 1, n -> n - 2), J = (gx^2, gx gy, gy^2)
// (tensor.py:66-69), planar float64 outputs

__device__ __forceinline__ int reflect(int i, int n) {
  if (n == 1) return 0;
  return i < 0 ? -i : (i >= n ? 2 * n - 2 - i : i);
}

template <int DT>
__device__ __forceinline__ double px(const void *f, int64_t i) {
  if constexpr (DT == 1)
    return __ldg(static_cast<const double *>(f) + i);
  else
    return (double)__ldg(static_cast<const float *>(f) + i);
}

template <int DT>
__global__ void grad_tensor_kernel(const void *f, int H, int W, int64_t ld, double *j11,
                                   double *j12, double *j22) {
  const int64_t n = (int64_t)H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / W), c = (int)(i - (int64_t)r * W);
    const int64_t row = (int64_t)r * ld;
    const double gx = 0.5 * (px<DT>(f, row + reflect(c + 1, W)) - px<DT>(f, row + reflect(c - 1, W)));
    const double gy = 0.5 * (px<DT>(f, (int64_t)reflect(r + 1, H) * ld + c) -
                             px<DT>(f, (int64_t)reflect(r - 1, H) * ld + c));
    j11[i] = gx * gx;
    j12[i] = gx * gy;
    j22[i] = gy * gy;
  }
}

__global__ void interleave3_kernel(const double *a, const double *b, const double *c, int64_t n,
                                   double *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[3 * i] = a[i];
    out[3 * i + 1] = b[i];
    out[3 * i + 2] = c[i];
  }
}

// ---------------------------------------------------------------------------
// exact order statistics of the trace J11 + J22: radix select over the
// order-preserving unsigned image of the float64 bits, 8 bits per pass, up
// to four ranks at once (np.percentile needs v[floor(i)], v[floor(i) + 1]
// for each of the 5th and 95th percentiles)

__device__ __forceinline__ uint64_t order_key(double v) {
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

inline double key_value(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double v;
  memcpy(&v, &b, sizeof v);
  return v;
}

// Radix-select state, on the device: the selected key prefix and the
// remaining rank of each of the (up to 4) wanted order statistics.
struct SelectState {
  unsigned long long prefix[4];
  long long left[4];
};

// tr = J11 + J22 (tensor.py:117), compacted once for the select passes
__global__ void trace_kernel(const double *j, int64_t n, double *tr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    tr[i] = j[3 * i] + j[3 * i + 2];
}

// One 8-bit digit: counts of the keys that match each rank's prefix above
// the digit (bits >= shift + 8).
__global__ void select_hist_kernel(const double *tr, int64_t n, int nr, int shift,
                                   const SelectState *ss, unsigned *hist) {
  __shared__ unsigned h[4][256];
  __shared__ unsigned long long pre[4];
  for (int t = threadIdx.x; t < 4 * 256; t += blockDim.x) (&h[0][0])[t] = 0;
  if (threadIdx.x < 4) pre[threadIdx.x] = ss->prefix[threadIdx.x];
  __syncthreads();
  const int hi = shift + 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = order_key(tr[i]);
    const unsigned byte = (unsigned)(k >> shift) & 255u;
    for (int r = 0; r < nr; ++r)
      if (hi >= 64 || (k >> hi) == (pre[r] >> hi)) atomicAdd(&h[r][byte], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nr * 256; t += blockDim.x) {
    const unsigned v = (&h[0][0])[t];
    if (v) atomicAdd(hist + t, v);
  }
}

// Pick each rank's bucket of this digit, extend its prefix, and clear the
// histogram for the next digit -- no host round trip per digit.  One CTA of
// 256 threads: an inclusive scan of the 256 counts in shared memory, then the
// bin whose [exclusive, inclusive) count range holds the remaining rank.
__global__ void __launch_bounds__(256) select_pick_kernel(int nr, int shift, SelectState *ss,
                                                          unsigned *hist) {
  __shared__ unsigned long long c[256];
  __shared__ long long s_left;
  const int t = threadIdx.x;
  for (int r = 0; r < nr; ++r) {
    const unsigned long long own = hist[r * 256 + t];
    c[t] = own;
    if (t == 0) s_left = ss->left[r];  // read before the selected thread rewrites it
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {  // Hillis-Steele inclusive scan
      const unsigned long long v = t >= o ? c[t - o] : 0ull;
      __syncthreads();
      c[t] += v;
      __syncthreads();
    }
    const long long left = s_left;
    const long long inc = (long long)c[t], exc = inc - (long long)own;
    // the first bin whose inclusive count exceeds the rank (bin 255 takes
    // any remainder) -- the host loop's `while (left >= h[b]) left -= h[b++]`
    if (exc <= left && (left < inc || t == 255)) {
      ss->left[r] = left - exc;
      ss->prefix[r] |= (unsigned long long)t << shift;
    }
    __syncthreads();
  }
  for (int i = t; i < nr * 256; i += blockDim.x) hist[i] = 0u;
}

// values[r] = the element of rank ranks[r] (0-based, ascending) of tr
int select_trace(const double *tr, int64_t n, const int64_t *ranks, int nr, double *values,
                 cudaStream_t s) {
  {
    int dev = 0;
    RT_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= rubs_internal::kMaxDevices)
      return set_error(RUBS_ECUDA, "device index beyond the per-device state table");
    t_ts_cur = dev;
  }
  if (!t_ts.d_hist) {
    RT_CUDA_TRY(cudaMalloc(&t_ts.d_hist, 4 * 256 * sizeof(unsigned) + sizeof(SelectState)));
    RT_CUDA_TRY(cudaMallocHost(&t_ts.h_hist, sizeof(SelectState)));
    RT_CUDA_TRY(cudaMemsetAsync(t_ts.d_hist, 0, 4 * 256 * sizeof(unsigned), s));
  }
  SelectState *ss = reinterpret_cast<SelectState *>(t_ts.d_hist + 4 * 256);
  SelectState *hs = reinterpret_cast<SelectState *>(t_ts.h_hist);
  for (int r = 0; r < 4; ++r) {
    hs->prefix[r] = 0;
    hs->left[r] = r < nr ? ranks[r] : 0;
  }
  RT_CUDA_TRY(cudaMemcpyAsync(ss, hs, sizeof(SelectState), cudaMemcpyHostToDevice, s));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 4 * sms);
  for (int shift = 56; shift >= 0; shift -= 8) {
    select_hist_kernel<<<grid, 256, 0, s>>>(tr, n, nr, shift, ss, t_ts.d_hist);
    select_pick_kernel<<<1, 256, 0, s>>>(nr, shift, ss, t_ts.d_hist);
    rubs_internal::count_launches(2);
    RT_CUDA_TRY(cudaGetLastError());
  }
  RT_CUDA_TRY(cudaMemcpyAsync(hs, ss, sizeof(SelectState), cudaMemcpyDeviceToHost, s));
  RT_CUDA_TRY(cudaStreamSynchronize(s));
  for (int r = 0; r < nr; ++r) values[r] = key_value(hs->prefix[r]);
  return RUBS_OK;
}

// np.percentile(tr, q), method "linear" (numpy's _lerp: a + (b - a) t,
// and b - (b - a)(1 - t) for t >= 0.5)
void percentile_ranks(int64_t n, double q, int64_t &lo, int64_t &hi, double &t) {
  const double vi = (q / 100.0) * (double)(n - 1);
  const double fl = std::floor(vi);
  lo = std::min<int64_t>((int64_t)fl, n - 1);
  hi = std::min<int64_t>(lo + 1, n - 1);
  t = vi - fl;
}

double lerp_np(double a, double b, double t) {
  const double d = b - a;
  return t >= 0.5 ? b - d * (1.0 - t) : a + d * t;
}

// ---------------------------------------------------------------------------
// anisotropy (tensor.py:114-171), elementwise

struct AnisoParams {
  double q05, q95, s_min, s_max, bound_fraction, size_iso, rho_cap;
  int has_spread;
};

__device__ __forceinline__ double elongation_bound_v(double phi) {  // tensor.py:77-86
  const double s2 = sin(2.0 * phi), c2 = cos(2.0 * phi);
  const double nu = fabs(c2 / s2);
  const double root = hypot(1.0, nu);
  const double out = (1.0 + nu + root) / (1.0 - 1.0 / (nu + root));
  return isfinite(nu) ? out : INFINITY;
}

__global__ void anisotropy_kernel(const double *j, int64_t n, AnisoParams p, double *size,
                                  double *rho, double *theta, unsigned char *iso) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double j11 = j[3 * i], j12 = j[3 * i + 1], j22 = j[3 * i + 2];
    const double tr = j11 + j22;
    const double disc = hypot(j11 - j22, 2.0 * j12);
    const double lmax = 0.5 * (tr + disc), lmin = 0.5 * (tr - disc);
    const double thr = kEigRel * tr + kEigAbs;
    const bool has_major = lmax > thr, has_minor = lmin > thr;
    double th = 0.5 * atan2(2.0 * j12, j11 - j22) + 0.5 * kPi;
    th = fmod(th, kPi);  // np.mod: th >= 0 here, so fmod agrees
    if (th < 0.0) th += kPi;
    if (!has_major) th = 0.0;
    double r = has_major && has_minor ? lmax / lmin : (has_major ? fmax(1.0, lmax) : 1.0);
    r = fmin(r, p.bound_fraction * elongation_bound_v(th));
    r = fmax(r, 1.0);
    double sz;
    if (p.has_spread)
      sz = p.s_max + (tr - p.q05) * (p.s_min - p.s_max) / (p.q95 - p.q05);
    else
      sz = 0.5 * (p.s_min + p.s_max);
    sz = fmin(fmax(sz, p.s_min), p.s_max);
    if (!has_major) {
      sz = p.size_iso;
      r = 1.0;
    }
    if (p.rho_cap > 0.0) r = fmin(r, p.rho_cap);  // adaptive_smooth (tensor.py:216)
    size[i] = sz;
    rho[i] = r;
    theta[i] = th;
    if (iso) iso[i] = has_major ? 0 : 1;
  }
}

// out <- out / gain where |gain| > 1e-6 (tensor.py:222-224)
__global__ void gain_correct_kernel(double *out, int64_t ld_out, const double *gain, int H,
                                    int W) {
  const int64_t n = (int64_t)H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / W), c = (int)(i - (int64_t)r * W);
    const double g = gain[i];
    double &o = out[(int64_t)r * ld_out + c];
    if (fabs(g) > 1e-6) o = o / (g == 0.0 ? 1.0 : g);
  }
}

template <class T>
__global__ void fill_kernel(T *p, int64_t n, T v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

int grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 8 * sms));
}

int anisotropy_impl(const double *j, int64_t H, int64_t W, double noise_sigma,
                    const double *size_range, double bound_fraction, double iso_gain,
                    double rho_cap, double *size, double *rho, double *theta, unsigned char *iso,
                    cudaStream_t s) {
  if (!(bound_fraction > 0.0 && bound_fraction < 1.0))
    return set_error(RUBS_EVALUE, "bound_fraction must lie in (0, 1)");
  double s_min = 0.5, s_max = 3.0 * noise_sigma * noise_sigma + 0.5;
  if (size_range) {
    s_min = size_range[0];
    s_max = size_range[1];
  }
  if (!(0.0 < s_min && s_min <= s_max))
    return set_error(RUBS_EVALUE, "size_range must be positive and ordered");
  const int64_t n = H * W;
  if (n == 0) return RUBS_OK;
  AnisoParams p{};
  int64_t r5lo, r5hi, r95lo, r95hi;
  double t5, t95;
  percentile_ranks(n, 5.0, r5lo, r5hi, t5);
  percentile_ranks(n, 95.0, r95lo, r95hi, t95);
  const int64_t ranks[4] = {r5lo, r5hi, r95lo, r95hi};
  double v[4];
  void *trb;
  int rc = tbuf(0, n * sizeof(double), &trb);
  if (rc) return rc;
  trace_kernel<<<grid_for(n), 256, 0, s>>>(j, n, static_cast<double *>(trb));
  rubs_internal::count_launches(1);
  RT_CUDA_TRY(cudaGetLastError());
  if ((rc = select_trace(static_cast<const double *>(trb), n, ranks, 4, v, s))) return rc;
  p.q05 = lerp_np(v[0], v[1], t5);
  p.q95 = lerp_np(v[2], v[3], t95);
  p.has_spread = (p.q95 - p.q05) > 1e-300;
  p.s_min = s_min;
  p.s_max = s_max;
  p.bound_fraction = bound_fraction;
  const double sigma_iso = std::max(iso_gain * noise_sigma * noise_sigma, 1.0);
  p.size_iso = sigma_iso * sigma_iso / 3.0;
  p.rho_cap = rho_cap;
  anisotropy_kernel<<<grid_for(n), 256, 0, s>>>(j, n, p, size, rho, theta, iso);
  rubs_internal::count_launches(1);
  RT_CUDA_TRY(cudaGetLastError());
  return RUBS_OK;
}

int structure_tensor_impl(const void *f, int f_dtype, int64_t H, int64_t W, int64_t ld_f,
                          double window_sigma, double *j, cudaStream_t s) {
  if (f_dtype != RUBS_F32 && f_dtype != RUBS_F64) return set_error(RUBS_EVALUE, "bad dtype");
  if (!(window_sigma >= 0.0)) return set_error(RUBS_EVALUE, "window_sigma must be >= 0");
  const int64_t n = H * W;
  if (n == 0) return RUBS_OK;
  void *b[6];
  int rc;
  for (int k = 0; k < 6; ++k)
    if ((rc = tbuf(k, n * sizeof(double), &b[k]))) return rc;
  double *g[3] = {(double *)b[0], (double *)b[1], (double *)b[2]};
  if (f_dtype == RUBS_F64)
    grad_tensor_kernel<1><<<grid_for(n), 256, 0, s>>>(f, (int)H, (int)W, ld_f, g[0], g[1], g[2]);
  else
    grad_tensor_kernel<0><<<grid_for(n), 256, 0, s>>>(f, (int)H, (int)W, ld_f, g[0], g[1], g[2]);
  rubs_internal::count_launches(1);
  RT_CUDA_TRY(cudaGetLastError());
  const double *src[3] = {g[0], g[1], g[2]};
  if (window_sigma > 0.0) {
    // isotropic scale-vector c (1,1,1,1): covariance c^2/6 I (tensor.py:72-74);
    // the three channels share the kernel: one three-channel pass
    const double c = std::max(window_sigma * std::sqrt(6.0), kScaleFloor);
    const double a[4] = {c, c, c, c};
    double *dst[3] = {(double *)b[3], (double *)b[4], (double *)b[5]};
    const double *chans[3] = {g[0], g[1], g[2]};
    if ((rc = rubs_internal::filter_uniform_multi(chans, 3, H, W, W, a, dst, W, s))) return rc;
    for (int k = 0; k < 3; ++k) src[k] = dst[k];
  }
  interleave3_kernel<<<grid_for(n), 256, 0, s>>>(src[0], src[1], src[2], n, j);
  rubs_internal::count_launches(1);
  RT_CUDA_TRY(cudaGetLastError());
  return RUBS_OK;
}

}  // namespace

extern "C" {

int rubs_b200_structure_tensor(const void *f, int f_dtype, int64_t H, int64_t W, int64_t ld_f,
                               double window_sigma, double *j, void *stream) {
  return structure_tensor_impl(f, f_dtype, H, W, ld_f, window_sigma, j,
                               static_cast<cudaStream_t>(stream));
}

int rubs_b200_anisotropy(const double *j, int64_t H, int64_t W, double noise_sigma,
                         const double *size_range, double bound_fraction, double iso_gain,
                         double *size, double *elong, double *orient, unsigned char *isotropic,
                         void *stream) {
  return anisotropy_impl(j, H, W, noise_sigma, size_range, bound_fraction, iso_gain, 0.0, size,
                         elong, orient, isotropic, static_cast<cudaStream_t>(stream));
}

int rubs_b200_adaptive_smooth(const void *f, int f_dtype, int64_t H, int64_t W, int64_t ld_f,
                              double noise_sigma, double window_sigma, int iterations,
                              const rubs_lut *lut, double bound_fraction,
                              const double *size_range, double iso_gain, double *out,
                              int64_t ld_out, void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!(noise_sigma >= 0.0)) return set_error(RUBS_EVALUE, "noise_sigma must be >= 0");
  if (!lut) return set_error(RUBS_EVALUE, "lut is NULL");
  const int64_t n = H * W;
  if (n == 0) return RUBS_OK;
  // scratch: J (3n), size / rho / theta (3n), flat image (n), gain (n)
  double *J, *maps, *ones, *gain;
  int rc;
  // buffers 0-5 are used by structure_tensor_impl; the pipeline's own go in
  // dedicated allocations of the same grow-only kind
  static thread_local std::vector<std::pair<void *, size_t>> own_dev[rubs_internal::kMaxDevices];
  int dev = 0;
  RT_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= rubs_internal::kMaxDevices)
    return set_error(RUBS_ECUDA, "device index beyond the per-device state table");
  auto &own = own_dev[dev];
  if (own.empty()) own.assign(4, {nullptr, 0});
  auto obuf = [&](int k, size_t bytes, double **o) -> int {
    if (bytes > own[k].second) {
      if (own[k].first) cudaFree(own[k].first);
      own[k].first = nullptr;
      RT_CUDA_TRY(cudaMalloc(&own[k].first, bytes));
      own[k].second = bytes;
    }
    *o = static_cast<double *>(own[k].first);
    return RUBS_OK;
  };
  if ((rc = obuf(0, 3 * n * sizeof(double), &J))) return rc;
  if ((rc = obuf(1, 3 * n * sizeof(double), &maps))) return rc;
  if ((rc = obuf(2, n * sizeof(double), &ones))) return rc;
  if ((rc = obuf(3, n * sizeof(double), &gain))) return rc;
  if ((rc = structure_tensor_impl(f, f_dtype, H, W, ld_f, window_sigma, J, s))) return rc;
  double *size = maps, *rho = maps + n, *theta = maps + 2 * n;
  if ((rc = anisotropy_impl(J, H, W, noise_sigma, size_range, bound_fraction, iso_gain,
                            rubs_internal::lut_rho_max(lut) * (1.0 - 1e-9), size, rho, theta,
                            nullptr, s)))
    return rc;
  // out = filter(f), gain = filter(1) with the same per-pixel kernels: one
  // two-channel pass (a flat image of f's dtype next to f) when possible
  if (f_dtype == RUBS_F32)
    fill_kernel<float><<<grid_for(n), 256, 0, s>>>(reinterpret_cast<float *>(ones), n, 1.0f);
  else
    fill_kernel<double><<<grid_for(n), 256, 0, s>>>(ones, n, 1.0);
  rubs_internal::count_launches(1);
  RT_CUDA_TRY(cudaGetLastError());
  if (iterations == 1 && ld_f == W && ld_out == W) {
    const void *chans[2] = {f, ones};
    double *dst[2] = {out, gain};
    if ((rc = rubs_internal::filter_params_multi(chans, f_dtype, 2, H, W, W, size, rho, theta,
                                                 RUBS_F64, W, lut, dst, W, s)))
      return rc;
  } else {
    if ((rc = rubs_b200_filter_params(f, f_dtype, H, W, ld_f, size, rho, theta, RUBS_F64, W, lut,
                                      iterations, out, ld_out, s)))
      return rc;
    if ((rc = rubs_b200_filter_params(ones, f_dtype, H, W, W, size, rho, theta, RUBS_F64, W, lut,
                                      iterations, gain, W, s)))
      return rc;
  }
  gain_correct_kernel<<<grid_for(n), 256, 0, s>>>(out, ld_out, gain, (int)H, (int)W);
  rubs_internal::count_launches(1);
  RT_CUDA_TRY(cudaGetLastError());
  return RUBS_OK;
}

}  // extern "C"
