/*
 * TEST INFRASTRUCTURE ONLY -- parity oracle, never part of the product path.
 * Only tests/ may load it, and only as the checker.  (SURVEY.md §8f rank 3:
 * whole-image validation at the BASELINE sizes instead of sampled pixels.)
 *
 * The exact dense filter of dense_oracle.c on the GPU, same arithmetic:
 *   out(n) = sum_m K_{a(n)}(n - m) f(m),  zero outside the image,
 *   K_a(x) = area([x1 +- a1/2] x [x2 +- a3/2]
 *                 intersect {|y1+y2| <= a2/sqrt2, |y1-y2| <= a4/sqrt2}) / (a1 a2 a3 a4)
 * (the reference's oracle.dense_convolve + _exact.kernel_values,
 * pkg/src/rubs/oracle.py:177-241, _exact.py:29-106; the area by
 * Sutherland-Hodgman clipping + shoelace, as in dense_oracle.c, which the
 * golden vectors pin).  One thread per output pixel, one pass (floor 0.05).
 * It shares no code with the product kernels: it evaluates the kernel
 * directly instead of pre-integrating.
 */
#include <cuda_runtime.h>
#include <stdint.h>

#define SQRT2 1.4142135623730951

__device__ double clipped_area(double rx0, double rx1, double ry0, double ry1, double hs,
                               double hd) {
  double px[16], py[16], qx[16], qy[16];
  int n = 4;
  px[0] = rx0; py[0] = ry0;
  px[1] = rx1; py[1] = ry0;
  px[2] = rx1; py[2] = ry1;
  px[3] = rx0; py[3] = ry1;
  const double hpn[4][2] = {{1.0, 1.0}, {-1.0, -1.0}, {1.0, -1.0}, {-1.0, 1.0}};
  const double hpc[4] = {hs, hs, hd, hd};
  for (int h = 0; h < 4 && n > 0; ++h) {
    int m = 0;
    for (int i = 0; i < n; ++i) {
      const int j = (i + 1) % n;
      const double dp = hpn[h][0] * px[i] + hpn[h][1] * py[i] - hpc[h];
      const double dq = hpn[h][0] * px[j] + hpn[h][1] * py[j] - hpc[h];
      if (dp <= 0.0) {
        qx[m] = px[i];
        qy[m] = py[i];
        ++m;
      }
      if ((dp < 0.0 && dq > 0.0) || (dp > 0.0 && dq < 0.0)) {
        const double t = dp / (dp - dq);
        qx[m] = px[i] + t * (px[j] - px[i]);
        qy[m] = py[i] + t * (py[j] - py[i]);
        ++m;
      }
    }
    n = m;
    for (int i = 0; i < n; ++i) {
      px[i] = qx[i];
      py[i] = qy[i];
    }
  }
  if (n < 3) return 0.0;
  double acc = 0.0;
  for (int i = 1; i + 1 < n; ++i) {
    const double ax = px[i] - px[0], ay = py[i] - py[0];
    const double bx = px[i + 1] - px[0], by = py[i + 1] - py[0];
    acc += ax * by - ay * bx;
  }
  return 0.5 * fabs(acc);
}

__device__ double kernel_value(const double a[4], double x1, double x2) {
  const double hs = a[1] / SQRT2, hd = a[3] / SQRT2;
  const double area = clipped_area(x1 - 0.5 * a[0], x1 + 0.5 * a[0], x2 - 0.5 * a[2],
                                   x2 + 0.5 * a[2], hs, hd);
  return area / (a[0] * a[1] * a[2] * a[3]);
}

// outputs for rows [r_lo, r_lo + rows) x cols [c_lo, c_lo + cols) of an
// H x W image (f, field: full arrays; out: rows x cols)
__global__ void dense_kernel(const double *f, int H, int W, const double *field, int uniform,
                             int r_lo, int c_lo, int rows, int cols, double *out) {
  const int64_t n = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int row = r_lo + (int)(i / cols), col = c_lo + (int)(i % cols);
    const double *src = uniform ? field : field + ((int64_t)row * W + col) * 4;
    double a[4];
    for (int k = 0; k < 4; ++k) a[k] = src[k] < 0.05 ? 0.05 : src[k];
    const double diag = (a[1] + a[3]) / SQRT2;
    const int rx = (int)ceil(0.5 * (a[0] + diag)) + 1;
    const int ry = (int)ceil(0.5 * (a[2] + diag)) + 1;
    const int r0 = max(0, row - ry), r1 = min(H - 1, row + ry);
    const int c0 = max(0, col - rx), c1 = min(W - 1, col + rx);
    double acc = 0.0;
    for (int r = r0; r <= r1; ++r)
      for (int c = c0; c <= c1; ++c) {
        const double k = kernel_value(a, (double)(col - c), (double)(row - r));
        if (k != 0.0) acc += k * f[(int64_t)r * W + c];
      }
    out[i] = acc;
  }
}


// One CTA per query point: the exact one-pass output at lattice point
// (row, col) (which may lie outside the image: iterated passes evaluate the
// intermediate on extended canvases), the point's own raw scale-vector
// floored at 0.05 and divided by div = sqrt(iterations).  The image is f32
// or f64 (zero outside).  The taps of the support window are split over the
// CTA's threads and summed by a fixed-order tree: deterministic.  Used for
// the BASELINE-size samples of configs 4 and 5 (tests/test_gpu_fullsize.py),
// where one point's support holds up to ~10^6 taps.
__global__ void __launch_bounds__(256) points_kernel(const void *f, int f32, int H, int W,
                                                     const double *field, double div,
                                                     const int64_t *pts, int n, double *out) {
  __shared__ double red[256];
  for (int p = blockIdx.x; p < n; p += gridDim.x) {
    const int row = (int)pts[2 * p], col = (int)pts[2 * p + 1];
    double a[4];
    for (int k = 0; k < 4; ++k) {
      const double v = field[4 * p + k];
      a[k] = (v < 0.05 ? 0.05 : v) / div;
    }
    const double diag = (a[1] + a[3]) / SQRT2;
    const int rx = (int)ceil(0.5 * (a[0] + diag)) + 1;
    const int ry = (int)ceil(0.5 * (a[2] + diag)) + 1;
    const int r0 = max(0, row - ry), r1 = min(H - 1, row + ry);
    const int c0 = max(0, col - rx), c1 = min(W - 1, col + rx);
    double acc = 0.0;
    if (r1 >= r0 && c1 >= c0) {
      const int nc = c1 - c0 + 1;
      const int64_t nt = (int64_t)(r1 - r0 + 1) * nc;
      for (int64_t t = threadIdx.x; t < nt; t += blockDim.x) {
        const int r = r0 + (int)(t / nc), c = c0 + (int)(t % nc);
        const double k = kernel_value(a, (double)(col - c), (double)(row - r));
        if (k != 0.0) {
          const int64_t i = (int64_t)r * W + c;
          const double v = f32 ? (double)((const float *)f)[i] : ((const double *)f)[i];
          acc += k * v;
        }
      }
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[p] = red[0];
    __syncthreads();
  }
}

extern "C" {

// Device pointers; one pass.  Returns 0 or a cudaError_t.
int rubs_oracle_cuda_dense(const double *f, int H, int W, const double *field, int uniform,
                           int r_lo, int c_lo, int rows, int cols, double *out) {
  const int64_t n = (int64_t)rows * cols;
  if (n <= 0) return 0;
  const int grid = (int)((n + 127) / 128);
  dense_kernel<<<grid, 128>>>(f, H, W, field, uniform, r_lo, c_lo, rows, cols, out);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return (int)e;
}


// Device pointers: f (H x W, f32 if f32 != 0 else f64), field (n x 4 raw
// scale-vectors, one per point), pts (n x 2 int64 row, col), out (n).
// Returns 0 or a cudaError_t.
int rubs_oracle_cuda_points(const void *f, int f32, int H, int W, const double *field,
                            double div, const int64_t *pts, int n, double *out) {
  if (n <= 0) return 0;
  points_kernel<<<n < 65535 ? n : 65535, 256>>>(f, f32, H, W, field, div, pts, n, out);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return (int)e;
}

}  // extern "C"
