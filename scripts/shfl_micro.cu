// Dev micro-benchmark: does SHFL consume L1 data-pipe wavefronts (the big
// gather's binding resource)?  ncu --metrics l1tex__data_pipe_lsu_wavefronts.sum,
// smsp__inst_executed.sum,gpu__time_duration.sum ./shfl_micro
#include <cstdio>
#include <cuda_runtime.h>
__global__ void shfl_kernel(double *out, int iters) {
  double v = threadIdx.x * 1.0;
  for (int i = 0; i < iters; ++i) {
    v += __shfl_down_sync(0xffffffffu, v, 1);
    v += __shfl_up_sync(0xffffffffu, v, 1);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = v;
}
__global__ void lds_kernel(double *out, int iters) {
  __shared__ double s[256 + 64];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  double v = 0;
  int k = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    v += s[(k + i) & 255];
    v += s[(k + i + 1) & 255];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = v;
}
int main() {
  double *d;
  cudaMalloc(&d, 148 * 8 * 256 * 8);
  for (int r = 0; r < 2; ++r) {
    shfl_kernel<<<148 * 8, 256>>>(d, 4096);
    lds_kernel<<<148 * 8, 256>>>(d, 4096);
  }
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); shfl_kernel<<<148 * 8, 256>>>(d, 4096); cudaEventRecord(b); cudaEventSynchronize(b);
  float t1; cudaEventElapsedTime(&t1, a, b);
  cudaEventRecord(a); lds_kernel<<<148 * 8, 256>>>(d, 4096); cudaEventRecord(b); cudaEventSynchronize(b);
  float t2; cudaEventElapsedTime(&t2, a, b);
  double n = 148.0 * 8 * 256 / 32 * 4096 * 2;  // warp instructions of each kind
  printf("shfl: %.3f ms, %.2f warp-shfl/clk/SM @1.965GHz; lds.64: %.3f ms, %.2f warp-lds/clk/SM\n", t1,
         n / (t1 * 1e-3) / 148 / 1.965e9, t2, n / (t2 * 1e-3) / 148 / 1.965e9);
  return 0;
}
