// Dev micro-benchmark: L1 data-pipe cost of one warp-wide global load (L1
// hits) as a function of the lanes' address pattern -- the large-halo
// gather (big_gather_kernel) is bound by that pipe at 5.4 wavefronts per
// request on config 5.  Each pattern is timed alone; the printed figure is
// clocks per warp request per SM at 1.965 GHz (= wavefronts per request when
// the pipe binds).   nvcc -arch=sm_100a -O3 -o ldg_micro ldg_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kPitch = 264;  // doubles per row (not a multiple of 16: rows start at different offsets)
constexpr int kRows = 40;

// (results are folded with integer XORs: a DADD per load would make the
// fp64 pipe, 2 warp instructions per clock per SM, the bound)
__device__ __forceinline__ unsigned long long ld8(const double *p) {
  unsigned long long v;
  asm volatile("ld.global.ca.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld16(const double *p) {
  unsigned long long a, b;
  asm volatile("ld.global.ca.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
  return a ^ b;
}

template <int PAT>
__device__ __forceinline__ int offset(int lane) {
  switch (PAT) {
    case 0: return lane;                                 // 32 contiguous doubles, 256 B aligned
    case 1: return lane + 1;                             // contiguous, 8 B off alignment
    case 2: return lane + 7;                             // contiguous, 56 B off
    case 3: return (lane / 16) * kPitch + lane;          // 2 rows (staircase)
    case 4: return (lane / 8) * kPitch + lane;           // 4 rows
    case 5: return (lane / 5) * kPitch + lane;           // 7 rows
    case 6: return (lane / 4) * kPitch + lane;           // 8 rows
    case 7: return (lane / 2) * kPitch + lane;           // 16 rows
    case 8: return lane * kPitch;                        // 32 rows, one element each
    case 9: return (lane / 8) * kPitch + (lane & 7);     // 8 x 4 block (same columns in 4 rows)
    case 10: return (lane / 16) * kPitch + (lane & 15);  // 16 x 2 block
    case 11: return (lane / 4) * kPitch + (lane & 3);    // 4 x 8 block
    case 12: return 2 * lane;                            // v2: 512 B contiguous
    case 13: return lane & ~1;                           // v2: pairs shared by two lanes (256 B span)
    case 14: return (lane / 5) * kPitch + (lane & ~1);   // v2: 7-row staircase, shared pairs
    case 15: return (lane / 8) * kPitch + (lane & ~1);   // v2: 4-row staircase
    case 16: return 0;                                   // broadcast
    case 17: return (lane & 1) * kPitch + (lane / 2);    // 2 rows interleaved lanes
    case 18: return lane * 2;                            // stride 2 (512 B span, 8 B each)
    case 19: return lane * 4;                            // stride 4 (1 KB span): one sector per lane
  }
  return 0;
}

template <int PAT, bool V2>
__global__ void __launch_bounds__(256) k(const double *buf, double *out, int iters) {
  const int lane = threadIdx.x & 31;
  const double *p = buf + 8 + offset<PAT>(lane) + (V2 ? 0 : 0);
  unsigned long long s = 0;
  for (int i = 0; i < iters; ++i) {
    // the address depends on the iteration (a loop-invariant asm is hoisted)
    const double *q = p + (i & 3) * (8 * kPitch);
#pragma unroll
    for (int u = 0; u < 8; ++u) s ^= V2 ? ld16(q + u * kPitch) : ld8(q + u * kPitch);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (double)s;
}

template <int PAT, bool V2>
void run(const char *name, const double *buf, double *out) {
  const int iters = 2048;
  k<PAT, V2><<<148 * 8, 256>>>(buf, out, iters);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<PAT, V2><<<148 * 8, 256>>>(buf, out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double req = 148.0 * 8 * 8 * iters * 8;  // warp requests
  printf("%-52s %6.2f clk / request / SM  (%.3f ms)\n", name, ms * 1e-3 * 1.965e9 * 148 / req, ms);
}

int main() {
  double *buf, *out;
  cudaMalloc(&buf, (kRows + 72) * kPitch * 8 + 4096);
  cudaMemset(buf, 0, (kRows + 72) * kPitch * 8 + 4096);
  cudaMalloc(&out, 148 * 8 * 256 * 8);
  run<0, false>("ld.64  32 contiguous, 256 B aligned", buf, out);
  run<1, false>("ld.64  32 contiguous, +8 B", buf, out);
  run<2, false>("ld.64  32 contiguous, +56 B", buf, out);
  run<3, false>("ld.64  staircase over 2 rows", buf, out);
  run<4, false>("ld.64  staircase over 4 rows", buf, out);
  run<5, false>("ld.64  staircase over 7 rows", buf, out);
  run<6, false>("ld.64  staircase over 8 rows", buf, out);
  run<7, false>("ld.64  staircase over 16 rows", buf, out);
  run<8, false>("ld.64  32 rows, one element each", buf, out);
  run<9, false>("ld.64  block 8 wide x 4 rows", buf, out);
  run<10, false>("ld.64  block 16 wide x 2 rows", buf, out);
  run<11, false>("ld.64  block 4 wide x 8 rows", buf, out);
  run<17, false>("ld.64  2 rows, lanes interleaved", buf, out);
  run<18, false>("ld.64  stride 2 (512 B span)", buf, out);
  run<19, false>("ld.64  stride 4 (1 KB span)", buf, out);
  run<16, false>("ld.64  broadcast", buf, out);
  run<12, true>("ld.128 512 B contiguous", buf, out);
  run<13, true>("ld.128 pairs shared by 2 lanes (256 B span)", buf, out);
  run<14, true>("ld.128 shared pairs, staircase over 7 rows", buf, out);
  run<15, true>("ld.128 shared pairs, staircase over 4 rows", buf, out);
  return 0;
}
