// Dev probe: isolate the 2-D TMA box load used by load_region.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>

struct Maps { CUtensorMap m[2]; unsigned valid; };

template <int VARIANT>
__global__ void k(const __grid_constant__ Maps tm, double *out, int P, int RH, int c0, int r0) {
  extern __shared__ __align__(128) double S[];
  __shared__ uint64_t s_mbar;
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&s_mbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
    if (VARIANT != 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nbox = (RH + 7) >> 3;
    const uint32_t bytes = (uint32_t)nbox * 64u * (uint32_t)P;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(S);
    const uint64_t map = reinterpret_cast<uint64_t>(&tm.m[0]);
    for (int b = 0; b < nbox; ++b) {
      if (VARIANT == 2)
        asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3}], [%4];" ::"r"(sb + (uint32_t)b * 64u * (uint32_t)P),
                     "l"(map), "r"(c0), "r"(r0 + 8 * b), "r"(mbar) : "memory");
      else
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3}], [%4];" ::"r"(sb + (uint32_t)b * 64u * (uint32_t)P),
                     "l"(map), "r"(c0), "r"(r0 + 8 * b), "r"(mbar) : "memory");
    }
  }
  asm volatile("{\n .reg .pred p;\nW%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(mbar), "r"(0) : "memory");
  for (int i = threadIdx.x; i < P * ((RH + 7) & ~7); i += blockDim.x) out[i] = S[i];
}

int main(int argc, char **argv) {
  int W = 48, H = 40, P = 20, RH = 12, c0 = -3, r0 = -2;
  int variant = argc > 1 ? atoi(argv[1]) : 0;
  if (argc > 2) P = atoi(argv[2]);
  if (argc > 3) c0 = atoi(argv[3]);
  if (argc > 4) r0 = atoi(argv[4]);
  int cluster = argc > 5 ? atoi(argv[5]) : 0;
  std::vector<double> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = i;
  double *d, *o;
  cudaMalloc(&d, W * H * 8);
  cudaMalloc(&o, 1 << 20);
  cudaMemcpy(d, h.data(), W * H * 8, cudaMemcpyHostToDevice);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  Maps mp{};
  cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
  cuuint64_t strides[1] = {(cuuint64_t)W * 8};
  cuuint32_t box[2] = {(cuuint32_t)P, 8};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode(&mp.m[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d fn %p q %d\n", (int)r, fn, (int)q);
  if (cluster) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 16 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaError_t le = variant == 2 ? cudaLaunchKernelEx(&cfg, k<2>, mp, o, P, RH, c0, r0)
                                  : cudaLaunchKernelEx(&cfg, k<0>, mp, o, P, RH, c0, r0);
    printf("launch %s\n", cudaGetErrorString(le));
  } else if (variant == 0) k<0><<<1, 128, 16 * 1024>>>(mp, o, P, RH, c0, r0);
  else if (variant == 2) k<2><<<1, 128, 16 * 1024>>>(mp, o, P, RH, c0, r0);
  else k<1><<<1, 128, 16 * 1024>>>(mp, o, P, RH, c0, r0);
  printf("launch err %s\n", cudaGetErrorString(cudaGetLastError()));
  cudaError_t e = cudaDeviceSynchronize();
  printf("variant %d P %d c0 %d r0 %d cluster %d: %s\n", variant, P, c0, r0, cluster, cudaGetErrorString(e));
  std::vector<double> ho(P * 16);
  cudaMemcpy(ho.data(), o, P * 16 * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int rr = 0; rr < 16; ++rr)
    for (int cc = 0; cc < P; ++cc) {
      int gr = r0 + rr, gc = c0 + cc;
      double want = (gr >= 0 && gr < H && gc >= 0 && gc < W) ? h[gr * W + gc] : 0.0;
      if (ho[rr * P + cc] != want) ++bad;
    }
  printf("mismatches %d\n", bad);
  for (int rr = 0; rr < 4; ++rr) {
    for (int cc = 0; cc < 8; ++cc) printf("%6.0f ", ho[rr * P + cc]);
    printf("\n");
  }
  return 0;
}
