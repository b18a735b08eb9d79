// tma_lat.cu — TMA load latency/throughput on sm_100a: 148 CTAs (optionally
// clusters of 2 with multicast) stream 16 KB boxes from a 256 MB buffer with
// `depth` loads in flight; report mean issue->complete latency (cycles).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx_sm100.cuh"
using namespace dmha;

template <bool MC>
__global__ void __launch_bounds__(32, 1) lat(const __grid_constant__ CUtensorMap tm, int depth, int n,
                                             unsigned long long* out, int rows_total) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[8];
  const uint32_t cr = MC ? ptx::cluster_ctarank() : 0;
  if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) ptx::mbar_init(&bar[i], 1); ptx::fence_mbar_init(); }
  if (MC) ptx::cluster_sync(); else __syncthreads();
  if (threadIdx.x == 0) {
    long long t_issue[8];
    uint32_t ph[8] = {0};
    unsigned long long sum = 0;
    int row = (blockIdx.x / (MC ? 2 : 1)) * 128;
    for (int i = 0; i < n + depth; ++i) {
      const int s = i % depth;
      if (i >= depth) {
        ptx::mbar_wait(&bar[s], ph[s]); ph[s] ^= 1;
        sum += clock64() - t_issue[s];
      }
      if (i < n) {
        ptx::mbar_arrive_expect_tx(&bar[s], 16384);
        t_issue[s] = clock64();
        if (MC) ptx::tma_load_3d_mc(&tm, &bar[s], smem + s * 16384 + cr * 8192, 0, 0, row + cr * 64, 0x3);
        else ptx::tma_load_3d(&tm, &bar[s], smem + s * 16384, 0, 0, row);
        row = (row + 128 * 148) % rows_total;
      }
    }
    out[blockIdx.x] = sum / n;
  }
  if (MC) ptx::cluster_sync();
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int rows = 1 << 21;  // 256 MB of 128-byte rows
  void* g; cudaMalloc(&g, size_t(rows) * 128); cudaMemset(g, 0, size_t(rows) * 128);
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  CUtensorMap m128, m64;
  cuuint64_t dims[3] = {64, 1, cuuint64_t(rows)}, str[2] = {128, 128};
  cuuint32_t b128[3] = {64, 1, 128}, b64[3] = {64, 1, 64}, es[3] = {1, 1, 1};
  auto enc = reinterpret_cast<EncodeTiledFn>(fp);
  enc(&m128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, g, dims, str, b128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&m64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, g, dims, str, b64, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  unsigned long long h[148];
  for (int mc = 0; mc < 2; ++mc)
    for (int depth : {1, 2, 4, 8}) {
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(148); cfg.blockDim = dim3(32); cfg.dynamicSmemBytes = 140 * 1024;
      cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = mc ? 2 : 1; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
      cfg.attrs = a; cfg.numAttrs = 1;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      const int n = 2000;
      if (mc) { cudaFuncSetAttribute(lat<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
                cudaLaunchKernelEx(&cfg, lat<true>, m64, depth, 50, d, rows);
                cudaEventRecord(e0); cudaLaunchKernelEx(&cfg, lat<true>, m64, depth, n, d, rows); cudaEventRecord(e1); }
      else { cudaFuncSetAttribute(lat<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
             cudaLaunchKernelEx(&cfg, lat<false>, m128, depth, 50, d, rows);
             cudaEventRecord(e0); cudaLaunchKernelEx(&cfg, lat<false>, m128, depth, n, d, rows); cudaEventRecord(e1); }
      cudaError_t err = cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
      const double bytes = 148.0 * n * (mc ? 8192 : 16384);  // bytes fetched from L2/DRAM
      printf("%s depth %d: %s  latency %.0f cycles  fetch %.0f GB/s (L2->SM delivered %.0f GB/s)\n",
             mc ? "multicast pair" : "unicast      ", depth, cudaGetErrorString(err), avg, bytes / ms / 1e6,
             148.0 * n * 16384 / ms / 1e6);
    }
  return 0;
}
