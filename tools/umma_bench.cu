// umma_bench.cu — microbenchmark of single-CTA tcgen05.mma issue rates on
// sm_100a under the kinds of concurrent traffic the attention kernel creates.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../paper_2302_06218_b200/csrc
//        umma_bench.cu -o umma_bench
// Thread 0 issues `iters` x (8 QK-shaped SS MMAs + 8 PV-shaped TS MMAs) on
// smem operands that hold garbage (values do not matter for timing).
// Optional background load from warps 1..4 (one per TMEM lane quarter):
//   BG_TMEM: tcgen05.ld/st loops on TMEM columns the MMAs do not touch
//   BG_SMEM: st.shared streams into a separate smem region (like TMA writes)
//   BG_MUFU: ex2.approx loops (softmax-like ALU/XU pressure, no memory)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx_sm100.cuh"

using namespace dmha;

enum { BG_NONE = 0, BG_TMEM = 1, BG_SMEM = 2, BG_MUFU = 3, BG_TMA = 4 };

__device__ volatile int g_sink;

template <int BG, bool CLUSTER>
__global__ void __launch_bounds__(160, 1) bench(unsigned long long* out, int iters,
                                                const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  __shared__ uint64_t tbar[4];
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) ptx::mbar_init(&tbar[i], 1);
    ptx::fence_mbar_init();
    stop = 0;
  }
  if (warp == 0) ptx::tmem_alloc<512>(&tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(smem), b = a + 32768;
    constexpr uint32_t id_qk = ptx::make_idesc(1, 128, 128, 0, 0);
    constexpr uint32_t id_pv = ptx::make_idesc(1, 128, 128, 0, 1);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
        ptx::mma_bf16_ss(tmem + (it & 1) * 128, ptx::smem_desc_sw128(a + off, 16, 1024),
                         ptx::smem_desc_sw128(b + off, 16, 1024), id_qk, kk > 0);
      }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        ptx::mma_bf16_ts(tmem + 256, tmem + ((it + 1) & 1) * 128 + kk * 8,
                         ptx::smem_desc_sw128(b + kk * 2048, 16384, 1024), id_pv, 1);
    }
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
    stop = 1;
  } else if (BG == BG_TMA && warp == 1) {
    // stream 16 KB boxes from global into 4 slots at smem + 96 KB, depth 4
    if ((threadIdx.x & 31) == 0) {
      uint32_t ph[4] = {0, 0, 0, 0};
      int row = blockIdx.x * 128;
      for (int n = 0; !stop; ++n) {
        const int sl = n & 3;
        if (n >= 4) { ptx::mbar_wait(&tbar[sl], ph[sl]); ph[sl] ^= 1; }
        ptx::mbar_arrive_expect_tx(&tbar[sl], 16384);
        ptx::tma_load_3d(&tm, &tbar[sl], smem + 98304 + sl * 16384, 0, 0, row);
        row = (row + 128 * 148) & ((1 << 19) - 1);
      }
      for (int sl = 0; sl < 4; ++sl) ptx::mbar_wait(&tbar[sl], ph[sl]);
    }
  } else if (warp >= 1 && warp <= 4) {
    const uint32_t lane_addr = static_cast<uint32_t>(((warp - 1) & 3) * 32) << 16;
    float acc = 0.f;
    while (!stop) {
      if (BG == BG_TMEM) {
        float v[32];
        ptx::tmem_ld32(tmem + lane_addr + 384, v);
        ptx::tmem_wait_ld();
        ptx::tmem_st32(tmem + lane_addr + 448, v);
        ptx::tmem_wait_st();
        acc += v[3];
      } else if (BG == BG_SMEM) {
        uint4* dst = reinterpret_cast<uint4*>(smem + 98304);
#pragma unroll 4
        for (int i = 0; i < 64; ++i) dst[(i * 128 + threadIdx.x - 32) & 4095] = make_uint4(i, i, i, i);
      } else if (BG == BG_MUFU) {
#pragma unroll
        for (int i = 0; i < 32; ++i) acc = ptx::ex2_approx(acc * 0.5f - 1.f);
      } else {
        break;
      }
    }
    if (acc == 12345.f) g_sink = 1;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}

CUtensorMap g_map;

template <int BG, bool CLUSTER>
void run(const char* name) {
  const int iters = 2048;
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  auto k = bench<BG, CLUSTER>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(160);
  cfg.dynamicSmemBytes = 200 * 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CLUSTER ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, d, 16, g_map);
  cudaLaunchKernelEx(&cfg, k, d, iters, g_map);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("%-34s %s  cycles per (QK+PV) pair %.0f  (ideal 1024)\n", name, cudaGetErrorString(e),
         avg / iters);
  cudaFree(d);
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  {  // 2^19 rows x 64 bf16 (64 MB) global buffer viewed as (64, 1, rows)
    void* g = nullptr;
    cudaMalloc(&g, (size_t(1) << 19) * 128);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    cuuint64_t dims[3] = {64, 1, cuuint64_t(1) << 19};
    cuuint64_t strides[2] = {128, 128};
    cuuint32_t box[3] = {64, 1, 128}, es[3] = {1, 1, 1};
    reinterpret_cast<EncodeTiledFn>(fp)(&g_map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, g, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  run<BG_NONE, false>("no background");
  run<BG_NONE, true>("no background, cluster 2");
  run<BG_TMEM, false>("TMEM ld/st background");
  run<BG_SMEM, false>("smem store background");
  run<BG_MUFU, false>("MUFU background");
  run<BG_TMEM, true>("TMEM ld/st background, cluster 2");
  run<BG_TMA, false>("TMA stream background");
  return 0;
}
