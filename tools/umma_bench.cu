// umma_bench.cu — microbenchmark of single-CTA tcgen05.mma issue rates on
// sm_100a, to size the attention kernel's MMA pipeline.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../paper_2302_06218_b200/csrc
//        umma_bench.cu -o umma_bench -lcuda
// Each CTA (one per SM) issues `iters` batches of MMAs on smem operands that
// were never loaded (garbage values are fine for timing) and reports cycles
// per 128x128x16 MMA-equivalent.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx_sm100.cuh"

using namespace dmha;

template <int MODE>
__global__ void __launch_bounds__(128, 1) bench(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc<512>(&tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(smem), b = a + 65536;
    // MODE 0: SS  M128 N128 K16, A,B K-major (QK^T)
    // MODE 1: TS  M128 N128 K16, A tmem, B MN-major (PV)
    // MODE 2: SS  M128 N256 K16 (QK^T with 256 keys)
    // MODE 3: alternating 8x MODE0 + 8x MODE1 (the attention pattern)
    constexpr uint32_t id_qk = ptx::make_idesc(1, 128, 128, 0, 0);
    constexpr uint32_t id_pv = ptx::make_idesc(1, 128, 128, 0, 1);
    constexpr uint32_t id_qk256 = ptx::make_idesc(1, 128, 256, 0, 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
        if (MODE == 0 || MODE == 3)
          ptx::mma_bf16_ss(tmem, ptx::smem_desc_sw128(a + off, 16, 1024),
                           ptx::smem_desc_sw128(b + off, 16, 1024), id_qk, kk > 0);
        if (MODE == 1 || MODE == 3)
          ptx::mma_bf16_ts(tmem + 256, tmem + 128 + kk * 8,
                           ptx::smem_desc_sw128(b + kk * 2048, 16384, 1024), id_pv, 1);
        if (MODE == 2)
          ptx::mma_bf16_ss(tmem, ptx::smem_desc_sw128(a + off, 16, 1024),
                           ptx::smem_desc_sw128(b + off, 16, 1024), id_qk256, kk > 0);
      }
    }
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}

template <int MODE>
void run(const char* name, double mma_equiv_per_iter) {
  const int iters = 4096;
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  bench<MODE><<<148, 128, 200 * 1024>>>(d, 16);
  bench<MODE><<<148, 128, 200 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("%-40s %s cycles/iter %.1f  cycles per 128x128x16-equiv %.2f (ideal 64 at 8192 FLOP/clk)\n",
         name, cudaGetErrorString(e), avg / iters, avg / iters / mma_equiv_per_iter);
  cudaFree(d);
}

int main() {
  run<0>("SS M128 N128 K16 (QK^T)", 8);
  run<1>("TS M128 N128 K16 (PV, B MN-major)", 8);
  run<2>("SS M128 N256 K16", 16);
  run<3>("SS+TS alternating", 16);
  return 0;
}
