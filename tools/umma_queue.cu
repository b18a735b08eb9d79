// umma_queue.cu — how many tcgen05.mma a single thread can issue before the
// issue itself blocks: t_issue(K) = cycles to issue K back-to-back 128x128x16
// SS MMAs (one clock read after the last issue), t_done(K) = until the commit
// arrives.  Slope 0 then ~64 cycles/MMA once the hardware queue is full.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx_sm100.cuh"
using namespace dmha;

template <int K, int KIND>
__global__ void __launch_bounds__(128, 1) q(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(smem), b = a + 65536;
    constexpr uint32_t id = ptx::make_idesc(1, 128, 128, 0, KIND);
    long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (KIND == 0)
        ptx::mma_bf16_ss(tmem, ptx::smem_desc_sw128(a + (i & 3) * 32, 16, 1024),
                         ptx::smem_desc_sw128(b + (i & 3) * 32, 16, 1024), id, 1);
      else
        ptx::mma_bf16_ts(tmem, tmem + 256 + (i & 7) * 8,
                         ptx::smem_desc_sw128(b + (i & 7) * 2048, 16384, 1024), id, 1);
    }
    long long t1 = clock64();
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[2 * blockIdx.x] = t1 - t0;
    out[2 * blockIdx.x + 1] = t2 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}

template <int K, int KIND>
void run(long long* d) {
  auto k = q<K, KIND>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  k<<<148, 128, 140 * 1024>>>(d);
  k<<<148, 128, 140 * 1024>>>(d);
  cudaDeviceSynchronize();
  long long h[2 * 148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double a = 0, b = 0;
  for (int i = 0; i < 148; ++i) { a += h[2 * i]; b += h[2 * i + 1]; }
  printf("%s K=%2d  issue %6.0f cycles  done %6.0f cycles\n", KIND ? "TS" : "SS", K, a / 148, b / 148);
}

int main() {
  long long* d;
  cudaMalloc(&d, 2 * 148 * 8);
  run<1, 0>(d); run<2, 0>(d); run<4, 0>(d); run<8, 0>(d); run<12, 0>(d); run<16, 0>(d); run<24, 0>(d); run<32, 0>(d);
  run<1, 1>(d); run<4, 1>(d); run<8, 1>(d); run<16, 1>(d); run<32, 1>(d);
  return 0;
}
