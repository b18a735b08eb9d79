// umma_mix64.cu — tensor-pipe time of the MMA mix of a kBN = 64 / D = 128
// schedule: per "128 keys" 32 SS 128x64x16 (QK^T, two accumulators) issued by
// one thread and 16 TS 128x128x16 (PV, two accumulators) issued by another,
// versus today's 16 SS 128x128x16 + 16 TS 128x128x16 from one thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx_sm100.cuh"
using namespace dmha;

template <int MODE>  // 0: today's mix, one issuer; 1: kBN=64 mix, S and PV issuers
__global__ void __launch_bounds__(128, 1) bench(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar[0], 1); ptx::mbar_init(&bar[1], 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  const int w = threadIdx.x / 32;
  const uint32_t a = ptx::smem_u32(smem), b = a + 65536;
  constexpr uint32_t id64 = ptx::make_idesc(1, 128, 64, 0, 0);
  constexpr uint32_t id128 = ptx::make_idesc(1, 128, 128, 0, 0);
  constexpr uint32_t idpv = ptx::make_idesc(1, 128, 128, 0, 1);
  long long t0 = clock64();
  if ((threadIdx.x & 31) == 0) {
    if (MODE == 0 && w == 0) {
      for (int it = 0; it < iters; ++it)
        for (int g = 0; g < 2; ++g) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            ptx::mma_bf16_ts(tmem + 256 + g * 128, tmem + g * 128 + kk * 8,
                             ptx::smem_desc_sw128(b + kk * 2048, 16384, 1024), idpv, 1);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            ptx::mma_bf16_ss(tmem + g * 128, ptx::smem_desc_sw128(a + off, 16, 1024),
                             ptx::smem_desc_sw128(b + off, 16, 1024), id128, 1);
          }
        }
      ptx::mma_commit(&bar[0]);
      ptx::mbar_wait(&bar[0], 0);
    }
    if (MODE == 1 && w == 0) {  // S issuer: per 128 keys, 2 tiles x 2 Q tiles x 8 K-steps of N = 64
      for (int it = 0; it < iters; ++it)
        for (int t = 0; t < 4; ++t) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            ptx::mma_bf16_ss(tmem + (t & 1) * 64 + (t >> 1) * 256, ptx::smem_desc_sw128(a + off, 16, 1024),
                             ptx::smem_desc_sw128(b + off, 16, 1024), id64, 1);
          }
        }
      ptx::mma_commit(&bar[0]);
      ptx::mbar_wait(&bar[0], 0);
    }
    if (MODE == 1 && w == 1) {  // PV issuer: per 128 keys, 2 tiles x 2 Q tiles x 4 K-steps
      for (int it = 0; it < iters; ++it)
        for (int t = 0; t < 4; ++t) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            ptx::mma_bf16_ts(tmem + 128 + (t >> 1) * 256, tmem + (t & 1) * 64 + (t >> 1) * 256 + kk * 8,
                             ptx::smem_desc_sw128(b + kk * 2048, 16384, 1024), idpv, 1);
        }
      ptx::mma_commit(&bar[1]);
      ptx::mbar_wait(&bar[1], 0);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}

template <int MODE>
void run(long long* d) {
  auto k = bench<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  const int iters = 256;
  k<<<148, 128, 140 * 1024>>>(d, iters);
  k<<<148, 128, 140 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
  printf("%s: %.0f cycles per 128 keys x 256 rows (%s)\n",
         MODE ? "kBN=64 mix, S + PV issuers" : "today's mix, one issuer", s / 148 / iters,
         cudaGetErrorString(e));
}
int main() { long long* d; cudaMalloc(&d, 148 * 8); run<0>(d); run<1>(d); return 0; }
