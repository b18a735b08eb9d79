// umma_multi.cu — can two issuing warps drive one SM's tensor core faster
// than one?  W warps (lane 0 of each) issue n MMAs each into their own
// accumulator; reports aggregate cycles per MMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx_sm100.cuh"
using namespace dmha;

template <int KIND, int N, int W>
__global__ void __launch_bounds__(128, 1) bench(long long* out, int n) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) ptx::mbar_init(&bar[i], 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  const int w = threadIdx.x / 32;
  long long t0 = clock64();
  if (w < W && (threadIdx.x & 31) == 0) {
    const uint32_t a = ptx::smem_u32(smem), b = a + 65536;
    constexpr uint32_t id = ptx::make_idesc(1, 128, N, 0, KIND);
    const uint32_t acc = tmem + w * (KIND ? 64 : 128);
    for (int i = 0; i < n; ++i) {
      if (KIND == 0)
        ptx::mma_bf16_ss(acc, ptx::smem_desc_sw128(a + (i & 3) * 32, 16, 1024),
                         ptx::smem_desc_sw128(b + (i & 3) * 32, 16, 1024), id, 1);
      else
        ptx::mma_bf16_ts(acc, tmem + 256 + (i & 7) * 8,
                         ptx::smem_desc_sw128(b + (i & 7) * 2048, 16384, 1024), id, 1);
    }
    ptx::mma_commit(&bar[w]);
    ptx::mbar_wait(&bar[w], 0);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}

template <int KIND, int N, int W>
void run(long long* d) {
  auto k = bench<KIND, N, W>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  const int n = 512;
  k<<<148, 128, 140 * 1024>>>(d, n);
  k<<<148, 128, 140 * 1024>>>(d, n);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
  printf("%s N=%3d issuers=%d: %.1f cycles per MMA (aggregate) %s\n", KIND ? "TS" : "SS", N, W, s / 148 / (n * W), cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  run<0, 64, 1>(d); run<0, 64, 2>(d); run<0, 128, 1>(d); run<0, 128, 2>(d);
  run<1, 64, 1>(d); run<1, 64, 2>(d); run<1, 64, 4>(d); run<1, 128, 1>(d); run<1, 128, 2>(d);
  return 0;
}
