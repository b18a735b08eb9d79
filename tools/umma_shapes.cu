// umma_shapes.cu — tcgen05.mma cycles per instruction by shape (SS / TS,
// N = 64 / 128 / 256, M = 128, K = 16) and the issue-queue depth: thread 0
// stamps clock64 after each issue, so the stamp where issue starts to track
// completion shows how many MMAs the hardware queue accepts ahead.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../paper_2302_06218_b200/csrc umma_shapes.cu -o umma_shapes
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx_sm100.cuh"
using namespace dmha;

// NACC accumulators used round-robin (independent D regions)
template <int KIND, int N, int NACC, bool ZERO, bool STAMP>  // KIND 0 = SS, 1 = TS (A from TMEM)
__global__ void __launch_bounds__(128, 1) bench(long long* out, int n) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (ZERO) for (int i = threadIdx.x; i < 32768; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(smem), b = a + 65536;
    constexpr uint32_t acc_stride = (KIND == 1) ? 64 : (N > 128 ? 256 : 128) / (NACC > 2 ? 2 : 1);
    constexpr uint32_t id = ptx::make_idesc(1, 128, N, 0, KIND);
    long long st[48];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      if (KIND == 0)
        ptx::mma_bf16_ss(tmem + (i % NACC) * acc_stride, ptx::smem_desc_sw128(a + (i & 3) * 32, 16, 1024),
                         ptx::smem_desc_sw128(b + (i & 3) * 32, 16, 1024), id, 1);
      else
        ptx::mma_bf16_ts(tmem + (i % NACC) * acc_stride, tmem + 256 + (i & 7) * 8,
                         ptx::smem_desc_sw128(b + (i & 7) * 2048, 16384, 1024), id, 1);
      if (STAMP && i < 48) st[i] = clock64();
    }
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x * 64 + 0] = t1 - t0;
    for (int i = 0; STAMP && i < 48 && i < n; ++i) out[blockIdx.x * 64 + 1 + i] = st[i] - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}

template <int KIND, int N, int NACC = 1, bool ZERO = false, bool STAMP = false>
void run(const char* name, long long* d) {
  auto k = bench<KIND, N, NACC, ZERO, STAMP>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  const int n = 512;
  k<<<148, 128, 140 * 1024>>>(d, n);
  k<<<148, 128, 140 * 1024>>>(d, n);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  long long h[64];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-10s %.1f cycles/MMA  issue stamps:", name, double(h[0]) / n);
  for (int i = 0; i < 24; ++i) printf(" %lld", h[1 + i]);
  printf("\n");
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 64 * 8);
  run<0, 64>("SS N=64", d);
  run<0, 128>("SS N=128", d);
  run<0, 256>("SS N=256", d);
  run<1, 64>("TS N=64", d);
  run<1, 128>("TS N=128", d);
  run<1, 256>("TS N=256", d);
  run<0, 64, 2>("SS N=64 x2acc", d);
  run<0, 128, 2>("SS N=128 x2acc", d);
  run<1, 64, 2>("TS N=64 x2acc", d);
  run<1, 64, 4>("TS N=64 x4acc", d);
  run<1, 128, 2>("TS N=128 x2acc", d);
  run<0, 64, 1, true, true>("SS N=64 stamped", d);
  run<0, 128, 1, true>("SS N=128 init", d);
  run<1, 64, 1, true>("TS N=64 init", d);
  run<1, 128, 1, true>("TS N=128 init", d);
  return 0;
}
