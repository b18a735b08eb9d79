// tf32_kernel_probe.cu — the 3xTF32 attention kernel (attn_fwd_tf32.cu) with a
// bounded mbarrier wait: a CTA that waits > ~2^26 polls records (block, tag)
// in mapped host memory and traps, so a stall is located instead of hanging.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../include tf32_kernel_probe.cu -o tf32_kernel_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ int* g_dbg;
#define TF32_WAIT_UNUSED(bar, phase, tag) \
  do {                                                                                     \
    long _n = 0;                                                                           \
    while (!ptx::mbar_try_wait(bar, phase)) {                                              \
      if (++_n > (1l << 26)) {                                                             \
        if (threadIdx.x == 0) { g_dbg[0] = 1; g_dbg[1] = blockIdx.x; g_dbg[2] = blockIdx.y; g_dbg[3] = (tag); __threadfence_system(); } \
        asm volatile("trap;");                                                             \
      }                                                                                    \
    }                                                                                      \
  } while (0)
#include "../paper_2302_06218_b200/csrc/ptx_sm100.cuh"
#include "../paper_2302_06218_b200/csrc/attn_fwd_tf32.cu"

int main(int argc, char** argv) {
  const int L = argc > 1 ? atoi(argv[1]) : 128, H = 1, D = argc > 2 ? atoi(argv[2]) : 64;
  int* hdbg; int* ddbg;
  cudaHostAlloc(&hdbg, 64, cudaHostAllocMapped);
  for (int i = 0; i < 16; ++i) hdbg[i] = 0;
  cudaHostGetDevicePointer(&ddbg, hdbg, 0);
  cudaMemcpyToSymbol(g_dbg, &ddbg, sizeof(ddbg));
  float *q, *k, *v, *o, *lse;
  size_t n = (size_t)L * H * D;
  cudaMalloc(&q, n * 4); cudaMalloc(&k, n * 4); cudaMalloc(&v, n * 4); cudaMalloc(&o, n * 4);
  cudaMalloc(&lse, (size_t)H * L * 4);
  cudaMemset(q, 0, n * 4); cudaMemset(k, 0, n * 4); cudaMemset(v, 0, n * 4);
  dmha::LocalAttnArgs a;
  a.q = q; a.k = k; a.v = v; a.out = o; a.lse = lse; a.Lq = L; a.Lk = L; a.D = D; a.H = H;
  a.causal = 0; a.qmap = {0, L, L}; a.kmap = {0, L, L}; a.out_mode = dmha::OUT_FINAL;
  cudaError_t e = dmha::launch_attn_fwd_tf32x3(a, 0);
  printf("launch: %s\n", cudaGetErrorString(e));
  e = cudaDeviceSynchronize();
  printf("sync: %s  dbg: stalled=%d block=(%d,%d) tag=%d\n", cudaGetErrorString(e), hdbg[0], hdbg[1], hdbg[2], hdbg[3]);
  float ho[8];
  if (e == cudaSuccess) { cudaMemcpy(ho, o, 32, cudaMemcpyDeviceToHost); printf("out[0..3] %g %g %g %g\n", ho[0], ho[1], ho[2], ho[3]); }
  return e == cudaSuccess ? 0 : 1;
}
