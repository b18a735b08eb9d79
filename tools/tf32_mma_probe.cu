// tf32_mma_probe.cu — does one tcgen05.mma kind::tf32 (M=128, N=64, K=8, both
// operands K-major 128B-swizzled in shared memory) complete, and with what
// result?  Bounded mbarrier wait (no hang), bf16 kind::f16 as the control.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I ../paper_2302_06218_b200/csrc tf32_mma_probe.cu -o tf32_mma_probe
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include "ptx_sm100.cuh"

using namespace dmha;

__global__ void probe(int mode, int* status, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = sm;            // 128 rows x 128 B
  uint8_t* sb = sm + 16384;    // 64 rows x 128 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 16384 + 8192);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x;
  // fill: every element of row r of A = 1 (+ r/1024), B = 1  (tf32: fp32 bits; bf16: bf16 bits)
  for (int i = tid; i < 128 * 32; i += 128) {
    const int r = i / 32;
    if (mode == 0) reinterpret_cast<float*>(sa)[i] = 1.0f + r / 1024.0f;
    else reinterpret_cast<__nv_bfloat16*>(sa)[i] = __float2bfloat16(1.0f);
  }
  for (int i = tid; i < 64 * 32; i += 128) {
    if (mode == 0) reinterpret_cast<float*>(sb)[i] = 1.0f;
    else reinterpret_cast<__nv_bfloat16*>(sb)[i] = __float2bfloat16(1.0f);
  }
  if (tid == 0) { ptx::mbar_init(bar, 1); ptx::fence_mbar_init(); }
  if (tid < 32) ptx::tmem_alloc<256>(slot);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  if (tid == 0) {
    const uint64_t da = ptx::smem_desc_sw128(ptx::smem_u32(sa), 16, 1024);
    const uint64_t db = ptx::smem_desc_sw128(ptx::smem_u32(sb), 16, 1024);
    if (mode == 0) ptx::mma_tf32_ss(tmem, da, db, ptx::make_idesc(2, 128, 64, 0, 0), 0);
    else ptx::mma_bf16_ss(tmem, da, db, ptx::make_idesc(1, 128, 64, 0, 0), 0);
    ptx::mma_commit(bar);
  }
  bool ok = false;
  for (long it = 0; it < (1l << 26); ++it)
    if (ptx::mbar_try_wait(bar, 0)) { ok = true; break; }
  if (tid == 0) status[mode] = ok ? 1 : -1;
  __syncwarp();
  ptx::tc_fence_after();
  if (ok) {
    float v[32];
    ptx::tmem_ld32(tmem + ((tid & ~31) << 16), v);
    ptx::tmem_wait_ld();
    out[mode * 128 + tid] = v[0];
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (tid < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc<256>(tmem); }
}

int main() {
  int* st; float* out;
  cudaMalloc(&st, 8); cudaMemset(st, 0, 8);
  cudaMalloc(&out, 256 * 4); cudaMemset(out, 0, 1024);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int mode = 1; mode >= 0; --mode) {
    probe<<<1, 128, 64 * 1024>>>(mode, st, out);
    cudaError_t e = cudaDeviceSynchronize();
    int h[2]; float o[256];
    cudaMemcpy(h, st, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(o, out, 1024, cudaMemcpyDeviceToHost);
    printf("mode %s: err=%s status=%d  D[row0]=%g D[row127]=%g (expect %s)\n", mode ? "bf16" : "tf32",
           cudaGetErrorString(e), h[mode], o[mode * 128], o[mode * 128 + 127],
           mode ? "16 (K=16)" : "8*(1+r/1024) (K=8)");
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
