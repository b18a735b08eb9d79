// mufu_rate.cu — measured ex2.approx throughput per SM on sm_100a, and the
// same with the FFMA + F2FP (bf16 pack) companions of the softmax loop.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
__global__ void k_ex2(float* out, int iters) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) out[gridDim.x * blockDim.x + blockIdx.x] = float(t1 - t0);
}
__global__ void k_softmaxlike(float* out, int iters) {
  float a[16]; unsigned pk[8];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      float x0 = fmaf(a[i], 0.17f, -1.f), x1 = fmaf(a[i + 1], 0.17f, -1.f);
      asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0));
      asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
      __nv_bfloat162 b = __floats2bfloat162_rn(x0, x1);
      pk[i / 2] ^= *reinterpret_cast<unsigned*>(&b);
      a[i] += x0; a[i + 1] += x1;
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  for (int i = 0; i < 8; ++i) s += pk[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) out[gridDim.x * blockDim.x + blockIdx.x] = float(t1 - t0);
}
int main() {
  float* d; cudaMalloc(&d, 148 * 1024 * 4 + 148 * 4);
  float h[148];
  for (int kind = 0; kind < 2; ++kind)
    for (int warps : {4, 8, 16, 32}) {
      const int iters = 2000;
      if (kind == 0) { k_ex2<<<148, warps * 32>>>(d, 10); k_ex2<<<148, warps * 32>>>(d, iters); }
      else { k_softmaxlike<<<148, warps * 32>>>(d, 10); k_softmaxlike<<<148, warps * 32>>>(d, iters); }
      cudaDeviceSynchronize();
      cudaMemcpy(h, d + 148 * warps * 32, 148 * 4, cudaMemcpyDeviceToHost);
      double cyc = 0; for (int i = 0; i < 148; ++i) cyc += h[i]; cyc /= 148;
      const double ex = double(warps) * 32 * iters * 16;
      printf("%s warps/SM %2d: %.2f exp2/clk/SM\n", kind ? "softmax-like" : "ex2 only    ", warps, ex / cyc);
    }
  return 0;
}
