// ex2_bf16.cu — throughput of ex2.approx.ftz.bf16x2 / ex2.approx.f16x2 vs ex2.approx.ftz.f32 (exps/clk/SM).
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
template <int MODE>
__global__ void k(float* out, int iters) {
  unsigned a[16]; float f[16];
  for (int i = 0; i < 16; ++i) { a[i] = 0x3f003f00u + threadIdx.x + i; f[i] = threadIdx.x * 1e-3f + i; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      else if (MODE == 1) asm("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
      else asm("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += f[i] + a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) out[gridDim.x * blockDim.x + blockIdx.x] = float(t1 - t0);
}
template <int MODE> void run(const char* name, float* d) {
  float h[148];
  for (int warps : {4, 8, 16}) {
    const int iters = 2000;
    k<MODE><<<148, warps * 32>>>(d, 10); k<MODE><<<148, warps * 32>>>(d, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d + 148 * warps * 32, 148 * 4, cudaMemcpyDeviceToHost);
    double cyc = 0; for (int i = 0; i < 148; ++i) cyc += h[i]; cyc /= 148;
    const double per = MODE == 0 ? 1 : 2;
    printf("%-22s warps/SM %2d: %.2f exps/clk/SM\n", name, warps, per * warps * 32 * iters * 16 / cyc);
  }
}
int main() {
  float* d;
  cudaMalloc(&d, 148 * 1024 * 4 + 148 * 4);
  run<0>("ex2.f32", d);
  run<1>("ex2.bf16x2", d);
  run<2>("ex2.f16x2", d);
  return 0;
}
