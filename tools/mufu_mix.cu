// mufu_mix.cu — which companions of ex2.approx slow it down (sm_100a):
// per thread 16 independent chains; variants add FFMA, F2FP (bf16 pack),
// FADD, or an ALU-only bf16 pack (PRMT/IADD) next to each ex2.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
template <int MODE>
__global__ void k(float* out, int iters) {
  float a[16]; unsigned acc = 0;
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      float x0 = a[i], x1 = a[i + 1];
      if (MODE & 1) { x0 = fmaf(x0, 0.17f, -1.f); x1 = fmaf(x1, 0.17f, -1.f); }
      asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0));
      asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
      if (MODE & 2) { __nv_bfloat162 b = __floats2bfloat162_rn(x0, x1); acc ^= *reinterpret_cast<unsigned*>(&b); }
      if (MODE & 4) {  // ALU bf16 pack (round-to-nearest-even by integer ops)
        unsigned u0 = __float_as_uint(x0), u1 = __float_as_uint(x1);
        u0 += 0x7FFFu + ((u0 >> 16) & 1u); u1 += 0x7FFFu + ((u1 >> 16) & 1u);
        acc ^= __byte_perm(u0, u1, 0x7632);
      }
      a[i] = x0 * 0.5f; a[i + 1] = x1 * 0.5f;
    }
  }
  long long t1 = clock64();
  float s = acc; for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) out[gridDim.x * blockDim.x + blockIdx.x] = float(t1 - t0);
}
template <int MODE> void run(const char* name, float* d) {
  float h[148];
  for (int warps : {4, 8}) {
    const int iters = 2000;
    k<MODE><<<148, warps * 32>>>(d, 10); k<MODE><<<148, warps * 32>>>(d, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d + 148 * warps * 32, 148 * 4, cudaMemcpyDeviceToHost);
    double cyc = 0; for (int i = 0; i < 148; ++i) cyc += h[i]; cyc /= 148;
    printf("%-26s warps/SM %d: %.2f exp2/clk/SM\n", name, warps, double(warps) * 32 * iters * 16 / cyc);
  }
}
int main() {
  float* d; cudaMalloc(&d, 148 * 1024 * 4 + 148 * 4);
  run<0>("ex2 + fmul", d);
  run<1>("ex2 + ffma + fmul", d);
  run<2>("ex2 + F2FP pack + fmul", d);
  run<4>("ex2 + ALU pack + fmul", d);
  run<3>("ex2 + ffma + F2FP + fmul", d);
  run<5>("ex2 + ffma + ALU pack + fmul", d);
  return 0;
}
