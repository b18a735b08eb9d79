// tf32_abi_probe.cpp — the fp32 path through the C ABI (libdmha.so) without
// Python: dmha_init(fp32) + dmha_forward on random data, with a host
// watchdog that reports a hang (exit 3) instead of blocking.
//   g++ -O2 tf32_abi_probe.cpp -I../include -I/usr/local/cuda/include -L../paper_2302_06218_b200 -ldmha
//       -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$ORIGIN/../paper_2302_06218_b200 -o tf32_abi_probe
#include <cuda_runtime.h>
#include <unistd.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include "dmha.h"

int main(int argc, char** argv) {
  const int L = argc > 1 ? atoi(argv[1]) : 128, H = 1, D = argc > 2 ? atoi(argv[2]) : 64;
  std::atomic<bool> done{false};
  std::thread wd([&] {
    for (int i = 0; i < 200 && !done; ++i) usleep(100000);
    if (!done) { printf("HANG (L=%d D=%d)\n", L, D); fflush(stdout); _exit(3); }
  });
  if (dmha_init(1, 0, nullptr, 0, DMHA_FP32, DMHA_LAYOUT_CONTIGUOUS, nullptr)) { printf("init: %s\n", dmha_last_error()); return 1; }
  size_t n = (size_t)L * H * D;
  std::vector<float> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = (float)((i * 2654435761u) % 1000) / 1000.f - 0.5f;
  float *q, *k, *v, *o, *lse;
  cudaMalloc(&q, n * 4); cudaMalloc(&k, n * 4); cudaMalloc(&v, n * 4); cudaMalloc(&o, n * 4); cudaMalloc(&lse, (size_t)H * L * 4);
  cudaMemcpy(q, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(k, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(v, h.data(), n * 4, cudaMemcpyHostToDevice);
  int rc = dmha_forward(q, k, v, o, lse, L, D, H, 0);
  printf("forward rc=%d %s\n", rc, rc ? dmha_last_error() : "");
  cudaError_t e = cudaDeviceSynchronize();
  done = true;
  float ho[4];
  cudaMemcpy(ho, o, 16, cudaMemcpyDeviceToHost);
  printf("sync: %s out[0..3] %g %g %g %g\n", cudaGetErrorString(e), ho[0], ho[1], ho[2], ho[3]);
  wd.join();
  dmha_finalize();
  return 0;
}
