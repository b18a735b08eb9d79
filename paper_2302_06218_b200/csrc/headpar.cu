// headpar.cu — pack/unpack kernels of the paper's own exchange (SURVEY §8(f)
// NEXT-1; §10.4): the sequence-sharded Q/K/V are shuffled
// to head-parallel (every rank gets ALL L rows of H/P heads), each rank
// runs full-L attention for its heads, and the output is shuffled
// back to sequence-parallel.  The shuffles ("COSTA" in the paper) are
// all-to-alls; these kernels lay the blocks out so that every peer's block is
// one contiguous message, and scatter received rows to their GLOBAL positions
// (which for the zigzag layout are not contiguous per rank).
//
// All kernels are HBM-bound copies: one thread moves 16 bytes; D * elem bytes
// per (row, head) is a multiple of 16.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace dmha {
namespace {

__device__ __forceinline__ int64_t gpos(const HeadparGeom& g, int rank, int64_t i) {
  if (g.zigzag) {
    const int64_t c = g.Lloc / 2;
    return i < c ? rank * c + i : static_cast<int64_t>(2 * g.P - 1 - rank) * c + (i - c);
  }
  return rank * g.Lloc + i;
}

// x_t [Lloc, H, D] (t = q, k, v) -> send [P(dest)][3][Lloc][Hp][D]
__global__ void pack_qkv_kernel(const uint4* __restrict__ q, const uint4* __restrict__ k,
                                const uint4* __restrict__ v, uint4* __restrict__ send,
                                HeadparGeom g, int vec) {
  const int Hp = g.H / g.P;
  const int64_t n = static_cast<int64_t>(g.P) * 3 * g.Lloc * Hp * vec;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t r = e;
    const int w = static_cast<int>(r % vec); r /= vec;
    const int hh = static_cast<int>(r % Hp); r /= Hp;
    const int64_t i = r % g.Lloc; r /= g.Lloc;
    const int t = static_cast<int>(r % 3); r /= 3;
    const int d = static_cast<int>(r);
    const uint4* src = t == 0 ? q : (t == 1 ? k : v);
    send[e] = src[(i * g.H + d * Hp + hh) * vec + w];
  }
}

// recv [P(src)][3][Lloc][Hp][D] -> X_t [L, Hp, D] in global row order
__global__ void unpack_qkv_kernel(const uint4* __restrict__ recv, uint4* __restrict__ xq,
                                  uint4* __restrict__ xk, uint4* __restrict__ xv, HeadparGeom g,
                                  int vec) {
  const int Hp = g.H / g.P;
  const int64_t n = static_cast<int64_t>(g.P) * 3 * g.Lloc * Hp * vec;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t r = e;
    const int w = static_cast<int>(r % vec); r /= vec;
    const int hh = static_cast<int>(r % Hp); r /= Hp;
    const int64_t i = r % g.Lloc; r /= g.Lloc;
    const int t = static_cast<int>(r % 3); r /= 3;
    const int s = static_cast<int>(r);
    uint4* dst = t == 0 ? xq : (t == 1 ? xk : xv);
    dst[(gpos(g, s, i) * Hp + hh) * vec + w] = recv[e];
  }
}

// out_g [L, Hp, D] (global order) -> send [P(dest)][Lloc][Hp][D]; lse_g [Hp, L] ->
// send_lse [P(dest)][Hp][Lloc]
__global__ void pack_out_kernel(const uint4* __restrict__ outg, uint4* __restrict__ send,
                                const float* __restrict__ lseg, float* __restrict__ send_lse,
                                HeadparGeom g, int vec) {
  const int Hp = g.H / g.P;
  const int64_t n = static_cast<int64_t>(g.P) * g.Lloc * Hp * vec;
  const int64_t nl = static_cast<int64_t>(g.P) * Hp * g.Lloc;
  const int64_t L = g.Lloc * g.P;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n + nl;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (e < n) {
      int64_t r = e;
      const int w = static_cast<int>(r % vec); r /= vec;
      const int hh = static_cast<int>(r % Hp); r /= Hp;
      const int64_t i = r % g.Lloc; r /= g.Lloc;
      const int d = static_cast<int>(r);
      send[e] = outg[(gpos(g, d, i) * Hp + hh) * vec + w];
    } else {
      int64_t r = e - n;
      const int64_t i = r % g.Lloc; r /= g.Lloc;
      const int hh = static_cast<int>(r % Hp); r /= Hp;
      const int d = static_cast<int>(r);
      send_lse[e - n] = lseg[hh * L + gpos(g, d, i)];
    }
  }
}

// recv [P(src)][Lloc][Hp][D] -> out [Lloc, H, D] (head block of src)
__global__ void unpack_out_kernel(const uint4* __restrict__ recv, uint4* __restrict__ out,
                                  HeadparGeom g, int vec) {
  const int Hp = g.H / g.P;
  const int64_t n = static_cast<int64_t>(g.P) * g.Lloc * Hp * vec;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t r = e;
    const int w = static_cast<int>(r % vec); r /= vec;
    const int hh = static_cast<int>(r % Hp); r /= Hp;
    const int64_t i = r % g.Lloc; r /= g.Lloc;
    const int s = static_cast<int>(r);
    out[(i * g.H + s * Hp + hh) * vec + w] = recv[e];
  }
}

unsigned grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = 148 * 8;
  if (b > cap) b = cap;
  return static_cast<unsigned>(b < 1 ? 1 : b);
}

}  // namespace

cudaError_t launch_headpar_pack_qkv(const void* q, const void* k, const void* v, void* send,
                                    const HeadparGeom& g, int elem_bytes, cudaStream_t st) {
  const int vec = g.D * elem_bytes / 16;
  const int64_t n = static_cast<int64_t>(g.P) * 3 * g.Lloc * (g.H / g.P) * vec;
  pack_qkv_kernel<<<grid_for(n), 256, 0, st>>>(static_cast<const uint4*>(q),
                                                static_cast<const uint4*>(k),
                                                static_cast<const uint4*>(v),
                                                static_cast<uint4*>(send), g, vec);
  return cudaGetLastError();
}

cudaError_t launch_headpar_unpack_qkv(const void* recv, void* xq, void* xk, void* xv,
                                      const HeadparGeom& g, int elem_bytes, cudaStream_t st) {
  const int vec = g.D * elem_bytes / 16;
  const int64_t n = static_cast<int64_t>(g.P) * 3 * g.Lloc * (g.H / g.P) * vec;
  unpack_qkv_kernel<<<grid_for(n), 256, 0, st>>>(static_cast<const uint4*>(recv),
                                                  static_cast<uint4*>(xq), static_cast<uint4*>(xk),
                                                  static_cast<uint4*>(xv), g, vec);
  return cudaGetLastError();
}

cudaError_t launch_headpar_pack_out(const void* outg, void* send, const float* lseg,
                                    float* send_lse, const HeadparGeom& g, int elem_bytes,
                                    cudaStream_t st) {
  const int vec = g.D * elem_bytes / 16;
  const int64_t n = static_cast<int64_t>(g.P) * g.Lloc * (g.H / g.P) * (vec + 1);
  pack_out_kernel<<<grid_for(n), 256, 0, st>>>(static_cast<const uint4*>(outg),
                                                static_cast<uint4*>(send), lseg, send_lse, g, vec);
  return cudaGetLastError();
}

cudaError_t launch_headpar_unpack_out(const void* recv, void* out, const HeadparGeom& g,
                                      int elem_bytes, cudaStream_t st) {
  const int vec = g.D * elem_bytes / 16;
  const int64_t n = static_cast<int64_t>(g.P) * g.Lloc * (g.H / g.P) * vec;
  unpack_out_kernel<<<grid_for(n), 256, 0, st>>>(static_cast<const uint4*>(recv),
                                                  static_cast<uint4*>(out), g, vec);
  return cudaGetLastError();
}

}  // namespace dmha
