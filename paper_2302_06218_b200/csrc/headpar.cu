// headpar.cu — pack/unpack kernels of the paper's own exchange (SURVEY §8(f)
// NEXT-1; §10.4): the sequence-sharded Q/K/V are shuffled
// to head-parallel (every rank gets ALL L rows of H/P heads), each rank
// runs full-L attention for its heads, and the output is shuffled
// back to sequence-parallel.  The shuffles ("COSTA" in the paper) are
// all-to-alls; these kernels lay the blocks out so that every peer's block is
// one contiguous message, and scatter received rows to their GLOBAL positions
// (which for the zigzag layout are not contiguous per rank).
//
// All kernels are HBM-bound copies.  The unit of work is one row SEGMENT: the
// Hp = H/P heads of one (peer, tensor, row), Hp*D*elem contiguous bytes on
// both sides (a multiple of 16).  One warp copies a segment with 16-byte
// loads/stores; the (peer, tensor) pair comes from blockIdx.z / blockIdx.y and
// the row from a warp-strided loop, so there is no per-element div/mod.
// Algorithmic bytes: 2x the bytes moved (read + write), see DESIGN.md.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace dmha {
namespace {

constexpr int kWarps = 8;  // warps (= row segments in flight) per block

__device__ __forceinline__ int64_t gpos(const HeadparGeom& g, int rank, int64_t i) {
  if (g.zigzag) {
    const int64_t c = g.Lloc / 2;
    return i < c ? rank * c + i : static_cast<int64_t>(2 * g.P - 1 - rank) * c + (i - c);
  }
  return rank * g.Lloc + i;
}

// Rows [0, Lloc) of one (peer, tensor) plane.  Segments of >= 32 vectors: one
// warp per row.  Shorter power-of-two segments (e.g. 2 heads x 64 bf16 = 16
// vectors): the block copies a flat run of (row, vector) pairs, so every lane
// moves 16 bytes per step instead of half the warp idling.
template <typename DstRow, typename SrcRow>
__device__ __forceinline__ void copy_rows(int64_t Lloc, int seg, int seg_shift, DstRow dst_row,
                                          SrcRow src_row) {
  if (seg >= 32 || seg_shift < 0) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5); i < Lloc;
         i += static_cast<int64_t>(gridDim.x) * kWarps) {
      uint4* d = dst_row(i);
      const uint4* s = src_row(i);
      for (int w = lane; w < seg; w += 32) d[w] = s[w];
    }
    return;
  }
  const int64_t n = Lloc << seg_shift;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e >> seg_shift;
    const int w = static_cast<int>(e & (seg - 1));
    dst_row(i)[w] = src_row(i)[w];
  }
}

// x_t [Lloc, H, D] (t = q, k, v) -> send [P(dest)][3][Lloc][Hp][D];
// blockIdx.z = dest d, blockIdx.y = t
__global__ void pack_qkv_kernel(const uint4* __restrict__ q, const uint4* __restrict__ k,
                                const uint4* __restrict__ v, uint4* __restrict__ send,
                                HeadparGeom g, int vec, int seg_shift) {
  const int Hp = g.H / g.P, seg = Hp * vec;
  const int d = blockIdx.z, t = blockIdx.y;
  const uint4* src = t == 0 ? q : (t == 1 ? k : v);
  uint4* dst = send + (static_cast<int64_t>(d) * 3 + t) * g.Lloc * seg;
  copy_rows(g.Lloc, seg, seg_shift, [&](int64_t i) { return dst + i * seg; },
            [&](int64_t i) { return src + (i * g.H + d * Hp) * vec; });
}

// recv [P(src)][3][Lloc][Hp][D] -> X_t [L, Hp, D] in global row order;
// blockIdx.z = source s, blockIdx.y = t
__global__ void unpack_qkv_kernel(const uint4* __restrict__ recv, uint4* __restrict__ xq,
                                  uint4* __restrict__ xk, uint4* __restrict__ xv, HeadparGeom g,
                                  int vec, int seg_shift) {
  const int Hp = g.H / g.P, seg = Hp * vec;
  const int s = blockIdx.z, t = blockIdx.y;
  uint4* dst = t == 0 ? xq : (t == 1 ? xk : xv);
  const uint4* src = recv + (static_cast<int64_t>(s) * 3 + t) * g.Lloc * seg;
  copy_rows(g.Lloc, seg, seg_shift, [&](int64_t i) { return dst + gpos(g, s, i) * seg; },
            [&](int64_t i) { return src + i * seg; });
}

// out_g [L, Hp, D] (global order) -> send [P(dest)][Lloc][Hp][D] (blockIdx.y = 0);
// lse_g [Hp, L] -> send_lse [P(dest)][Hp][Lloc] (blockIdx.y = 1, thread per row)
__global__ void pack_out_kernel(const uint4* __restrict__ outg, uint4* __restrict__ send,
                                const float* __restrict__ lseg, float* __restrict__ send_lse,
                                HeadparGeom g, int vec, int seg_shift) {
  const int Hp = g.H / g.P, seg = Hp * vec;
  const int d = blockIdx.z;
  if (blockIdx.y == 0) {
    uint4* dst = send + static_cast<int64_t>(d) * g.Lloc * seg;
    copy_rows(g.Lloc, seg, seg_shift, [&](int64_t i) { return dst + i * seg; },
              [&](int64_t i) { return outg + gpos(g, d, i) * seg; });
  } else {
    const int64_t L = g.Lloc * g.P;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < g.Lloc;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int64_t gp = gpos(g, d, i);
      for (int hh = 0; hh < Hp; ++hh)
        send_lse[(static_cast<int64_t>(d) * Hp + hh) * g.Lloc + i] = lseg[hh * L + gp];
    }
  }
}

// recv [P(src)][Lloc][Hp][D] -> out [Lloc, H, D] (head block of src); blockIdx.z = s
__global__ void unpack_out_kernel(const uint4* __restrict__ recv, uint4* __restrict__ out,
                                  HeadparGeom g, int vec, int seg_shift) {
  const int Hp = g.H / g.P, seg = Hp * vec;
  const int s = blockIdx.z;
  const uint4* src = recv + static_cast<int64_t>(s) * g.Lloc * seg;
  copy_rows(g.Lloc, seg, seg_shift, [&](int64_t i) { return out + (i * g.H + s * Hp) * vec; },
            [&](int64_t i) { return src + i * seg; });
}

// log2(segment length in 16-byte vectors) when it is a power of two, else -1.
int seg_shift_of(const HeadparGeom& g, int vec) {
  const int seg = g.H / g.P * vec;
  return (seg & (seg - 1)) == 0 ? __builtin_ctz(static_cast<unsigned>(seg)) : -1;
}

// About 8 resident blocks per SM over the whole (x, y, z) grid.
dim3 grid_for(const HeadparGeom& g, int planes_y) {
  const int64_t planes = static_cast<int64_t>(g.P) * planes_y;
  int64_t bx = (g.Lloc + kWarps - 1) / kWarps;
  const int64_t cap = (148 * 8 + planes - 1) / planes;
  if (bx > cap) bx = cap;
  return dim3(static_cast<unsigned>(bx < 1 ? 1 : bx), planes_y, g.P);
}

}  // namespace

cudaError_t launch_headpar_pack_qkv(const void* q, const void* k, const void* v, void* send,
                                    const HeadparGeom& g, int elem_bytes, cudaStream_t st) {
  const int vec = g.D * elem_bytes / 16;
  pack_qkv_kernel<<<grid_for(g, 3), 32 * kWarps, 0, st>>>(
      static_cast<const uint4*>(q), static_cast<const uint4*>(k), static_cast<const uint4*>(v),
      static_cast<uint4*>(send), g, vec, seg_shift_of(g, vec));
  return cudaGetLastError();
}

cudaError_t launch_headpar_unpack_qkv(const void* recv, void* xq, void* xk, void* xv,
                                      const HeadparGeom& g, int elem_bytes, cudaStream_t st) {
  const int vec = g.D * elem_bytes / 16;
  unpack_qkv_kernel<<<grid_for(g, 3), 32 * kWarps, 0, st>>>(
      static_cast<const uint4*>(recv), static_cast<uint4*>(xq), static_cast<uint4*>(xk),
      static_cast<uint4*>(xv), g, vec, seg_shift_of(g, vec));
  return cudaGetLastError();
}

cudaError_t launch_headpar_pack_out(const void* outg, void* send, const float* lseg,
                                    float* send_lse, const HeadparGeom& g, int elem_bytes,
                                    cudaStream_t st) {
  const int vec = g.D * elem_bytes / 16;
  pack_out_kernel<<<grid_for(g, 2), 32 * kWarps, 0, st>>>(
      static_cast<const uint4*>(outg), static_cast<uint4*>(send), lseg, send_lse, g, vec,
      seg_shift_of(g, vec));
  return cudaGetLastError();
}

cudaError_t launch_headpar_unpack_out(const void* recv, void* out, const HeadparGeom& g,
                                      int elem_bytes, cudaStream_t st) {
  const int vec = g.D * elem_bytes / 16;
  unpack_out_kernel<<<grid_for(g, 1), 32 * kWarps, 0, st>>>(static_cast<const uint4*>(recv),
                                                             static_cast<uint4*>(out), g, vec,
                                                             seg_shift_of(g, vec));
  return cudaGetLastError();
}

}  // namespace dmha
