// selector.cu — the token Selector s_{psi,tau}: X_{L x D} -> X'_{L' x D}
// (§10.2, Eq. `selector` P:630-634), run on
// this rank's rows before attention, plus the re-aggregation scatter
// (P:622).  Readings R18-R21: untrained scorer ||x_t||_2 or
// |x_t . psi|, keep iff score >= tau in original order, never empty.
//
// Three HBM-bound passes over 256-row tiles:
//   1. score   — one warp per row, 16-byte loads, fp64 accumulation of the
//                exact bf16 products (the keep/drop decision is taken in fp64
//                like the oracle's, R20); writes the fp64 score, a keep flag
//                and the tile's kept count;
//   2. scan    — one block: exclusive scan of the tile counts -> tile offsets
//                and the total;
//   3. compact — per tile: block-wide exclusive scan of the flags gives each
//                kept row its output slot (order preserving); warps copy the
//                kept rows (16-byte vectors) and write their row indices.
// Traffic per call: read n*w*2 (twice: score + copy of kept rows only) +
// write kept*w*2 + 8 n (scores) + 8 kept (indices).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "kernels.h"

namespace dmha {
namespace {

constexpr int kTile = 256;     // rows per block (8 warps x 32 rows)
constexpr int kThreads = 256;

__device__ __forceinline__ void bf16x8_to_f32(const uint4 u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

template <int kScorer>
__global__ void __launch_bounds__(kThreads) sel_score_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ psi, int64_t n, int w,
    double tau, double* __restrict__ scores, uint8_t* __restrict__ flags,
    int* __restrict__ tile_counts) {
  __shared__ int s_count;
  if (threadIdx.x == 0) s_count = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tile0 = static_cast<int64_t>(blockIdx.x) * kTile;
  int kept = 0;
  for (int i = 0; i < kTile / 8; ++i) {
    const int64_t row = tile0 + warp * (kTile / 8) + i;
    if (row >= n) break;
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * w);
    double acc = 0.0;
    for (int c = lane; c < w / 8; c += 32) {
      float f[8];
      bf16x8_to_f32(__ldg(xr + c), f);
      if (kScorer == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          acc = __fma_rn(static_cast<double>(f[e]), static_cast<double>(f[e]), acc);
      } else {
        float p[8];
        bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(psi) + c), p);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          acc = __fma_rn(static_cast<double>(f[e]), static_cast<double>(p[e]), acc);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const double sc = kScorer == 0 ? sqrt(acc) : fabs(acc);
    const bool keep = sc >= tau;
    if (lane == 0) {
      scores[row] = sc;
      flags[row] = keep ? 1 : 0;
    }
    kept += keep ? 1 : 0;
  }
  if (lane == 0 && kept) atomicAdd(&s_count, kept);
  __syncthreads();
  if (threadIdx.x == 0) tile_counts[blockIdx.x] = s_count;
}

// One block of 1024 threads: offsets[b] = sum_{b' < b} counts[b'], *total.
__global__ void __launch_bounds__(1024) sel_scan_kernel(const int* __restrict__ counts, int nb,
                                                        int64_t* __restrict__ offsets,
                                                        int64_t* __restrict__ total) {
  __shared__ int64_t s_warp[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int per = (nb + 1023) / 1024;
  const int b0 = t * per, b1 = min(nb, b0 + per);
  int64_t local = 0;
  for (int b = b0; b < b1; ++b) local += counts[b];
  int64_t incl = local;  // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t v = s_warp[lane], vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, vi, o);
      if (lane >= o) vi += y;
    }
    s_warp[lane] = vi - v;  // exclusive prefix of warp sums
    if (lane == 31) *total = vi;
  }
  __syncthreads();
  int64_t run = s_warp[warp] + incl - local;
  for (int b = b0; b < b1; ++b) {
    offsets[b] = run;
    run += counts[b];
  }
}

__global__ void __launch_bounds__(kThreads) sel_compact_kernel(
    const __nv_bfloat16* __restrict__ x, int64_t n, int w, const uint8_t* __restrict__ flags,
    const int64_t* __restrict__ offsets, __nv_bfloat16* __restrict__ x_out,
    int64_t* __restrict__ idx_out) {
  __shared__ int s_warp[kThreads / 32];
  __shared__ int64_t s_rows[kTile];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * kTile + t;
  const bool keep = row < n && flags[row];
  const unsigned bal = __ballot_sync(0xffffffffu, keep);
  if (lane == 0) s_warp[warp] = __popc(bal);
  __syncthreads();
  int before = 0, k = 0;
#pragma unroll
  for (int i = 0; i < kThreads / 32; ++i) {
    before += i < warp ? s_warp[i] : 0;
    k += s_warp[i];
  }
  const int slot = before + __popc(bal & ((1u << lane) - 1u));
  const int64_t base = offsets[blockIdx.x];
  if (keep) {
    s_rows[slot] = row;
    idx_out[base + slot] = row;
  }
  __syncthreads();
  for (int i = warp; i < k; i += kThreads / 32) {
    const uint4* src = reinterpret_cast<const uint4*>(x + s_rows[i] * w);
    uint4* dst = reinterpret_cast<uint4*>(x_out + (base + i) * w);
    for (int c = lane; c < w / 8; c += 32) dst[c] = __ldg(src + c);
  }
}

// Single block: the first row with the largest score (never-empty rule, R19).
__global__ void __launch_bounds__(1024) sel_argmax_kernel(const double* __restrict__ scores,
                                                          int64_t n, double* __restrict__ best,
                                                          int64_t* __restrict__ best_row) {
  __shared__ double s_v[32];
  __shared__ int64_t s_i[32];
  double v = -INFINITY;
  int64_t idx = INT64_MAX;
  for (int64_t r = threadIdx.x; r < n; r += blockDim.x) {
    const double s = scores[r];
    if (s > v || (s == v && r < idx)) { v = s; idx = r; }
  }
  auto better = [](double a, int64_t ia, double b, int64_t ib) { return a > b || (a == b && ia < ib); };
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (better(ov, oi, v, idx)) { v = ov; idx = oi; }
  }
  if ((threadIdx.x & 31) == 0) { s_v[threadIdx.x >> 5] = v; s_i[threadIdx.x >> 5] = idx; }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x / 32;
    v = threadIdx.x < nw ? s_v[threadIdx.x] : -INFINITY;
    idx = threadIdx.x < nw ? s_i[threadIdx.x] : INT64_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (better(ov, oi, v, idx)) { v = ov; idx = oi; }
    }
    if (threadIdx.x == 0) { *best = v; *best_row = idx; }
  }
}

__global__ void __launch_bounds__(kThreads) sel_scatter_kernel(
    const __nv_bfloat16* __restrict__ y_sel, const int64_t* __restrict__ idx, int64_t k, int w,
    __nv_bfloat16* __restrict__ y_full) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + (threadIdx.x >> 5); i < k;
       i += warps) {
    const uint4* src = reinterpret_cast<const uint4*>(y_sel + i * w);
    uint4* dst = reinterpret_cast<uint4*>(y_full + idx[i] * w);
    for (int c = lane; c < w / 8; c += 32) dst[c] = __ldg(src + c);
  }
}

}  // namespace

int64_t selector_tiles(int64_t n) { return (n + kTile - 1) / kTile; }

cudaError_t launch_selector_score(const void* x, const void* psi, int64_t n, int w, int scorer,
                                  double tau, double* scores, uint8_t* flags, int* tile_counts,
                                  cudaStream_t st) {
  const int64_t nb = selector_tiles(n);
  if (nb <= 0) return cudaSuccess;
  const auto* xb = static_cast<const __nv_bfloat16*>(x);
  const auto* pb = static_cast<const __nv_bfloat16*>(psi);
  if (scorer == 0)
    sel_score_kernel<0><<<static_cast<unsigned>(nb), kThreads, 0, st>>>(xb, pb, n, w, tau, scores,
                                                                       flags, tile_counts);
  else
    sel_score_kernel<1><<<static_cast<unsigned>(nb), kThreads, 0, st>>>(xb, pb, n, w, tau, scores,
                                                                       flags, tile_counts);
  return cudaGetLastError();
}

cudaError_t launch_selector_scan(const int* tile_counts, int64_t n, int64_t* offsets,
                                 int64_t* total, cudaStream_t st) {
  const int64_t nb = selector_tiles(n);
  sel_scan_kernel<<<1, 1024, 0, st>>>(tile_counts, static_cast<int>(nb), offsets, total);
  return cudaGetLastError();
}

cudaError_t launch_selector_compact(const void* x, int64_t n, int w, const uint8_t* flags,
                                    const int64_t* offsets, void* x_out, int64_t* idx_out,
                                    cudaStream_t st) {
  const int64_t nb = selector_tiles(n);
  if (nb <= 0) return cudaSuccess;
  sel_compact_kernel<<<static_cast<unsigned>(nb), kThreads, 0, st>>>(
      static_cast<const __nv_bfloat16*>(x), n, w, flags, offsets,
      static_cast<__nv_bfloat16*>(x_out), idx_out);
  return cudaGetLastError();
}

cudaError_t launch_selector_argmax(const double* scores, int64_t n, double* best,
                                   int64_t* best_row, cudaStream_t st) {
  sel_argmax_kernel<<<1, 1024, 0, st>>>(scores, n, best, best_row);
  return cudaGetLastError();
}

cudaError_t launch_scatter_rows(const void* y_sel, const int64_t* idx, int64_t k, int w,
                                void* y_full, cudaStream_t st) {
  if (k <= 0) return cudaSuccess;
  int64_t blocks = (k + kThreads / 32 - 1) / (kThreads / 32);
  if (blocks > 148 * 8) blocks = 148 * 8;
  sel_scatter_kernel<<<static_cast<unsigned>(blocks), kThreads, 0, st>>>(
      static_cast<const __nv_bfloat16*>(y_sel), idx, k, w, static_cast<__nv_bfloat16*>(y_full));
  return cudaGetLastError();
}

}  // namespace dmha
