// lse_combine.cu — log-sum-exp merge of a ring-step partial into the running
// accumulator (north_star (3)).
//
// Row softmax needs every key of a row; the ring delivers the
// keys in P blocks, so each step yields a partial (O_s = softmax over the
// block's keys . V, lse_s) and the exact full-row result is
//   lse = M + ln(e^{lse_acc - M} + e^{lse_s - M}),   M = max(lse_acc, lse_s)
//   O   = O_acc e^{lse_acc - lse} + O_s e^{lse_s - lse}
// A -inf lse (no usable key) weighs 0; two -inf stay -inf with O = 0.
//
// HBM-bound: per element it reads O_acc and O_s (fp32) and writes O_acc
// (fp32) or the final output (bf16/fp32): 12 B/elem (10 B on the bf16 final
// step) + 12 B per (row, head) of lse.  One thread per 4 consecutive
// elements (16-byte vector accesses, coalesced along D); grid sized to a
// multiple of the 148 SMs and grid-strided.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "combine_math.cuh"
#include "kernels.h"

namespace dmha {
namespace {

// Every iteration is warp-uniform (the index space is rounded up to whole
// warps) so the __syncwarp between the lse_acc reads of a row's lanes and the
// lead lane's in-place write is executed by the full warp.  A row's D/4 lanes
// (16 or 32) always sit in one warp: blocks start at multiples of 256 lanes.
template <int D, bool kFinal, bool kBf16>
__global__ void __launch_bounds__(256) lse_combine_kernel(float* __restrict__ o_acc,
                                                          float* __restrict__ lse_acc,
                                                          const float* __restrict__ o_part,
                                                          const float* __restrict__ lse_part,
                                                          void* __restrict__ out,
                                                          float* __restrict__ lse_out,
                                                          int64_t Lq, int H, float lse_bias) {
  constexpr int kVecPerRow = D / 4;
  const int64_t n_vec = Lq * H * kVecPerRow;
  const int64_t n_pad = (n_vec + 31) & ~static_cast<int64_t>(31);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_pad;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const bool ok = i < n_vec;
    const int64_t rh = i / kVecPerRow;  // (row, head) pair in [L, H] order
    const int64_t row = rh / H;
    const int head = static_cast<int>(rh - row * H);
    const int64_t li = static_cast<int64_t>(head) * Lq + row;
    float wa = 0.f, wp = 0.f, lnew = 0.f;
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ok) {
      merge_weights(lse_acc[li], lse_part[li] + lse_bias, wa, wp, lnew);
      const float4 a = reinterpret_cast<const float4*>(o_acc)[i];
      const float4 b = reinterpret_cast<const float4*>(o_part)[i];
      r.x = combine_one(a.x, b.x, wa, wp);
      r.y = combine_one(a.y, b.y, wa, wp);
      r.z = combine_one(a.z, b.z, wa, wp);
      r.w = combine_one(a.w, b.w, wa, wp);
    }
    __syncwarp();  // every lane of the row has read lse_acc[li] before it is rewritten
    if (!ok) continue;
    const bool lead = (i - rh * kVecPerRow) == 0;
    if (kFinal) {
      if (kBf16) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(r.x, r.y);
        __nv_bfloat162 hi = __floats2bfloat162_rn(r.z, r.w);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&lo);
        w.y = *reinterpret_cast<uint32_t*>(&hi);
        reinterpret_cast<uint2*>(out)[i] = w;
      } else {
        reinterpret_cast<float4*>(out)[i] = r;
      }
      if (lead) lse_out[li] = lnew;
    } else {
      reinterpret_cast<float4*>(o_acc)[i] = r;
      if (lead) lse_acc[li] = lnew;
    }
  }
}

template <int D>
cudaError_t launch_d(float* o_acc, float* lse_acc, const float* o_part, const float* lse_part,
                     void* out, float* lse_out, int64_t Lq, int H, int final_step, int bf16,
                     cudaStream_t stream, float bias) {
  const int64_t n_vec = Lq * H * (D / 4);
  int64_t blocks = (n_vec + 255) / 256;
  const int64_t cap = 148 * 8;  // 8 resident 256-thread blocks per SM, grid-strided
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const unsigned g = static_cast<unsigned>(blocks);
  if (!final_step)
    lse_combine_kernel<D, false, false><<<g, 256, 0, stream>>>(o_acc, lse_acc, o_part, lse_part,
                                                                out, lse_out, Lq, H, bias);
  else if (bf16)
    lse_combine_kernel<D, true, true><<<g, 256, 0, stream>>>(o_acc, lse_acc, o_part, lse_part,
                                                              out, lse_out, Lq, H, bias);
  else
    lse_combine_kernel<D, true, false><<<g, 256, 0, stream>>>(o_acc, lse_acc, o_part, lse_part,
                                                               out, lse_out, Lq, H, bias);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_lse_combine(float* o_acc, float* lse_acc, const float* o_part,
                               const float* lse_part, void* out, float* lse_out, int64_t Lq,
                               int D, int H, int final_step, int out_dtype_bf16,
                               cudaStream_t stream, float lse_bias) {
  if (Lq <= 0) return cudaSuccess;
  if (D == 64)
    return launch_d<64>(o_acc, lse_acc, o_part, lse_part, out, lse_out, Lq, H, final_step,
                        out_dtype_bf16, stream, lse_bias);
  if (D == 128)
    return launch_d<128>(o_acc, lse_acc, o_part, lse_part, out, lse_out, Lq, H, final_step,
                         out_dtype_bf16, stream, lse_bias);
  return cudaErrorInvalidValue;
}

}  // namespace dmha
