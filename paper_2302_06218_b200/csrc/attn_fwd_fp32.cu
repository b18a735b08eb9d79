// attn_fwd_fp32.cu — fp32-storage attention forward (the DMHA_FP32 path,
// BASELINE config C1: L=512, D=64, H=4, rel-L2 <= 1e-4).
//
// Same operation and the same global-position causal rule as the bf16
// tcgen05 kernel (north_star 1/sqrt(D)), computed in fp32 on
// the FMA pipes: one warp per (query row, head).  Keys are processed 32 at a
// time: lane t computes the full dot product of key j0+t (q row held in
// registers), the chunk max / sum are warp-shuffle reductions, and each lane
// accumulates D/32 output columns with the broadcast probabilities.
// The default fp32 path is the 3xTF32 tensor-core kernel (attn_fwd_tf32.cu);
// this SIMT kernel is the independent cross-check behind DMHA_FP32_SIMT=1.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "kernels.h"

namespace dmha {
namespace {

__device__ __forceinline__ int64_t pos_of32(const PosMap& m, int64_t i) {
  return i < m.chunk ? m.base0 + i : m.base1 + (i - m.chunk);
}

template <int D>
__global__ void __launch_bounds__(256) attn_fwd_fp32_kernel(const float* __restrict__ q,
                                                            const float* __restrict__ k,
                                                            const float* __restrict__ v,
                                                            float* __restrict__ out,
                                                            float* __restrict__ lse, int64_t Lq,
                                                            int64_t Lk, int H, int causal,
                                                            PosMap qmap, PosMap kmap) {
  constexpr int kPer = D / 32;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (gw >= Lq * H) return;
  const int64_t row = gw / H;
  const int head = static_cast<int>(gw % H);
  const float scale = rsqrtf(static_cast<float>(D));

  // keys usable by this row: a prefix of [0, Lk) because kpos is increasing
  int64_t klim = Lk;
  if (causal) {
    const int64_t qp = pos_of32(qmap, row);
    if (Lk > kmap.chunk && qp >= kmap.base1) {
      klim = kmap.chunk + (qp - kmap.base1) + 1;
    } else if (qp >= kmap.base0) {
      klim = qp - kmap.base0 + 1;
      if (klim > kmap.chunk) klim = kmap.chunk;
    } else {
      klim = 0;
    }
    if (klim > Lk) klim = Lk;
  }

  float qr[D];
  const float* qrow = q + (row * H + head) * D;
#pragma unroll
  for (int d = 0; d < D; ++d) qr[d] = qrow[d] * scale;

  float m = -INFINITY, l = 0.f;
  float acc[kPer];
#pragma unroll
  for (int e = 0; e < kPer; ++e) acc[e] = 0.f;

  for (int64_t j0 = 0; j0 < klim; j0 += 32) {
    const int64_t j = j0 + lane;
    float s = -INFINITY;
    if (j < klim) {
      const float4* kr = reinterpret_cast<const float4*>(k + (j * H + head) * D);
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
      for (int d4 = 0; d4 < D / 4; ++d4) {
        const float4 kv = kr[d4];
        a0 = fmaf(qr[4 * d4], kv.x, a0);
        a1 = fmaf(qr[4 * d4 + 1], kv.y, a1);
        a2 = fmaf(qr[4 * d4 + 2], kv.z, a2);
        a3 = fmaf(qr[4 * d4 + 3], kv.w, a3);
      }
      s = (a0 + a1) + (a2 + a3);
    }
    float cm = s;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
    const float m_new = fmaxf(m, cm);
    const float alpha = (m == -INFINITY) ? 0.f : expf(m - m_new);
    const float pj = (s == -INFINITY) ? 0.f : expf(s - m_new);
    float cs = pj;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
    l = l * alpha + cs;
#pragma unroll
    for (int e = 0; e < kPer; ++e) acc[e] *= alpha;
    const int nk = static_cast<int>((klim - j0) < 32 ? (klim - j0) : 32);
    for (int t = 0; t < nk; ++t) {
      const float pt = __shfl_sync(0xffffffffu, pj, t);
      const float* vr = v + ((j0 + t) * H + head) * D;
#pragma unroll
      for (int e = 0; e < kPer; ++e) acc[e] = fmaf(pt, vr[lane + 32 * e], acc[e]);
    }
    m = m_new;
  }
  const bool empty = !(l > 0.f);
  const float inv = empty ? 0.f : 1.f / l;
  float* orow = out + (row * H + head) * D;
#pragma unroll
  for (int e = 0; e < kPer; ++e) orow[lane + 32 * e] = acc[e] * inv;
  if (lane == 0) lse[static_cast<int64_t>(head) * Lq + row] = empty ? -INFINITY : m + logf(l);
}

}  // namespace

static bool fp32_simt() {
  const char* e = std::getenv("DMHA_FP32_SIMT");
  return e && std::atoi(e) != 0;
}

int fp32_launches_per_call(int64_t Lq, int64_t Lk) {
  if (Lq <= 0) return 0;
  return fp32_simt() ? 1 : (Lk > 0 ? 2 : 1);
}

cudaError_t launch_attn_fwd_fp32(const LocalAttnArgs& a, cudaStream_t stream) {
  if (!fp32_simt()) return launch_attn_fwd_tf32x3(a, stream);
  if (a.Lq <= 0) return cudaSuccess;
  const int64_t warps = a.Lq * a.H;
  const int64_t blocks = (warps * 32 + 255) / 256;
  if (a.D == 64) {
    attn_fwd_fp32_kernel<64><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
        static_cast<const float*>(a.q), static_cast<const float*>(a.k),
        static_cast<const float*>(a.v), static_cast<float*>(a.out), a.lse, a.Lq, a.Lk, a.H,
        a.causal, a.qmap, a.kmap);
  } else if (a.D == 128) {
    attn_fwd_fp32_kernel<128><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
        static_cast<const float*>(a.q), static_cast<const float*>(a.k),
        static_cast<const float*>(a.v), static_cast<float*>(a.out), a.lse, a.Lq, a.Lk, a.H,
        a.causal, a.qmap, a.kmap);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace dmha
