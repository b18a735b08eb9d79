// softmax_sm100.cuh — exponential helpers shared by the attention kernels:
// P = exp2(S*scale*log2e - m) for one 128-column score row per thread, on
// MUFU.EX2 or (for EMU of every 8 column pairs) on the FMA pipe, packed to bf16
// and stored to TMEM — the numerator of the row softmax of PAPER.md:198-201
// (online form with a running max m, readings R11/R16).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

#include "ptx_sm100.cuh"

namespace dmha {
namespace sm {

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  return fmaxf(fmaxf(a, b), c);  // ptxas fuses to FMNMX3
}

// 2^x for a pair on MUFU.EX2.
__device__ __forceinline__ float2 exp2_mufu2(float2 x) {
  return make_float2(ptx::ex2_approx(x.x), ptx::ex2_approx(x.y));
}

// 2^x for a pair on the FMA pipe (FADD2/FFMA2 + 2 ALU ops per element):
// n = round(x) via the 1.5*2^23 magic add, f = x - n in [-0.5, 0.5],
// 2^f by a degree-3 minimax polynomial (max rel. error 7.5e-5, below the
// 2^-9 bf16 rounding P gets anyway), exponent added as (n << 23).
// x is clamped at -126 so the exponent cannot wrap (only used on unmasked
// tiles, whose entries are finite).
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  const float2 magic = make_float2(12582912.f, 12582912.f);
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = __fadd2_rn(x, magic);
  const float2 j = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-j.x, -j.y));
  float2 p = __ffma2_rn(f, make_float2(0.055171459913253784f, 0.055171459913253784f),
                        make_float2(0.2426108568906784f, 0.2426108568906784f));
  p = __ffma2_rn(p, f, make_float2(0.6932609677314758f, 0.6932609677314758f));
  p = __ffma2_rn(p, f, make_float2(0.9999281167984009f, 0.9999281167984009f));
  const uint32_t rx = __float_as_uint(p.x) + (__float_as_uint(t.x) << 23);
  const uint32_t ry = __float_as_uint(p.y) + (__float_as_uint(t.y) << 23);
  return make_float2(__uint_as_float(rx), __uint_as_float(ry));
}

// P = exp2(S*scale*log2e - m) for one 128-column score row, packed to bf16 and
// written over the first 64 TMEM columns of the S buffer (16-column chunks, so
// the fp32 scores die as P is produced).  Returns the fp32 sum of P.
// EMU of every 8 column pairs use exp2_poly2 (FMA pipe), the rest MUFU.
template <int EMU>
__device__ __forceinline__ float exp_tile(float (&s)[128], float sl2, float m_use, uint32_t tP) {
  const float2 sc2 = make_float2(sl2, sl2);
  const float2 nm2 = make_float2(-m_use, -m_use);
  float2 sum_a = make_float2(0.f, 0.f), sum_b = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      // x = S*scale*log2e - m on the packed FP32x2 pipe (FFMA2)
      const float2 x = __ffma2_rn(make_float2(s[32 * c + 2 * e], s[32 * c + 2 * e + 1]), sc2, nm2);
      const float2 pe = (((c * 16 + e) & 7) < EMU) ? exp2_poly2(x) : exp2_mufu2(x);
      if (e & 1)
        sum_b = __fadd2_rn(sum_b, pe);
      else
        sum_a = __fadd2_rn(sum_a, pe);
      __nv_bfloat162 b = __floats2bfloat162_rn(pe.x, pe.y);
      pk[e] = *reinterpret_cast<uint32_t*>(&b);
    }
    ptx::tmem_st16(tP + c * 16, pk);
  }
  return (sum_a.x + sum_a.y) + (sum_b.x + sum_b.y);
}

// Same for one half row (64 columns -> 32 P columns at tP).
__device__ __forceinline__ float exp_half(float (&s)[64], float sl2, float m_use, uint32_t tP) {
  const float2 sc2 = make_float2(sl2, sl2);
  const float2 nm2 = make_float2(-m_use, -m_use);
  float2 sum_a = make_float2(0.f, 0.f), sum_b = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const float2 x = __ffma2_rn(make_float2(s[32 * c + 2 * e], s[32 * c + 2 * e + 1]), sc2, nm2);
      const float2 pe = exp2_mufu2(x);
      if (e & 1)
        sum_b = __fadd2_rn(sum_b, pe);
      else
        sum_a = __fadd2_rn(sum_a, pe);
      __nv_bfloat162 b = __floats2bfloat162_rn(pe.x, pe.y);
      pk[e] = *reinterpret_cast<uint32_t*>(&b);
    }
    ptx::tmem_st16(tP + c * 16, pk);
  }
  return (sum_a.x + sum_a.y) + (sum_b.x + sum_b.y);
}

__device__ __forceinline__ float row_max64(const float (&s)[64]) {
  float m[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) m[i] = fmaxf(fmaxf(s[i], s[8 + i]), s[16 + i]);
#pragma unroll
  for (int i = 0; i < 8; ++i) m[i] = fmaxf(fmaxf(m[i], s[24 + i]), s[32 + i]);
#pragma unroll
  for (int i = 0; i < 8; ++i) m[i] = fmaxf(fmaxf(m[i], s[40 + i]), s[48 + i]);
#pragma unroll
  for (int i = 0; i < 8; ++i) m[i] = fmaxf(m[i], s[56 + i]);
  const float a = fmaxf(fmaxf(m[0], m[1]), m[2]), b = fmaxf(fmaxf(m[3], m[4]), m[5]);
  return fmaxf(fmaxf(a, b), fmaxf(m[6], m[7]));
}

// Two-pass variant: all 128 exponentials first (in place, long independent
// MUFU streams), then bf16 packing and the TMEM stores.
__device__ __forceinline__ float exp_tile_2pass(float (&s)[128], float sl2, float m_use,
                                                uint32_t tP) {
  const float2 sc2 = make_float2(sl2, sl2);
  const float2 nm2 = make_float2(-m_use, -m_use);
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    const float2 x = __ffma2_rn(make_float2(s[2 * i], s[2 * i + 1]), sc2, nm2);
    s[2 * i] = ptx::ex2_approx(x.x);
    s[2 * i + 1] = ptx::ex2_approx(x.y);
  }
  float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                   make_float2(0.f, 0.f)};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const float2 pe = make_float2(s[32 * c + 2 * e], s[32 * c + 2 * e + 1]);
      acc[e & 3] = __fadd2_rn(acc[e & 3], pe);
      __nv_bfloat162 b = __floats2bfloat162_rn(pe.x, pe.y);
      pk[e] = *reinterpret_cast<uint32_t*>(&b);
    }
    ptx::tmem_st16(tP + c * 16, pk);
  }
  const float2 t = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
  return t.x + t.y;
}

// In-place exponentials of one 128-column score row (pass 1 of the split
// exp / store used by the D = 64 schedule, so the wait for the P buffer sits
// after the MUFU work): s <- exp2(s*scale*log2e - m).  EMU of every 8 column
// pairs on the FMA-pipe polynomial (finite inputs only), the rest on MUFU.
template <int EMU>
__device__ __forceinline__ void exp_inplace(float (&s)[128], float sl2, float m_use) {
  const float2 sc2 = make_float2(sl2, sl2);
  const float2 nm2 = make_float2(-m_use, -m_use);
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    const float2 x = __ffma2_rn(make_float2(s[2 * i], s[2 * i + 1]), sc2, nm2);
    const float2 pe = ((i & 7) < EMU) ? exp2_poly2(x) : exp2_mufu2(x);
    s[2 * i] = pe.x;
    s[2 * i + 1] = pe.y;
  }
}

// Pass 2: pack the 128 exponentials to bf16, store them as 64 TMEM columns at
// tP (16-column chunks) and return their fp32 sum.
__device__ __forceinline__ float store_p(const float (&s)[128], uint32_t tP) {
  float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                   make_float2(0.f, 0.f)};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const float2 pe = make_float2(s[32 * c + 2 * e], s[32 * c + 2 * e + 1]);
      acc[e & 3] = __fadd2_rn(acc[e & 3], pe);
      __nv_bfloat162 b = __floats2bfloat162_rn(pe.x, pe.y);
      pk[e] = *reinterpret_cast<uint32_t*>(&b);
    }
    ptx::tmem_st16(tP + c * 16, pk);
  }
  const float2 t = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
  return t.x + t.y;
}

// Pass 2 for P in shared memory (D = 128, kPS): pack the 128 exponentials of
// row r to bf16 and store them as row r of a 128 x 128 K-major tile in the
// 128-byte-swizzled layout an SS MMA operand descriptor (SWIZZLE_128B) reads
// — two 64-key panels of 128 rows x 128 B, 16-byte chunk c of row r stored
// at chunk c ^ (r & 7) — with 16 vector stores (a warp's 32 rows of one chunk
// take the minimum 4 wavefronts).  Returns the fp32 sum.  The caller fences
// (fence.proxy.async) before signalling the MMA issuer.
__device__ __forceinline__ float store_p_smem(const float (&s)[128], uint8_t* tile, int r) {
  float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                   make_float2(0.f, 0.f)};
  uint8_t* row = tile + r * 128;
  const int sw = r & 7;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    uint32_t w[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float2 pe = make_float2(s[8 * c + 2 * t], s[8 * c + 2 * t + 1]);
      acc[t] = __fadd2_rn(acc[t], pe);
      __nv_bfloat162 b = __floats2bfloat162_rn(pe.x, pe.y);
      w[t] = *reinterpret_cast<uint32_t*>(&b);
    }
    *reinterpret_cast<uint4*>(row + (c >> 3) * (128 * 128) + (((c & 7) ^ sw) << 4)) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
  const float2 t = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
  return t.x + t.y;
}

// Half-row versions (64 columns, split softmax): exponentials in place, then
// pack + store 32 P columns at tP and return the fp32 sum.
template <int EMU = 0>  // EMU of every 8 column pairs on the FMA-pipe polynomial (finite inputs)
__device__ __forceinline__ void exp_inplace64(float (&s)[64], float sl2, float m_use) {
  const float2 sc2 = make_float2(sl2, sl2);
  const float2 nm2 = make_float2(-m_use, -m_use);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const float2 x = __ffma2_rn(make_float2(s[2 * i], s[2 * i + 1]), sc2, nm2);
    const float2 pe = ((i & 7) < EMU) ? exp2_poly2(x) : exp2_mufu2(x);
    s[2 * i] = pe.x;
    s[2 * i + 1] = pe.y;
  }
}
__device__ __forceinline__ float store_p64(const float (&s)[64], uint32_t tP) {
  float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const float2 pe = make_float2(s[32 * c + 2 * e], s[32 * c + 2 * e + 1]);
      acc[e & 1] = __fadd2_rn(acc[e & 1], pe);
      __nv_bfloat162 b = __floats2bfloat162_rn(pe.x, pe.y);
      pk[e] = *reinterpret_cast<uint32_t*>(&b);
    }
    ptx::tmem_st16(tP + c * 16, pk);
  }
  const float2 t = __fadd2_rn(acc[0], acc[1]);
  return t.x + t.y;
}

// Row max of 128 scores as a shallow tree: 16 independent 3-input max chains
// of depth 4, then a 3-level tree (instead of 4 serial chains of depth 32).
__device__ __forceinline__ float row_max128(const float (&s)[128]) {
  float m[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) m[i] = fmax3(s[i], s[16 + i], s[32 + i]);
#pragma unroll
  for (int i = 0; i < 16; ++i) m[i] = fmax3(m[i], s[48 + i], s[64 + i]);
#pragma unroll
  for (int i = 0; i < 16; ++i) m[i] = fmax3(m[i], s[80 + i], s[96 + i]);
#pragma unroll
  for (int i = 0; i < 16; ++i) m[i] = fmaxf(m[i], s[112 + i]);
  float t[6];
#pragma unroll
  for (int i = 0; i < 5; ++i) t[i] = fmax3(m[3 * i], m[3 * i + 1], m[3 * i + 2]);
  t[5] = m[15];
  return fmaxf(fmax3(t[0], t[1], t[2]), fmax3(t[3], t[4], t[5]));
}

}  // namespace sm
}  // namespace dmha
