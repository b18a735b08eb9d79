// attn_fwd_tf32.cu — the fp32 path (dtype DMHA_FP32; BASELINE config C1:
// L=512, D=64, H=4, fp32, rel L2 <= 1e-4) on the tcgen05 tensor cores with
// 3xTF32 split arithmetic for BOTH contractions (SURVEY §8(c) reading 13,
// DESIGN.md R13: one-pass TF32 misses 1e-4, 3xTF32 on QK^T and PV passes):
//   x = hi + lo,  hi = x rounded to tf32 (nearest, ties away),  lo = x - hi
//   S  = Qlo Khi^T + Qhi Klo^T + Qhi Khi^T
//   O += Plo Vhi   + Phi Vlo   + Phi Vhi
// (small terms first; lo*lo is below fp32 rounding), accumulated in fp32 in
// TMEM.  The row softmax runs in fp32 with the same
// global-position causal rule, 1/sqrt(D) scale and lazy rescale rule as the
// bf16 kernel.
//
// Two launches per local attention call:
//  1. tf32_split_kv_kernel: K -> K hi / lo ([Lk, H, D]) and V -> V^T hi / lo
//     ([H, D, Lk4], keys contiguous) in the caller's scratch (the tf32 MMA
//     reads both operands K-major, so V is transposed once here instead of in
//     every CTA).
//  2. attn_fwd_tf32x3_kernel: CTA = one 128-row query tile of one head,
//     12 warps (D = 64) / 8 warps (D = 128):
//       warp 0     TMA producer of K hi / lo     (kKST-slot ring)
//       warp 1     TMEM allocator + MMA issuer
//       warp 2     TMA producer of V^T hi / lo   (kVST-slot ring)
//       warps 4-7  softmax + epilogue (thread <-> TMEM lane <-> query row);
//                  D = 64: warps 4-7 and 8-11 each take half of every
//                  row's score and output columns
//     Both A operands live in TMEM (Q hi / lo written once by the softmax
//     threads; P hi over the S columns it came from, P lo in its own
//     columns), so the tensor core reads only the K / V^T tiles from shared
//     memory.  S and P are double-buffered: the issuer runs QK^T one tile
//     ahead of PV, and softmax(j) overlaps PV(j-1) + QK^T(j+1).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "kernels.h"
#include "ptx_sm100.cuh"
#include "tma_map.h"

// TF32_WAIT: the kernel's mbarrier wait (a probe build can redefine it as a
// bounded wait that reports where a CTA stalls).
// -DDMHA_TF32_BOUNDED=1 (debug build): give up after ~2^28 polls, print the
// tag (which wait, which tile) and trap, so a protocol bug is an error, not
// a hung GPU.
#ifndef TF32_WAIT
#if DMHA_TF32_BOUNDED
#include <cstdio>
#define TF32_WAIT(bar, phase, tag)                                                         \
  do {                                                                                     \
    uint32_t n_ = 0;                                                                       \
    while (!ptx::mbar_try_wait(bar, phase)) {                                              \
      if (++n_ == (1u << 28)) {                                                            \
        printf("tf32 wait timeout tag %d block (%d,%d) thread %d\n", (tag), blockIdx.x,     \
               blockIdx.y, threadIdx.x);                                                   \
        __trap();                                                                          \
      }                                                                                    \
    }                                                                                      \
  } while (0)
#else
#define TF32_WAIT(bar, phase, tag) ptx::mbar_wait(bar, phase)
#endif
#endif

// Keys per TMEM accumulation chunk of O (see kFlush; measurement knob).
#ifndef DMHA_TF32_FLUSH_KEYS
#define DMHA_TF32_FLUSH_KEYS 512
#endif
// K / V^T ring slots (measurement knobs; 2 + 2 measured fastest at both D)
#ifndef DMHA_TF32_KST
#define DMHA_TF32_KST 2
#endif
#ifndef DMHA_TF32_VST
#define DMHA_TF32_VST 2
#endif

namespace dmha {
namespace {

constexpr int kBM = 128;
constexpr float kTf32RescaleThreshold = 8.0f;  // log2 units, as the bf16 kernel

template <int D>
struct Tf32Cfg {
  static constexpr int kBN = D == 64 ? 64 : 32;  // keys per tile
  static constexpr int kKST = DMHA_TF32_KST, kVST = DMHA_TF32_VST;  // ring slots
  static constexpr int kKOp = kBN * D * 4;        // one of K hi / lo
  static constexpr int kVOp = D * kBN * 4;        // one of V^T hi / lo
  static constexpr int kKOff = 0;
  static constexpr int kVOff = kKOff + kKST * 2 * kKOp;
  // fp32 master copy of O (one 128-row tile; 16-byte chunks XOR-swizzled by
  // row so a warp's row-per-thread accesses are conflict-free)
  static constexpr int kMOff = kVOff + kVST * 2 * kVOp;
  // D = 64: two softmax warpgroups split each row's score columns (the
  // per-row chain, not issue, bounds one warp per SMSP); they exchange row
  // maxima (2 tiles x 2 halves x 128) and, at the end, row sums (2 x 128)
  static constexpr int kHalves = D == 64 ? 2 : 1;
  static constexpr int kThreads = 128 + 128 * kHalves;
  static constexpr int kCols = kBN / kHalves;  // score columns per half
  static constexpr int kRedOff = kMOff + kBM * D * 4;
  static constexpr int kBarOff = kRedOff + (kHalves == 2 ? 6 * kBM * 4 : 0);
  // PV restarts its TMEM accumulator every kFlush tiles (512 keys) after the
  // softmax threads have added the partial into the master copy (see the
  // kernel): error 3.6e-6 (D = 64) / 3.8e-6 (D = 128) rel L2 at any length,
  // the flush's wait for PV(j-1) paid once per 512 keys
  static constexpr int kFlush = DMHA_TF32_FLUSH_KEYS / kBN;
  static_assert(kFlush >= 1, "flush interval");
  // kfull[KST] kempty[KST] vfull[VST] vempty[VST] sfull[2] pready[2] oready
  // ofinal qready
  static constexpr int kNumBars = 2 * kKST + 2 * kVST + 7;
  static constexpr int kSmem = kBarOff + kNumBars * 8 + 16 + 1024;
  // TMEM columns (fp32 / tf32: one element per column)
  static constexpr int cQh = 0, cQl = D, cS = 2 * D, cPl = cS + 2 * kBN, cO = cPl + 2 * kBN;
  static constexpr uint32_t kIdescS = ptx::make_idesc(2, kBM, kBN, 0, 0);  // tf32, K-major
  static constexpr uint32_t kIdescO = ptx::make_idesc(2, kBM, D, 0, 0);
  static_assert(cO + D <= 512, "TMEM budget");
  static_assert(kSmem <= 232448, "shared memory budget");
  static_assert(kBN % 32 == 0 && D % 32 == 0, "32-column TMEM chunks");
};

// x = hi + lo with hi = x rounded to tf32 (10 mantissa bits, nearest, ties
// away from zero on the magnitude) and lo = x - hi exact in fp32.
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
  lo = x - hi;
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

__device__ __forceinline__ float lds32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}

__device__ __forceinline__ int64_t pos_tf(const PosMap& m, int64_t i) {
  return i < m.chunk ? m.base0 + i : m.base1 + (i - m.chunk);
}

// Keys usable by a query at global position qp: a prefix of [0, Lk).
__device__ __forceinline__ int64_t klimit_tf(int causal, const PosMap& km, int64_t Lk, int64_t qp) {
  if (!causal) return Lk;
  int64_t lim;
  if (Lk > km.chunk && qp >= km.base1) {
    lim = km.chunk + (qp - km.base1) + 1;
  } else if (qp >= km.base0) {
    lim = qp - km.base0 + 1;
    if (lim > km.chunk) lim = km.chunk;
  } else {
    lim = 0;
  }
  return lim < Lk ? lim : Lk;
}

// D[tmem] (+)= A[tmem] * B[smem desc]  (kind::tf32, A read from tensor
// memory).  Whole-warp issue: every lane of the converged issuer warp runs it
// with the same operands and elect.sync picks the issuing lane; the smem
// descriptor is given as its low word (start address >> 4 | LBO) plus the
// constant high word, so per-MMA descriptor math is one 32-bit add.  The
// issue rate matters here: a 128 x 64 x 8 tf32 MMA is ~32 tensor cycles (16
// at N = 32), and a one-thread loop building 64-bit descriptors per MMA
// measured slower than that (tensor pipe 36 % active, softmax starved).
__device__ __forceinline__ void mma_tf32_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo,
                                              uint32_t desc_hi, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 db;\n\t"
      "mov.b64 db, {%2, %3};\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], db, %4, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "r"(b_lo), "r"(desc_hi), "r"(idesc), "r"(acc)
      : "memory");
}

// 128-byte-swizzle K-major smem descriptor words (SBO = 1024 B: 8 rows x 128 B)
constexpr uint32_t kDescHi = (1024u >> 4) | (1u << 14) | (2u << 29);
__device__ __forceinline__ uint32_t desc_lo(uint32_t saddr) {
  return ((saddr >> 4) & 0x3FFFu) | (1u << 16);  // LBO = 16 B (unused with swizzle)
}

// D (+)= A * B^T over K = kKdim: A = kKdim TMEM columns from a_col, B = a
// K-major 128-byte-swizzled shared-memory operand of kBRows rows (panels of
// 32 fp32 along K) whose descriptor low word is b_lo.  Eight K elements per
// instruction, fully unrolled (constant descriptor offsets).
template <int kKdim, int kBRows>
__device__ __forceinline__ void mma_tf32_kloop(uint32_t d, uint32_t a_col, uint32_t b_lo,
                                               uint32_t idesc, bool acc) {
#pragma unroll
  for (int kk = 0; kk < kKdim / 8; ++kk) {
    constexpr int kPanel = kBRows * 128;
    const uint32_t off = static_cast<uint32_t>((kk >> 2) * kPanel + (kk & 3) * 32) >> 4;
    mma_tf32_ts_w(d, a_col + kk * 8, b_lo + off, kDescHi, idesc, (acc || kk > 0) ? 1u : 0u);
  }
}

// ---------------------------------------------------------------- launch 1
// Block = 32 keys of one head: K split elementwise (coalesced along D), V
// split and transposed through shared memory (one 128-byte row of 32 keys
// per warp store).  Keys in [Lk, Lk4) of V^T are written as zeros.
template <int D>
__global__ void __launch_bounds__(256) tf32_split_kv_kernel(
    const float* __restrict__ k, const float* __restrict__ v, float* __restrict__ kh,
    float* __restrict__ kl, float* __restrict__ vth, float* __restrict__ vtl, int64_t Lk,
    int64_t Lk4, int H) {
  __shared__ float tile[32][D + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int head = blockIdx.y;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * 32;
  for (int i = tid; i < 32 * (D / 4); i += 256) {
    const int r = i / (D / 4), c = i % (D / 4);
    const int64_t key = j0 + r;
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    if (key < Lk) {
      const int64_t e4 = (key * H + head) * (D / 4) + c;
      const float4 x = reinterpret_cast<const float4*>(k)[e4];
      float4 h, l;
      split_tf32(x.x, h.x, l.x);
      split_tf32(x.y, h.y, l.y);
      split_tf32(x.z, h.z, l.z);
      split_tf32(x.w, h.w, l.w);
      reinterpret_cast<float4*>(kh)[e4] = h;
      reinterpret_cast<float4*>(kl)[e4] = l;
      y = reinterpret_cast<const float4*>(v)[e4];
    }
    tile[r][4 * c] = y.x;
    tile[r][4 * c + 1] = y.y;
    tile[r][4 * c + 2] = y.z;
    tile[r][4 * c + 3] = y.w;
  }
  __syncthreads();
  const int64_t key = j0 + lane;
  if (key >= Lk4) return;
  for (int d = warp; d < D; d += 8) {
    float h, l;
    split_tf32(tile[lane][d], h, l);
    const int64_t o = (static_cast<int64_t>(head) * D + d) * Lk4 + key;
    vth[o] = h;
    vtl[o] = l;
  }
}

// ---------------------------------------------------------------- launch 2
template <int D>
__global__ void __launch_bounds__(Tf32Cfg<D>::kThreads, 1)
    attn_fwd_tf32x3_kernel(const __grid_constant__ CUtensorMap tm_kh,
                           const __grid_constant__ CUtensorMap tm_kl,
                           const __grid_constant__ CUtensorMap tm_vh,
                           const __grid_constant__ CUtensorMap tm_vl, const float* __restrict__ q,
                           float* __restrict__ out, float* __restrict__ lse, int64_t Lq,
                           int64_t Lk, int H, int causal, PosMap qmap, PosMap kmap,
                           float scale_log2) {
  using C = Tf32Cfg<D>;
  constexpr int kBN = C::kBN, kKST = C::kKST, kVST = C::kVST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::kBarOff);
  uint64_t* kfull = bars;
  uint64_t* kempty = kfull + kKST;
  uint64_t* vfull = kempty + kKST;
  uint64_t* vempty = vfull + kVST;
  uint64_t* sfull = vempty + kVST;
  uint64_t* pready = sfull + 2;
  uint64_t* oready = pready + 2;
  uint64_t* ofinal = oready + 1;
  uint64_t* qready = ofinal + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qready + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int head = blockIdx.y;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * kBM;
  // tiles this CTA visits: the key prefix its last row may use
  const int64_t last = (m0 + kBM - 1 < Lq - 1) ? m0 + kBM - 1 : Lq - 1;
  const int64_t kmax = klimit_tf(causal, kmap, Lk, pos_tf(qmap, last));
  const int ntiles = static_cast<int>((kmax + kBN - 1) / kBN);

  if (tid == 0) {
    for (int i = 0; i < kKST; ++i) {
      ptx::mbar_init(&kfull[i], 1);
      ptx::mbar_init(&kempty[i], 1);
    }
    for (int i = 0; i < kVST; ++i) {
      ptx::mbar_init(&vfull[i], 1);
      ptx::mbar_init(&vempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&sfull[i], 1);
      ptx::mbar_init(&pready[i], 128 * C::kHalves);
    }
    ptx::mbar_init(oready, 1);
    ptx::mbar_init(ofinal, 1);
    ptx::mbar_init(qready, 128 * C::kHalves);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = ptx::smem_u32(sm);

  if (warp == 0) {
    // ---- K hi / lo producer
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tm_kh);
      ptx::tma_prefetch_desc(&tm_kl);
    }
    for (int j = 0; j < ntiles; ++j) {
      const int st = j % kKST;
      if (j >= kKST) TF32_WAIT(&kempty[st], ((j / kKST) - 1) & 1, 100);
      if (lane == 0) {
        ptx::mbar_arrive_expect_tx(&kfull[st], 2 * C::kKOp);
        uint8_t* dst = sm + C::kKOff + st * 2 * C::kKOp;
#pragma unroll
        for (int p = 0; p < D / 32; ++p) {
          ptx::tma_load_3d(&tm_kh, &kfull[st], dst + p * kBN * 128, p * 32, head, j * kBN);
          ptx::tma_load_3d(&tm_kl, &kfull[st], dst + C::kKOp + p * kBN * 128, p * 32, head,
                           j * kBN);
        }
      }
      __syncwarp();
    }
  } else if (warp == 2) {
    // ---- V^T hi / lo producer
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tm_vh);
      ptx::tma_prefetch_desc(&tm_vl);
    }
    for (int j = 0; j < ntiles; ++j) {
      const int st = j % kVST;
      if (j >= kVST) TF32_WAIT(&vempty[st], ((j / kVST) - 1) & 1, 200);
      if (lane == 0) {
        ptx::mbar_arrive_expect_tx(&vfull[st], 2 * C::kVOp);
        uint8_t* dst = sm + C::kVOff + st * 2 * C::kVOp;
#pragma unroll
        for (int p = 0; p < kBN / 32; ++p) {
          ptx::tma_load_3d(&tm_vh, &vfull[st], dst + p * D * 128, j * kBN + p * 32, 0, head);
          ptx::tma_load_3d(&tm_vl, &vfull[st], dst + C::kVOp + p * D * 128, j * kBN + p * 32, 0,
                           head);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---- MMA issuer: QK(0), QK(1), then PV(j), QK(j+2) ...  The whole warp
    // waits on the barriers and runs the issue code; elect.sync picks the
    // lane that issues (no lane spins alone, descriptors stay uniform).
    auto issue_qk = [&](int j) {
      const int st = j % kKST;
      TF32_WAIT(&kfull[st], (j / kKST) & 1, 300);
      ptx::tc_fence_after();
      const uint32_t d = tmem + C::cS + (j & 1) * kBN;
      const uint32_t kh = desc_lo(sbase + C::kKOff + st * 2 * C::kKOp);
      const uint32_t kl = kh + (C::kKOp >> 4);
      mma_tf32_kloop<D, kBN>(d, tmem + C::cQl, kh, C::kIdescS, false);
      mma_tf32_kloop<D, kBN>(d, tmem + C::cQh, kl, C::kIdescS, true);
      mma_tf32_kloop<D, kBN>(d, tmem + C::cQh, kh, C::kIdescS, true);
      ptx::mma_commit_w(&kempty[st]);
      ptx::mma_commit_w(&sfull[j & 1]);
      __syncwarp();
    };
    auto issue_pv = [&](int j) {
      const int b = j & 1, st = j % kVST;
      TF32_WAIT(&pready[b], (j >> 1) & 1, 400);
      TF32_WAIT(&vfull[st], (j / kVST) & 1, 500);
      ptx::tc_fence_after();
      const uint32_t d = tmem + C::cO;
      const uint32_t vh = desc_lo(sbase + C::kVOff + st * 2 * C::kVOp);
      const uint32_t vl = vh + (C::kVOp >> 4);
      const uint32_t ph = tmem + C::cS + b * kBN, pl = tmem + C::cPl + b * kBN;
      mma_tf32_kloop<kBN, D>(d, pl, vh, C::kIdescO, (j % C::kFlush) != 0);
      mma_tf32_kloop<kBN, D>(d, ph, vl, C::kIdescO, true);
      mma_tf32_kloop<kBN, D>(d, ph, vh, C::kIdescO, true);
      ptx::mma_commit_w(&vempty[st]);
      ptx::mma_commit_w(oready);
      if (j == ntiles - 1) ptx::mma_commit_w(ofinal);
      __syncwarp();
    };
    if (ntiles > 0) {
      TF32_WAIT(qready, 0, 600);
      ptx::tc_fence_after();
      issue_qk(0);
      if (ntiles > 1) issue_qk(1);
      for (int j = 0; j < ntiles; ++j) {
        issue_pv(j);
        if (j + 2 < ntiles) issue_qk(j + 2);
      }
    }
  } else if (warp >= 4) {
    // ---- softmax + epilogue: thread <-> TMEM lane <-> query row.  With two
    // halves (D = 64) warpgroup h owns score columns [32h, 32h + 32) of each
    // tile and O / Q columns [32h, 32h + 32); the halves agree on the row max
    // through shared memory once per tile (named barrier 1).
    constexpr int kH = C::kHalves, kCols = C::kCols, kOCols = D / kH;
    const int h = kH == 2 ? (warp - 4) >> 2 : 0;
    const int wq = warp & 3;
    const int r = wq * 32 + lane;
    const int64_t row = m0 + r;
    const bool row_ok = row < Lq;
    const uint32_t lane_addr = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t tl = tmem + lane_addr;
    const int scol = h * kCols, ocol = h * kOCols;
    if (ntiles > 0) {
      // Q row -> TMEM hi / lo (rows past Lq are zero)
      const float4* qr = reinterpret_cast<const float4*>(q + (row * H + head) * D + ocol);
#pragma unroll
      for (int c = 0; c < kOCols / 32; ++c) {
        float hi[32], lo[32];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float4 x = row_ok ? qr[c * 8 + e] : make_float4(0.f, 0.f, 0.f, 0.f);
          split_tf32(x.x, hi[4 * e], lo[4 * e]);
          split_tf32(x.y, hi[4 * e + 1], lo[4 * e + 1]);
          split_tf32(x.z, hi[4 * e + 2], lo[4 * e + 2]);
          split_tf32(x.w, hi[4 * e + 3], lo[4 * e + 3]);
        }
        ptx::tmem_st32(tl + C::cQh + ocol + c * 32, hi);
        ptx::tmem_st32(tl + C::cQl + ocol + c * 32, lo);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(qready);
    }
    // O = master + TMEM partial.  The tensor core's fp32 accumulation
    // truncates, and its bias grows with the number of accumulate steps
    // (measured: rel L2 1.1e-4 at 16384 keys with one accumulator); moving
    // the partial into the master with round-to-nearest FADDs every kFlush
    // tiles bounds that to kFlush tiles' worth.
    // (16-byte chunk c4 of this row's master at mrow + 16 * (c4 ^ (r & 7));
    // the XOR keeps each half's chunks in its own half of the row)
    const uint32_t mrow = sbase + C::kMOff + static_cast<uint32_t>(r) * D * 4;
    auto mchunk = [&](int c4) { return mrow + static_cast<uint32_t>((c4 ^ (r & 7)) << 4); };
#pragma unroll
    for (int c4 = 0; c4 < kOCols / 4; ++c4) sts128(mchunk(ocol / 4 + c4), make_float4(0.f, 0.f, 0.f, 0.f));
    const uint32_t red = sbase + C::kRedOff;  // [2 tiles][2 halves][kBM] maxima, then [2][kBM] sums
    const int64_t qp = pos_tf(qmap, row_ok ? row : Lq - 1);
    const int64_t klim = klimit_tf(causal, kmap, Lk, qp);
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < ntiles; ++j) {
      const int b = j & 1;
      TF32_WAIT(&sfull[b], (j >> 1) & 1, 700);
      ptx::tc_fence_after();
      float s[kCols];
#pragma unroll
      for (int c = 0; c < kCols / 32; ++c)
        ptx::tmem_ld32(tl + C::cS + b * kBN + scol + c * 32,
                       *reinterpret_cast<float(*)[32]>(&s[32 * c]));
      ptx::tmem_wait_ld();
      // row max of the raw scores (the scale is positive), 8 independent
      // partial maxima (one softmax warp per SMSP per half: latency binds);
      // keys past the row's limit (causal / ragged tail) are -inf
      const int64_t nv = klim - static_cast<int64_t>(j) * kBN - scol;
      if (nv < kCols) {
#pragma unroll
        for (int c = 0; c < kCols; ++c) s[c] = (c < nv) ? s[c] : -INFINITY;
      }
      float pm[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) pm[i] = s[i];
#pragma unroll
      for (int c = 8; c < kCols; ++c) pm[c & 7] = fmaxf(pm[c & 7], s[c]);
      float rmax = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                         fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
      if constexpr (kH == 2) {
        const uint32_t slot = red + static_cast<uint32_t>(((b * 2 + h) * kBM + r) * 4);
        sts32(slot, rmax);
        asm volatile("bar.sync 1, 256;" ::: "memory");
        rmax = fmaxf(rmax, lds32(red + static_cast<uint32_t>(((b * 2 + (h ^ 1)) * kBM + r) * 4)));
      }
      const float mx = rmax * scale_log2;
      // lazy rescale: move the reference max only when a score exceeds it by
      // more than 2^8 (P <= 256 otherwise); warp-uniform because the O
      // rescale is a warp-collective tcgen05.ld / st, and the same in both
      // halves (same rows, same max)
      const bool need = mx > m_run + kTf32RescaleThreshold;
      const bool rescale = __any_sync(0xffffffffu, need);
      const bool flush = j > 0 && (j % C::kFlush) == 0;  // PV(j) restarts the accumulator
      float alpha = 1.f;
      if (rescale) {
        const float m_new = fmaxf(m_run, mx);
        alpha = (m_run == -INFINITY) ? 1.f : exp2f(m_run - m_new);
        l_run *= alpha;
        m_run = m_new;
      }
      if (j > 0 && (rescale || flush)) {
        // PV(j-1) complete: O is final so far.  Unambiguous parity: S(j)'s
        // commit covered PV(j-2), and PV(j) waits for this tile's P.
        TF32_WAIT(oready, (j - 1) & 1, 800);
        ptx::tc_fence_after();
#pragma unroll
        for (int c = 0; c < kOCols / 32; ++c) {
          float o[32];
          ptx::tmem_ld32(tl + C::cO + ocol + c * 32, o);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e4 = 0; e4 < 8; ++e4) {
            const uint32_t a = mchunk(ocol / 4 + c * 8 + e4);
            const float4 m = lds128(a);
            if (flush) {  // master = (master + partial) * alpha
              sts128(a, make_float4((m.x + o[4 * e4]) * alpha, (m.y + o[4 * e4 + 1]) * alpha,
                                    (m.z + o[4 * e4 + 2]) * alpha, (m.w + o[4 * e4 + 3]) * alpha));
            } else {
              sts128(a, make_float4(m.x * alpha, m.y * alpha, m.z * alpha, m.w * alpha));
            }
          }
          if (!flush) {
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] *= alpha;
            ptx::tmem_st32(tl + C::cO + ocol + c * 32, o);
          }
        }
      }
      const float neg_m = (m_run == -INFINITY) ? 0.f : -m_run;
      float ps[4] = {0.f, 0.f, 0.f, 0.f};  // independent partial sums
#pragma unroll
      for (int c = 0; c < kCols / 32; ++c) {
        float hi[32], lo[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float p = exp2f(fmaf(s[32 * c + e], scale_log2, neg_m));
          ps[e & 3] += p;
          split_tf32(p, hi[e], lo[e]);
        }
        ptx::tmem_st32(tl + C::cS + b * kBN + scol + c * 32, hi);  // P hi over S(j)
        ptx::tmem_st32(tl + C::cPl + b * kBN + scol + c * 32, lo);
      }
      l_run += (ps[0] + ps[1]) + (ps[2] + ps[3]);
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&pready[b]);
    }
    // ---- epilogue: O / l, lse = ln l + m (natural log of the scaled scores)
    // (ofinal, not oready: up to two PVs may be outstanding here, so an
    // oready parity would be ambiguous)
    if (ntiles > 0) {
      TF32_WAIT(ofinal, 0, 900);
      ptx::tc_fence_after();
    }
    float l_tot = l_run;
    if constexpr (kH == 2) {
      const uint32_t lred = red + static_cast<uint32_t>(4 * kBM * 4);
      sts32(lred + static_cast<uint32_t>((h * kBM + r) * 4), l_run);
      asm volatile("bar.sync 1, 256;" ::: "memory");
      l_tot += lds32(lred + static_cast<uint32_t>(((h ^ 1) * kBM + r) * 4));
    }
    const bool empty = !(l_tot > 0.f);
    const float inv = empty ? 0.f : 1.f / l_tot;
#pragma unroll
    for (int c = 0; c < kOCols / 32; ++c) {
      float o[32];
      if (ntiles > 0) {
        ptx::tmem_ld32(tl + C::cO + ocol + c * 32, o);
        ptx::tmem_wait_ld();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = 0.f;
      }
      if (row_ok) {
        float4* dst = reinterpret_cast<float4*>(out + (row * H + head) * D + ocol + c * 32);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float4 m = lds128(mchunk(ocol / 4 + c * 8 + e));
          dst[e] = make_float4((m.x + o[4 * e]) * inv, (m.y + o[4 * e + 1]) * inv,
                               (m.z + o[4 * e + 2]) * inv, (m.w + o[4 * e + 3]) * inv);
        }
      }
    }
    if (row_ok && h == 0)
      lse[static_cast<int64_t>(head) * Lq + row] =
          empty ? -INFINITY : (m_run + log2f(l_tot)) * 0.69314718055994530942f;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

int64_t lk4_of(int64_t Lk) { return (Lk + 3) / 4 * 4; }

template <int D>
cudaError_t launch_tf32(const LocalAttnArgs& a, cudaStream_t stream) {
  using C = Tf32Cfg<D>;
  if (a.Lk > 0 && (!a.scratch || a.scratch_bytes < tf32_scratch_bytes(a.Lk, a.H, D)))
    return cudaErrorInvalidValue;
  const int64_t Lk4 = lk4_of(a.Lk);
  const size_t kel = static_cast<size_t>(a.Lk) * a.H * D, vel = static_cast<size_t>(a.H) * D * Lk4;
  float* kh = static_cast<float*>(a.scratch);
  float* kl = kh + kel;
  float* vth = kl + kel;
  float* vtl = vth + vel;
  if (a.Lk > 0) {
    dim3 g1(static_cast<unsigned>((a.Lk + 31) / 32), a.H);
    tf32_split_kv_kernel<D><<<g1, 256, 0, stream>>>(static_cast<const float*>(a.k),
                                                    static_cast<const float*>(a.v), kh, kl, vth,
                                                    vtl, a.Lk, Lk4, a.H);
  }
  // K hi / lo: [Lk, H, D] as (D, H, Lk), boxes of 32 fp32 x 1 head x kBN keys;
  // V^T hi / lo: [H, D, Lk4] as (Lk, D, H), boxes of 32 keys x D rows x 1 head
  // (keys past Lk read as zeros).  128-byte swizzle, as the descriptors expect.
  const cuuint64_t lk = static_cast<cuuint64_t>(a.Lk > 0 ? a.Lk : 1);
  const cuuint64_t kdims[3] = {D, static_cast<cuuint64_t>(a.H), lk};
  const cuuint64_t kstr[2] = {D * 4ull, static_cast<cuuint64_t>(a.H) * D * 4};
  const cuuint32_t kbox[3] = {32, 1, static_cast<cuuint32_t>(C::kBN)};
  const cuuint64_t vdims[3] = {lk, D, static_cast<cuuint64_t>(a.H)};
  const cuuint64_t vstr[2] = {static_cast<cuuint64_t>(Lk4) * 4, static_cast<cuuint64_t>(Lk4) * D * 4};
  const cuuint32_t vbox[3] = {32, D, 1};
  CUtensorMap tkh{}, tkl{}, tvh{}, tvl{};  // Lk = 0: no tile is loaded, maps unused
  if (a.Lk > 0 && (!make_tma_map_f32(&tkh, kh, kdims, kstr, kbox) ||
                   !make_tma_map_f32(&tkl, kl, kdims, kstr, kbox) ||
                   !make_tma_map_f32(&tvh, vth, vdims, vstr, vbox) ||
                   !make_tma_map_f32(&tvl, vtl, vdims, vstr, vbox)))
    return cudaErrorInvalidValue;
  static int attr_dev = -1;
  int cur = 0;
  cudaGetDevice(&cur);
  if (attr_dev != cur) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_tf32x3_kernel<D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    attr_dev = cur;
  }
  dim3 grid(static_cast<unsigned>((a.Lq + kBM - 1) / kBM), a.H);
  attn_fwd_tf32x3_kernel<D><<<grid, C::kThreads, C::kSmem, stream>>>(
      tkh, tkl, tvh, tvl, static_cast<const float*>(a.q), static_cast<float*>(a.out), a.lse, a.Lq,
      a.Lk, a.H, a.causal, a.qmap, a.kmap,
      static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(D))));
  return cudaGetLastError();
}

}  // namespace

size_t tf32_scratch_bytes(int64_t Lk, int H, int D) {
  if (Lk <= 0) return 0;
  return (2 * static_cast<size_t>(Lk) * H * D + 2 * static_cast<size_t>(H) * D * lk4_of(Lk)) * 4;
}

cudaError_t launch_attn_fwd_tf32x3(const LocalAttnArgs& a, cudaStream_t stream) {
  if (a.Lq <= 0) return cudaSuccess;
  if (a.out_mode != OUT_FINAL && a.out_mode != OUT_PARTIAL_F32) return cudaErrorInvalidValue;
  if (a.D == 64) return launch_tf32<64>(a, stream);
  if (a.D == 128) return launch_tf32<128>(a, stream);
  return cudaErrorInvalidValue;
}

}  // namespace dmha
