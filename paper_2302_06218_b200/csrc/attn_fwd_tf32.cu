// attn_fwd_tf32.cu — the fp32 path (dtype DMHA_FP32; BASELINE config C1:
// L=512, D=64, H=4, fp32, rel L2 <= 1e-4) on the tcgen05 tensor cores with
// 3xTF32 split arithmetic for BOTH contractions (SURVEY §8(c) reading 13,
// DESIGN.md R13: one-pass TF32 misses 1e-4, 3xTF32 on QK^T and PV passes):
//   x = hi + lo,  hi = tf32_rna(x),  lo = x - hi          (exact in fp32)
//   S  = Qlo Khi^T + Qhi Klo^T + Qhi Khi^T
//   O += Plo Vhi   + Phi Vlo   + Phi Vhi
// (small terms first; lo*lo is below fp32 rounding), accumulated in fp32 in
// TMEM.  The row softmax runs in fp32 with the same
// global-position causal rule and 1/sqrt(D) scale as the bf16 kernel, and P is
// split hi/lo the same way before the PV product.
//
// CTA = one 128-row query tile of one head, 4 warps (thread t <-> TMEM lane t
// <-> query row t).  Per 64-key (D = 64) / 32-key (D = 128) tile: all threads
// load K and V from global memory (coalesced 16-byte loads), split them and
// store hi / lo into shared memory in the 128-byte-swizzled K-major layout the
// tcgen05 descriptors read (V transposed, so both operands are K-major); one
// thread issues the three QK^T products; the softmax threads read S from TMEM,
// rescale O when the running max grows, write P hi / lo to shared memory; one
// thread issues the three PV products.  The steps are not overlapped: C1 is
// 512 x 512 x 4 heads (latency-bound), and the kernel exists for exactness on
// the tensor cores, not for the bf16 path's throughput.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "kernels.h"
#include "ptx_sm100.cuh"

// TF32_WAIT: the kernel's mbarrier wait (tools/tf32_kernel_probe.cu
// redefines it as a bounded wait that reports where a CTA stalls).
#ifndef TF32_WAIT
#define TF32_WAIT(bar, phase, tag) ptx::mbar_wait(bar, phase)
#endif

namespace dmha {
namespace {

constexpr int kBM = 128;

template <int D>
struct Tf32Cfg {
  static constexpr int kBN = D == 64 ? 64 : 32;      // keys per tile
  static constexpr int kQBytes = kBM * D * 4;         // one of Q hi / lo
  static constexpr int kKBytes = kBN * D * 4;         // one of K hi / lo
  static constexpr int kVBytes = D * kBN * 4;         // one of V^T hi / lo
  static constexpr int kPBytes = kBM * kBN * 4;       // one of P hi / lo
  static constexpr int kQh = 0, kQl = kQh + kQBytes;
  static constexpr int kKh = kQl + kQBytes, kKl = kKh + kKBytes;
  static constexpr int kVh = kKl + kKBytes, kVl = kVh + kVBytes;
  static constexpr int kPh = kVl + kVBytes, kPl = kPh + kPBytes;
  static constexpr int kBar = kPl + kPBytes;
  static constexpr int kSmem = kBar + 64 + 1024;
  static constexpr uint32_t kIdescS = ptx::make_idesc(2, kBM, kBN, 0, 0);  // tf32, K-major
  static constexpr uint32_t kIdescO = ptx::make_idesc(2, kBM, D, 0, 0);
  static constexpr int kTmemS = 0, kTmemO = 128;  // S: kBN columns, O: D columns
  static_assert(kSmem <= 232448, "shared memory budget");
};

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Byte offset of 16-byte chunk c (4 fp32 along K) of row `row` in a K-major
// operand of `rows` rows, 128-byte swizzle: 32 fp32 of K per 128-byte panel
// row, panels of rows x 128 B, chunk index XOR (row % 8).
__device__ __forceinline__ uint32_t sw_off(int rows, int row, int c) {
  return static_cast<uint32_t>((c >> 3) * rows * 128 + row * 128 + (((c & 7) ^ (row & 7)) << 4));
}

__device__ __forceinline__ void split4(float4 x, float4& hi, float4& lo) {
  hi = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
  lo = make_float4(x.x - hi.x, x.y - hi.y, x.z - hi.z, x.w - hi.w);
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

// D[tmem] (+)= A * B^T over K = kdim (K-major tf32 operands of ra / rb rows)
__device__ __forceinline__ void mma_tf32_kloop(uint32_t d, uint32_t a, int ra, uint32_t b, int rb,
                                               int kdim, uint32_t idesc, bool acc) {
  for (int kk = 0; kk < kdim / 8; ++kk) {
    const uint32_t off_a = (kk >> 2) * ra * 128 + (kk & 3) * 32;
    const uint32_t off_b = (kk >> 2) * rb * 128 + (kk & 3) * 32;
    ptx::mma_tf32_ss(d, ptx::smem_desc_sw128(a + off_a, 16, 1024),
                     ptx::smem_desc_sw128(b + off_b, 16, 1024), idesc, (acc || kk > 0) ? 1u : 0u);
  }
}

template <int D>
__global__ void __launch_bounds__(128, 1)
    attn_fwd_tf32x3_kernel(const float* __restrict__ q, const float* __restrict__ k,
                           const float* __restrict__ v, float* __restrict__ out,
                           float* __restrict__ lse, int64_t Lq, int64_t Lk, int H, int causal,
                           PosMap qmap, PosMap kmap, float scale_log2) {
  using C = Tf32Cfg<D>;
  constexpr int kBN = C::kBN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::kBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x;
  const int head = blockIdx.y;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * kBM;

  if (tid == 0) {
    ptx::mbar_init(bar, 1);
    ptx::fence_mbar_init();
  }
  if (tid < 32) ptx::tmem_alloc<256>(tmem_slot);
  // Q tile -> hi / lo (rows past Lq are zero)
  for (int i = tid; i < kBM * (D / 4); i += 128) {
    const int r = i / (D / 4), c = i % (D / 4);
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (m0 + r < Lq) x = reinterpret_cast<const float4*>(q + ((m0 + r) * H + head) * D)[c];
    float4 hi, lo;
    split4(x, hi, lo);
    *reinterpret_cast<float4*>(sm + C::kQh + sw_off(kBM, r, c)) = hi;
    *reinterpret_cast<float4*>(sm + C::kQl + sw_off(kBM, r, c)) = lo;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = ptx::smem_u32(sm);

  const int64_t row = m0 + tid;
  const bool row_ok = row < Lq;
  const int64_t qp = pos_tf(qmap, row_ok ? row : Lq - 1);
  const int64_t klim = klimit_tf(causal, kmap, Lk, qp);
  // tiles this CTA visits: the prefix its last row may use
  const int64_t last = (m0 + kBM - 1 < Lq - 1) ? m0 + kBM - 1 : Lq - 1;
  const int64_t kmax = klimit_tf(causal, kmap, Lk, pos_tf(qmap, last));
  const int ntiles = static_cast<int>((kmax + kBN - 1) / kBN);
  const uint32_t lane_addr = static_cast<uint32_t>((tid & ~31) << 16);
  const uint32_t tS = tmem + lane_addr + C::kTmemS;
  const uint32_t tO = tmem + lane_addr + C::kTmemO;

  float m_run = -INFINITY, l_run = 0.f;
  uint32_t phase = 0;
  for (int jt = 0; jt < ntiles; ++jt) {
    const int64_t j0 = static_cast<int64_t>(jt) * kBN;
    // K_j, V_j -> hi / lo (keys past Lk are zero; they are masked below)
    for (int i = tid; i < kBN * (D / 4); i += 128) {
      const int r = i / (D / 4), c = i % (D / 4);
      float4 kx = make_float4(0.f, 0.f, 0.f, 0.f), vx = kx;
      if (j0 + r < Lk) {
        kx = reinterpret_cast<const float4*>(k + ((j0 + r) * H + head) * D)[c];
        vx = reinterpret_cast<const float4*>(v + ((j0 + r) * H + head) * D)[c];
      }
      float4 hi, lo;
      split4(kx, hi, lo);
      *reinterpret_cast<float4*>(sm + C::kKh + sw_off(kBN, r, c)) = hi;
      *reinterpret_cast<float4*>(sm + C::kKl + sw_off(kBN, r, c)) = lo;
      // V^T: row d, K index = key r (element (d, r) of a D-row operand)
      split4(vx, hi, lo);
      const float hs[4] = {hi.x, hi.y, hi.z, hi.w}, ls[4] = {lo.x, lo.y, lo.z, lo.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int d = 4 * c + e;
        const uint32_t o = sw_off(D, d, r >> 2) + (r & 3) * 4;
        *reinterpret_cast<float*>(sm + C::kVh + o) = hs[e];
        *reinterpret_cast<float*>(sm + C::kVl + o) = ls[e];
      }
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    // one thread issues; the rest of its warp waits at __syncwarp (not in the
    // mbarrier spin below, which could starve the issuing lane)
    if (tid < 32) {
      if (tid == 0) {
        ptx::tc_fence_after();
        const uint32_t d = tmem + C::kTmemS;
        mma_tf32_kloop(d, sbase + C::kQl, kBM, sbase + C::kKh, kBN, D, C::kIdescS, false);
        mma_tf32_kloop(d, sbase + C::kQh, kBM, sbase + C::kKl, kBN, D, C::kIdescS, true);
        mma_tf32_kloop(d, sbase + C::kQh, kBM, sbase + C::kKh, kBN, D, C::kIdescS, true);
        ptx::mma_commit(bar);
      }
      __syncwarp();
    }
    TF32_WAIT(bar, phase, 1000 + jt);
    phase ^= 1;
    ptx::tc_fence_after();
    // ---- online softmax of this row (fp32, exp2 domain)
    float s[kBN];
#pragma unroll
    for (int c = 0; c < kBN / 32; ++c)
      ptx::tmem_ld32(tS + c * 32, *reinterpret_cast<float(*)[32]>(&s[32 * c]));
    ptx::tmem_wait_ld();
    const int64_t nv = klim - j0;
    float mx = -INFINITY;
#pragma unroll
    for (int c = 0; c < kBN; ++c) {
      s[c] = (c < nv) ? s[c] * scale_log2 : -INFINITY;
      mx = fmaxf(mx, s[c]);
    }
    const float m_new = fmaxf(m_run, mx);
    const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
    const float alpha = (m_run == -INFINITY) ? 0.f : exp2f(m_run - m_use);
    float sum = 0.f;
#pragma unroll
    for (int c = 0; c < kBN; c += 4) {
      float4 pv, hi, lo;
      pv.x = exp2f(s[c] - m_use);
      pv.y = exp2f(s[c + 1] - m_use);
      pv.z = exp2f(s[c + 2] - m_use);
      pv.w = exp2f(s[c + 3] - m_use);
      sum += (pv.x + pv.y) + (pv.z + pv.w);
      split4(pv, hi, lo);
      *reinterpret_cast<float4*>(sm + C::kPh + sw_off(kBM, tid, c >> 2)) = hi;
      *reinterpret_cast<float4*>(sm + C::kPl + sw_off(kBM, tid, c >> 2)) = lo;
    }
    l_run = l_run * alpha + sum;
    // O (complete: the previous PV was waited for) *= alpha.  tcgen05.ld/st are
    // warp-collective (.sync.aligned): the whole warp takes the branch when any
    // of its rows needs it (alpha = 1 for the others).
    if (__any_sync(0xffffffffu, jt > 0 && m_new > m_run)) {
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        float o[32];
        ptx::tmem_ld32(tO + c * 32, o);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] *= alpha;
        ptx::tmem_st32(tO + c * 32, o);
      }
      ptx::tmem_wait_st();
    }
    m_run = m_new;
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    if (tid < 32) {
      if (tid == 0) {
        ptx::tc_fence_after();
        const uint32_t d = tmem + C::kTmemO;
        mma_tf32_kloop(d, sbase + C::kPl, kBM, sbase + C::kVh, D, kBN, C::kIdescO, jt > 0);
        mma_tf32_kloop(d, sbase + C::kPh, kBM, sbase + C::kVl, D, kBN, C::kIdescO, true);
        mma_tf32_kloop(d, sbase + C::kPh, kBM, sbase + C::kVh, D, kBN, C::kIdescO, true);
        ptx::mma_commit(bar);
      }
      __syncwarp();
    }
    TF32_WAIT(bar, phase, 2000 + jt);  // PV done: K/V/P buffers free, O complete
    phase ^= 1;
    ptx::tc_fence_after();
  }
  // ---- epilogue: O / l, lse = ln l + m (natural log of the scaled scores)
  const bool empty = !(l_run > 0.f);
  const float inv = empty ? 0.f : 1.f / l_run;
#pragma unroll
  for (int c = 0; c < D / 32; ++c) {
    float o[32];
    if (ntiles > 0) {
      ptx::tmem_ld32(tO + c * 32, o);
      ptx::tmem_wait_ld();
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e) o[e] = 0.f;
    }
    if (row_ok) {
      float4* dst = reinterpret_cast<float4*>(out + (row * H + head) * D + c * 32);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        dst[e] = make_float4(o[4 * e] * inv, o[4 * e + 1] * inv, o[4 * e + 2] * inv,
                             o[4 * e + 3] * inv);
    }
  }
  if (row_ok)
    lse[static_cast<int64_t>(head) * Lq + row] =
        empty ? -INFINITY : (m_run + log2f(l_run)) * 0.69314718055994530942f;
  ptx::tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<256>(tmem);
  }
}

template <int D>
cudaError_t launch_tf32(const LocalAttnArgs& a, cudaStream_t stream) {
  using C = Tf32Cfg<D>;
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
  attn_fwd_tf32x3_kernel<D><<<grid, 128, C::kSmem, stream>>>(
      static_cast<const float*>(a.q), static_cast<const float*>(a.k),
      static_cast<const float*>(a.v), static_cast<float*>(a.out), a.lse, a.Lq, a.Lk, a.H, a.causal,
      a.qmap, a.kmap, static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(D))));
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_fwd_tf32x3(const LocalAttnArgs& a, cudaStream_t stream) {
  if (a.Lq <= 0) return cudaSuccess;
  if (a.out_mode != OUT_FINAL && a.out_mode != OUT_PARTIAL_F32) return cudaErrorInvalidValue;
  if (a.D == 64) return launch_tf32<64>(a, stream);
  if (a.D == 128) return launch_tf32<128>(a, stream);
  return cudaErrorInvalidValue;
}

}  // namespace dmha
