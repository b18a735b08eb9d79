// attn_fwd_sm100_v2.cu — "dbuf" flash-attention forward for sm_100a: two
// 128-row query tiles per CTA (like the ping-pong kernel, so one K/V tile
// feeds 256 query rows), 64-key K/V tiles, and a DOUBLE-BUFFERED score tile
// per query tile, so QK^T of tile j+1 runs on the tensor core while the
// softmax works on tile j.  This removes the serial chain of the ping-pong
// kernel (softmax(j) -> PV(j) -> QK^T(j+1) -> softmax(j+1), DESIGN.md lesson
// 7) at the price of N = 64 QK^T MMAs (48.8 instead of 32 cycles per
// 128x64x16 step: shared-memory operand bound, lesson 8).
//
// Computes, for one query block against one key/value block (one ring step,
// SURVEY §8(a) a2), per head h and query row i:
//   S = Q K^T / sqrt(D)                      PAPER.md:193-196 Eq. `unnormalized`
//   A = row softmax(S) over the usable keys
//   Z = A V                                  PAPER.md:203-211 Eq. `attn-sum`
//   lse = ln sum_j exp(S_j)                  (reading R9)
// with the causal rule "key j usable by row i iff kpos(j) <= qpos(i)" on
// GLOBAL positions, and the same output modes as the ping-pong kernel
// (final / fp32 partial / NEXT-2 fused combine).
//
// CTA = 2 query tiles (256 rows) of one head; 12 warps:
//   warps 0-3 / 4-7  softmax for Q tile 0 / 1 (thread <-> TMEM lane <-> row)
//   warp  8          TMA producer (Q once; K_j, V_j through a 10-slot ring)
//   warp  9          TMEM allocator + QK^T issuer (both Q tiles)
//   warp 10          PV issuer (both Q tiles)
//   warp 11          idle
// TMEM (512 cols): per Q tile g: S_g[0] [256g, 256g+64), S_g[1] [256g+64,
// 256g+128), O_g [256g+128, 256g+128+D).  P_g(j) (bf16x2, 32 cols) is written
// over the first half of S_g[j%2] after the softmax has loaded S_g(j).
// Buffer reuse: S_g(j) overwrites P_g(j-2), so the QK^T issuer waits for
// PV_g(j-2) to COMPLETE (pv_done[g][j%2]) — the two issuers are different
// threads, so only completion orders them.  (One issuer per Q tile, issuing
// PV_g(j) then S_g(j+2) in program order, measured slower: 1012 vs 1083 TF/s
// at C4.)  Every per-tile barrier is kept per buffer (index j%2, parity
// (j>>1)&1) so no waiter can fall two phases behind.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "combine_math.cuh"
#include "kernels.h"
#include "tma_map.h"
#include "ptx_sm100.cuh"

namespace dmha {
extern unsigned long long* g_trace;
namespace {

constexpr int kBM = 128;   // query rows per tile (MMA M)
constexpr int kBN = 64;    // keys per K/V tile (QK^T N, PV K)
constexpr int kThreads = 384;
constexpr int kProducerWarp = 8;
constexpr int kSWarp = 9;
constexpr int kPVWarp = 10;
constexpr float kRescaleThreshold = 8.0f;  // log2 units (factor 256), as in v1

template <int D>
struct Cfg {
  static constexpr int kPanels = D / 64;                    // 128-byte swizzle panels per row
  static constexpr int kQPanelBytes = kBM * 128;            // 128 rows x 128 B
  static constexpr int kQTileBytes = kPanels * kQPanelBytes;
  static constexpr int kKVPanelBytes = kBN * 128;           // 64 rows x 128 B
  static constexpr int kKVTileBytes = kPanels * kKVPanelBytes;
  static constexpr int kStages = D == 128 ? 10 : 18;        // K/V ring slots (even: K/V keep parity)
  static constexpr int kQOff = 0;
  static constexpr int kKVOff = 2 * kQTileBytes;
  static constexpr int kBarOff = kKVOff + kStages * kKVTileBytes;
  static constexpr int kSmemBytes = kBarOff + 512 + 1024;   // barriers + align slack
  static constexpr uint32_t kIdescQK = ptx::make_idesc(1, kBM, kBN, 0, 0);
  static constexpr uint32_t kIdescPV = ptx::make_idesc(1, kBM, D, 0, 1);  // V is MN-major
  static_assert(kStages % 2 == 0, "K and V must keep their slot parity");
};

struct Params {
  int64_t Lq, Lk;
  int H;
  int causal;
  PosMap qmap, kmap;
  float scale_log2;  // log2(e) / sqrt(D)
  void* out;
  float* lse;
  int out_mode;
  float* acc_o;
  float* acc_lse;
  int n_mblk;
  unsigned long long* trace;  // debug timeline (dmha_debug_set_trace), usually null
};

// Timeline stamps, [cta < 2][event < 9][tile < 64], head 0:
//  0/2 softmax Q tile 0/1 saw S(j)   1/3 Q tile 0/1 arrived P(j)
//  4 QK^T issuer issued S0(j), S1(j)   5/6 PV issuer saw P0(j) / P1(j)
//  7 softmax 0 loaded S(j)   8 softmax 0 starts the exponentials of tile j
__device__ __forceinline__ void trace_stamp(const Params& p, int ev, int j) {
  if (p.trace != nullptr && blockIdx.y == 0 && blockIdx.x < 2 && j < 64)
    p.trace[(blockIdx.x * 9 + ev) * 64 + j] = clock64();
}

__device__ __forceinline__ int64_t pos_of(const PosMap& m, int64_t i) {
  return i < m.chunk ? m.base0 + i : m.base1 + (i - m.chunk);
}

// Number of leading keys (a prefix: kpos is increasing) usable at position qp.
__device__ __forceinline__ int64_t key_limit(const Params& p, int64_t qp) {
  if (!p.causal) return p.Lk;
  const PosMap& m = p.kmap;
  int64_t lim;
  if (p.Lk > m.chunk && qp >= m.base1) {
    lim = m.chunk + (qp - m.base1) + 1;
  } else if (qp >= m.base0) {
    lim = qp - m.base0 + 1;
    if (lim > m.chunk) lim = m.chunk;
  } else {
    lim = 0;
  }
  return lim < p.Lk ? lim : p.Lk;
}

__device__ __forceinline__ int num_kv_tiles(const Params& p, int64_t m0) {
  int64_t last = m0 + 2 * kBM - 1;
  if (last > p.Lq - 1) last = p.Lq - 1;
  const int64_t lim = key_limit(p, pos_of(p.qmap, last));
  return static_cast<int>((lim + kBN - 1) / kBN);
}

// Softmax warpgroup alternation (kAlt): WG g runs its exponentials only after
// the other WG finished its own (named barriers 1 / 2, 256 threads), so one
// WG's load / max / store overlaps the other's MUFU phase.
__device__ __forceinline__ void nbar_sync(int id) {
  asm volatile("bar.sync %0, 256;" ::"r"(id) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id) {
  asm volatile("bar.arrive %0, 256;" ::"r"(id) : "memory");
}

template <int D, bool kAlt>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_dbuf_kernel(const __grid_constant__ CUtensorMap tm_q,
                         const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const Params p) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem + C::kQOff;
  uint8_t* sKV = smem + C::kKVOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_full = bars;                       // [1]
  uint64_t* kv_full = q_full + 1;                // [kStages]
  uint64_t* kv_empty = kv_full + C::kStages;     // [kStages]
  uint64_t* s_full = kv_empty + C::kStages;      // [2 g][2 buf]
  uint64_t* p_ready = s_full + 4;                // [2 g][2 buf]
  uint64_t* pv_done = p_ready + 4;               // [2 g][2 buf]
  uint64_t* o_final = pv_done + 4;               // [2 g]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_final + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  const int mblk = p.causal ? (p.n_mblk - 1 - static_cast<int>(blockIdx.x))
                            : static_cast<int>(blockIdx.x);  // causal: heaviest first
  const int64_t m0 = static_cast<int64_t>(mblk) * (2 * kBM);
  const int nkv = num_kv_tiles(p, m0);

  if (warp == kProducerWarp && lane == 0) {
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);  // K slots: QK^T issuer; V slots: PV issuer
    }
    for (int i = 0; i < 4; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&p_ready[i], kBM);
      ptx::mbar_init(&pv_done[i], 1);
    }
    ptx::mbar_init(&o_final[0], 1);
    ptx::mbar_init(&o_final[1], 1);
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == kSWarp) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto slot_of = [](int item) { return item % C::kStages; };
  auto par_of = [](int item) { return static_cast<uint32_t>((item / C::kStages) & 1); };

  if (warp == kProducerWarp) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && nkv > 0) {
      ptx::mbar_arrive_expect_tx(q_full, 2 * C::kQTileBytes);
      for (int g = 0; g < 2; ++g)
        for (int pn = 0; pn < C::kPanels; ++pn)
          ptx::tma_load_3d(&tm_q, q_full, sQ + g * C::kQTileBytes + pn * C::kQPanelBytes, pn * 64,
                           head, static_cast<int32_t>(m0 + g * kBM));
      for (int item = 0; item < 2 * nkv; ++item) {  // K_j = item 2j, V_j = item 2j+1
        const int s = slot_of(item);
        ptx::mbar_wait(&kv_empty[s], par_of(item) ^ 1);
        ptx::mbar_arrive_expect_tx(&kv_full[s], C::kKVTileBytes);
        const CUtensorMap* tm = (item & 1) ? &tm_v : &tm_k;
        for (int pn = 0; pn < C::kPanels; ++pn)
          ptx::tma_load_3d(tm, &kv_full[s], sKV + s * C::kKVTileBytes + pn * C::kKVPanelBytes,
                           pn * 64, head, (item >> 1) * kBN);
      }
    }
  } else if (warp == kSWarp) {
    // ------------------------------------------------------------ QK^T issuer
    if (lane == 0 && nkv > 0) {
      const uint32_t sq = ptx::smem_u32(sQ);
      const uint32_t skv = ptx::smem_u32(sKV);
      ptx::mbar_wait(q_full, 0);
      for (int j = 0; j < nkv; ++j) {
        const int ik = 2 * j, b = j & 1;
        ptx::mbar_wait(&kv_full[slot_of(ik)], par_of(ik));
        for (int g = 0; g < 2; ++g) {
          // S_g(j) overwrites P_g(j-2): PV_g(j-2) (issued by the other warp)
          // must be COMPLETE.  PV_g(j) (same barrier, next phase) needs S_g(j),
          // so this waiter is never two phases behind.
          if (j >= 2)
            ptx::mbar_wait(&pv_done[2 * g + b], static_cast<uint32_t>(((j - 2) >> 1) & 1));
          ptx::tc_fence_after();
          const uint32_t a0 = sq + g * C::kQTileBytes;
          const uint32_t b0 = skv + slot_of(ik) * C::kKVTileBytes;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            ptx::mma_bf16_ss(
                tmem + 256 * g + 64 * b,
                ptx::smem_desc_sw128(a0 + (kk >> 2) * C::kQPanelBytes + (kk & 3) * 32, 16, 1024),
                ptx::smem_desc_sw128(b0 + (kk >> 2) * C::kKVPanelBytes + (kk & 3) * 32, 16, 1024),
                C::kIdescQK, kk > 0);
          }
          ptx::mma_commit(&s_full[2 * g + b]);
        }
        trace_stamp(p, 4, j);
        ptx::mma_commit(&kv_empty[slot_of(ik)]);
      }
    }
  } else if (warp == kPVWarp) {
    // ------------------------------------------------------------ PV issuer
    if (lane == 0 && nkv > 0) {
      const uint32_t skv = ptx::smem_u32(sKV);
      for (int j = 0; j < nkv; ++j) {
        const int iv = 2 * j + 1, b = j & 1;
        ptx::mbar_wait(&kv_full[slot_of(iv)], par_of(iv));
        for (int g = 0; g < 2; ++g) {
          // p_ready[g][b] phase j>>1: the softmax cannot arrive for j+2 before
          // PV_g(j) completed (S_g(j+2) waits for it), so no 2-phase lag.
          ptx::mbar_wait(&p_ready[2 * g + b], static_cast<uint32_t>((j >> 1) & 1));
          trace_stamp(p, 5 + g, j);
          ptx::tc_fence_after();
          const uint32_t b0 = skv + slot_of(iv) * C::kKVTileBytes;
#pragma unroll
          for (int kk = 0; kk < kBN / 16; ++kk) {
            ptx::mma_bf16_ts(tmem + 256 * g + 128, tmem + 256 * g + 64 * b + kk * 8,
                             ptx::smem_desc_sw128(b0 + kk * 16 * 128, C::kKVPanelBytes, 1024),
                             C::kIdescPV, (j > 0 || kk > 0) ? 1u : 0u);
          }
          ptx::mma_commit(&pv_done[2 * g + b]);
          if (j == nkv - 1) ptx::mma_commit(&o_final[g]);
        }
        ptx::mma_commit(&kv_empty[slot_of(iv)]);
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------ softmax
    const int g = warp >> 2;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int64_t row = m0 + g * kBM + r;
    const bool row_ok = row < p.Lq;
    const int64_t qp = pos_of(p.qmap, row_ok ? row : p.Lq - 1);
    const int64_t klim = key_limit(p, qp);
    const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tO = tmem + lane_addr + 256 * g + 128;
    const float sl2 = p.scale_log2;
    float m_run = -INFINITY;
    float l_run = 0.f;
    if (kAlt && g == 1 && nkv > 0) nbar_arrive(1);  // WG0 takes the first turn
    for (int j = 0; j < nkv; ++j) {
      const int b = j & 1;
      const uint32_t tS = tmem + lane_addr + 256 * g + 64 * b;
      // s_full[g][b] phase j>>1: S_g(j+2) needs PV_g(j), which needs this
      // softmax's P_g(j), so the barrier cannot run two phases ahead.
      ptx::mbar_wait(&s_full[2 * g + b], static_cast<uint32_t>((j >> 1) & 1));
      if (threadIdx.x % 128 == 0) trace_stamp(p, 2 * g, j);
      ptx::tc_fence_after();
      float s[64];
      ptx::tmem_ld32(tS, *reinterpret_cast<float(*)[32]>(&s[0]));
      ptx::tmem_ld32(tS + 32, *reinterpret_cast<float(*)[32]>(&s[32]));
      ptx::tmem_wait_ld();
      if (g == 0 && threadIdx.x == 0) trace_stamp(p, 7, j);

      const int64_t nv64 = klim - static_cast<int64_t>(j) * kBN;
      const int nvalid = nv64 < 0 ? 0 : (nv64 > kBN ? kBN : static_cast<int>(nv64));
      const bool masked = !__all_sync(0xffffffffu, nvalid >= kBN);
      if (masked) {
#pragma unroll
        for (int c = 0; c < 64; ++c) s[c] = c < nvalid ? s[c] : -INFINITY;
      }
      float mx[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx[i] = fmaxf(fmaxf(s[i], s[8 + i]), s[16 + i]);
#pragma unroll
      for (int i = 0; i < 8; ++i) mx[i] = fmaxf(fmaxf(mx[i], s[24 + i]), s[32 + i]);
#pragma unroll
      for (int i = 0; i < 8; ++i) mx[i] = fmaxf(fmaxf(mx[i], s[40 + i]), s[48 + i]);
#pragma unroll
      for (int i = 0; i < 8; ++i) mx[i] = fmaxf(mx[i], s[56 + i]);
      const float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                             fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))) * sl2;
      const bool need = mt > m_run + kRescaleThreshold;
      const bool warp_rescale = __any_sync(0xffffffffu, need);
      float alpha = 1.f;
      if (warp_rescale) {
        const float m_new = fmaxf(m_run, mt);
        alpha = (m_new == -INFINITY) ? 1.f : ptx::ex2_approx(m_run - m_new);
        l_run *= alpha;
        m_run = m_new;
      }
      const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
      if (kAlt) nbar_sync(1 + g);  // my turn on MUFU
      if (g == 0 && threadIdx.x == 0) trace_stamp(p, 8, j);
      // P = exp2(S*scale*log2e - m) -> bf16 over the first 32 columns of S_g[b]
      float sum0 = 0.f, sum1 = 0.f;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float e0 = ptx::ex2_approx(fmaf(s[32 * c + 2 * e], sl2, -m_use));
          const float e1 = ptx::ex2_approx(fmaf(s[32 * c + 2 * e + 1], sl2, -m_use));
          sum0 += e0;
          sum1 += e1;
          __nv_bfloat162 hb = __floats2bfloat162_rn(e0, e1);
          pk[e] = *reinterpret_cast<uint32_t*>(&hb);
        }
        ptx::tmem_st16(tS + c * 16, pk);
      }
      l_run += sum0 + sum1;
      if (kAlt) nbar_arrive(2 - g);  // the other WG's turn
      // Rescale O in place: it must hold PV_g(j-1) completely (PV_g(j) is not
      // issued before this tile's p_ready).  pv_done[g][(j-1)&1] phase
      // (j-1)>>1 cannot be two phases ahead: PV_g(j+1) needs P_g(j+1).
      if (warp_rescale && j > 0) {
        ptx::mbar_wait(&pv_done[2 * g + ((j - 1) & 1)], static_cast<uint32_t>(((j - 1) >> 1) & 1));
        ptx::tc_fence_after();
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          float o[32];
          ptx::tmem_ld32(tO + c * 32, o);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] *= alpha;
          ptx::tmem_st32(tO + c * 32, o);
        }
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      if (threadIdx.x % 128 == 0) trace_stamp(p, 2 * g + 1, j);
      ptx::mbar_arrive(&p_ready[2 * g + b]);
    }
    if (kAlt && g == 0 && nkv > 0) nbar_sync(1);  // consume WG1's last hand-over
    if (nkv > 0) {
      ptx::mbar_wait(&o_final[g], 0);
      ptx::tc_fence_after();
    }
    // ---------------------------------------------------------- epilogue
    const bool empty = !(l_run > 0.f);
    const float inv_l = empty ? 0.f : 1.f / l_run;
    const float lse_s = empty ? -INFINITY : (m_run + __log2f(l_run)) * 0.69314718055994530942f;
    const int64_t li = static_cast<int64_t>(head) * p.Lq + row;
    const bool fused = p.out_mode >= OUT_COMBINE_ACC;
    float wa = 0.f, wp = 0.f, lnew = lse_s;
    if (fused && row_ok) merge_weights(p.acc_lse[li], lse_s, wa, wp, lnew);
    if (row_ok) {
      if (p.out_mode == OUT_COMBINE_ACC) p.acc_lse[li] = lnew;
      else p.lse[li] = lnew;
    }
    const int64_t obase = (row * p.H + head) * static_cast<int64_t>(D);
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      float o[32];
      if (nkv > 0) {
        ptx::tmem_ld32(tO + c * 32, o);
        ptx::tmem_wait_ld();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = 0.f;
      }
      if (!row_ok) continue;
      float rr[32];
      if (fused) {
        const float4* acc = reinterpret_cast<const float4*>(p.acc_o + obase + c * 32);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float4 a4 = acc[e];
          rr[4 * e + 0] = combine_one(a4.x, __fmul_rn(o[4 * e + 0], inv_l), wa, wp);
          rr[4 * e + 1] = combine_one(a4.y, __fmul_rn(o[4 * e + 1], inv_l), wa, wp);
          rr[4 * e + 2] = combine_one(a4.z, __fmul_rn(o[4 * e + 2], inv_l), wa, wp);
          rr[4 * e + 3] = combine_one(a4.w, __fmul_rn(o[4 * e + 3], inv_l), wa, wp);
        }
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) rr[e] = __fmul_rn(o[e], inv_l);
      }
      if (p.out_mode == OUT_PARTIAL_F32 || p.out_mode == OUT_COMBINE_ACC) {
        float4* dst = reinterpret_cast<float4*>(
            (p.out_mode == OUT_COMBINE_ACC ? p.acc_o : reinterpret_cast<float*>(p.out)) + obase +
            c * 32);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          dst[e] = make_float4(rr[4 * e], rr[4 * e + 1], rr[4 * e + 2], rr[4 * e + 3]);
      } else {
        uint4* dst =
            reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.out) + obase + c * 32);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          uint32_t w[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            __nv_bfloat162 hb = __floats2bfloat162_rn(rr[8 * e + 2 * t], rr[8 * e + 2 * t + 1]);
            w[t] = *reinterpret_cast<uint32_t*>(&hb);
          }
          dst[e] = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kSWarp) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------- host side
template <int D, bool kAlt>
cudaError_t launch_d(const LocalAttnArgs& a, cudaStream_t stream) {
  using C = Cfg<D>;
  CUtensorMap tq, tk, tv;
  if (!make_tma_map_bf16(&tq, a.q, a.Lq, a.H, D, kBM) || !make_tma_map_bf16(&tk, a.k, a.Lk, a.H, D, kBN) ||
      !make_tma_map_bf16(&tv, a.v, a.Lk, a.H, D, kBN))
    return cudaErrorInvalidValue;
  // the dynamic shared-memory limit is a per-device function attribute
  static int attr_dev = -1;
  int cur_dev = 0;
  cudaGetDevice(&cur_dev);
  if (attr_dev != cur_dev) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_dbuf_kernel<D, kAlt>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_dev = cur_dev;
  }
  Params p;
  p.Lq = a.Lq;
  p.Lk = a.Lk;
  p.H = a.H;
  p.causal = a.causal;
  p.qmap = a.qmap;
  p.kmap = a.kmap;
  p.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(D)));
  p.out = a.out;
  p.lse = a.lse;
  p.out_mode = a.out_mode;
  p.acc_o = a.acc_o;
  p.acc_lse = a.acc_lse;
  p.n_mblk = static_cast<int>((a.Lq + 2 * kBM - 1) / (2 * kBM));
  p.trace = g_trace;
  dim3 grid(p.n_mblk, a.H);
  attn_fwd_dbuf_kernel<D, kAlt><<<grid, kThreads, C::kSmemBytes, stream>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_fwd_bf16_dbuf(const LocalAttnArgs& a, cudaStream_t stream) {
  if (a.Lq <= 0) return cudaSuccess;
  if (a.Lq > INT32_MAX || a.Lk > INT32_MAX) return cudaErrorInvalidValue;
  // DMHA_DBUF_ALT=1: alternate the two softmax warpgroups' exponential phases
  const char* e = std::getenv("DMHA_DBUF_ALT");
  const bool alt = e && std::atoi(e) != 0;
  if (a.D == 64) return alt ? launch_d<64, true>(a, stream) : launch_d<64, false>(a, stream);
  if (a.D == 128) return alt ? launch_d<128, true>(a, stream) : launch_d<128, false>(a, stream);
  return cudaErrorInvalidValue;
}

}  // namespace dmha
