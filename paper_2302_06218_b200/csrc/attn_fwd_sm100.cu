// attn_fwd_sm100.cu — fused flash-attention forward for sm_100a (B200).
//
// Computes, for one query block against one key/value block (one ring step,
// SURVEY §8(a) a2), per head h and query row i:
//   S = Q K^T / sqrt(D)                      PAPER.md:193-196 Eq. `unnormalized`
//   A = row softmax(S) over the usable keys
//   Z = A V                                  PAPER.md:203-211 Eq. `attn-sum`
//   lse = ln sum_j exp(S_j)                  (reading R9)
// with the causal rule "key j usable by row i iff kpos(j) <= qpos(i)" on
// GLOBAL positions (north_star), so the same kernel serves every ring step and
// both shard layouts.  S, P and O never leave the SM: S and O accumulate in
// TMEM, P is written back to TMEM as bf16 and consumed from there.
//
// CTA = 2 query tiles of 128 rows (256 rows) of one head; 20 warps:
//   warps 0-15  softmax: warpgroup w = warp/4 handles Q tile g = w/2 and score
//               columns [64h, 64h+64) with h = w%2 (two warpgroups share each
//               row: thread t <-> TMEM lane t <-> row t; the row max is
//               exchanged through shared memory once per KV tile)
//   warp  16    TMA producer (Q once; K_j, V_j through an NST-slot ring)
//   warp  17    TMEM allocator + single-thread tcgen05.mma issuer
//   warps 18-19 idle (keep the CTA at whole warpgroups for setmaxnreg)
// Splitting each row over two warpgroups halves the softmax latency, which is
// the serial part of every tile: S_g(j+1) cannot start before PV_g(j) has read
// P_g(j) (they share TMEM columns), so per Q tile the loop is
// softmax -> PV + QK^T -> softmax, and the two Q tiles ping-pong on the tensor
// core.  (Timeline measured with dmha_debug_set_trace.)
// TMEM (512 cols): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [384,384+D);
// P_g (bf16x2) aliases the first 64 columns of S_g (half h writes [32h,32h+32)).
// MMA order per KV tile j:  PV0_{j-1}, S0_j, PV1_{j-1}, S1_j — S_g(j) is issued
// after PV_g(j-1) read P_g(j-1) (tcgen05.mma executes in issue order), and the
// commit that signals S_g(j) also covers PV_g(j-1), so the softmax warps can
// rescale O_g right after they see S_g(j) (warpgroup h = 0 does it).
// Online softmax in the exp2 domain with a stale running max: O is rescaled
// only when the tile max exceeds the running max by more than 8 (factor 256);
// exact because l and O always share the max that was subtracted.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "kernels.h"
#include "ptx_sm100.cuh"

namespace dmha {
extern unsigned long long* g_trace;
namespace {

constexpr int kBM = 128;          // query rows per tile (MMA M)
constexpr int kBN = 128;          // keys per tile (MMA N of QK^T, K of PV)
constexpr int kSoftmaxWarps = 16;
constexpr int kThreads = 640;     // 20 warps
constexpr int kProducerWarp = 16;
constexpr int kMmaWarp = 17;
constexpr float kRescaleThreshold = 8.0f;  // log2 units: rescale when max grows by > 2^8
// Register split (65536 per SM, 1 CTA/SM, 96 per thread at launch): the control
// warpgroup (TMA, MMA, 2 idle warps) gives registers to the four softmax
// warpgroups: 4*104 + 56 <= 512.
constexpr uint32_t kRegsCtl = 56;
constexpr uint32_t kRegsSoftmax = 104;

template <int D>
struct Cfg {
  static constexpr int kPanels = D / 64;                    // 128-byte swizzle panels per row
  static constexpr int kPanelBytes = 128 * 128;             // 128 rows x 128 B
  static constexpr int kTileBytes = kPanels * kPanelBytes;  // one 128 x D bf16 tile
  static constexpr int kStages = (D == 128) ? 4 : 6;        // K/V ring slots
  static constexpr int kQOff = 0;
  static constexpr int kKVOff = 2 * kTileBytes;
  static constexpr int kRedOff = kKVOff + kStages * kTileBytes;  // row-max exchange [2][2][128] f32
  static constexpr int kBarOff = kRedOff + 2 * 2 * 128 * 4;
  static constexpr int kSmemBytes = kBarOff + 256 + 1024;   // + barriers + align slack
  // Default number (of every 8) of score-column pairs whose exp2 runs as a
  // polynomial on the FMA pipe instead of MUFU (D=64 has half the MMA work
  // per exponential of D=128).  Overridable per launch for measurement.
  static constexpr int kEmuDefault = (D == 128) ? 2 : 4;
  static constexpr uint32_t kIdescQK = ptx::make_idesc(1, kBM, kBN, 0, 0);
  static constexpr uint32_t kIdescPV = ptx::make_idesc(1, kBM, D, 0, 1);  // V is MN-major
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
  int n_mblk;
  unsigned long long* trace;  // debug timeline (dmha_debug_set_trace), usually null
};

// Timeline trace (measurement hook): clock64 stamps for the first kTraceCtas
// CTAs of head 0 and their first kTraceTiles KV tiles.  Events:
//  0/2: softmax WG0/WG1 saw S full   1/3: WG0/WG1 arrive P ready
//  4/5: MMA warp saw P0/P1 ready     6: MMA warp issued S1(j+1)
constexpr int kTraceCtas = 4, kTraceEvents = 7, kTraceTiles = 64;
__device__ __forceinline__ void trace_stamp(const Params& p, int ev, int j) {
  if (p.trace != nullptr && blockIdx.y == 0 && blockIdx.x < kTraceCtas && j < kTraceTiles)
    p.trace[(blockIdx.x * kTraceEvents + ev) * kTraceTiles + j] = clock64();
}

// 2^x for a pair on MUFU.EX2.
__device__ __forceinline__ float2 exp2_mufu2(float2 x) {
  return make_float2(ptx::ex2_approx(x.x), ptx::ex2_approx(x.y));
}

// 2^x for a pair on the FMA pipe (FADD2/FFMA2 + 2 ALU ops per element):
// n = round(x) via the 1.5*2^23 magic add, f = x - n in [-0.5, 0.5],
// 2^f by a degree-3 minimax polynomial (max rel. error 7.5e-5, below the
// 2^-9 bf16 rounding P gets anyway), exponent added as (n << 23).
// x is clamped at -126 so -inf (masked) gives ~0 and the exponent cannot wrap.
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

// P = exp2(S*scale*log2e - m) for this thread's 64 score columns, packed to
// bf16 and written to its 32 P columns in TMEM (16-column chunks, so the fp32
// scores die as P is produced).  Returns the fp32 sum of the 64 P values.
// EMU of every 8 column pairs use exp2_poly2 (FMA pipe), the rest MUFU.
template <int EMU>
__device__ __forceinline__ float exp_tile(float (&s)[64], float sl2, float m_use, uint32_t tP) {
  const float2 sc2 = make_float2(sl2, sl2);
  const float2 nm2 = make_float2(-m_use, -m_use);
  float2 sum_a = make_float2(0.f, 0.f), sum_b = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
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

// Named barrier over the 256 threads (two warpgroups) that share Q tile g.
__device__ __forceinline__ void pair_sync(int g) {
  asm volatile("bar.sync %0, 256;" ::"r"(1 + g) : "memory");
}

__device__ __forceinline__ int64_t pos_of(const PosMap& m, int64_t i) {
  return i < m.chunk ? m.base0 + i : m.base1 + (i - m.chunk);
}

// Number of leading keys (a prefix, since kpos is increasing) that a query at
// global position qp may use.
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

// KV tiles this CTA has to visit (a prefix of the key tiles).
__device__ __forceinline__ int num_kv_tiles(const Params& p, int64_t m0) {
  int64_t last = m0 + 2 * kBM - 1;
  if (last > p.Lq - 1) last = p.Lq - 1;
  const int64_t lim = key_limit(p, pos_of(p.qmap, last));
  return static_cast<int>((lim + kBN - 1) / kBN);
}

template <int D, int kEmu, bool kRegSplit>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q,
                          const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const Params p) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem + C::kQOff;
  uint8_t* sKV = smem + C::kKVOff;
  float* red = reinterpret_cast<float*>(smem + C::kRedOff);  // [g][h][row]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + C::kStages;
  uint64_t* s_full = kv_empty + C::kStages;   // [2]
  uint64_t* p_ready = s_full + 2;             // [2]
  uint64_t* o_final = p_ready + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_final + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  // Causal: heaviest query blocks first.
  const int mblk = p.causal ? (p.n_mblk - 1 - static_cast<int>(blockIdx.x))
                            : static_cast<int>(blockIdx.x);
  const int64_t m0 = static_cast<int64_t>(mblk) * (2 * kBM);
  const int nkv = num_kv_tiles(p, m0);

  if (warp == kProducerWarp && lane == 0) {
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    for (int g = 0; g < 2; ++g) {
      ptx::mbar_init(&s_full[g], 1);
      ptx::mbar_init(&p_ready[g], 2 * kBM);  // both column halves of every row
      ptx::mbar_init(&o_final[g], 1);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == kMmaWarp) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kProducerWarp) {
    // ------------------------------------------------------------ TMA producer
    if (kRegSplit) ptx::setmaxnreg_dec<kRegsCtl>();
    if (lane == 0 && nkv > 0) {
      ptx::mbar_arrive_expect_tx(q_full, 2 * C::kTileBytes);
      for (int g = 0; g < 2; ++g)
        for (int pn = 0; pn < C::kPanels; ++pn)
          ptx::tma_load_3d(&tm_q, q_full, sQ + g * C::kTileBytes + pn * C::kPanelBytes, pn * 64,
                           head, static_cast<int32_t>(m0 + g * kBM));
      int stage = 0;
      uint32_t phase = 0;
      for (int j = 0; j < nkv; ++j) {
        for (int which = 0; which < 2; ++which) {
          ptx::mbar_wait(&kv_empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&kv_full[stage], C::kTileBytes);
          const CUtensorMap* tm = which == 0 ? &tm_k : &tm_v;
          for (int pn = 0; pn < C::kPanels; ++pn)
            ptx::tma_load_3d(tm, &kv_full[stage], sKV + stage * C::kTileBytes + pn * C::kPanelBytes,
                             pn * 64, head, j * kBN);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    if (kRegSplit) ptx::setmaxnreg_dec<kRegsCtl>();
    if (lane == 0 && nkv > 0) {
      const uint32_t sq = ptx::smem_u32(sQ);
      const uint32_t skv = ptx::smem_u32(sKV);
      auto qk = [&](int g, int slot) {
        const uint32_t a0 = sq + g * C::kTileBytes;
        const uint32_t b0 = skv + slot * C::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::kPanelBytes + (kk & 3) * 32;
          ptx::mma_bf16_ss(tmem + g * kBN, ptx::smem_desc_sw128(a0 + off, 16, 1024),
                           ptx::smem_desc_sw128(b0 + off, 16, 1024), C::kIdescQK, kk > 0);
        }
      };
      auto pv = [&](int g, int slot, bool acc) {
        const uint32_t b0 = skv + slot * C::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          ptx::mma_bf16_ts(tmem + 256 + g * 128, tmem + g * kBN + kk * 8,
                           ptx::smem_desc_sw128(b0 + kk * 16 * 128, C::kPanelBytes, 1024),
                           C::kIdescPV, (acc || kk > 0) ? 1u : 0u);
        }
      };
      int stage = 0;
      uint32_t phase = 0;
      auto advance = [&]() { if (++stage == C::kStages) { stage = 0; phase ^= 1; } };

      ptx::mbar_wait(q_full, 0);
      // j = 0
      int slotK = stage;
      ptx::mbar_wait(&kv_full[slotK], phase);
      advance();
      ptx::tc_fence_after();
      qk(0, slotK);
      ptx::mma_commit(&s_full[0]);
      qk(1, slotK);
      ptx::mma_commit(&s_full[1]);
      ptx::mma_commit(&kv_empty[slotK]);
      for (int j = 1; j <= nkv; ++j) {
        const int slotV = stage;  // V_{j-1}
        ptx::mbar_wait(&kv_full[slotV], phase);
        advance();
        const bool more = j < nkv;
        int slotK2 = -1;
        if (more) {
          slotK2 = stage;  // K_j
          ptx::mbar_wait(&kv_full[slotK2], phase);
          advance();
        }
        const uint32_t ppar = static_cast<uint32_t>((j - 1) & 1);
        ptx::mbar_wait(&p_ready[0], ppar);
        trace_stamp(p, 4, j - 1);
        ptx::tc_fence_after();
        pv(0, slotV, j > 1);
        if (more) {
          qk(0, slotK2);
          ptx::mma_commit(&s_full[0]);
        } else {
          ptx::mma_commit(&o_final[0]);
        }
        ptx::mbar_wait(&p_ready[1], ppar);
        trace_stamp(p, 5, j - 1);
        ptx::tc_fence_after();
        pv(1, slotV, j > 1);
        ptx::mma_commit(&kv_empty[slotV]);
        if (more) {
          qk(1, slotK2);
          ptx::mma_commit(&s_full[1]);
          trace_stamp(p, 6, j);
          ptx::mma_commit(&kv_empty[slotK2]);
        } else {
          ptx::mma_commit(&o_final[1]);
        }
      }
    }
    __syncwarp();
  } else if (warp >= kSoftmaxWarps) {
    if (kRegSplit) ptx::setmaxnreg_dec<kRegsCtl>();  // idle warps of the control warpgroup
  } else {
    // ------------------------------------------------------------ softmax
    if (kRegSplit) ptx::setmaxnreg_inc<kRegsSoftmax>();
    const int wg = warp >> 2;
    const int g = wg >> 1;                    // Q tile of this warpgroup
    const int h = wg & 1;                     // score-column half / output-column half
    const int quarter = warp & 3;             // TMEM lane quarter
    const int r = quarter * 32 + lane;        // row within the tile
    const int64_t row = m0 + g * kBM + r;     // local query row
    const bool row_ok = row < p.Lq;
    const int64_t qp = pos_of(p.qmap, row_ok ? row : p.Lq - 1);
    const int64_t klim = key_limit(p, qp);
    const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_addr + g * kBN + h * 64;  // this half's 64 score columns
    const uint32_t tP = tmem + lane_addr + g * kBN + h * 32;  // this half's 32 P columns
    const uint32_t tO = tmem + lane_addr + 256 + g * 128;
    float* red_mine = red + (g * 2 + h) * kBM + r;
    const float* red_other = red + (g * 2 + (h ^ 1)) * kBM + r;
    const float sl2 = p.scale_log2;
    const bool leader = (threadIdx.x % 256) == 0;  // one stamp per Q tile

    float m_run = -INFINITY;  // running max, log2 units (scaled); equal in both halves
    float l_run = 0.f;        // this half's share of the row sum
    for (int j = 0; j < nkv; ++j) {
      ptx::mbar_wait(&s_full[g], static_cast<uint32_t>(j & 1));
      if (leader) trace_stamp(p, 2 * g, j);
      ptx::tc_fence_after();
      float s[64];
      ptx::tmem_ld32(tS, *reinterpret_cast<float(*)[32]>(&s[0]));
      ptx::tmem_ld32(tS + 32, *reinterpret_cast<float(*)[32]>(&s[32]));
      ptx::tmem_wait_ld();

      const int64_t nv64 = klim - static_cast<int64_t>(j) * kBN - h * 64;
      const int nvalid = nv64 < 0 ? 0 : (nv64 > 64 ? 64 : static_cast<int>(nv64));
      // Warp-uniform in both halves of a row: masked iff any row of the Q tile
      // has fewer than all 128 keys of the tile visible.
      const bool masked = !__all_sync(0xffffffffu, klim - static_cast<int64_t>(j) * kBN >= kBN);
      if (masked) {
#pragma unroll
        for (int c = 0; c < 64; ++c) s[c] = c < nvalid ? s[c] : -INFINITY;
      }
      float mx0 = s[0], mx1 = s[1], mx2 = s[2], mx3 = s[3];
#pragma unroll
      for (int c = 4; c < 64; c += 4) {
        mx0 = fmaxf(mx0, s[c]);
        mx1 = fmaxf(mx1, s[c + 1]);
        mx2 = fmaxf(mx2, s[c + 2]);
        mx3 = fmaxf(mx3, s[c + 3]);
      }
      const float pmax = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
      *red_mine = pmax;
      pair_sync(g);  // the other half reads this slot before tile j+1 can be
                     // written: S_g(j+1) needs both halves' P_g(j) first.
      const float mt = fmaxf(pmax, *red_other) * sl2;
      const bool need = mt > m_run + kRescaleThreshold;
      const bool warp_rescale = __any_sync(0xffffffffu, need);  // same in both halves
      float alpha = 1.f;
      if (warp_rescale) {
        const float m_new = fmaxf(m_run, mt);
        alpha = (m_new == -INFINITY) ? 1.f : ptx::ex2_approx(m_run - m_new);
        l_run *= alpha;
        m_run = m_new;
      }
      const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
      // Unmasked tiles send kEmu of every 8 column pairs to the FMA-pipe
      // polynomial; masked tiles (-inf entries, must give exactly 0) use MUFU only.
      if (masked)
        l_run += exp_tile<0>(s, sl2, m_use, tP);
      else
        l_run += exp_tile<kEmu>(s, sl2, m_use, tP);
      // O_g holds PV_g(j-1) (complete: covered by the S_g(j) commit) and PV_g(j)
      // is not issued before p_ready, so O can be rescaled in place here.
      if (warp_rescale && j > 0 && h == 0) {
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
      if (leader) trace_stamp(p, 2 * g + 1, j);
      ptx::mbar_arrive(&p_ready[g]);
    }
    if (nkv > 0) {
      ptx::mbar_wait(&o_final[g], 0);
      ptx::tc_fence_after();
    }
    // ---------------------------------------------------------- epilogue
    // Row sum = both halves' shares (same m_run); each half writes D/2 columns.
    *red_mine = l_run;
    pair_sync(g);
    const float l_tot = l_run + *red_other;
    const bool empty = !(l_tot > 0.f);
    const float inv_l = empty ? 0.f : 1.f / l_tot;
    if (row_ok && h == 0)
      p.lse[static_cast<int64_t>(head) * p.Lq + row] =
          empty ? -INFINITY : (m_run + __log2f(l_tot)) * 0.69314718055994530942f;
    const int64_t obase = (row * p.H + head) * static_cast<int64_t>(D) + h * (D / 2);
#pragma unroll
    for (int c = 0; c < D / 64; ++c) {
      float o[32];
      if (nkv > 0) {
        ptx::tmem_ld32(tO + h * (D / 2) + c * 32, o);
        ptx::tmem_wait_ld();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = 0.f;
      }
      if (row_ok) {
        if (p.out_mode == OUT_PARTIAL_F32) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + obase + c * 32);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            dst[e] = make_float4(o[4 * e] * inv_l, o[4 * e + 1] * inv_l, o[4 * e + 2] * inv_l,
                                 o[4 * e + 3] * inv_l);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.out) + obase +
                                                c * 32);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint32_t w[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              __nv_bfloat162 b = __floats2bfloat162_rn(o[8 * e + 2 * t] * inv_l,
                                                       o[8 * e + 2 * t + 1] * inv_l);
              w[t] = *reinterpret_cast<uint32_t*>(&b);
            }
            dst[e] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------- host side
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// [L, H, D] bf16 viewed as a 3-D tensor (D, H, L); box (64, 1, 128), 128B swizzle.
bool make_map(CUtensorMap* map, const void* base, int64_t L, int H, int D) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  // A zero-length block is never loaded (nkv = 0) but the map must be valid.
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(L > 0 ? L : 1)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2,
                           static_cast<cuuint64_t>(D) * H * 2};
  cuuint32_t box[3] = {64, 1, 128};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Kernel variant (measurement knob): DMHA_EMU=<pairs of 8 on the FMA pipe>,
// DMHA_REGSPLIT=0/1.  Defaults: Cfg<D>::kEmuDefault, register split on.
struct Variant {
  int emu;
  bool regsplit;
};

template <int D>
Variant variant() {
  static Variant v = [] {
    Variant x{Cfg<D>::kEmuDefault, true};
    if (const char* e = std::getenv("DMHA_EMU")) x.emu = std::atoi(e);
    if (const char* r = std::getenv("DMHA_REGSPLIT")) x.regsplit = std::atoi(r) != 0;
    return x;
  }();
  return v;
}

template <int D, int E, bool R>
cudaError_t launch_v(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                     const Params& p, dim3 grid, cudaStream_t stream) {
  using C = Cfg<D>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_sm100_kernel<D, E, R>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  attn_fwd_sm100_kernel<D, E, R><<<grid, kThreads, C::kSmemBytes, stream>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

template <int D>
cudaError_t launch_d(const LocalAttnArgs& a, cudaStream_t stream) {
  CUtensorMap tq, tk, tv;
  if (!make_map(&tq, a.q, a.Lq, a.H, D) || !make_map(&tk, a.k, a.Lk, a.H, D) ||
      !make_map(&tv, a.v, a.Lk, a.H, D))
    return cudaErrorInvalidValue;
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
  p.n_mblk = static_cast<int>((a.Lq + 2 * kBM - 1) / (2 * kBM));
  p.trace = g_trace;
  dim3 grid(p.n_mblk, a.H);
  const Variant v = variant<D>();
  if (!v.regsplit) return launch_v<D, Cfg<D>::kEmuDefault, false>(tq, tk, tv, p, grid, stream);
  switch (v.emu) {
    case 0: return launch_v<D, 0, true>(tq, tk, tv, p, grid, stream);
    case 1: return launch_v<D, 1, true>(tq, tk, tv, p, grid, stream);
    case 2: return launch_v<D, 2, true>(tq, tk, tv, p, grid, stream);
    case 3: return launch_v<D, 3, true>(tq, tk, tv, p, grid, stream);
    case 4: return launch_v<D, 4, true>(tq, tk, tv, p, grid, stream);
    default: return launch_v<D, Cfg<D>::kEmuDefault, true>(tq, tk, tv, p, grid, stream);
  }
}

}  // namespace

unsigned long long* g_trace = nullptr;

cudaError_t launch_attn_fwd_bf16(const LocalAttnArgs& a, cudaStream_t stream) {
  if (a.Lq <= 0) return cudaSuccess;
  if (a.Lq > INT32_MAX || a.Lk > INT32_MAX) return cudaErrorInvalidValue;
  if (a.D == 64) return launch_d<64>(a, stream);
  if (a.D == 128) return launch_d<128>(a, stream);
  return cudaErrorInvalidValue;
}

}  // namespace dmha
