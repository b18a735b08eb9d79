// attn_fwd_sm100.cu — "ping-pong" flash-attention forward for sm_100a:
// two 128-row query tiles per CTA share every K/V tile in shared memory (so
// L2->SMEM traffic is one K/V tile per 256 query rows) and alternate on the
// tensor core.  The attention kernel of libdmha.so for both head dims (the
// measured-slower cluster / cta_group::2 / 64-key "dbuf" variants of round 1
// are archived under tools/variants/, DESIGN.md §5 lessons 3-4, 9).
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
// CTA = 2 query tiles of 128 rows (256 rows) of one head; 12 warps:
//   warps 0-3  softmax for Q tile 0 (thread t <-> TMEM lane t <-> row t)
//   warps 4-7  softmax for Q tile 1
//   warp  8    TMA producer (Q once; K_j, V_j through an NST-slot ring)
//   warp  9    TMEM allocator + single-thread tcgen05.mma issuer
//   warps 10-11 idle (keep the CTA at 3 warpgroups)
// TMEM (512 cols): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [384,384+D);
// P_g (bf16x2) aliases the first 64 columns of S_g.
// MMA order per KV tile j:  PV0_{j-1}, S0_j, PV1_{j-1}, S1_j — S_g(j) is issued
// after PV_g(j-1) read P_g(j-1) (tcgen05.mma executes in issue order), and the
// commit that signals S_g(j) also covers PV_g(j-1), so the softmax warps can
// rescale O_g right after they see S_g(j).
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

#include "combine_math.cuh"
#include "kernels.h"
#include "tma_map.h"
#include "ptx_sm100.cuh"
#include "softmax_sm100.cuh"

namespace dmha {
extern unsigned long long* g_trace;
namespace {

constexpr int kBM = 128;          // query rows per tile (MMA M)
constexpr int kBN = 128;          // keys per tile (MMA N of QK^T, K of PV)
// Warp roles: kSm softmax warps (8, or 16 with the split softmax), then the
// TMA producer, the MMA warp and two idle warps.
template <bool kSplit>
struct Roles {
  static constexpr int kSm = kSplit ? 16 : 8;
  static constexpr int kProducerWarp = kSm;
  static constexpr int kMmaWarp = kSm + 1;
  static constexpr int kThreads = (kSm + 4) * 32;
};
constexpr float kRescaleThreshold = 8.0f;  // log2 units: rescale when max grows by > 2^8
#ifndef DMHA_KST64
#define DMHA_KST64 3  // D = 64 K ring slots
#endif
#ifndef DMHA_VST64
#define DMHA_VST64 3  // D = 64 V ring slots
#endif
#ifndef DMHA_EXPFORM
#define DMHA_EXPFORM 0  // D = 128 exponential loop: 0 scalar FFMA, 1 FFMA2/FADD2, 2 immediate-scale FFMA
#endif
#ifndef DMHA_SOFTMAX_REGS
#define DMHA_SOFTMAX_REGS 0
#endif
constexpr int kSmRegs = DMHA_SOFTMAX_REGS;  // 0: no re-balancing
constexpr int kOtherRegs = kSmRegs > 0 ? ((384 * 168 - 256 * kSmRegs) / 128) / 8 * 8 : 0;
static_assert(kSmRegs == 0 || (kSmRegs % 8 == 0 && kSmRegs <= 256 && kOtherRegs >= 24),
              "setmaxnreg budget");


// kPS (D = 128 only): P_g(j) goes to shared memory instead of over S_g's TMEM
// columns, so QK^T(j+1) can run during softmax(j) (the separate-P schedule of
// D = 64, whose P fits in TMEM).  Shared memory then holds Q (2 tiles), ONE K
// slot, two V slots and the two P tiles: 224 KB of the 227 KB.
template <int D, bool kPS>
struct Cfg {
  static constexpr int kPanels = D / 64;                    // 128-byte swizzle panels per row
  static constexpr int kPanelBytes = 128 * 128;             // 128 rows x 128 B
  static constexpr int kTileBytes = kPanels * kPanelBytes;  // one 128 x D bf16 tile
  // Separate-P schedule: K and V in their own rings (kKSt / kVSt slots);
  // otherwise one K/V ring of kStages slots (K_j, V_j alternate).
  static constexpr bool kSepP = (D == 64) || kPS;
  static constexpr int kKSt = (D == 64) ? DMHA_KST64 : 1;
  static constexpr int kVSt = (D == 64) ? DMHA_VST64 : 2;
  static constexpr int kStages = kSepP ? kKSt + kVSt : 4;
  static constexpr int kQOff = 0;
  static constexpr int kKVOff = 2 * kTileBytes;
  static constexpr int kPOff = kKVOff + kStages * kTileBytes;     // kPS: P_0, P_1 (128 x 128 bf16)
  static constexpr int kRedOff = kPOff + (kPS ? 2 * 128 * 128 * 2 : 0);
  // split softmax: [2][2][2][128] f32 row maxima + l [2][2][128]
  static constexpr int kRedBytes = kPS ? 0 : 12 * 128 * 4;
  static constexpr int kBarOff = kRedOff + kRedBytes;
  static constexpr int kSmemBytes = kBarOff + 256 + 1024;   // + barriers + align slack
  static_assert(kSmemBytes <= 232448, "shared memory budget (227 KB)");
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
  float* acc_o;    // OUT_COMBINE_*: running accumulator (read; ACC also writes it)
  float* acc_lse;
  void* out2;      // kv_split = 2: the z = 1 CTAs' partial output / lse
  float* lse2;
  int kv_split;    // 1, or 2: blockIdx.z picks one half of each CTA's key tiles
  int n_mblk;
  float lse_bias;  // fault injection (DMHA_FAULT=perturb_lse): added to lse_s in the combine; 0
  int alt;         // D = 128: the two softmax warpgroups take turns on MUFU (DMHA_ALT)
  unsigned long long* trace;  // debug timeline (dmha_debug_set_trace), usually null
};

// Timeline trace (measurement hook, same buffer layout as the other variants:
// [cta < 4][event < 9][tile < 64] clock64 stamps, head 0 only).  Events:
//  0/2: softmax of Q tile 0/1 saw S(j)   1/3: Q tile 0/1 arrive P(j) ready
//  4/5: MMA thread saw P0(j)/P1(j) ready   6: MMA thread issued S1(j)
// Per-tile stamps exist only in a measurement build (-DDMHA_TRACE=1,
// tools/trace.py builds it): compiled in, the disabled checks and clock reads
// cost the product kernel 2.6 % at C4 and 2.1 % C5-shaped (one of them sits
// in the single-thread MMA issue path) — DESIGN.md §5 lesson 32.
#ifndef DMHA_TRACE
#define DMHA_TRACE 0
#endif
__device__ __forceinline__ void trace_stamp(const Params& p, int ev, int j) {
  if (DMHA_TRACE && p.trace != nullptr && blockIdx.y == 0 && blockIdx.x < 2 && j < 64)
    p.trace[(blockIdx.x * 9 + ev) * 64 + j] = clock64();
}
// Extra events 0..17 of CTA 0 (stored where CTAs 2-3 would be).
__device__ __forceinline__ void trace_x(const Params& p, int ev, int j) {
  if (DMHA_TRACE && p.trace != nullptr && blockIdx.y == 0 && blockIdx.x == 0 && j < 64)
    p.trace[(18 + ev) * 64 + j] = clock64();
}

// Per-CTA wall-clock stamps (%globaltimer, ns) at words 4096 + 2*id (+1).
#ifndef DMHA_CTA_STAMPS
#define DMHA_CTA_STAMPS 0  // measurement builds only: they cost the 96-register D = 64 kernel 20 %
#endif
__device__ __forceinline__ void cta_stamp(const Params& p, int which) {
  if (!DMHA_CTA_STAMPS || p.trace == nullptr) return;
  const unsigned id = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (id >= 16384) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  p.trace[4096 + 2 * id + which] = t;
}

// Sub-phase stamps of the D = 64 split softmax, compiled only into the
// measurement build (-DDMHA_TRACE_PHASES=1, tools/trace.py via DMHA_LIB):
// trace_x events 0-5 of the (g = 0, h = 0) warpgroup's thread 0.
#ifndef DMHA_TRACE_PHASES
#define DMHA_TRACE_PHASES 0
#endif
#define PHASE(ev)                                                                 \
  do {                                                                            \
    if (DMHA_TRACE_PHASES && g == 0 && h == 0 && threadIdx.x % 128 == 0) trace_x(p, ev, j); \
  } while (0)

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

// mbarrier wait of the attention kernel: D = 128 (power-capped, chain-bound)
// sleeps on the barrier, D = 64 (wake-up latency on the critical path)
// polls — measured, see ptx::mbar_try_wait_sleep.
template <int D, int kSleepD64 = 0>
__device__ __forceinline__ void kwait(uint64_t* bar, uint32_t parity) {
  if constexpr (D == 128 || kSleepD64)
    ptx::mbar_wait_sleep(bar, parity);
  else
    ptx::mbar_wait(bar, parity);
}
#ifndef DMHA_PROD_SLEEP
#define DMHA_PROD_SLEEP 0  // measurement knob: D = 64 TMA producer sleeps too
#endif
#ifndef DMHA_MMA_SLEEP
#define DMHA_MMA_SLEEP 0   // measurement knob: D = 64 MMA issuer sleeps too
#endif

template <int D, int kEmu, bool kSplit, int kIss, bool kPS>
__global__ void __launch_bounds__(Roles<kSplit>::kThreads, 1)
    attn_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q,
                          const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const Params p) {
  using C = Cfg<D, kPS>;
  using R = Roles<kSplit>;
  constexpr int kProducerWarp = R::kProducerWarp;
  constexpr int kMmaWarp = R::kMmaWarp;
  // Separate P buffers decouple S_g(j+1) from PV_g(j): in TMEM for D = 64
  // (room next to O_g), in shared memory for D = 128 (kPS).
  constexpr bool kSepP = C::kSepP;
  static_assert(!kPS || (D == 128 && !kSplit), "P in shared memory: D = 128, one warpgroup per tile");
  constexpr uint32_t kPCol = 256 + 64;  // P_g at kPCol + 128 g (D = 64 only)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem + C::kQOff;
  uint8_t* sKV = smem + C::kKVOff;
  uint8_t* sP = smem + C::kPOff;  // kPS only
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + C::kStages;
  uint64_t* s_full = kv_empty + C::kStages;   // [2]
  uint64_t* p_ready = s_full + 2;             // [2]
  uint64_t* o_final = p_ready + 2;            // [2]
  // D = 64 only (separate P buffers): softmax loaded S_g / PV_g complete.
  uint64_t* s_free = o_final + 2;             // [2]
  uint64_t* pv_done = s_free + 2;             // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  // Causal: heaviest query blocks first.
  const int mblk = p.causal ? (p.n_mblk - 1 - static_cast<int>(blockIdx.x))
                            : static_cast<int>(blockIdx.x);
  const int64_t m0 = static_cast<int64_t>(mblk) * (2 * kBM);
  // Split-KV (small grids): CTA z of a split covers tiles [jt0, jt0 + nkv) of
  // its row block's visible key tiles and writes an fp32 partial (out2/lse2
  // for z = 1) that the log-sum-exp combine merges.
  const int nkv_all = num_kv_tiles(p, m0);
  const int kv_half = (nkv_all + p.kv_split - 1) / p.kv_split;
  const int jt0 = min(nkv_all, static_cast<int>(blockIdx.z) * kv_half);
  const int nkv = min(nkv_all, jt0 + kv_half) - jt0;
  void* const out_ptr = blockIdx.z ? p.out2 : p.out;
  float* const lse_ptr = blockIdx.z ? p.lse2 : p.lse;

  if (warp == kProducerWarp && lane == 0) {
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      // one release per issuer that reads the slot: separate-P rings hold K in
      // slots [0, kKSt) (read by the S issuers) and V after them (read by the
      // PV issuers; two for kIss = 2 and 4); the single ring is read by every
      // issuer
      const bool v_slot = kSepP && s >= C::kKSt;
      const int readers = kSepP ? ((kIss == 2 || (kIss == 4 && v_slot)) ? 2 : 1) : (kIss == 2 ? 2 : 1);
      ptx::mbar_init(&kv_empty[s], readers);
    }
    for (int g = 0; g < 2; ++g) {
      ptx::mbar_init(&s_full[g], 1);
      ptx::mbar_init(&p_ready[g], kSplit ? 2 * kBM : kBM);  // every softmax thread of the Q tile
      ptx::mbar_init(&o_final[g], 1);
      ptx::mbar_init(&s_free[g], kSplit ? 2 * kBM : kBM);
      ptx::mbar_init(&pv_done[g], 1);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (threadIdx.x == 0) cta_stamp(p, 0);
  if (warp == kMmaWarp) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Register re-balancing (one-warpgroup-per-tile schedule): the producer /
  // MMA / idle warpgroup (warps 8-11, all four execute the dec) hands
  // registers to the two softmax warpgroups, whose 128-score rows otherwise
  // leave ptxas too few registers to keep several MUFU results in flight
  // (ncu: short-scoreboard stalls on MUFU.EX2 with a reused destination).
  // 384 threads x 168 = 256 x kSmRegs + 128 x kOtherRegs.
  if constexpr (!kSplit && kSmRegs > 0) {
    if (warp >= 8) ptx::setmaxnreg_dec<kOtherRegs>();
    else ptx::setmaxnreg_inc<kSmRegs>();
  }

  if (warp == kProducerWarp) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && nkv > 0) {
      ptx::mbar_arrive_expect_tx(q_full, 2 * C::kTileBytes);
      for (int g = 0; g < 2; ++g)
        for (int pn = 0; pn < C::kPanels; ++pn)
          ptx::tma_load_3d(&tm_q, q_full, sQ + g * C::kTileBytes + pn * C::kPanelBytes, pn * 64,
                           head, static_cast<int32_t>(m0 + g * kBM));
      if constexpr (kSepP) {
        // K_j -> K ring slot j % kKSt, V_j -> V ring slot j % kVSt (separate
        // rings: K_{j+1} only waits for S(j), not for PV(j-1))
        for (int j = 0; j < nkv; ++j) {
          for (int which = 0; which < 2; ++which) {
            const int nst = which == 0 ? C::kKSt : C::kVSt;
            const int slot = (which == 0 ? 0 : C::kKSt) + j % nst;
            const uint32_t ph = static_cast<uint32_t>((j / nst) & 1);
            trace_x(p, 5 + 9 * which, j);
            kwait<D, DMHA_PROD_SLEEP>(&kv_empty[slot], ph ^ 1);
            trace_x(p, 6 + 9 * which, j);
            ptx::mbar_arrive_expect_tx(&kv_full[slot], C::kTileBytes);
            const CUtensorMap* tm = which == 0 ? &tm_k : &tm_v;
            for (int pn = 0; pn < C::kPanels; ++pn)
              ptx::tma_load_3d(tm, &kv_full[slot], sKV + slot * C::kTileBytes + pn * C::kPanelBytes,
                               pn * 64, head, (jt0 + j) * kBN);
          }
        }
      } else {
        int stage = 0;
        uint32_t phase = 0;
        for (int j = 0; j < nkv; ++j) {
          for (int which = 0; which < 2; ++which) {
            trace_x(p, 5 + 9 * which, j);
            kwait<D, DMHA_PROD_SLEEP>(&kv_empty[stage], phase ^ 1);
            trace_x(p, 6 + 9 * which, j);
            ptx::mbar_arrive_expect_tx(&kv_full[stage], C::kTileBytes);
            const CUtensorMap* tm = which == 0 ? &tm_k : &tm_v;
            for (int pn = 0; pn < C::kPanels; ++pn)
              ptx::tma_load_3d(tm, &kv_full[stage], sKV + stage * C::kTileBytes + pn * C::kPanelBytes,
                               pn * 64, head, (jt0 + j) * kBN);
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == kMmaWarp || (kIss > 1 && warp == kMmaWarp + 1) ||
             (kIss == 4 && warp == kMmaWarp + 2)) {
    // ------------------------------------------------------------ MMA issuer(s)
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
      // D = 64: P_g lives at columns [320 + 128g, 384 + 128g) (the unused half
      // of O_g's 128-column slot).
      // D = 128 with kPS: P_g is a 128 x 128 bf16 K-major tile in shared
      // memory (the 128-byte-swizzled layout TMA gives Q), an SS MMA operand.
      const uint32_t sp = ptx::smem_u32(sP);
      auto pv_sep = [&](int g, int slot, bool acc) {
        const uint32_t b0 = skv + slot * C::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          const uint64_t bdesc = ptx::smem_desc_sw128(b0 + kk * 16 * 128, C::kPanelBytes, 1024);
          if constexpr (kPS) {
            const uint32_t a0 = sp + g * (kBM * kBN * 2) + (kk >> 2) * C::kPanelBytes + (kk & 3) * 32;
            ptx::mma_bf16_ss(tmem + 256 + g * 128, ptx::smem_desc_sw128(a0, 16, 1024), bdesc,
                             C::kIdescPV, (acc || kk > 0) ? 1u : 0u);
          } else {
            ptx::mma_bf16_ts(tmem + 256 + g * 128, tmem + kPCol + g * 128 + kk * 8, bdesc,
                             C::kIdescPV, (acc || kk > 0) ? 1u : 0u);
          }
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
      if constexpr (kSepP) {
        // D = 64: P_g has its own TMEM columns, so S_g(j) only waits for the
        // softmax to have LOADED S_g(j-1) (s_free) and runs on the tensor core
        // during that softmax's exponentials; PV_g(j-1) follows when P is ready.
        // One issuing warp per Q tile (warp kMmaWarp + g): a single thread
        // issues A-from-TMEM MMAs at only ~69 cycles each whatever N is
        // (tools/umma_multi.cu: two issuers reach 39, the N = 64 PV needs 32),
        // and each Q tile's chain no longer waits behind the other's barriers.
        // K_t sits in K ring slot t % kKSt, V_t in V ring slot kKSt + t % kVSt
        // (separate rings, see the producer); each slot is released by every
        // issuer that reads it (kv_empty counts).
        // kIss = 1: one thread issues both Q tiles (S0 S1, then PV0 PV1);
        // kIss = 2: warp kMmaWarp + g issues Q tile g (S_g and PV_g);
        // kIss = 3: warp kMmaWarp issues S0 S1, warp kMmaWarp + 1 PV0 PV1.
        // kIss = 4: warp kMmaWarp issues S0 S1, warp kMmaWarp + 1 + g PV_g.
        const int role = warp - kMmaWarp;
        const int g_lo = kIss == 2 ? role : (kIss == 4 && role > 0 ? role - 1 : 0);
        const int g_hi = (kIss == 2 || (kIss == 4 && role > 0)) ? g_lo + 1 : 2;
        const bool do_s = (kIss != 3 && kIss != 4) || role == 0;
        const bool do_pv = (kIss != 3 && kIss != 4) || role >= 1;
        auto kslot = [](int t) { return t % C::kKSt; };
        auto kpar = [](int t) { return static_cast<uint32_t>((t / C::kKSt) & 1); };
        auto vslot = [](int t) { return C::kKSt + t % C::kVSt; };
        auto vpar = [](int t) { return static_cast<uint32_t>((t / C::kVSt) & 1); };
        kwait<D, DMHA_MMA_SLEEP>(q_full, 0);
        if (do_s) {
          kwait<D, DMHA_MMA_SLEEP>(&kv_full[kslot(0)], kpar(0));
          ptx::tc_fence_after();
          for (int g = g_lo; g < g_hi; ++g) {
            qk(g, kslot(0));
            ptx::mma_commit(&s_full[g]);
          }
          ptx::mma_commit(&kv_empty[kslot(0)]);
        }
        for (int j = 1; j <= nkv; ++j) {
          const uint32_t ppar = static_cast<uint32_t>((j - 1) & 1);
          if (do_s && j < nkv) {  // S_g(j): needs K_j and S_g(j-1) consumed
            trace_x(p, 9 * g_lo + 0, j);
            kwait<D, DMHA_MMA_SLEEP>(&kv_full[kslot(j)], kpar(j));
            trace_x(p, 9 * g_lo + 1, j);
            for (int g = g_lo; g < g_hi; ++g) {
              kwait<D, DMHA_MMA_SLEEP>(&s_free[g], ppar);
              if (g == g_lo) trace_x(p, 9 * g_lo + 2, j);
              ptx::tc_fence_after();
              qk(g, kslot(j));
              ptx::mma_commit(&s_full[g]);
            }
            if (g_lo == 0) trace_stamp(p, 6, j);
            ptx::mma_commit(&kv_empty[kslot(j)]);
          }
          if (do_pv) {  // PV_g(j-1): needs V_{j-1} and P_g(j-1)
            kwait<D, DMHA_MMA_SLEEP>(&kv_full[vslot(j - 1)], vpar(j - 1));
            trace_x(p, 9 * g_lo + 3, j - 1);
            for (int g = g_lo; g < g_hi; ++g) {
              kwait<D, DMHA_MMA_SLEEP>(&p_ready[g], ppar);
              trace_stamp(p, 4 + g, j - 1);
              ptx::tc_fence_after();
              pv_sep(g, vslot(j - 1), j > 1);
              ptx::mma_commit(&pv_done[g]);
              if (j == nkv) ptx::mma_commit(&o_final[g]);
            }
            trace_x(p, 9 * g_lo + 4, j - 1);
            ptx::mma_commit(&kv_empty[vslot(j - 1)]);
          }
        }
      } else if constexpr (kIss == 2) {
        // D = 128, one issuing warp per Q tile: warp kMmaWarp + g issues
        // PV_g(j-1) then S_g(j) (same thread, so S_g(j) still follows the PV
        // that reads P_g(j-1) from S_g's columns, and the S_g(j) commit covers
        // both).  Every K/V slot is released by both issuers (kv_empty count 2).
        const int g = warp - kMmaWarp;
        auto slot_of = [](int item) { return item % C::kStages; };
        auto par_of = [](int item) { return static_cast<uint32_t>((item / C::kStages) & 1); };
        kwait<D, DMHA_MMA_SLEEP>(q_full, 0);
        kwait<D, DMHA_MMA_SLEEP>(&kv_full[slot_of(0)], par_of(0));
        ptx::tc_fence_after();
        qk(g, slot_of(0));
        ptx::mma_commit(&s_full[g]);
        ptx::mma_commit(&kv_empty[slot_of(0)]);
        for (int j = 1; j <= nkv; ++j) {
          const uint32_t ppar = static_cast<uint32_t>((j - 1) & 1);
          const int iv = 2 * (j - 1) + 1, ik = 2 * j;
          kwait<D, DMHA_MMA_SLEEP>(&kv_full[slot_of(iv)], par_of(iv));
          if (j < nkv) kwait<D, DMHA_MMA_SLEEP>(&kv_full[slot_of(ik)], par_of(ik));
          kwait<D, DMHA_MMA_SLEEP>(&p_ready[g], ppar);
          trace_stamp(p, 4 + g, j - 1);
          ptx::tc_fence_after();
          pv(g, slot_of(iv), j > 1);
          ptx::mma_commit(&kv_empty[slot_of(iv)]);
          if (j < nkv) {
            qk(g, slot_of(ik));
            ptx::mma_commit(&s_full[g]);
            if (g == 1) trace_stamp(p, 6, j);
            ptx::mma_commit(&kv_empty[slot_of(ik)]);
          } else {
            ptx::mma_commit(&o_final[g]);
          }
        }
      } else {
      int stage = 0;
      uint32_t phase = 0;
      auto advance = [&]() { if (++stage == C::kStages) { stage = 0; phase ^= 1; } };

      kwait<D, DMHA_MMA_SLEEP>(q_full, 0);
      // j = 0
      int slotK = stage;
      kwait<D, DMHA_MMA_SLEEP>(&kv_full[slotK], phase);
      advance();
      ptx::tc_fence_after();
      qk(0, slotK);
      ptx::mma_commit(&s_full[0]);
      qk(1, slotK);
      ptx::mma_commit(&s_full[1]);
      ptx::mma_commit(&kv_empty[slotK]);
      for (int j = 1; j <= nkv; ++j) {
        const int slotV = stage;  // V_{j-1}
        kwait<D, DMHA_MMA_SLEEP>(&kv_full[slotV], phase);
        advance();
        const bool more = j < nkv;
        int slotK2 = -1;
        if (more) {
          slotK2 = stage;  // K_j
          kwait<D, DMHA_MMA_SLEEP>(&kv_full[slotK2], phase);
          advance();
        }
        const uint32_t ppar = static_cast<uint32_t>((j - 1) & 1);
        kwait<D, DMHA_MMA_SLEEP>(&p_ready[0], ppar);
        trace_stamp(p, 4, j - 1);
        ptx::tc_fence_after();
        pv(0, slotV, j > 1);
        if (more) {
          qk(0, slotK2);
          ptx::mma_commit(&s_full[0]);
        } else {
          ptx::mma_commit(&o_final[0]);
        }
        kwait<D, DMHA_MMA_SLEEP>(&p_ready[1], ppar);
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
      }
    __syncwarp();
  } else if (kSplit && warp < R::kSm) {
    // ------------------------------------------------------------ split softmax
    // Two warpgroups per Q tile: warpgroup (g, h) handles score columns
    // [64h, 64h+64) of every row of Q tile g, so 8 warps (2 per SMSP) feed
    // MUFU during a tile's exponentials.  The row max is swapped through
    // shared memory (slot by tile parity); each half keeps its share of l and
    // rescales / writes half of O's columns.
    float* red = reinterpret_cast<float*>(smem + C::kRedOff);  // [parity][g][h][128]
    float* redl = red + 8 * kBM;                               // [g][h][128]
    const int wg = warp >> 2;
    const int g = wg & 1;                     // Q tile
    const int h = wg >> 1;                    // column half
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int64_t row = m0 + g * kBM + r;
    const bool row_ok = row < p.Lq;
    const int64_t qp = pos_of(p.qmap, row_ok ? row : p.Lq - 1);
    // this row's key limit relative to the launch's first key tile, 32-bit (a
    // launch's keys fit one GPU: < 2^31): the 64-bit form spilled at the
    // 96-register cap and was reloaded from local memory every tile
    const int klim_t =
        static_cast<int>(key_limit(p, qp) - static_cast<int64_t>(jt0) * kBN);
    const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_addr + g * kBN;
    const uint32_t tO = tmem + lane_addr + 256 + g * 128 + h * (D / 2);
    const uint32_t tP = (kSepP ? (tmem + lane_addr + kPCol + g * 128) : tS) + h * 32;
    const float sl2 = p.scale_log2;
    float m_run = -INFINITY;
    float l_run = 0.f;
    for (int j = 0; j < nkv; ++j) {
      kwait<D>(&s_full[g], static_cast<uint32_t>(j & 1));
      if (h == 0 && threadIdx.x % 128 == 0) trace_stamp(p, 2 * g, j);
      ptx::tc_fence_after();
      float s[64];
      ptx::tmem_ld32(tS + h * 64, *reinterpret_cast<float(*)[32]>(&s[0]));
      ptx::tmem_ld32(tS + h * 64 + 32, *reinterpret_cast<float(*)[32]>(&s[32]));
      ptx::tmem_wait_ld();
      PHASE(0);
      if constexpr (kSepP) {
        ptx::tc_fence_before();
        ptx::mbar_arrive(&s_free[g]);
      }
      const int tile_lim = klim_t - j * kBN;
      const bool masked = !__all_sync(0xffffffffu, tile_lim >= kBN);  // same in both halves
      if (masked) {
        const int nv = tile_lim - h * 64;
        const int nvalid = nv < 0 ? 0 : (nv > 64 ? 64 : nv);
#pragma unroll
        for (int c = 0; c < 64; ++c) s[c] = c < nvalid ? s[c] : -INFINITY;
      }
      const float pmax = sm::row_max64(s);
      float* red_t = red + ((j & 1) * 2 + g) * 2 * kBM;
      red_t[h * kBM + r] = pmax;
      PHASE(1);
      asm volatile("bar.sync %0, 256;" ::"r"(1 + g) : "memory");
      PHASE(2);
      const float mt = fmaxf(pmax, red_t[(h ^ 1) * kBM + r]) * sl2;
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
      if constexpr (kSepP) {
        // exponentials first, then wait for PV_g(j-1) to have read P_g(j-1)
        if (kEmu == 0 || masked)
          sm::exp_inplace64<0>(s, sl2, m_use);
        else
          sm::exp_inplace64<(kEmu > 4 ? 4 : kEmu)>(s, sl2, m_use);
        PHASE(3);
        if (j > 0) {
          kwait<D>(&pv_done[g], static_cast<uint32_t>((j - 1) & 1));
          ptx::tc_fence_after();
        }
        PHASE(4);
        l_run += sm::store_p64(s, tP);
      } else {
        l_run += sm::exp_half(s, sl2, m_use, tP);
      }
      if (warp_rescale && j > 0) {  // this half's D/2 columns of O
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          float o[32];
          ptx::tmem_ld32(tO + c * 32, o);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] *= alpha;
          ptx::tmem_st32(tO + c * 32, o);
        }
      }
      ptx::tmem_wait_st();
      PHASE(5);
      ptx::tc_fence_before();
      if (h == 0 && threadIdx.x % 128 == 0) trace_stamp(p, 2 * g + 1, j);
      ptx::mbar_arrive(&p_ready[g]);
    }
    if (nkv > 0) {
      kwait<D>(&o_final[g], 0);
      ptx::tc_fence_after();
    }
    const int64_t li = static_cast<int64_t>(head) * p.Lq + row;
    const bool fused = p.out_mode >= OUT_COMBINE_ACC;
    // both halves read lse_acc before the barrier; h = 0 writes it after
    const float la = (fused && row_ok) ? p.acc_lse[li] : 0.f;
    redl[(g * 2 + h) * kBM + r] = l_run;
    asm volatile("bar.sync %0, 256;" ::"r"(1 + g) : "memory");
    const float l_tot = l_run + redl[(g * 2 + (h ^ 1)) * kBM + r];
    const bool empty = !(l_tot > 0.f);
    const float inv_l = empty ? 0.f : 1.f / l_tot;
    const float lse_s = empty ? -INFINITY : (m_run + __log2f(l_tot)) * 0.69314718055994530942f;
    float wa = 0.f, wp = 0.f, lnew = lse_s;
    if (fused && row_ok) merge_weights(la, lse_s + p.lse_bias, wa, wp, lnew);
    if (row_ok && h == 0) {
      if (p.out_mode == OUT_COMBINE_ACC) p.acc_lse[li] = lnew;
      else lse_ptr[li] = lnew;
    }
    const int64_t obase = (row * p.H + head) * static_cast<int64_t>(D) + h * (D / 2);
#pragma unroll
    for (int c = 0; c < D / 64; ++c) {
      float o[32];
      if (nkv > 0) {
        ptx::tmem_ld32(tO + c * 32, o);
        ptx::tmem_wait_ld();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = 0.f;
      }
      if (row_ok && fused) {
        float4* acc = reinterpret_cast<float4*>(p.acc_o + obase + c * 32);
        float rr[32];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float4 a4 = acc[e];
          rr[4 * e + 0] = combine_one(a4.x, __fmul_rn(o[4 * e + 0], inv_l), wa, wp);
          rr[4 * e + 1] = combine_one(a4.y, __fmul_rn(o[4 * e + 1], inv_l), wa, wp);
          rr[4 * e + 2] = combine_one(a4.z, __fmul_rn(o[4 * e + 2], inv_l), wa, wp);
          rr[4 * e + 3] = combine_one(a4.w, __fmul_rn(o[4 * e + 3], inv_l), wa, wp);
        }
        if (p.out_mode == OUT_COMBINE_ACC) {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            acc[e] = make_float4(rr[4 * e], rr[4 * e + 1], rr[4 * e + 2], rr[4 * e + 3]);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out_ptr) + obase +
                                                c * 32);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint32_t wd[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              __nv_bfloat162 b = __floats2bfloat162_rn(rr[8 * e + 2 * t], rr[8 * e + 2 * t + 1]);
              wd[t] = *reinterpret_cast<uint32_t*>(&b);
            }
            dst[e] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
          }
        }
      } else if (row_ok) {
        if (p.out_mode == OUT_PARTIAL_F32) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(out_ptr) + obase + c * 32);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            dst[e] = make_float4(__fmul_rn(o[4 * e], inv_l), __fmul_rn(o[4 * e + 1], inv_l),
                                 __fmul_rn(o[4 * e + 2], inv_l), __fmul_rn(o[4 * e + 3], inv_l));
        } else {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out_ptr) + obase +
                                                c * 32);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint32_t wd[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              __nv_bfloat162 b = __floats2bfloat162_rn(o[8 * e + 2 * t] * inv_l,
                                                       o[8 * e + 2 * t + 1] * inv_l);
              wd[t] = *reinterpret_cast<uint32_t*>(&b);
            }
            dst[e] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
          }
        }
      }
    }
  } else if (!kSplit && warp < 8) {
    // ------------------------------------------------------------ softmax
    const int g = warp >> 2;                  // Q tile of this warpgroup
    const int quarter = warp & 3;             // TMEM lane quarter
    const int r = quarter * 32 + lane;        // row within the tile
    const int64_t row = m0 + g * kBM + r;     // local query row
    const bool row_ok = row < p.Lq;
    const int64_t qp = pos_of(p.qmap, row_ok ? row : p.Lq - 1);
    const int64_t klim = key_limit(p, qp);
    const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_addr + g * kBN;
    const uint32_t tO = tmem + lane_addr + 256 + g * 128;
    const float sl2 = p.scale_log2;

    float m_run = -INFINITY;  // running max, log2 units (scaled)
    float l_run = 0.f;
    for (int j = 0; j < nkv; ++j) {
      kwait<D>(&s_full[g], static_cast<uint32_t>(j & 1));
      if (threadIdx.x % 128 == 0) trace_stamp(p, 2 * g, j);
      ptx::tc_fence_after();
      // Turn-taking (p.alt, DMHA_ALT=1): the two softmax warpgroups run their
      // exponentials one after the other — WG1 starts tile j when WG0 has
      // finished it, WG0 starts tile j+1 when WG1 has finished tile j (named
      // barriers 1 = "WG0 may go", 2 = "WG1 may go"; 128 arrive + 128 sync).
      const bool alt = !kSepP && p.alt;
      auto turn_wait = [&]() {
        if (alt && (g == 1 || j > 0)) asm volatile("bar.sync %0, 256;" ::"r"(1 + g) : "memory");
      };
      auto turn_done = [&]() {
        if (alt) asm volatile("bar.arrive %0, 256;" ::"r"(2 - g) : "memory");
      };
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        ptx::tmem_ld32(tS + c * 32, *reinterpret_cast<float(*)[32]>(&s[c * 32]));
      ptx::tmem_wait_ld();
      if (g == 0 && threadIdx.x == 0) trace_stamp(p, 7, j);
      if constexpr (kSepP) {  // S_g is in registers: the tensor core may overwrite it
        ptx::tc_fence_before();
        ptx::mbar_arrive(&s_free[g]);
      }

      int64_t nv64 = klim - static_cast<int64_t>(jt0 + j) * kBN;
      const int nvalid = nv64 < 0 ? 0 : (nv64 > kBN ? kBN : static_cast<int>(nv64));
      const bool masked = !__all_sync(0xffffffffu, nvalid >= kBN);
      if (masked) {
#pragma unroll
        for (int c = 0; c < 128; ++c) s[c] = c < nvalid ? s[c] : -INFINITY;
      }
      const float mt = sm::row_max128(s) * sl2;
      const bool need = mt > m_run + kRescaleThreshold;
      const bool warp_rescale = __any_sync(0xffffffffu, need);
      float alpha = 1.f;
      if (warp_rescale) {
        const float m_new = fmaxf(m_run, mt);
        alpha = (m_new == -INFINITY) ? 1.f : ptx::ex2_approx(m_run - m_new);
        l_run *= alpha;
        m_run = m_new;
      }
      // only the exponential phase is serialised by the turn-taking: the S
      // load and row max above overlap the other warpgroup's exponentials
      turn_wait();
      // P = exp2(S*scale*log2e - m) -> bf16, written over the first 64 columns
      // of S (D = 64: into P_g) in 16-column chunks so the fp32 scores die as P
      // is produced.
      if (g == 0 && threadIdx.x == 0) trace_stamp(p, 8, j);
      const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
      const uint32_t tP = kSepP ? (tmem + lane_addr + kPCol + g * 128) : tS;
      // Unmasked tiles send kEmu of every 8 column pairs to the FMA-pipe
      // polynomial; masked tiles (-inf entries, exact zeros needed) use MUFU only.
      if constexpr (kSepP) {
        // D = 64: exponentials first (in registers), THEN wait for PV_g(j-1) to
        // have read P_g(j-1) (and to have finished O_g, for the rescale), then
        // store P_g(j): the PV latency hides behind the MUFU work instead of
        // sitting between the row max and the exponentials.
        if (kEmu == 0 || masked)
          sm::exp_inplace<0>(s, sl2, m_use);
        else
          sm::exp_inplace<(kEmu > 4 ? 4 : kEmu)>(s, sl2, m_use);
        if (j > 0) {
          kwait<D>(&pv_done[g], static_cast<uint32_t>((j - 1) & 1));
          ptx::tc_fence_after();
        }
        if constexpr (kPS) {
          l_run += sm::store_p_smem(s, sP + g * (kBM * kBN * 2), r);
          ptx::fence_proxy_async_smem();
        } else {
          l_run += sm::store_p(s, tP);
        }
      } else if (kEmu == 0 || masked) {
#if DMHA_EXPFORM == 1
        // packed FFMA2 / FADD2 (two scores per FMA-pipe instruction)
        l_run += sm::exp_tile<0>(s, sl2, m_use, tP);
#else
        // scalar FFMA + MUFU.EX2; DMHA_EXPFORM == 2: the scale as an immediate
        // (FFMA R, R, imm, R) and FADD2 sums
#if DMHA_EXPFORM == 2
        constexpr float kSl2 = D == 64 ? 0.18033688011112042f : 0.12751743082459868f;
        float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#else
        const float kSl2 = sl2;
        float sum0 = 0.f, sum1 = 0.f;
#endif
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float e0 = ptx::ex2_approx(fmaf(s[32 * c + 2 * e], kSl2, -m_use));
            const float e1 = ptx::ex2_approx(fmaf(s[32 * c + 2 * e + 1], kSl2, -m_use));
#if DMHA_EXPFORM == 2
            acc2[e & 1] = __fadd2_rn(acc2[e & 1], make_float2(e0, e1));
#else
            sum0 += e0;
            sum1 += e1;
#endif
            __nv_bfloat162 b = __floats2bfloat162_rn(e0, e1);
            pk[e] = *reinterpret_cast<uint32_t*>(&b);
          }
          ptx::tmem_st16(tP + c * 16, pk);
        }
#if DMHA_EXPFORM == 2
        l_run += (acc2[0].x + acc2[0].y) + (acc2[1].x + acc2[1].y);
#else
        l_run += sum0 + sum1;
#endif
#endif
      } else {
        l_run += sm::exp_tile<kEmu>(s, sl2, m_use, tP);
      }
      turn_done();
      // O_g holds PV_g(j-1) (complete: covered by the S_g(j) commit, or by the
      // pv_done wait when D = 64) and PV_g(j) is not issued before p_ready, so
      // O can be rescaled in place here.
      if (warp_rescale && j > 0) {
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
      ptx::mbar_arrive(&p_ready[g]);
    }
    // WG0 consumes WG1's hand-over of the last tile (no dangling arrival)
    if (!kSepP && p.alt && g == 0 && nkv > 0) asm volatile("bar.sync 1, 256;" ::: "memory");
    if (nkv > 0) {
      kwait<D>(&o_final[g], 0);
      ptx::tc_fence_after();
    }
    // ---------------------------------------------------------- epilogue
    const bool empty = !(l_run > 0.f);
    const float inv_l = empty ? 0.f : 1.f / l_run;
    const float lse_s = empty ? -INFINITY : (m_run + __log2f(l_run)) * 0.69314718055994530942f;
    const int64_t li = static_cast<int64_t>(head) * p.Lq + row;
    // NEXT-2 fused combine: merge with the running accumulator here instead of
    // writing an fp32 partial for lse_combine (same arithmetic, same bits).
    const bool fused = p.out_mode >= OUT_COMBINE_ACC;
    float wa = 0.f, wp = 0.f, lnew = lse_s;
    if (fused && row_ok) merge_weights(p.acc_lse[li], lse_s + p.lse_bias, wa, wp, lnew);
    if (row_ok) {
      if (p.out_mode == OUT_COMBINE_ACC) p.acc_lse[li] = lnew;
      else lse_ptr[li] = lnew;
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
      if (row_ok && fused) {
        float4* acc = reinterpret_cast<float4*>(p.acc_o + obase + c * 32);
        float r[32];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float4 a4 = acc[e];
          r[4 * e + 0] = combine_one(a4.x, __fmul_rn(o[4 * e + 0], inv_l), wa, wp);
          r[4 * e + 1] = combine_one(a4.y, __fmul_rn(o[4 * e + 1], inv_l), wa, wp);
          r[4 * e + 2] = combine_one(a4.z, __fmul_rn(o[4 * e + 2], inv_l), wa, wp);
          r[4 * e + 3] = combine_one(a4.w, __fmul_rn(o[4 * e + 3], inv_l), wa, wp);
        }
        if (p.out_mode == OUT_COMBINE_ACC) {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            acc[e] = make_float4(r[4 * e], r[4 * e + 1], r[4 * e + 2], r[4 * e + 3]);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out_ptr) + obase +
                                                c * 32);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint32_t w[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              __nv_bfloat162 b = __floats2bfloat162_rn(r[8 * e + 2 * t], r[8 * e + 2 * t + 1]);
              w[t] = *reinterpret_cast<uint32_t*>(&b);
            }
            dst[e] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      } else if (row_ok) {
        if (p.out_mode == OUT_PARTIAL_F32) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(out_ptr) + obase + c * 32);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            dst[e] = make_float4(__fmul_rn(o[4 * e], inv_l), __fmul_rn(o[4 * e + 1], inv_l),
                                 __fmul_rn(o[4 * e + 2], inv_l), __fmul_rn(o[4 * e + 3], inv_l));
        } else {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out_ptr) + obase +
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
  if (threadIdx.x == 0) cta_stamp(p, 1);
}

// ---------------------------------------------------------------- host side
template <int D, int E, bool S, int I = 2, bool PS = false>
cudaError_t launch_de(const LocalAttnArgs& a, cudaStream_t stream) {
  using C = Cfg<D, PS>;
  CUtensorMap tq, tk, tv;
  if (!make_tma_map_bf16(&tq, a.q, a.Lq, a.H, D, kBM) || !make_tma_map_bf16(&tk, a.k, a.Lk, a.H, D, kBN) ||
      !make_tma_map_bf16(&tv, a.v, a.Lk, a.H, D, kBN))
    return cudaErrorInvalidValue;
  // the dynamic shared-memory limit is a per-device function attribute
  static int attr_dev = -1;
  int cur_dev = 0;
  cudaGetDevice(&cur_dev);
  if (attr_dev != cur_dev) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_sm100_kernel<D, E, S, I, PS>,
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
  p.out2 = a.out2;
  p.lse2 = a.lse2;
  p.kv_split = a.kv_split == 2 ? 2 : 1;
  p.n_mblk = static_cast<int>((a.Lq + 2 * kBM - 1) / (2 * kBM));
  p.lse_bias = a.lse_bias;
  p.alt = 0;
  if (const char* e = std::getenv("DMHA_ALT")) p.alt = std::atoi(e) != 0;
  p.trace = g_trace;
  dim3 grid(p.n_mblk, a.H, p.kv_split);
  attn_fwd_sm100_kernel<D, E, S, I, PS><<<grid, Roles<S>::kThreads, C::kSmemBytes, stream>>>(tq, tk, tv, p);
  return cudaGetLastError();
}


// Measurement knobs (defaults = the measured-fastest configuration):
//  DMHA_EMU     = pairs (of every 8) of score columns on the FMA-pipe exp2 (0)
//  DMHA_ISSUERS = MMA-issuing threads: 1 = one for both Q tiles (D = 128
//                 default), 2 = one per Q tile, 3 = split S / PV issuers
//                 (D = 64 default), 4 = S issuer + one PV issuer per Q tile
//                 (3 and 4: separate-P schedules only)
//  DMHA_SPLIT   = 1: split-row softmax (16 softmax warps; D = 64 default)
//  DMHA_PS      = 1: D = 128 with P in shared memory (separate-P schedule)
struct PingpongConfig {
  bool split;
  int iss;
  bool ps;
};
PingpongConfig pingpong_config(int D) {
  // D = 64 default: the split softmax (16 softmax warps, two per row) with
  // split S / PV issuing warps (DESIGN.md §5 lessons 16-17, 33: one issuer
  // per Q tile was the round-1 choice; on the final build the S / PV split is
  // +5 % on small grids and level at million scale)
  PingpongConfig c{D == 64, 1, false};
  if (const char* e = std::getenv("DMHA_SPLIT")) c.split = std::atoi(e) != 0;
  if (const char* e = std::getenv("DMHA_PS")) c.ps = D == 128 && std::atoi(e) != 0;
  if (c.ps) c.split = false;
  c.iss = D == 64 ? 3 : 1;
  if (const char* e = std::getenv("DMHA_ISSUERS")) c.iss = std::atoi(e);
  return c;
}

template <int D, bool S, int I, bool PS = false>
cudaError_t launch_emu(int emu, const LocalAttnArgs& a, cudaStream_t stream) {
  switch (emu) {
    case 1: return launch_de<D, 1, S, I, PS>(a, stream);
    case 2: return launch_de<D, 2, S, I, PS>(a, stream);
    case 3: return launch_de<D, 3, S, I, PS>(a, stream);
    default: return launch_de<D, 0, S, I, PS>(a, stream);
  }
}

template <int D>
cudaError_t launch_d(const LocalAttnArgs& a, cudaStream_t stream) {
  int emu = 0;
  if (const char* e = std::getenv("DMHA_EMU")) emu = std::atoi(e);
  const PingpongConfig cfg = pingpong_config(D);
  const int iss = cfg.iss;
  if constexpr (D == 128) {
    if (cfg.ps) {  // separate-P schedule, P in shared memory
      switch (iss) {
        case 2: return launch_emu<D, false, 2, true>(emu, a, stream);
        case 3: return launch_de<D, 0, false, 3, true>(a, stream);
        case 4: return launch_de<D, 0, false, 4, true>(a, stream);
        default: return launch_emu<D, false, 1, true>(emu, a, stream);
      }
    }
  }
  if (cfg.split) {
    if (iss == 2) {
      if constexpr (D == 64) return launch_emu<D, true, 2>(emu, a, stream);
      return launch_de<D, 0, true, 2>(a, stream);
    }
    if constexpr (D == 64) {
      if (iss == 4) return launch_de<D, 0, true, 4>(a, stream);
      if (iss == 3) return launch_emu<D, true, 3>(emu, a, stream);
    }
    if (a.out_mode >= OUT_COMBINE_ACC) return cudaErrorInvalidValue;  // see pingpong_fused_combine_ok
    return launch_de<D, 0, true, 1>(a, stream);
  }
  if (iss == 2) return launch_emu<D, false, 2>(emu, a, stream);
  if constexpr (D == 64) {
    if (iss == 4) return launch_de<D, 0, false, 4>(a, stream);
    if (iss == 3) return launch_emu<D, false, 3>(emu, a, stream);
  }
  return launch_emu<D, false, 1>(emu, a, stream);
}

}  // namespace

unsigned long long* g_trace = nullptr;

bool pingpong_fused_combine_ok(int D) {
  // The one-thread-per-row epilogue merges; so does the split softmax's when
  // it runs with per-tile or split issuers (the D = 64 configurations).  The
  // D = 128 split softmax (single issuer) keeps the separate combine pass.
  const PingpongConfig c = pingpong_config(D);
  return c.ps || !c.split || (D == 64 && (c.iss == 2 || c.iss == 3 || c.iss == 4));
}

bool attn_fused_combine_supported(int D) {
  return (D == 64 || D == 128) && pingpong_fused_combine_ok(D);
}

bool attn_kv_split_supported(int D) { return attn_fused_combine_supported(D); }

cudaError_t launch_attn_fwd_bf16(const LocalAttnArgs& a, cudaStream_t stream) {
  if (a.Lq <= 0) return cudaSuccess;
  if (a.kv_split != 1 && (!attn_kv_split_supported(a.D) || a.out_mode != OUT_PARTIAL_F32))
    return cudaErrorInvalidValue;
  if (a.out_mode >= OUT_COMBINE_ACC && !attn_fused_combine_supported(a.D))
    return cudaErrorInvalidValue;
  if (a.Lq > INT32_MAX || a.Lk > INT32_MAX) return cudaErrorInvalidValue;
  if (a.D == 64) return launch_d<64>(a, stream);
  if (a.D == 128) return launch_d<128>(a, stream);
  return cudaErrorInvalidValue;
}

}  // namespace dmha
