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
// Structure:
//  * CTA = one 128-row query tile of one head; CTAs run in clusters of 2 that
//    work on adjacent query tiles of the same head and share every K/V tile:
//    each CTA TMA-loads half of the tile's rows and multicasts it into both
//    CTAs' shared memory, so L2 -> SM traffic is one K/V tile per 256 rows.
//  * S is triple-buffered in TMEM, so QK^T of tiles j+1, j+2 runs on the
//    tensor core while the softmax of tile j runs; the per-tile loop is bounded
//    by max(tensor core, softmax) instead of their sum (the single-buffer
//    design measured ~3300 cycles/tile for 2048 cycles of MMA).
//  * 12 warps: 0-7 softmax (warpgroup w owns the KV tiles j = w mod 2 and
//    S buffer w; thread t <-> TMEM lane t <-> row t, a full 128-column score
//    row per thread; only the running max is handed between the warpgroups),
//    8 TMA producer, 9 TMEM allocator + tcgen05.mma issuer (whole warp,
//    elect.sync issues), 10-11 idle.
//  * TMEM (512 cols): S buffers [0,128), [128,256), [256,384); O [384, 384+D).
//    P(j) (bf16x2) overwrites the first 64 columns of S buffer j%3.
//  * MMA issue order (tcgen05.mma executes in order): S(0), S(1), S(2), then
//    per tile j: PV(j) [after P(j) ready], S(j+3) into the buffer PV(j) just
//    read.  K/V ring slots are loaded in exactly this order (K0 K1 K2 V0 K3 V1
//    K4 ...).
//  * Online softmax in the exp2 domain with a stale running max: O is rescaled
//    only when the tile max exceeds the running max by more than 8 (factor
//    256) — exact because l and O always share the subtracted max.  The rare
//    rescale first waits for PV(j-1) (pv_done barrier).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "tma_map.h"
#include "ptx_sm100.cuh"
#include "softmax_sm100.cuh"

namespace dmha {
extern unsigned long long* g_trace;
namespace {

constexpr int kBM = 128;          // query rows per CTA (MMA M)
constexpr int kBN = 128;          // keys per tile (MMA N of QK^T, K of PV)
constexpr int kThreads = 384;     // 12 warps
constexpr int kProducerWarp = 8;
constexpr int kMmaWarp = 9;       // TMEM allocator; MMA issuer (pair path: S = QK^T only)
constexpr int kPvWarp = 10;       // pair path: issues PV MMAs
constexpr float kRescaleThreshold = 8.0f;  // log2 units: rescale when max grows by > 2^8
constexpr int kNB = 3;            // S buffers in TMEM (S(t+3) reuses buffer t%3 after PV(t))
constexpr int kOCol = kNB * kBN;  // first TMEM column of O

// K2 = true: CTA-pair MMA (tcgen05 cta_group::2, M = 256).  Each CTA holds
// its own 128 query rows and HALF of every K/V tile (64 keys of K, D/2 columns
// of V), so L2->SMEM traffic is one K/V tile per 256 query rows and the pair
// leader issues one MMA per 256 rows.  K2 = false: each CTA issues its own
// M = 128 MMAs; the pair still shares K/V tiles by TMA multicast (each CTA
// loads half and multicasts it into both).
template <int D, bool K2>
struct Cfg {
  static constexpr int kPanels = D / 64;                    // 128-byte swizzle panels per row
  static constexpr int kPanelBytes = 128 * 128;             // 128 rows x 128 B
  static constexpr int kTileBytes = kPanels * kPanelBytes;  // one 128 x D bf16 tile
  static constexpr int kHalfBytes = kPanelBytes / 2;        // 64 rows of one panel
  static constexpr int kQBytes = kTileBytes;                // this CTA's query tile
  static constexpr int kSlotBytes = K2 ? kTileBytes / 2 : kTileBytes;  // one K/V ring slot
  static constexpr int kKPanelStride = K2 ? kHalfBytes : kPanelBytes;   // K panel stride in a slot
  static constexpr int kStages = K2 ? 11 : ((D == 128) ? 5 : 10);       // K/V ring slots
  static constexpr int kQOff = 0;
  static constexpr int kKVOff = kQBytes;
  static constexpr int kRedOff = kKVOff + kStages * kSlotBytes;  // m hand-off [2][128] + l/m [2][2][128]
  static constexpr int kBarOff = kRedOff + 6 * 128 * 4;
  static constexpr int kSmemBytes = kBarOff + 512 + 1024;   // + barriers + align slack
  // Default number (of every 8) of score-column pairs whose exp2 runs as a
  // polynomial on the FMA pipe instead of MUFU (D=64 has half the MMA work per
  // exponential of D=128).  Overridable per launch for measurement (DMHA_EMU).
  static constexpr int kEmuDefault = 0;  // measured best on B200 for both D
  static constexpr uint32_t kM = K2 ? 256 : kBM;
  static constexpr uint32_t kIdescQK = ptx::make_idesc(1, kM, kBN, 0, 0);
  static constexpr uint32_t kIdescPV = ptx::make_idesc(1, kM, D, 0, 1);  // V is MN-major
  static_assert(!K2 || D == 128, "the CTA-pair path splits V by 64-column panels (D = 128)");
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
  int n_pairs;  // CTA pairs along the query axis
  unsigned long long* trace;  // debug timeline (dmha_debug_set_trace), usually null
};

// Timeline trace (measurement hook): clock64 stamps for the first kTraceCtas
// CTAs of head 0 and their first kTraceTiles KV tiles.  Events:
//  0/2: softmax WG0/WG1 saw S(j)   1/3: WG0/WG1 arrive P(j) ready
//  4: MMA saw P(j) ready   5: MMA issued PV(j)   6: MMA issued S(j)
//  7: MMA saw V_j landed    8: producer issued the V_j load
constexpr int kTraceCtas = 4, kTraceEvents = 9, kTraceTiles = 64;
__device__ __forceinline__ void trace_stamp(const Params& p, int ev, int j) {
  if (p.trace != nullptr && blockIdx.y == 0 && blockIdx.x < kTraceCtas && j < kTraceTiles)
    p.trace[(blockIdx.x * kTraceEvents + ev) * kTraceTiles + j] = clock64();
}

// Named barrier over the 256 softmax threads (both warpgroups).
__device__ __forceinline__ void halves_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

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

// KV tiles the query rows [r0, r0 + n) need (a prefix of the key tiles).
__device__ __forceinline__ int tiles_for_rows(const Params& p, int64_t r0, int64_t n) {
  if (r0 >= p.Lq) return 0;
  int64_t last = r0 + n - 1;
  if (last > p.Lq - 1) last = p.Lq - 1;
  const int64_t lim = key_limit(p, pos_of(p.qmap, last));
  return static_cast<int>((lim + kBN - 1) / kBN);
}

// The K/V load/consume sequence shared by producer and MMA issuer:
//   K0, K1, K2, V0, K3, V1, K4, ..., V_{n-1}   (K_{t+3} right after V_t)
// item i -> (is_v, tile).
__device__ __forceinline__ void seq_item(int i, int n, bool& is_v, int& t) {
  const int lead = n < kNB ? n : kNB;  // leading K loads
  if (i < lead) {
    is_v = false;
    t = i;
    return;
  }
  const int k = i - lead;  // pairs (V_t, K_{t+kNB}) while t + kNB < n, then V only
  const int paired = n > kNB ? n - kNB : 0;
  if (k < 2 * paired) {
    is_v = (k & 1) == 0;
    t = is_v ? (k >> 1) : (k >> 1) + kNB;
  } else {
    is_v = true;
    t = paired + (k - 2 * paired);
  }
}

template <int D, int kEmu, bool K2>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q,
                          const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const Params p) {
  using C = Cfg<D, K2>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem + C::kQOff;
  uint8_t* sKV = smem + C::kKVOff;
  float* red = reinterpret_cast<float*>(smem + C::kRedOff);  // [tile parity][half][row]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + C::kStages;
  // Every barrier below is indexed so that its waiter can never be two phases
  // behind (parity waits are only exact within one phase):
  //  s_full[t%3]  S(t) written      — S(t+3) needs PV(t), i.e. P(t) consumed
  //  p_ready[t%3] P(t) written      — P(t+3) needs S(t+3), issued after PV(t)
  //  pv_done[..]  PV(t) complete    — per-CTA path: pv_done[t%2], waited (for
  //               the rare O rescale) by tile t+1's softmax, when PV(t-2) is
  //               known complete (S(t+1) was issued after it) and PV(t+2)
  //               cannot have been issued.  Pair path: pv_done[t%3], also
  //               waited by the S issuer before S(t+3) reuses buffer t%3.
  //  o_final      last PV complete  — one phase
  uint64_t* s_full = kv_empty + C::kStages;  // [3]
  uint64_t* p_ready = s_full + kNB;          // [3]
  uint64_t* pv_done = p_ready + kNB;         // [3]
  uint64_t* o_final = pv_done + 3;           // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_final + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  const uint32_t crank = ptx::cluster_ctarank();
  // Causal: heaviest query pairs first.
  const int pair = p.causal ? (p.n_pairs - 1 - static_cast<int>(blockIdx.x >> 1))
                            : static_cast<int>(blockIdx.x >> 1);
  const int64_t m_pair = static_cast<int64_t>(pair) * (2 * kBM);
  const int64_t m0 = m_pair + crank * kBM;
  const int n_load = tiles_for_rows(p, m_pair, 2 * kBM);  // tiles the pair streams
  // With the pair MMA both CTAs step through the pair's tiles together (rows a
  // tile does not reach are masked); otherwise a CTA stops at its own last tile.
  const int n_own = K2 ? n_load : tiles_for_rows(p, m0, kBM);
  const int n_items = 2 * n_load;

  if (warp == kProducerWarp && lane == 0) {
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], K2 ? 1 : 2);  // released by the MMA issuer(s) of the pair
    }
    for (int b = 0; b < kNB; ++b) {
      ptx::mbar_init(&s_full[b], 1);
      // K2: one arrive per softmax warp of both CTAs (on the leader's barrier);
      // else the 128 threads of the tile's warpgroup.
      ptx::mbar_init(&p_ready[b], K2 ? 8 : kBM);
    }
    for (int b = 0; b < 3; ++b) ptx::mbar_init(&pv_done[b], 1);
    ptx::mbar_init(o_final, 1);
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == kMmaWarp) {
    if (K2)
      ptx::tmem_alloc_2cta<512>(tmem_slot);
    else
      ptx::tmem_alloc<512>(tmem_slot);
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();  // peer barriers initialised before any multicast lands
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kProducerWarp) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && K2) {
      // Pair MMA: each CTA loads its own Q rows and its half of every K/V tile
      // into its own shared memory; completion is counted on the leader's
      // barriers (the leader alone waits on them and issues the MMAs).
      const uint32_t q_full_l = ptx::mapa_cluster(q_full, 0);
      if (n_load > 0) {
        if (crank == 0) ptx::mbar_arrive_expect_tx(q_full, 2 * C::kQBytes);
        for (int pn = 0; pn < C::kPanels; ++pn)
          ptx::tma_load_3d_2sm(&tm_q, q_full_l, sQ + pn * C::kPanelBytes, pn * 64, head,
                               static_cast<int32_t>(m0));
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < n_items; ++i) {
        bool is_v;
        int t;
        seq_item(i, n_load, is_v, t);
        ptx::mbar_wait(&kv_empty[stage], phase ^ 1);
        if (is_v) trace_stamp(p, 8, t);
        if (crank == 0) ptx::mbar_arrive_expect_tx(&kv_full[stage], 2 * C::kSlotBytes);
        const uint32_t full_l = ptx::mapa_cluster(&kv_full[stage], 0);
        uint8_t* slot = sKV + stage * C::kSlotBytes;
        if (!is_v) {  // K: keys [64*crank, 64*crank+64) of the tile, all D columns
          for (int pn = 0; pn < C::kPanels; ++pn)
            ptx::tma_load_3d_2sm(&tm_k, full_l, slot + pn * C::kKPanelStride, pn * 64, head,
                                 t * kBN + static_cast<int>(crank) * 64);
        } else {      // V: all 128 keys of the tile, columns [64*crank, 64*crank+64)
          ptx::tma_load_3d_2sm(&tm_v, full_l, slot, static_cast<int>(crank) * 64, head, t * kBN);
        }
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      }
      for (int i = 0; i < C::kStages; ++i) {  // drain (see below)
        ptx::mbar_wait(&kv_empty[stage], phase ^ 1);
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      }
    } else if (lane == 0) {
      if (n_own > 0) {
        ptx::mbar_arrive_expect_tx(q_full, C::kQBytes);
        for (int pn = 0; pn < C::kPanels; ++pn)
          ptx::tma_load_3d(&tm_q, q_full, sQ + pn * C::kPanelBytes, pn * 64, head,
                           static_cast<int32_t>(m0));
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < n_items; ++i) {
        bool is_v;
        int t;
        seq_item(i, n_load, is_v, t);
        ptx::mbar_wait(&kv_empty[stage], phase ^ 1);
        if (is_v) trace_stamp(p, 8, t);
        ptx::mbar_arrive_expect_tx(&kv_full[stage], C::kTileBytes);
        // This CTA loads rows [64*crank, 64*crank+64) of the tile into both CTAs.
        const CUtensorMap* tm = is_v ? &tm_v : &tm_k;
        for (int pn = 0; pn < C::kPanels; ++pn)
          ptx::tma_load_3d_mc(tm, &kv_full[stage],
                              sKV + stage * C::kSlotBytes + pn * C::kPanelBytes +
                                  crank * C::kHalfBytes,
                              pn * 64, head, t * kBN + static_cast<int>(crank) * 64, 0x3);
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      }
      // Drain: every slot's last fill released by the pair, so no remote
      // arrive can target this CTA's shared memory after it exits.
      for (int i = 0; i < C::kStages; ++i) {
        ptx::mbar_wait(&kv_empty[stage], phase ^ 1);
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs this loop (converged, warp-uniform operands); one
    // elected lane issues each tcgen05 instruction.
    // Operands are kept warp-uniform and 32-bit: descriptors are passed as
    // their low word (start address >> 4 in [0,14), LBO >> 4 in [16,30)) plus
    // a constant high word (SBO = 1024 B, version 1, SWIZZLE_128B).  The start
    // field holds the shared address modulo 2^18 (a CTA of a cluster can sit
    // above 256 KB in the shared window), hence the 14-bit mask.
    constexpr uint32_t kDescHi = (1024u >> 4) | (1u << 14) | (2u << 29);
    constexpr uint32_t kLboK = (16u >> 4) << 16;                        // K-major: unused
    constexpr uint32_t kLboV = (uint32_t(C::kPanelBytes) >> 4) << 16;   // MN-major V: panel stride
    const uint32_t sal = ptx::smem_u32(smem);
    const uint32_t q_lo = (((sal + C::kQOff) >> 4) & 0x3FFFu) | kLboK;
    const uint32_t k_lo = (((sal + C::kKVOff) >> 4) & 0x3FFFu) | kLboK;
    const uint32_t v_lo = (((sal + C::kKVOff) >> 4) & 0x3FFFu) | kLboV;
    if (!K2) {
      if (n_own > 0) ptx::mbar_wait(q_full, 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < n_items; ++i) {
        bool is_v;
        int t;
        seq_item(i, n_load, is_v, t);
        ptx::mbar_wait(&kv_full[stage], phase);
        if (is_v && lane == 0) trace_stamp(p, 7, t);
        ptx::tc_fence_after();
        const uint32_t soff = static_cast<uint32_t>(stage) * (C::kSlotBytes >> 4);
        if (t < n_own) {
          const uint32_t sbuf = tmem + static_cast<uint32_t>(t % kNB) * kBN;  // S(t) columns
          if (!is_v) {
            // S(t) = Q K_t^T into S buffer t%3 (after PV(t-3) read P(t-3) there)
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t aoff = ((kk >> 2) * C::kPanelBytes + (kk & 3) * 32) >> 4;
              const uint32_t boff = ((kk >> 2) * C::kKPanelStride + (kk & 3) * 32) >> 4;
              ptx::mma_bf16_ss_lo(sbuf, q_lo + aoff, k_lo + soff + boff, kDescHi, C::kIdescQK, kk > 0);
            }
            ptx::mma_commit_w(&s_full[t % kNB]);
            if (lane == 0) trace_stamp(p, 6, t);
          } else {
            // O += P(t) V_t, P(t) read from TMEM (S buffer t%3)
            ptx::mbar_wait(&p_ready[t % kNB], static_cast<uint32_t>((t / kNB) & 1));
            if (lane == 0) trace_stamp(p, 4, t);
            ptx::tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < kBN / 16; ++kk)
              ptx::mma_bf16_ts_lo(tmem + kOCol, sbuf + kk * 8, v_lo + soff + ((kk * 16 * 128) >> 4),
                                  kDescHi, C::kIdescPV, (t > 0 || kk > 0) ? 1u : 0u);
            ptx::mma_commit_w(&pv_done[t & 1]);
            if (t == n_own - 1) ptx::mma_commit_w(o_final);
            if (lane == 0) trace_stamp(p, 5, t);
          }
        }
        ptx::mma_commit_mc_w(&kv_empty[stage], 0x3);  // release the slot in both CTAs
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      }
    } else if (crank == 0) {
      // Pair path, S issuer (leader only): S(t) = Q K_t^T for the whole pair.
      // S(t) reuses buffer t%3 once PV(t-3) — issued by the PV warp — is
      // complete; the two issuers keep the tensor core's short queue fed.
      if (n_own > 0) ptx::mbar_wait(q_full, 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < n_items; ++i) {
        bool is_v;
        int t;
        seq_item(i, n_load, is_v, t);
        if (!is_v) {
          ptx::mbar_wait(&kv_full[stage], phase);
          if (t >= kNB) ptx::mbar_wait(&pv_done[t % kNB], static_cast<uint32_t>(((t - kNB) / kNB) & 1));
          ptx::tc_fence_after();
          const uint32_t soff = static_cast<uint32_t>(stage) * (C::kSlotBytes >> 4);
          const uint32_t sbuf = tmem + static_cast<uint32_t>(t % kNB) * kBN;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t aoff = ((kk >> 2) * C::kPanelBytes + (kk & 3) * 32) >> 4;
            const uint32_t boff = ((kk >> 2) * C::kKPanelStride + (kk & 3) * 32) >> 4;
            ptx::mma2_bf16_ss_lo(sbuf, q_lo + aoff, k_lo + soff + boff, kDescHi, C::kIdescQK, kk > 0);
          }
          ptx::mma2_commit_mc_w(&s_full[t % kNB], 0x3);
          ptx::mma2_commit_mc_w(&kv_empty[stage], 0x3);
          if (lane == 0) trace_stamp(p, 6, t);
        }
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (K2 && warp == kPvWarp && crank == 0) {
    // ------------------------------------------------------------ PV issuer
    // Pair path (leader only): O += P(t) V_t once P(t) of both CTAs is ready.
    const uint32_t sal = ptx::smem_u32(smem);
    constexpr uint32_t kDescHi = (1024u >> 4) | (1u << 14) | (2u << 29);
    constexpr uint32_t kLboV = (uint32_t(C::kPanelBytes) >> 4) << 16;
    const uint32_t v_lo = (((sal + C::kKVOff) >> 4) & 0x3FFFu) | kLboV;
    int stage = 0;
    uint32_t phase = 0;
    for (int i = 0; i < n_items; ++i) {
      bool is_v;
      int t;
      seq_item(i, n_load, is_v, t);
      if (is_v) {
        ptx::mbar_wait(&kv_full[stage], phase);
        if (lane == 0) trace_stamp(p, 7, t);
        ptx::mbar_wait(&p_ready[t % kNB], static_cast<uint32_t>((t / kNB) & 1));
        if (lane == 0) trace_stamp(p, 4, t);
        ptx::tc_fence_after();
        const uint32_t soff = static_cast<uint32_t>(stage) * (C::kSlotBytes >> 4);
        const uint32_t sbuf = tmem + static_cast<uint32_t>(t % kNB) * kBN;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk)
          ptx::mma2_bf16_ts_lo(tmem + kOCol, sbuf + kk * 8, v_lo + soff + ((kk * 16 * 128) >> 4),
                               kDescHi, C::kIdescPV, (t > 0 || kk > 0) ? 1u : 0u);
        ptx::mma2_commit_mc_w(&pv_done[t % kNB], 0x3);
        if (t == n_own - 1) ptx::mma2_commit_mc_w(o_final, 0x3);
        ptx::mma2_commit_mc_w(&kv_empty[stage], 0x3);
        if (lane == 0) trace_stamp(p, 5, t);
      }
      if (++stage == C::kStages) { stage = 0; phase ^= 1; }
    }
    __syncwarp();
  } else if (warp < 8) {
    // ------------------------------------------------------------ softmax
    // Warpgroup w handles the KV tiles j = w (mod 2) — it always reads S
    // buffer w — with one full 128-column score row per thread.  The only
    // hand-off between the two warpgroups is the running max m: the warpgroup
    // of tile j publishes m_j (per row) right after its row max, and the other
    // warpgroup reads it before the exponentials of tile j+1.  Each keeps its
    // own partial row sum l_w (relative to the m of its last tile); they are
    // merged in the epilogue.  The two warpgroups' MUFU phases thus overlap
    // instead of both waiting on a per-tile exchange.
    const int w = warp >> 2;                  // tile parity this warpgroup owns
    const int quarter = warp & 3;             // TMEM lane quarter
    const int r = quarter * 32 + lane;        // row within the tile
    const int64_t row = m0 + r;               // local query row
    const bool row_ok = row < p.Lq;
    const int64_t qp = pos_of(p.qmap, row_ok ? row : p.Lq - 1);
    const int64_t klim = key_limit(p, qp);
    const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tO = tmem + lane_addr + kOCol;
    const float sl2 = p.scale_log2;
    const bool leader = (threadIdx.x % 128) == 0;
    float* mrow = red;  // [tile parity][row]: m_j published by tile j's warpgroup

    float m_prev = -INFINITY;  // m of this warpgroup's last tile (log2 units, scaled)
    float l_run = 0.f;         // this warpgroup's partial row sum, relative to m_prev
    for (int j = w; j < n_own; j += 2) {
      const uint32_t sbuf = tmem + lane_addr + (j % kNB) * kBN;  // S(j), then P(j)
      ptx::mbar_wait(&s_full[j % kNB], static_cast<uint32_t>((j / kNB) & 1));
      if (leader) trace_stamp(p, 2 * w, j);
      ptx::tc_fence_after();
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        ptx::tmem_ld32(sbuf + c * 32, *reinterpret_cast<float(*)[32]>(&s[c * 32]));
      ptx::tmem_wait_ld();

      const int64_t nv64 = klim - static_cast<int64_t>(j) * kBN;
      const int nvalid = nv64 < 0 ? 0 : (nv64 > kBN ? kBN : static_cast<int>(nv64));
      const bool masked = !__all_sync(0xffffffffu, nvalid >= kBN);
      if (masked) {
#pragma unroll
        for (int c = 0; c < 128; ++c) s[c] = c < nvalid ? s[c] : -INFINITY;
      }
      float mx0 = s[0], mx1 = s[1], mx2 = s[2], mx3 = s[3];
#pragma unroll
      for (int c = 4; c < 128; c += 4) {
        mx0 = fmaxf(mx0, s[c]);
        mx1 = fmaxf(mx1, s[c + 1]);
        mx2 = fmaxf(mx2, s[c + 2]);
        mx3 = fmaxf(mx3, s[c + 3]);
      }
      const float mt = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * sl2;
      // m_{j-1} from the other warpgroup (tile j-1), published on barrier 2+(1-w).
      float m_in = -INFINITY;
      if (j > 0) {
        asm volatile("bar.sync %0, 256;" ::"r"(2 + (w ^ 1)) : "memory");
        m_in = mrow[((j - 1) & 1) * kBM + r];
      }
      const bool need = mt > m_in + kRescaleThreshold;
      const float m_cur = __any_sync(0xffffffffu, need) ? fmaxf(m_in, mt) : m_in;
      if (j + 1 < n_own) {  // hand m_j to the warpgroup of tile j+1
        mrow[(j & 1) * kBM + r] = m_cur;
        asm volatile("bar.arrive %0, 256;" ::"r"(2 + w) : "memory");
      }
      // This warpgroup's partial sum was accumulated relative to m_prev.
      if (m_cur != m_prev) {
        l_run *= (m_prev == -INFINITY) ? 0.f : ptx::ex2_approx(m_prev - m_cur);
      }
      const float m_use = (m_cur == -INFINITY) ? 0.f : m_cur;
      // Unmasked tiles send kEmu of every 8 column pairs to the FMA-pipe
      // polynomial; masked tiles (-inf entries, must give exactly 0) use MUFU only.
      if (masked)
        l_run += sm::exp_tile<0>(s, sl2, m_use, sbuf);
      else
        l_run += sm::exp_tile<kEmu>(s, sl2, m_use, sbuf);
      // O holds PV(0..j-2) and possibly PV(j-1) in flight; PV(j) waits for
      // p_ready.  If this warp's max moved, rescale its O rows after PV(j-1)
      // completes (at most one pv_done phase can be pending here).
      if (j > 0 && __any_sync(0xffffffffu, m_cur != m_in)) {
        const float alpha = (m_in == -INFINITY || m_cur == m_in) ? 1.f : ptx::ex2_approx(m_in - m_cur);
        if (K2)
          ptx::mbar_wait(&pv_done[(j - 1) % kNB], static_cast<uint32_t>(((j - 1) / kNB) & 1));
        else
          ptx::mbar_wait(&pv_done[(j - 1) & 1], static_cast<uint32_t>(((j - 1) >> 1) & 1));
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
      m_prev = m_cur;
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      if (leader) trace_stamp(p, 2 * w + 1, j);
      if (K2) {  // one arrive per warp on the pair leader's barrier
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa_cluster(&p_ready[j % kNB], 0));
      } else {
        ptx::mbar_arrive(&p_ready[j % kNB]);
      }
    }
    if (n_own > 0) {
      ptx::mbar_wait(o_final, 0);
      ptx::tc_fence_after();
    }
    // ---------------------------------------------------------- epilogue
    // Merge the two partial sums at the final max; each warpgroup then writes
    // D/2 output columns of every row.
    float* lx = red + 2 * kBM;  // [w][row] (l, m) pairs
    lx[(w * 2 + 0) * kBM + r] = l_run;
    lx[(w * 2 + 1) * kBM + r] = m_prev;
    halves_sync();
    const float l_o = lx[((w ^ 1) * 2 + 0) * kBM + r];
    const float m_o = lx[((w ^ 1) * 2 + 1) * kBM + r];
    const float m_fin = fmaxf(m_prev, m_o);
    float l_tot = 0.f;
    if (m_fin != -INFINITY) {
      l_tot = (m_prev == -INFINITY ? 0.f : l_run * ptx::ex2_approx(m_prev - m_fin)) +
              (m_o == -INFINITY ? 0.f : l_o * ptx::ex2_approx(m_o - m_fin));
    }
    const bool empty = !(l_tot > 0.f);
    const float inv_l = empty ? 0.f : 1.f / l_tot;
    if (row_ok && w == 0)
      p.lse[static_cast<int64_t>(head) * p.Lq + row] =
          empty ? -INFINITY : (m_fin + __log2f(l_tot)) * 0.69314718055994530942f;
    const int64_t obase = (row * p.H + head) * static_cast<int64_t>(D) + w * (D / 2);
#pragma unroll
    for (int c = 0; c < D / 64; ++c) {
      float o[32];
      if (n_own > 0) {
        ptx::tmem_ld32(tO + w * (D / 2) + c * 32, o);
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
  }
  ptx::tc_fence_before();
  if (K2) {
    ptx::cluster_sync();  // both CTAs done with the pair's TMEM and each other's barriers
    if (warp == kMmaWarp) {
      ptx::tc_fence_after();
      ptx::tmem_dealloc_2cta<512>(tmem);
    }
  } else {
    __syncthreads();
    if (warp == kMmaWarp) {
      ptx::tc_fence_after();
      ptx::tmem_dealloc<512>(tmem);
    }
    ptx::cluster_sync();  // the peer may still multicast into / arrive on this CTA until here
  }
}

// ---------------------------------------------------------------- host side
// Kernel variant (measurement knobs): DMHA_EMU=<pairs of 8 on the FMA pipe>,
// DMHA_PAIR_MMA=0 to use the per-CTA MMA path for D = 128.
template <int D>
int emu_variant() {
  static int v = [] {
    int x = Cfg<D, false>::kEmuDefault;
    if (const char* e = std::getenv("DMHA_EMU")) x = std::atoi(e);
    return x;
  }();
  return v;
}
// Kernel choice: DMHA_KERNEL = pingpong | cluster | pair (default pingpong,
// the measured fastest on C3/C4/C5).
enum KernelKind { K_PINGPONG, K_CLUSTER, K_PAIR, K_DBUF };
inline KernelKind kernel_kind(int D) {
  const char* e = std::getenv("DMHA_KERNEL");
  if (e) {
    if (!strcmp(e, "pingpong")) return K_PINGPONG;
    if (!strcmp(e, "cluster")) return K_CLUSTER;
    if (!strcmp(e, "pair")) return D == 128 ? K_PAIR : K_CLUSTER;
    if (!strcmp(e, "dbuf")) return K_DBUF;
  }
  return K_PINGPONG;
}

template <int D, int E, bool K2>
cudaError_t launch_v(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                     const Params& p, dim3 grid, cudaStream_t stream) {
  using C = Cfg<D, K2>;
  // the dynamic shared-memory limit is a per-device function attribute
  static int attr_dev = -1;
  int cur_dev = 0;
  cudaGetDevice(&cur_dev);
  if (attr_dev != cur_dev) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_sm100_kernel<D, E, K2>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_dev = cur_dev;
  }
  attn_fwd_sm100_kernel<D, E, K2><<<grid, kThreads, C::kSmemBytes, stream>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

template <int D, bool K2>
cudaError_t launch_e(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                     const Params& p, dim3 grid, cudaStream_t stream) {
  switch (emu_variant<D>()) {
    case 0: return launch_v<D, 0, K2>(tq, tk, tv, p, grid, stream);
    case 1: return launch_v<D, 1, K2>(tq, tk, tv, p, grid, stream);
    case 2: return launch_v<D, 2, K2>(tq, tk, tv, p, grid, stream);
    case 3: return launch_v<D, 3, K2>(tq, tk, tv, p, grid, stream);
    case 4: return launch_v<D, 4, K2>(tq, tk, tv, p, grid, stream);
    default: return launch_v<D, Cfg<D, K2>::kEmuDefault, K2>(tq, tk, tv, p, grid, stream);
  }
}

template <int D>
cudaError_t launch_d(const LocalAttnArgs& a, cudaStream_t stream) {
  const bool k2 = (D == 128) && kernel_kind(D) == K_PAIR;
  CUtensorMap tq, tk, tv;
  // K: 64-key half tiles (pair MMA: own half; multicast path: half per CTA).
  // V: pair MMA loads all 128 keys x 64 columns; multicast path 64-key halves.
  if (!make_tma_map_bf16(&tq, a.q, a.Lq, a.H, D, kBM) || !make_tma_map_bf16(&tk, a.k, a.Lk, a.H, D, kBN / 2) ||
      !make_tma_map_bf16(&tv, a.v, a.Lk, a.H, D, k2 ? kBN : kBN / 2))
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
  p.n_pairs = static_cast<int>((a.Lq + 2 * kBM - 1) / (2 * kBM));
  p.trace = g_trace;
  dim3 grid(2 * p.n_pairs, a.H);
  if constexpr (D == 128) {
    if (k2) return launch_e<D, true>(tq, tk, tv, p, grid, stream);
  }
  return launch_e<D, false>(tq, tk, tv, p, grid, stream);
}

}  // namespace

unsigned long long* g_trace = nullptr;

bool pingpong_fused_combine_ok(int D);  // attn_fwd_sm100_v1.cu

bool attn_fused_combine_supported(int D) {
  if (D != 64 && D != 128) return false;
  const KernelKind k = kernel_kind(D);
  return k == K_DBUF || (k == K_PINGPONG && pingpong_fused_combine_ok(D));
}

bool attn_kv_split_supported(int D) {
  return (D == 64 || D == 128) && kernel_kind(D) == K_PINGPONG && pingpong_fused_combine_ok(D);
}

cudaError_t launch_attn_fwd_bf16(const LocalAttnArgs& a, cudaStream_t stream) {
  if (a.Lq <= 0) return cudaSuccess;
  if (a.kv_split != 1 && (!attn_kv_split_supported(a.D) || a.out_mode != OUT_PARTIAL_F32))
    return cudaErrorInvalidValue;
  if (a.out_mode >= OUT_COMBINE_ACC && !attn_fused_combine_supported(a.D))
    return cudaErrorInvalidValue;
  if (a.Lq > INT32_MAX || a.Lk > INT32_MAX) return cudaErrorInvalidValue;
  if (kernel_kind(a.D) == K_PINGPONG) return launch_attn_fwd_bf16_pingpong(a, stream);
  if (kernel_kind(a.D) == K_DBUF) return launch_attn_fwd_bf16_dbuf(a, stream);
  if (a.D == 64) return launch_d<64>(a, stream);
  if (a.D == 128) return launch_d<128>(a, stream);
  return cudaErrorInvalidValue;
}

}  // namespace dmha
