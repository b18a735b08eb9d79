// dmha_api.cu — the C ABI (include/dmha.h) and the sequence-sharded ring
// distribution layer.
//
// PAPER.md §10.4 splits X along the sequence into N partitions and
// needs every key of a row for its softmax.  Here each rank keeps its
// L/P query rows; the K/V blocks circulate around a ring of P ranks by NCCL
// send/recv over NVLink (north_star (3)), P-1 steps, on a high-priority comm
// stream overlapped with the local tcgen05 attention kernel on the compute
// stream; per-step partials are merged by the fp32 log-sum-exp combine kernel.
//
// Per rank r, step s (0 <= s < P): source rank src = (r - s) mod P, K/V block
// kv_s (kv_0 = the user's k/v, kv_s = ring buffer s % 2 for s >= 1).
//   comm  (s < P-1): send kv_s -> r+1, recv kv_{s+1} <- r-1 into buffer (s+1)%2,
//                    after the compute of step s-1 (last reader of that buffer).
//   compute:         attention(q_r, kv_s, positions of src) -> partial;
//                    s = 0 writes the accumulator, s >= 1 combines into it, the
//                    last step writes out/lse.  P = 1 writes out/lse directly.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dmha.h"
#include "kernels.h"
#include "peer_link.h"

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CK_CUDA(expr)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return fail(DMHA_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                  __FILE__, __LINE__);                                                  \
  } while (0)

#define CK_NCCL(expr)                                                                     \
  do {                                                                                    \
    ncclResult_t _r = (expr);                                                             \
    if (_r != ncclSuccess)                                                                \
      return fail(DMHA_ERR_NCCL, "%s failed: %s (%s:%d)", #expr, ncclGetErrorString(_r), \
                  __FILE__, __LINE__);                                                    \
  } while (0)

struct State {
  bool inited = false;
  int world = 1, rank = 0, device = 0, dtype = DMHA_BF16, layout = DMHA_LAYOUT_CONTIGUOUS;
  cudaStream_t stream = nullptr;  // compute stream (user's)
  cudaStream_t comm = nullptr;    // NCCL stream (library-owned, high priority)
  ncclComm_t nccl = nullptr;
  // K/V transport of the ring at world size > 1 (DMHA_TRANSPORT at init):
  // 0 = NCCL send/recv (default), 1 = copy-engine pulls from peer memory
  // (CUDA IPC, NEXT-2).  With the peer transport the NCCL communicator is
  // created lazily, only for the entry points that need a collective.
  int transport = 0;
  dmha::PeerLink* peer = nullptr;
  unsigned char uid[128] = {};
  cudaEvent_t ev_start = nullptr, ev_recv[2] = {nullptr, nullptr},
              ev_done[2] = {nullptr, nullptr}, ev_comm_end = nullptr;
  // host path pipelining (dmha_forward_host at world size 1)
  cudaStream_t d2h = nullptr;
  cudaEvent_t ev_h2d[8] = {}, ev_comp[8] = {}, ev_kv[8] = {};
  // ring workspace
  void* kvbuf[2] = {nullptr, nullptr};  // each: K block then V block
  float* o_acc = nullptr;
  float* o_part = nullptr;
  float* lse_acc = nullptr;
  float* lse_part = nullptr;
  size_t kv_bytes = 0, acc_elems = 0, lse_elems = 0, part_elems = 0, part_lse_elems = 0;
  // head-parallel exchange workspace (dmha_forward_headpar*)
  void* hp = nullptr;
  size_t hp_bytes = 0;
  // NEXT-3 layer workspace (dmha_mha_forward): q, k, v, o, lse
  void* mha = nullptr;
  size_t mha_bytes = 0;
  void* sel = nullptr;  // NEXT-4 selector workspace
  size_t sel_bytes = 0;
  // fp32 path: split K / V^T operands of the current key block (3xTF32)
  void* tf32 = nullptr;
  size_t tf32_bytes = 0;
  // host-path staging
  void* st_qkv = nullptr;  // q, k, v back to back
  void* st_out = nullptr;
  float* st_lse = nullptr;
  size_t st_bytes = 0, st_lse_elems = 0;
  dmha_stats stats{};
  // Fault injection (DMHA_FAULT=perturb_lse, read at every forward): the
  // log-sum-exp combine adds this to each partial's lse, so the merged
  // output is wrong whenever a combine runs (test that the suite notices).
  float fault_lse_bias = 0.f;
  // profiling (dmha_set_profiling)
  bool profile = false;
  struct Rec {
    cudaEvent_t a, b;
    int kind;  // 0 attention, 1 combine, 2 exchange, 3 head-parallel pack/unpack, 4 GEMM
    uint64_t bytes;
    double flop = 0.0;
  };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
};

State g;

cudaEvent_t pool_event() {
  if (!g.pool.empty()) {
    cudaEvent_t e = g.pool.back();
    g.pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  return e;
}

// Bracket the launches enqueued by `fn` on `stream` with profiling events.
template <typename F>
int timed(int kind, cudaStream_t stream, F&& fn, uint64_t bytes = 0) {
  if (!g.profile) return fn();
  cudaEvent_t a = pool_event(), b = pool_event();
  if (a) cudaEventRecord(a, stream);
  int rc = fn();
  if (b) cudaEventRecord(b, stream);
  if (a && b) g.pending.push_back({a, b, kind, bytes, 0.0});
  return rc;
}

void resolve_profiles() {
  for (auto& r : g.pending) {
    float ms = 0.f;
    if (cudaEventSynchronize(r.b) == cudaSuccess && cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
      if (r.kind == 0) {
        g.stats.attn_ms += ms;
        g.stats.attn_launches++;
      } else if (r.kind == 1) {
        g.stats.combine_ms += ms;
        g.stats.combine_launches++;
      } else if (r.kind == 4) {
        g.stats.gemm_ms += ms;
        g.stats.gemm_launches++;
        g.stats.gemm_flop += r.flop;
      } else if (r.kind == 3) {
        g.stats.pack_ms += ms;
        g.stats.pack_launches++;
        g.stats.pack_bytes += r.bytes;
      } else {
        g.stats.exchange_ms += ms;
        g.stats.exchanges++;
      }
    }
    g.pool.push_back(r.a);
    g.pool.push_back(r.b);
  }
  g.pending.clear();
}

size_t elem_bytes(int dtype) { return dtype == DMHA_BF16 ? 2 : 4; }

int check_state() {
  if (!g.inited) return fail(DMHA_ERR_STATE, "dmha: not initialised (call dmha_init)");
  return DMHA_OK;
}

void free_ptr(void*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}
void free_ptr(float*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

void update_ws_stat() {
  g.stats.workspace_bytes = 2 * g.kv_bytes + (g.acc_elems + g.part_elems) * 4 +
                            (g.lse_elems + g.part_lse_elems) * 4 +
                            g.st_bytes + g.st_lse_elems * 4 + g.hp_bytes + g.mha_bytes +
                            g.sel_bytes + g.tf32_bytes +
                            (g.peer ? dmha::peer_pub_bytes(g.peer) : 0);
}

int alloc_or_oom(void** p, size_t bytes, const char* what) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear the sticky-free allocation error
    *p = nullptr;
    return fail(DMHA_ERR_OOM, "dmha: cudaMalloc(%zu) for %s failed: %s", bytes, what,
                cudaGetErrorString(e));
  }
  return DMHA_OK;
}

// NEXT-2: the attention epilogue merges each ring-step partial into the
// accumulator itself (bf16 ping-pong kernel; DMHA_FUSED_COMBINE=0 forces the
// separate lse_combine pass for A/B), so O_part / lse_part are not needed.
bool fused_combine(int D) {
  const char* e = std::getenv("DMHA_FUSED_COMBINE");
  if (e && std::atoi(e) == 0) return false;
  return g.dtype == DMHA_BF16 && dmha::attn_fused_combine_supported(D);
}

// Split-KV for a P = 1 forward on a small grid (fewer than 4 waves of
// 256-row CTAs, Lloc >= 2048; DMHA_KV_SPLIT=0 disables): two fp32 partials
// merged by the log-sum-exp combine (DESIGN.md §5 lesson 14).
bool split_kv_active(int64_t Lloc, int D, int H) {
  const int64_t ctas = (Lloc + 255) / 256 * H;
  const char* e = std::getenv("DMHA_KV_SPLIT");
  return g.dtype == DMHA_BF16 && ctas < 4 * 148 && Lloc >= 2048 && !(e && std::atoi(e) == 0) &&
         dmha::attn_kv_split_supported(D);
}

// Device bytes a forward at world size P holds (the buffers ensure_ring_ws
// allocates for it): P = 1 only the split-KV partials (O_acc, O_part,
// lse_acc, lse_part) when split_kv_active; P > 1 two K/V ring buffers, O_acc
// and lse_acc, plus O_part / lse_part when the combine is not fused.
size_t ring_ws_bytes(int P, int64_t Lloc, int D, int H) {
  const size_t elems = static_cast<size_t>(Lloc) * H * D;
  const size_t lse = static_cast<size_t>(Lloc) * H;
  // fp32: the 3xTF32 split operands of one key block (at most Lloc keys)
  const size_t tf32 = g.dtype == DMHA_FP32 ? dmha::tf32_scratch_bytes(Lloc, H, D) : 0;
  if (P == 1) return (split_kv_active(Lloc, D, H) ? 2 * (elems * 4 + lse * 4) : 0) + tf32;
  const size_t parts = fused_combine(D) ? 1 : 2;
  // + the published K/V block of the peer transport (NEXT-2)
  const size_t pub = g.transport == 1 ? 2 * elems * elem_bytes(g.dtype) : 0;
  return 2 * (2 * elems * elem_bytes(g.dtype)) + parts * (elems * 4 + lse * 4) + pub + tf32;
}

// fp32 path scratch for a key block of Lk rows (grow-only).
int ensure_tf32_ws(int64_t Lk, int D, int H) {
  const size_t need = dmha::tf32_scratch_bytes(Lk, H, D);
  if (need <= g.tf32_bytes) return DMHA_OK;
  free_ptr(g.tf32);
  g.tf32_bytes = 0;
  int rc = alloc_or_oom(&g.tf32, need, "fp32 split K/V scratch");
  if (rc == DMHA_OK) g.tf32_bytes = need;
  update_ws_stat();
  return rc;
}

// Ring accumulators (always), the partial buffers (unfused combine only) and
// the K/V ring buffers (need_kv).
int ensure_ring_ws(int64_t Lloc, int D, int H, bool need_kv, bool force_part = false) {
  const size_t elems = static_cast<size_t>(Lloc) * H * D;
  const size_t lse = static_cast<size_t>(Lloc) * H;
  const bool need_part = force_part || !fused_combine(D);
  if (elems > g.acc_elems) {
    free_ptr(g.o_acc);
    g.acc_elems = 0;
    if (int rc = alloc_or_oom(reinterpret_cast<void**>(&g.o_acc), elems * 4, "O_acc")) {
      update_ws_stat();
      return rc;
    }
    g.acc_elems = elems;
  }
  if (need_part && elems > g.part_elems) {
    free_ptr(g.o_part);
    g.part_elems = 0;
    if (int rc = alloc_or_oom(reinterpret_cast<void**>(&g.o_part), elems * 4, "O_part")) {
      update_ws_stat();
      return rc;
    }
    g.part_elems = elems;
  }
  if (lse > g.lse_elems) {
    free_ptr(g.lse_acc);
    g.lse_elems = 0;
    if (int rc = alloc_or_oom(reinterpret_cast<void**>(&g.lse_acc), lse * 4, "lse_acc")) {
      update_ws_stat();
      return rc;
    }
    g.lse_elems = lse;
  }
  if (need_part && lse > g.part_lse_elems) {
    free_ptr(g.lse_part);
    g.part_lse_elems = 0;
    if (int rc = alloc_or_oom(reinterpret_cast<void**>(&g.lse_part), lse * 4, "lse_part")) {
      update_ws_stat();
      return rc;
    }
    g.part_lse_elems = lse;
  }
  if (need_kv) {
    const size_t kvb = 2 * elems * elem_bytes(g.dtype);
    if (kvb > g.kv_bytes) {
      free_ptr(g.kvbuf[0]);
      free_ptr(g.kvbuf[1]);
      g.kv_bytes = 0;
      int rc = alloc_or_oom(&g.kvbuf[0], kvb, "K/V ring buffer 0");
      if (!rc) rc = alloc_or_oom(&g.kvbuf[1], kvb, "K/V ring buffer 1");
      if (rc) {
        free_ptr(g.kvbuf[0]);
        free_ptr(g.kvbuf[1]);
        update_ws_stat();
        return rc;
      }
      g.kv_bytes = kvb;
    }
  }
  update_ws_stat();
  return DMHA_OK;
}

// Shard sizes ("equal as possible"):
// contiguous — rank r owns L/P rows, plus one of the first L % P ranks;
// zigzag — 2 chunks of L/(2P) rows (L % 2P == 0 required).
int64_t shard_rows(int64_t L, int P, int r, int layout) {
  if (layout == DMHA_LAYOUT_ZIGZAG) return L / P;
  return L / P + (r < L % P ? 1 : 0);
}
int64_t max_shard_rows(int64_t L, int P, int layout) {
  return layout == DMHA_LAYOUT_ZIGZAG ? L / P : (L + P - 1) / P;
}

dmha::PosMap posmap(int64_t L, int P, int r, int layout) {
  dmha::PosMap m;
  if (layout == DMHA_LAYOUT_ZIGZAG) {
    const int64_t c = L / (2 * P);
    m.base0 = r * c;
    m.base1 = static_cast<int64_t>(2 * P - 1 - r) * c;
    m.chunk = c;
  } else {
    const int64_t rows = shard_rows(L, P, r, layout);
    m.base0 = r * (L / P) + std::min<int64_t>(r, L % P);
    m.base1 = m.base0 + rows;
    m.chunk = rows;
  }
  return m;
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const char* pa = static_cast<const char*>(a);
  const char* pb = static_cast<const char*>(b);
  return pa < pb + nb && pb < pa + na;
}

// nshards: how many shards each buffer holds back to back (the emulated entry
// points pass P rank-major shards of max_shard_rows rows), for the overlap
// check; rows: the rows of one shard (this rank's by default).
int validate(const void* q, const void* k, const void* v, const void* out, const float* lse,
             int64_t L, int D, int H, int P, int layout, int nshards = 1, int64_t rows = -1) {
  if (!q || !k || !v || !out || !lse) return fail(DMHA_ERR_INVALID, "dmha: null pointer");
  if (L < 1 || H < 1) return fail(DMHA_ERR_INVALID, "dmha: need L >= 1 and H >= 1");
  if (D != 64 && D != 128)
    return fail(DMHA_ERR_UNSUPPORTED, "dmha: per-head dim D=%d unsupported (64 or 128)", D);
  if (layout != DMHA_LAYOUT_CONTIGUOUS && layout != DMHA_LAYOUT_ZIGZAG)
    return fail(DMHA_ERR_INVALID, "dmha: unknown layout %d", layout);
  if (layout == DMHA_LAYOUT_ZIGZAG && L % (2LL * P) != 0)
    return fail(DMHA_ERR_INVALID, "dmha: L=%lld not divisible by 2P=%d (zigzag layout)",
                static_cast<long long>(L), 2 * P);
  // contiguous shards may be uneven (L % P != 0): the first L % P ranks hold
  // one row more
  const int64_t Lloc = rows >= 0 ? rows : max_shard_rows(L, P, layout);
  if (Lloc > (1LL << 31) - 1) return fail(DMHA_ERR_INVALID, "dmha: L/P too large");
  const void* ptrs[5] = {q, k, v, out, lse};
  for (const void* p : ptrs)
    if (reinterpret_cast<uintptr_t>(p) % 16 != 0)
      return fail(DMHA_ERR_INVALID, "dmha: base pointers must be 16-byte aligned");
  const size_t tb = static_cast<size_t>(Lloc) * H * D * elem_bytes(g.dtype) * nshards;
  const size_t lb = static_cast<size_t>(Lloc) * H * 4 * nshards;
  const void* ins[3] = {q, k, v};
  for (const void* in : ins)
    if (overlaps(out, tb, in, tb) || overlaps(lse, lb, in, tb))
      return fail(DMHA_ERR_INVALID, "dmha: out/lse overlap q/k/v");
  if (overlaps(out, tb, lse, lb)) return fail(DMHA_ERR_INVALID, "dmha: out overlaps lse");
  return DMHA_OK;
}

int run_local(const void* q, const void* k, const void* v, void* out, float* lse, int64_t Lq,
              int64_t Lk, int D, int H, int causal, dmha::PosMap qm, dmha::PosMap km,
              int out_mode, float* acc_o = nullptr, float* acc_lse = nullptr, int kv_split = 1,
              void* out2 = nullptr, float* lse2 = nullptr) {
  dmha::LocalAttnArgs a;
  a.acc_o = acc_o;
  a.acc_lse = acc_lse;
  a.kv_split = kv_split;
  a.out2 = out2;
  a.lse2 = lse2;
  a.lse_bias = g.fault_lse_bias;
  a.q = q;
  a.k = k;
  a.v = v;
  a.out = out;
  a.lse = lse;
  a.Lq = Lq;
  a.Lk = Lk;
  a.D = D;
  a.H = H;
  a.causal = causal;
  a.qmap = qm;
  a.kmap = km;
  a.out_mode = out_mode;
  if (g.dtype == DMHA_FP32) {
    if (int rc = ensure_tf32_ws(Lk, D, H)) return rc;
    a.scratch = g.tf32;
    a.scratch_bytes = g.tf32_bytes;
  }
  cudaError_t e = cudaSuccess;
  timed(0, g.stream, [&]() {
    e = g.dtype == DMHA_BF16 ? dmha::launch_attn_fwd_bf16(a, g.stream)
                             : dmha::launch_attn_fwd_fp32(a, g.stream);
    return 0;
  });
  if (e != cudaSuccess)
    return fail(DMHA_ERR_CUDA, "dmha: attention kernel launch failed: %s", cudaGetErrorString(e));
  g.stats.kernel_launches += g.dtype == DMHA_BF16 ? dmha::attn_launches_per_call()
                                                  : dmha::fp32_launches_per_call(Lq, Lk);
  return DMHA_OK;
}

int run_combine(float* o_part, float* lse_part, void* out, float* lse, int64_t Lq, int D, int H,
                int final_step) {
  cudaError_t e = cudaSuccess;
  timed(1, g.stream, [&]() {
    e = dmha::launch_lse_combine(g.o_acc, g.lse_acc, o_part, lse_part, out, lse, Lq, D, H,
                                 final_step, g.dtype == DMHA_BF16, g.stream, g.fault_lse_bias);
    return 0;
  });
  if (e != cudaSuccess)
    return fail(DMHA_ERR_CUDA, "dmha: combine launch failed: %s", cudaGetErrorString(e));
  g.stats.kernel_launches += 1;
  return DMHA_OK;
}

// The ring schedule of rank r at step s.  Pure function of
// (P, r, s, layout, L): shared by the NCCL ring, the single-GPU emulation and
// (exported as dmha_ring_plan) the multi-process CPU tests.
dmha_ring_plan make_plan(int P, int r, int s, int layout, int64_t L) {
  dmha_ring_plan pl;
  pl.src = ((r - s) % P + P) % P;
  pl.send_to = s < P - 1 ? (r + 1) % P : -1;
  pl.recv_from = s < P - 1 ? (r - 1 + P) % P : -1;
  pl.compute_buf = s == 0 ? -1 : (s & 1);
  pl.recv_buf = s < P - 1 ? ((s + 1) & 1) : -1;
  pl.recv_after_compute_of = (s < P - 1 && s >= 2) ? s - 1 : -1;
  pl.output = P == 1 ? DMHA_PLAN_FINAL : (s == 0 ? DMHA_PLAN_ACC : (s == P - 1 ? DMHA_PLAN_COMBINE_FINAL
                                                                              : DMHA_PLAN_COMBINE));
  const dmha::PosMap qm = posmap(L, P, r, layout), km = posmap(L, P, pl.src, layout);
  pl.q_base0 = qm.base0;
  pl.q_base1 = qm.base1;
  pl.q_chunk = qm.chunk;
  pl.k_base0 = km.base0;
  pl.k_base1 = km.base1;
  pl.k_chunk = km.chunk;
  return pl;
}

// Compute part of ring step s for rank r (shared by the NCCL and emulated rings
// so both run identical kernels in identical order).
int ring_compute_step(int s, int P, int r, int layout, const void* q, const void* ks,
                      const void* vs, void* out, float* lse, int64_t L, int D, int H, int causal) {
  const dmha_ring_plan pl = make_plan(P, r, s, layout, L);
  const int64_t Lloc = shard_rows(L, P, r, layout);    // query rows (this rank)
  const int64_t Lkv = shard_rows(L, P, pl.src, layout);  // key rows (the block's owner)
  const dmha::PosMap qm{pl.q_base0, pl.q_base1, pl.q_chunk}, km{pl.k_base0, pl.k_base1, pl.k_chunk};
  switch (pl.output) {
    case DMHA_PLAN_FINAL: {
      // Small grids (fewer than 4 waves of 256-row CTAs, e.g. C2) leave SMs
      // idle in the last wave: split each row block's keys over two CTAs
      // and merge the two fp32 partials with the log-sum-exp combine.
      if (!split_kv_active(Lloc, D, H))
        return run_local(q, ks, vs, out, lse, Lloc, Lkv, D, H, causal, qm, km, dmha::OUT_FINAL);
      if (int rc = ensure_ring_ws(Lloc, D, H, false, true)) return rc;  // P = 1: Lkv == Lloc
      if (int rc = run_local(q, ks, vs, g.o_acc, g.lse_acc, Lloc, Lkv, D, H, causal, qm, km,
                             dmha::OUT_PARTIAL_F32, nullptr, nullptr, 2, g.o_part, g.lse_part))
        return rc;
      return run_combine(g.o_part, g.lse_part, out, lse, Lloc, D, H, 1);
    }
    case DMHA_PLAN_ACC:
      return run_local(q, ks, vs, g.o_acc, g.lse_acc, Lloc, Lkv, D, H, causal, qm, km,
                       dmha::OUT_PARTIAL_F32);
    default: {
      const bool fin = pl.output == DMHA_PLAN_COMBINE_FINAL;
      if (fused_combine(D))  // NEXT-2: merge inside the attention epilogue
        return run_local(q, ks, vs, fin ? out : static_cast<void*>(g.o_acc), fin ? lse : g.lse_acc,
                         Lloc, Lkv, D, H, causal, qm, km,
                         fin ? dmha::OUT_COMBINE_FINAL : dmha::OUT_COMBINE_ACC, g.o_acc,
                         g.lse_acc);
      int rc = run_local(q, ks, vs, g.o_part, g.lse_part, Lloc, Lkv, D, H, causal, qm, km,
                         dmha::OUT_PARTIAL_F32);
      if (rc) return rc;
      return run_combine(g.o_part, g.lse_part, out, lse, Lloc, D, H,
                         pl.output == DMHA_PLAN_COMBINE_FINAL);
    }
  }
}

// The NCCL communicator (created at init with the NCCL transport, on first
// use with the peer transport).  Collective: every rank reaches it together.
int need_nccl() {
  if (g.world == 1 || g.nccl) return DMHA_OK;
  ncclUniqueId id;
  memcpy(&id, g.uid, sizeof(id));
  CK_NCCL(ncclCommInitRank(&g.nccl, g.world, id, g.rank));
  return DMHA_OK;
}

int poll_nccl() {
  if (!g.nccl) return DMHA_OK;
  ncclResult_t st = ncclSuccess;
  ncclResult_t r = ncclCommGetAsyncError(g.nccl, &st);
  if (r != ncclSuccess || st != ncclSuccess) {
    ncclCommAbort(g.nccl);
    g.nccl = nullptr;
    return fail(DMHA_ERR_NCCL, "dmha: NCCL async error: %s",
                ncclGetErrorString(r != ncclSuccess ? r : st));
  }
  return DMHA_OK;
}

// ---------------------------------------------------------------- a3 ring
// The K/V exchange of one ring step: at step s rank r sends
// the block it attends (kcur, vcur) to r+1 and receives the block of step
// s+1 from r-1 into ring buffer `dst` (K then V, blk bytes each), enqueued
// on the comm stream.  Two implementations share the loop below:
//   NcclTransport  grouped ncclSend / ncclRecv over NVLink (dmha_forward);
//   CopyTransport  the single-GPU emulation (dmha_forward_emulated): one
//                  cudaMemcpyAsync per K / V block from the shard rank r-1
//                  holds at step s (rank (r-1-s) mod P's original block).
// Block sizes: the block of ring step s belongs to rank src_s and holds its
// shard_rows(src_s) rows (uneven contiguous shards differ by one row); a ring
// buffer holds K at offset 0 and V at offset vo (the largest block's bytes).
struct Transport {
  virtual ~Transport() = default;
  virtual int exchange(const dmha_ring_plan& pl, int s, const void* kcur, const void* vcur,
                       size_t send_bytes, char* dst, size_t recv_bytes, size_t vo) = 0;
};

struct NcclTransport final : Transport {
  int exchange(const dmha_ring_plan& pl, int, const void* kcur, const void* vcur, size_t send_bytes,
               char* dst, size_t recv_bytes, size_t vo) override {
    CK_NCCL(ncclGroupStart());
    CK_NCCL(ncclSend(kcur, send_bytes, ncclChar, pl.send_to, g.nccl, g.comm));
    CK_NCCL(ncclSend(vcur, send_bytes, ncclChar, pl.send_to, g.nccl, g.comm));
    CK_NCCL(ncclRecv(dst, recv_bytes, ncclChar, pl.recv_from, g.nccl, g.comm));
    CK_NCCL(ncclRecv(dst + vo, recv_bytes, ncclChar, pl.recv_from, g.nccl, g.comm));
    CK_NCCL(ncclGroupEnd());
    return DMHA_OK;
  }
};

struct CopyTransport final : Transport {
  const char *k_all, *v_all;  // [P][max shard rows, H, D] shards, rank-major
  size_t shard;               // bytes per shard slot
  int P, r, layout;
  int64_t L;
  CopyTransport(const char* k, const char* v, size_t sh, int P_, int r_, int lay, int64_t L_)
      : k_all(k), v_all(v), shard(sh), P(P_), r(r_), layout(lay), L(L_) {}
  int exchange(const dmha_ring_plan& pl, int s, const void*, const void*, size_t, char* dst,
               size_t recv_bytes, size_t vo) override {
    // what rank recv_from sends at step s is the block it attends at step s,
    // i.e. rank (recv_from - s) mod P's shard == the src of our step s+1
    const int src_next = make_plan(P, r, s + 1, layout, L).src;
    if (src_next != ((pl.recv_from - s) % P + P) % P)
      return fail(DMHA_ERR_STATE, "dmha: ring plan inconsistent at rank %d step %d", r, s);
    CK_CUDA(cudaMemcpyAsync(dst, k_all + src_next * shard, recv_bytes, cudaMemcpyDeviceToDevice,
                            g.comm));
    CK_CUDA(cudaMemcpyAsync(dst + vo, v_all + src_next * shard, recv_bytes,
                            cudaMemcpyDeviceToDevice, g.comm));
    return DMHA_OK;
  }
};

// NEXT-2 peer transport: the block of ring step s+1 is rank src_next's own
// K/V, which that rank published in its IPC-shared buffer (K at 0, V at vo)
// at the start of the forward (see peer_forward); pull it with the copy
// engine once its "published" event has fired.  No relay: each block crosses
// the link once.
struct PeerTransport final : Transport {
  int P, r;
  PeerTransport(int P_, int r_) : P(P_), r(r_) {}
  int exchange(const dmha_ring_plan&, int s, const void*, const void*, size_t, char* dst,
               size_t recv_bytes, size_t vo) override {
    const int src_next = ((r - s - 1) % P + P) % P;
    const char* pub = static_cast<const char*>(dmha::peer_pub(g.peer, src_next));
    CK_CUDA(cudaStreamWaitEvent(g.comm, dmha::peer_pub_event(g.peer, src_next), 0));
    CK_CUDA(cudaMemcpyAsync(dst, pub, recv_bytes, cudaMemcpyDefault, g.comm));
    CK_CUDA(cudaMemcpyAsync(dst + vo, pub + vo, recv_bytes, cudaMemcpyDefault, g.comm));
    return DMHA_OK;
  }
};

// Per-forward accounting (dmha_stats.last_*): reset at every public forward,
// counted at each send (one exchange = one call).
void begin_forward() {
  g.stats.last_bytes_sent = 0;
  g.stats.last_exchanges = 0;
  const char* f = std::getenv("DMHA_FAULT");
  g.fault_lse_bias = (f && !strcmp(f, "perturb_lse")) ? 0.5f : 0.f;
}
void count_sent(uint64_t bytes) {
  g.stats.bytes_sent += bytes;
  g.stats.last_bytes_sent += bytes;
  g.stats.last_exchanges++;
}

// One rank's distributed forward: P-1 exchange steps on the comm
// stream, each overlapped with the attention of the current block on the
// compute stream.  Ordering (per buffer b in {0,1}):
//   recv into b at step s      waits ev_done[b] of the compute of step s-1
//                              (the buffer's last reader; plan field
//                              recv_after_compute_of) — the previous block
//                              is gone only after its attention finished;
//   compute of step s+1        waits ev_recv[b] (the block has landed).
int ring_forward(int P, int r, int layout, const void* q, const void* k, const void* v, void* out,
                 float* lse, int64_t L, int D, int H, int causal, Transport& tx) {
  if (P == 1) return ring_compute_step(0, 1, 0, layout, q, k, v, out, lse, L, D, H, causal);
  if (int rc = ensure_ring_ws(max_shard_rows(L, P, layout), D, H, true)) return rc;
  const size_t row_bytes = static_cast<size_t>(H) * D * elem_bytes(g.dtype);
  const size_t vo = static_cast<size_t>(max_shard_rows(L, P, layout)) * row_bytes;  // V offset
  CK_CUDA(cudaEventRecord(g.ev_start, g.stream));
  CK_CUDA(cudaStreamWaitEvent(g.comm, g.ev_start, 0));
  const void* kcur = k;
  const void* vcur = v;
  char name[64];
  for (int s = 0; s < P; ++s) {
    const dmha_ring_plan pl = make_plan(P, r, s, layout, L);
    snprintf(name, sizeof(name), "dmha ring rank %d step %d src %d", r, s, pl.src);
    nvtxRangePushA(name);
    if (pl.recv_buf >= 0) {
      const int nb = pl.recv_buf;
      if (pl.recv_after_compute_of >= 0) CK_CUDA(cudaStreamWaitEvent(g.comm, g.ev_done[nb], 0));
      char* dst = static_cast<char*>(g.kvbuf[nb]);
      const size_t send_bytes = static_cast<size_t>(shard_rows(L, P, pl.src, layout)) * row_bytes;
      const size_t recv_bytes =
          static_cast<size_t>(shard_rows(L, P, make_plan(P, r, s + 1, layout, L).src, layout)) *
          row_bytes;
      int rc = timed(2, g.comm, [&]() {
        return tx.exchange(pl, s, kcur, vcur, send_bytes, dst, recv_bytes, vo);
      });
      if (rc) {
        nvtxRangePop();
        return rc;
      }
      CK_CUDA(cudaEventRecord(g.ev_recv[nb], g.comm));
      count_sent(2 * send_bytes);
    }
    int rc = ring_compute_step(s, P, r, layout, q, kcur, vcur, out, lse, L, D, H, causal);
    nvtxRangePop();
    if (rc) return rc;
    if (pl.compute_buf >= 0) CK_CUDA(cudaEventRecord(g.ev_done[pl.compute_buf], g.stream));
    g.stats.ring_steps++;
    if (pl.recv_buf >= 0) {
      const int nb = pl.recv_buf;
      CK_CUDA(cudaStreamWaitEvent(g.stream, g.ev_recv[nb], 0));
      kcur = g.kvbuf[nb];
      vcur = static_cast<char*>(g.kvbuf[nb]) + vo;
    }
  }
  // The comm stream's last work must be ordered before any later reuse.
  CK_CUDA(cudaEventRecord(g.ev_comm_end, g.comm));
  CK_CUDA(cudaStreamWaitEvent(g.stream, g.ev_comm_end, 0));
  return DMHA_OK;
}

// Collective contract (dmha.h): every rank passes the same (L, D, H, causal).
// With DMHA_CHECK_COLLECTIVE=1 (debug) the values are cross-checked by a min
// and a max all-reduce before the ring starts (a mismatch would otherwise
// deadlock or corrupt the exchange).
int check_collective_contract(int64_t L, int D, int H, int causal) {
  const char* e = std::getenv("DMHA_CHECK_COLLECTIVE");
  if (!e || std::atoi(e) == 0 || g.world == 1) return DMHA_OK;
  if (int rc = need_nccl()) return rc;
  int64_t h[8] = {L, D, H, causal ? 1 : 0, -L, -D, -H, causal ? -1 : 0};
  int64_t* d = nullptr;
  CK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(h), g.stream));
  CK_CUDA(cudaMemcpyAsync(d, h, sizeof(h), cudaMemcpyHostToDevice, g.stream));
  CK_NCCL(ncclAllReduce(d, d, 8, ncclInt64, ncclMax, g.nccl, g.stream));
  CK_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, g.stream));
  CK_CUDA(cudaFreeAsync(d, g.stream));
  CK_CUDA(cudaStreamSynchronize(g.stream));
  if (h[0] != L || h[1] != D || h[2] != H || h[3] != (causal ? 1 : 0) || -h[4] != L || -h[5] != D ||
      -h[6] != H || -h[7] != (causal ? 1 : 0))
    return fail(DMHA_ERR_INVALID, "dmha: collective contract violated: ranks disagree on (L, D, H, causal)");
  return DMHA_OK;
}

// ---------------------------------------------------------------- head-parallel
// The paper's distributed MHA (§10.4):
//   pack -> all-to-all (seq-parallel -> head-parallel) -> unpack to global
//   order -> full-L attention for H/P heads -> pack -> all-to-all back ->
//   unpack.  `exchange(bytes_per_peer, send, recv)` moves block d of `send` to
// rank d and block s from rank s into `recv` (NCCL or the emulation).
struct HpLayout {
  size_t qkv_blk, out_blk, lse_blk;  // bytes per peer block
  size_t send1, recv1, xq, xk, xv, outg, lseg, send2, recv2, send_lse, total;
};

HpLayout hp_layout(int P, int64_t Lloc, int H, int D, size_t e) {
  HpLayout y{};
  const size_t rows_heads = static_cast<size_t>(Lloc) * (H / P);
  y.qkv_blk = 3 * rows_heads * D * e;
  y.out_blk = rows_heads * D * e;
  y.lse_blk = rows_heads * 4;
  size_t off = 0;
  auto take = [&](size_t n) { size_t o = off; off += (n + 255) & ~size_t(255); return o; };
  y.send1 = take(P * y.qkv_blk);
  y.recv1 = take(P * y.qkv_blk);
  y.xq = take(P * y.out_blk);
  y.xk = take(P * y.out_blk);
  y.xv = take(P * y.out_blk);
  y.outg = take(P * y.out_blk);
  y.lseg = take(P * y.lse_blk);
  y.send2 = take(P * y.out_blk);
  y.recv2 = take(P * y.out_blk);
  y.send_lse = take(P * y.lse_blk);
  y.total = off;
  return y;
}

int ensure_hp(size_t bytes) {
  if (bytes <= g.hp_bytes) return DMHA_OK;
  free_ptr(g.hp);
  g.hp_bytes = 0;
  if (int rc = alloc_or_oom(&g.hp, bytes, "head-parallel workspace")) return rc;
  g.hp_bytes = bytes;
  update_ws_stat();
  return DMHA_OK;
}

#define CK_LAUNCH(expr)                                                                   \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) return fail(DMHA_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
    g.stats.kernel_launches++;                                                            \
  } while (0)

// A head-parallel pack/unpack launch, timed as kind 3 when profiling; `bytes`
// = the bytes it reads + writes (algorithmic, for the GB/s roofline).
#define CK_PACK(expr, bytes)                                                                \
  do {                                                                                      \
    cudaError_t _pe = cudaSuccess;                                                          \
    timed(3, g.stream, [&]() { _pe = (expr); return 0; }, (bytes));                         \
    if (_pe != cudaSuccess) return fail(DMHA_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_pe)); \
    g.stats.kernel_launches++;                                                              \
  } while (0)

// Bytes one pack/unpack kernel moves (read + write): the Q/K/V shuffles copy
// 3 * L_loc*H*D elements, the output shuffles L_loc*H*D (+ the fp32 lse).
uint64_t hp_qkv_bytes(int64_t Lloc, int H, int D, size_t e) { return 2ull * 3 * Lloc * H * D * e; }
uint64_t hp_out_bytes(int64_t Lloc, int H, int D, size_t e, bool with_lse) {
  return 2ull * Lloc * H * (D * e + (with_lse ? 4 : 0));
}

// One rank's head-parallel forward; `ws` is this rank's workspace (layout y).
template <typename Ex1, typename Ex2>
int headpar_rank(int P, int r, int layout, const void* q, const void* k, const void* v,
                 void* out, float* lse, int64_t L, int D, int H, int causal, char* ws,
                 const HpLayout& y, Ex1&& exchange_qkv, Ex2&& exchange_out,
                 bool do_exchange_out_now) {
  (void)r;
  const int64_t Lloc = L / P;
  const int e = static_cast<int>(elem_bytes(g.dtype));
  const dmha::HeadparGeom geo{P, H, D, Lloc, layout == DMHA_LAYOUT_ZIGZAG ? 1 : 0};
  CK_PACK(dmha::launch_headpar_pack_qkv(q, k, v, ws + y.send1, geo, e, g.stream),
          hp_qkv_bytes(Lloc, H, D, e));
  if (int rc = exchange_qkv()) return rc;
  CK_PACK(dmha::launch_headpar_unpack_qkv(ws + y.recv1, ws + y.xq, ws + y.xk, ws + y.xv, geo,
                                          e, g.stream),
          hp_qkv_bytes(Lloc, H, D, e));
  const dmha::PosMap full{0, L, L};
  if (int rc = run_local(ws + y.xq, ws + y.xk, ws + y.xv, ws + y.outg,
                         reinterpret_cast<float*>(ws + y.lseg), L, L, D, H / P, causal, full, full,
                         dmha::OUT_FINAL))
    return rc;
  CK_PACK(dmha::launch_headpar_pack_out(ws + y.outg, ws + y.send2,
                                        reinterpret_cast<const float*>(ws + y.lseg),
                                        reinterpret_cast<float*>(ws + y.send_lse), geo, e,
                                        g.stream),
          hp_out_bytes(Lloc, H, D, e, true));
  if (do_exchange_out_now) {
    if (int rc = exchange_out()) return rc;
    CK_PACK(dmha::launch_headpar_unpack_out(ws + y.recv2, out, geo, e, g.stream),
            hp_out_bytes(Lloc, H, D, e, false));
  }
  (void)lse;
  return DMHA_OK;
}

int validate_headpar(int P, int64_t L, int H) {
  if (P < 1 || H % P != 0)
    return fail(DMHA_ERR_INVALID, "dmha headpar: H=%d must be divisible by the world size %d", H, P);
  if (L % P != 0)  // the all-to-all blocks are uniform
    return fail(DMHA_ERR_INVALID, "dmha headpar: L=%lld must be divisible by the world size %d",
                static_cast<long long>(L), P);
  return DMHA_OK;
}

}  // namespace

extern "C" {

const char* dmha_last_error(void) { return g_last_error.c_str(); }

int dmha_get_unique_id(void* id_out) {
  if (!id_out) return fail(DMHA_ERR_INVALID, "dmha_get_unique_id: null");
  static_assert(sizeof(ncclUniqueId) == DMHA_UNIQUE_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId id;
  CK_NCCL(ncclGetUniqueId(&id));
  memcpy(id_out, &id, sizeof(id));
  return DMHA_OK;
}

int dmha_init(int world_size, int rank, const void* unique_id, int device, int dtype, int layout,
              void* cuda_stream) {
  if (g.inited) return fail(DMHA_ERR_STATE, "dmha_init: already initialised");
  if (world_size < 1 || rank < 0 || rank >= world_size)
    return fail(DMHA_ERR_INVALID, "dmha_init: bad world_size/rank %d/%d", world_size, rank);
  if ((world_size > 1) != (unique_id != nullptr))
    return fail(DMHA_ERR_INVALID, "dmha_init: unique_id must be given iff world_size > 1");
  if (dtype != DMHA_BF16 && dtype != DMHA_FP32)
    return fail(DMHA_ERR_INVALID, "dmha_init: bad dtype %d", dtype);
  if (layout != DMHA_LAYOUT_CONTIGUOUS && layout != DMHA_LAYOUT_ZIGZAG)
    return fail(DMHA_ERR_INVALID, "dmha_init: bad layout %d", layout);
  int ndev = 0;
  CK_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev)
    return fail(DMHA_ERR_INVALID, "dmha_init: device %d of %d", device, ndev);
  CK_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(DMHA_ERR_UNSUPPORTED, "dmha_init: needs an sm_100 (B200) device, got sm_%d%d",
                prop.major, prop.minor);
  g = State();
  g.world = world_size;
  g.rank = rank;
  g.device = device;
  g.dtype = dtype;
  g.layout = layout;
  g.stream = static_cast<cudaStream_t>(cuda_stream);
  int lo = 0, hi = 0;
  CK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CK_CUDA(cudaStreamCreateWithPriority(&g.comm, cudaStreamNonBlocking, hi));
  CK_CUDA(cudaEventCreateWithFlags(&g.ev_start, cudaEventDisableTiming));
  CK_CUDA(cudaEventCreateWithFlags(&g.ev_comm_end, cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i) {
    CK_CUDA(cudaEventCreateWithFlags(&g.ev_recv[i], cudaEventDisableTiming));
    CK_CUDA(cudaEventCreateWithFlags(&g.ev_done[i], cudaEventDisableTiming));
  }
  if (const char* e = std::getenv("DMHA_TRANSPORT")) {
    if (!strcmp(e, "peer")) g.transport = 1;
    else if (strcmp(e, "nccl") != 0)
      return fail(DMHA_ERR_INVALID, "dmha_init: DMHA_TRANSPORT must be nccl or peer, got %s", e);
  }
  if (world_size > 1) {
    memcpy(g.uid, unique_id, sizeof(g.uid));
    if (g.transport == 1) {
      std::string err;
      if (int rc = dmha::peer_open(&g.peer, unique_id, world_size, rank, device, &err))
        return fail(rc, "%s", err.c_str());
    } else if (int rc = need_nccl()) {
      return rc;
    }
  }
  g.inited = true;
  g_last_error.clear();
  return DMHA_OK;
}

int dmha_set_stream(void* cuda_stream) {
  if (int rc = check_state()) return rc;
  g.stream = static_cast<cudaStream_t>(cuda_stream);
  return DMHA_OK;
}

int dmha_finalize(void) {
  if (!g.inited) return fail(DMHA_ERR_STATE, "dmha_finalize: not initialised");
  cudaDeviceSynchronize();
  free_ptr(g.kvbuf[0]);
  free_ptr(g.kvbuf[1]);
  free_ptr(g.o_acc);
  free_ptr(g.o_part);
  free_ptr(g.lse_acc);
  free_ptr(g.lse_part);
  free_ptr(g.st_qkv);
  free_ptr(g.st_out);
  free_ptr(g.st_lse);
  free_ptr(g.sel);
  free_ptr(g.hp);
  free_ptr(g.mha);
  free_ptr(g.tf32);
  resolve_profiles();
  for (cudaEvent_t e : g.pool) cudaEventDestroy(e);
  g.pool.clear();
  if (g.nccl) ncclCommDestroy(g.nccl);
  if (g.peer) dmha::peer_close(g.peer);
  cudaEvent_t evs[6] = {g.ev_start, g.ev_comm_end, g.ev_recv[0], g.ev_recv[1], g.ev_done[0],
                        g.ev_done[1]};
  for (cudaEvent_t e : evs)
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < 8; ++i) {
    if (g.ev_h2d[i]) cudaEventDestroy(g.ev_h2d[i]);
    if (g.ev_comp[i]) cudaEventDestroy(g.ev_comp[i]);
    if (g.ev_kv[i]) cudaEventDestroy(g.ev_kv[i]);
  }
  if (g.d2h) cudaStreamDestroy(g.d2h);
  if (g.comm) cudaStreamDestroy(g.comm);
  g = State();
  return DMHA_OK;
}

int dmha_workspace_bytes(int64_t L, int D, int H, size_t* bytes_out) {
  if (int rc = check_state()) return rc;
  return dmha_ring_workspace_bytes(g.world, L, D, H, bytes_out);
}

int dmha_ring_workspace_bytes(int world_size, int64_t L, int D, int H, size_t* bytes_out) {
  if (int rc = check_state()) return rc;
  if (!bytes_out || world_size < 1 || L < 1 || H < 1 ||
      (g.layout == DMHA_LAYOUT_ZIGZAG && L % (2LL * world_size)))
    return fail(DMHA_ERR_INVALID, "dmha_workspace_bytes: bad args");
  if (D != 64 && D != 128) return fail(DMHA_ERR_UNSUPPORTED, "dmha_workspace_bytes: D=%d", D);
  *bytes_out = ring_ws_bytes(world_size, max_shard_rows(L, world_size, g.layout), D, H);
  return DMHA_OK;
}

int dmha_reserve(int world_size, int64_t L, int D, int H) {
  if (int rc = check_state()) return rc;
  if (world_size < 1 || L < 1 || H < 1 || (g.layout == DMHA_LAYOUT_ZIGZAG && L % (2LL * world_size)))
    return fail(DMHA_ERR_INVALID, "dmha_reserve: bad args");
  if (D != 64 && D != 128) return fail(DMHA_ERR_UNSUPPORTED, "dmha_reserve: D=%d", D);
  const int64_t Lloc = max_shard_rows(L, world_size, g.layout);
  if (g.dtype == DMHA_FP32)
    if (int rc = ensure_tf32_ws(Lloc, D, H)) return rc;
  if (world_size == 1) {
    if (split_kv_active(Lloc, D, H)) return ensure_ring_ws(Lloc, D, H, false, true);
    return DMHA_OK;
  }
  if (int rc = ensure_ring_ws(Lloc, D, H, true)) return rc;
  if (g.peer && world_size == g.world) {
    std::string err;
    const size_t vo = static_cast<size_t>(Lloc) * H * D * elem_bytes(g.dtype);
    if (int rc = dmha::peer_ensure_pub(g.peer, 2 * vo, &err)) return fail(rc, "%s", err.c_str());
    update_ws_stat();
  }
  return DMHA_OK;
}

int dmha_get_stats(dmha_stats* s) {
  if (!s) return fail(DMHA_ERR_INVALID, "dmha_get_stats: null");
  resolve_profiles();
  *s = g.stats;
  return DMHA_OK;
}

int dmha_set_profiling(int enable) {
  if (int rc = check_state()) return rc;
  resolve_profiles();
  g.profile = enable != 0;
  g.stats.attn_launches = g.stats.combine_launches = g.stats.exchanges = 0;
  g.stats.attn_ms = g.stats.combine_ms = g.stats.exchange_ms = 0.0;
  g.stats.pack_launches = g.stats.pack_bytes = g.stats.gemm_launches = 0;
  g.stats.pack_ms = g.stats.gemm_ms = g.stats.gemm_flop = 0.0;
  return DMHA_OK;
}

int dmha_ring_plan_step(int world_size, int rank, int step, int layout, int64_t L,
                        struct dmha_ring_plan* plan_out) {
  if (!plan_out || world_size < 1 || rank < 0 || rank >= world_size || step < 0 ||
      step >= world_size || L < 1)
    return fail(DMHA_ERR_INVALID, "dmha_ring_plan_step: bad args");
  if ((layout != DMHA_LAYOUT_CONTIGUOUS && layout != DMHA_LAYOUT_ZIGZAG) ||
      (layout == DMHA_LAYOUT_ZIGZAG && L % (2LL * world_size)))
    return fail(DMHA_ERR_INVALID, "dmha_ring_plan_step: bad layout or L");
  *plan_out = make_plan(world_size, rank, step, layout, L);
  return DMHA_OK;
}

int dmha_shard_rows(int64_t L, int world_size, int rank, int layout, int64_t* rows_out) {
  if (!rows_out || world_size < 1 || rank < 0 || rank >= world_size || L < 1 ||
      (layout != DMHA_LAYOUT_CONTIGUOUS && layout != DMHA_LAYOUT_ZIGZAG) ||
      (layout == DMHA_LAYOUT_ZIGZAG && L % (2LL * world_size)))
    return fail(DMHA_ERR_INVALID, "dmha_shard_rows: bad args");
  *rows_out = shard_rows(L, world_size, rank, layout);
  return DMHA_OK;
}

int dmha_local_to_global(int64_t L, int world_size, int rank, int layout, int64_t i,
                         int64_t* global_out) {
  if (!global_out || world_size < 1 || rank < 0 || rank >= world_size || L < 1)
    return fail(DMHA_ERR_INVALID, "dmha_local_to_global: bad args");
  if ((layout != DMHA_LAYOUT_CONTIGUOUS && layout != DMHA_LAYOUT_ZIGZAG) ||
      (layout == DMHA_LAYOUT_ZIGZAG && L % (2LL * world_size)))
    return fail(DMHA_ERR_INVALID, "dmha_local_to_global: bad layout or L");
  if (i < 0 || i >= shard_rows(L, world_size, rank, layout))
    return fail(DMHA_ERR_INVALID, "dmha_local_to_global: i out of range");
  const dmha::PosMap m = posmap(L, world_size, rank, layout);
  *global_out = i < m.chunk ? m.base0 + i : m.base1 + (i - m.chunk);
  return DMHA_OK;
}

// One rank's forward with the peer transport (NEXT-2):
//   host barrier B1            every rank has issued its previous forward's
//                              "done pulling" record
//   stream waits done(peers)   nobody still reads my published buffer
//   copy k, v -> published buffer; record "published" on the stream
//   host barrier B2            every "published" record precedes the pulls
//   ring_forward(PeerTransport): step s+1's block pulled from its owner
//   record "done pulling" on the comm stream
int peer_forward(const void* q, const void* k, const void* v, void* out, float* lse, int64_t L,
                 int D, int H, int causal) {
  const int P = g.world, r = g.rank;
  const size_t row_bytes = static_cast<size_t>(H) * D * elem_bytes(g.dtype);
  const size_t vo = static_cast<size_t>(max_shard_rows(L, P, g.layout)) * row_bytes;  // V offset
  const size_t blk = static_cast<size_t>(shard_rows(L, P, r, g.layout)) * row_bytes;  // own rows
  std::string err;
  if (int rc = dmha::peer_ensure_pub(g.peer, 2 * vo, &err)) return fail(rc, "%s", err.c_str());
  update_ws_stat();
  if (int rc = dmha::peer_barrier(g.peer, &err)) return fail(rc, "%s", err.c_str());
  for (int p = 0; p < P; ++p)
    if (p != r) CK_CUDA(cudaStreamWaitEvent(g.stream, dmha::peer_done_event(g.peer, p), 0));
  char* pub = static_cast<char*>(dmha::peer_local_pub(g.peer));
  CK_CUDA(cudaMemcpyAsync(pub, k, blk, cudaMemcpyDeviceToDevice, g.stream));
  CK_CUDA(cudaMemcpyAsync(pub + vo, v, blk, cudaMemcpyDeviceToDevice, g.stream));
  CK_CUDA(cudaEventRecord(dmha::peer_pub_event(g.peer, r), g.stream));
  if (int rc = dmha::peer_barrier(g.peer, &err)) return fail(rc, "%s", err.c_str());
  PeerTransport tx(P, r);
  if (int rc = ring_forward(P, r, g.layout, q, k, v, out, lse, L, D, H, causal, tx)) return rc;
  CK_CUDA(cudaEventRecord(dmha::peer_done_event(g.peer, r), g.comm));
  return DMHA_OK;
}

int dmha_forward(const void* q, const void* k, const void* v, void* out, float* lse, int64_t L,
                 int D, int H, int causal) {
  if (int rc = check_state()) return rc;
  if (int rc = validate(q, k, v, out, lse, L, D, H, g.world, g.layout, 1,
                        shard_rows(L, g.world, g.rank, g.layout)))
    return rc;
  if (int rc = poll_nccl()) return rc;
  if (int rc = check_collective_contract(L, D, H, causal)) return rc;
  begin_forward();
  if (g.world > 1 && g.transport == 1) {
    if (int rc = peer_forward(q, k, v, out, lse, L, D, H, causal ? 1 : 0)) return rc;
  } else {
    NcclTransport tx;
    if (int rc = ring_forward(g.world, g.rank, g.layout, q, k, v, out, lse, L, D, H, causal ? 1 : 0, tx))
      return rc;
  }
  g.stats.forwards++;
  return DMHA_OK;
}

int dmha_forward_host(const void* q, const void* k, const void* v, void* out, float* lse,
                      int64_t L, int D, int H, int causal) {
  if (int rc = check_state()) return rc;
  if (!q || !k || !v || !out || !lse) return fail(DMHA_ERR_INVALID, "dmha_forward_host: null pointer");
  begin_forward();
  if (L < 1 || H < 1 || (g.layout == DMHA_LAYOUT_ZIGZAG && L % (2LL * g.world)))
    return fail(DMHA_ERR_INVALID, "dmha_forward_host: bad L/H");
  const int64_t Lloc = shard_rows(L, g.world, g.rank, g.layout);
  const size_t tb = static_cast<size_t>(Lloc) * H * D * elem_bytes(g.dtype);
  const size_t lb = static_cast<size_t>(Lloc) * H;
  if (3 * tb > g.st_bytes) {
    free_ptr(g.st_qkv);
    free_ptr(g.st_out);
    g.st_bytes = 0;
    int rc = alloc_or_oom(&g.st_qkv, 3 * tb, "host-path q/k/v staging");
    if (!rc) rc = alloc_or_oom(&g.st_out, tb, "host-path out staging");
    if (rc) {
      free_ptr(g.st_qkv);
      free_ptr(g.st_out);
      return rc;
    }
    g.st_bytes = 3 * tb;
  }
  if (lb > g.st_lse_elems) {
    free_ptr(g.st_lse);
    g.st_lse_elems = 0;
    if (int rc = alloc_or_oom(reinterpret_cast<void**>(&g.st_lse), lb * 4, "host-path lse")) return rc;
    g.st_lse_elems = lb;
  }
  update_ws_stat();
  char* dq = static_cast<char*>(g.st_qkv);
  const char* pipe_env = std::getenv("DMHA_HOST_PIPELINE");  // 0: unpipelined (A/B knob)
  if (g.world == 1 && L >= 2 * 32768 && !(pipe_env && std::atoi(pipe_env) == 0)) {
    // Single GPU: pipeline the copies with the compute.  Q arrives in row
    // chunks (non-causal) and K/V in key blocks, on a copy stream, in the order
    //   Q chunk 0, K/V block 0, ..., K/V block 3, Q chunk 1, Q chunk 2, ...
    // Chunk 0 is attended block by block as the K/V blocks land (the ring's
    // fused log-sum-exp combine, bit-for-bit the combine the ring uses);
    // later chunks attend all keys at once.  Each chunk's out/lse rows go back
    // on a third stream while the next chunk computes.  Only Q chunk 0, the
    // first K/V block and the last output chunk stay exposed.
    if (D != 64 && D != 128)
      return fail(DMHA_ERR_UNSUPPORTED, "dmha: per-head dim D=%d unsupported (64 or 128)", D);
    if (!g.d2h) {
      CK_CUDA(cudaStreamCreateWithFlags(&g.d2h, cudaStreamNonBlocking));
      for (int i = 0; i < 8; ++i) {
        CK_CUDA(cudaEventCreateWithFlags(&g.ev_h2d[i], cudaEventDisableTiming));
        CK_CUDA(cudaEventCreateWithFlags(&g.ev_comp[i], cudaEventDisableTiming));
        CK_CUDA(cudaEventCreateWithFlags(&g.ev_kv[i], cudaEventDisableTiming));
      }
    }
    causal = causal ? 1 : 0;
    const size_t row_b = static_cast<size_t>(H) * D * elem_bytes(g.dtype);
    // Causal: Q row chunks measured 4-8 % slower in the kernels (C5: 2830 ->
    // 2950-3050 ms of attention), so causal runs split only the K/V copy.
    int64_t nch = causal ? 1 : std::min<int64_t>(8, L / 32768);
    if (const char* e = std::getenv("DMHA_HOST_CHUNKS")) nch = std::max<int64_t>(1, std::min<int64_t>(8, std::atoi(e)));
    const int64_t per = ((L + nch - 1) / nch + 255) / 256 * 256;  // whole 256-row CTAs
    int nkb = fused_combine(D) ? 8 : 1;                           // K/V blocks for chunk 0
    if (const char* e = std::getenv("DMHA_HOST_KVBLOCKS")) nkb = std::max(1, std::min(nkb, std::atoi(e)));
    const int64_t kper = (L + nkb - 1) / nkb;
    const int64_t n0 = std::min<int64_t>(per, L);
    if (nkb > 1)
      if (int rc = ensure_ring_ws(n0, D, H, false)) return rc;
    // staging buffers are free once earlier work on the compute stream is done
    CK_CUDA(cudaEventRecord(g.ev_start, g.stream));
    CK_CUDA(cudaStreamWaitEvent(g.comm, g.ev_start, 0));
    CK_CUDA(cudaStreamWaitEvent(g.d2h, g.ev_start, 0));
    auto h2d = [&](int64_t r0, int64_t n, size_t off, const void* src) {
      return cudaMemcpyAsync(dq + off + r0 * row_b, static_cast<const char*>(src) + r0 * row_b,
                             n * row_b, cudaMemcpyHostToDevice, g.comm);
    };
    CK_CUDA(h2d(0, n0, 0, q));
    CK_CUDA(cudaEventRecord(g.ev_h2d[0], g.comm));
    for (int b = 0; b < nkb; ++b) {
      const int64_t k0 = b * kper, kn = std::min<int64_t>(kper, L - k0);
      CK_CUDA(h2d(k0, kn, tb, k));
      CK_CUDA(h2d(k0, kn, 2 * tb, v));
      CK_CUDA(cudaEventRecord(g.ev_kv[b], g.comm));
    }
    int c = 1;
    for (int64_t r0 = per; r0 < L; r0 += per, ++c) {
      CK_CUDA(h2d(r0, std::min<int64_t>(per, L - r0), 0, q));
      CK_CUDA(cudaEventRecord(g.ev_h2d[c], g.comm));
    }
    c = 0;
    for (int64_t r0 = 0; r0 < L; r0 += per, ++c) {
      const int64_t n = std::min<int64_t>(per, L - r0);
      const dmha::PosMap qm{r0, r0 + n, n};
      float* lse_c = g.st_lse + r0 * H;  // chunk-major [chunk][H][n]
      char* out_c = static_cast<char*>(g.st_out) + r0 * row_b;
      if (c == 0 && nkb > 1) {
        for (int b = 0; b < nkb; ++b) {
          const int64_t k0 = b * kper, kn = std::min<int64_t>(kper, L - k0);
          CK_CUDA(cudaStreamWaitEvent(g.stream, g.ev_kv[b], 0));  // (Q chunk 0 precedes)
          const dmha::PosMap km{k0, k0 + kn, kn};
          const bool last = b == nkb - 1;
          int rc = b == 0 ? run_local(dq, dq + tb, dq + 2 * tb, g.o_acc, g.lse_acc, n, kn, D, H,
                                      causal, qm, km, dmha::OUT_PARTIAL_F32)
                          : run_local(dq, dq + tb + k0 * row_b, dq + 2 * tb + k0 * row_b,
                                      last ? static_cast<void*>(out_c) : g.o_acc,
                                      last ? lse_c : g.lse_acc, n, kn, D, H, causal, qm, km,
                                      last ? dmha::OUT_COMBINE_FINAL : dmha::OUT_COMBINE_ACC,
                                      g.o_acc, g.lse_acc);
          if (rc) return rc;
        }
      } else {
        CK_CUDA(cudaStreamWaitEvent(g.stream, g.ev_h2d[c], 0));
        CK_CUDA(cudaStreamWaitEvent(g.stream, g.ev_kv[nkb - 1], 0));
        const dmha::PosMap km{0, L, L};
        if (int rc = run_local(dq + r0 * row_b, dq + tb, dq + 2 * tb, out_c, lse_c, n, L, D, H,
                               causal, qm, km, dmha::OUT_FINAL))
          return rc;
      }
      CK_CUDA(cudaEventRecord(g.ev_comp[c], g.stream));
      CK_CUDA(cudaStreamWaitEvent(g.d2h, g.ev_comp[c], 0));
      CK_CUDA(cudaMemcpyAsync(static_cast<char*>(out) + r0 * row_b, out_c, n * row_b,
                              cudaMemcpyDeviceToHost, g.d2h));
      CK_CUDA(cudaMemcpy2DAsync(lse + r0, static_cast<size_t>(L) * 4, lse_c,
                                static_cast<size_t>(n) * 4, static_cast<size_t>(n) * 4, H,
                                cudaMemcpyDeviceToHost, g.d2h));
    }
    CK_CUDA(cudaStreamSynchronize(g.d2h));
    CK_CUDA(cudaStreamSynchronize(g.stream));
    g.stats.forwards++;
    return DMHA_OK;
  }
  CK_CUDA(cudaMemcpyAsync(dq, q, tb, cudaMemcpyHostToDevice, g.stream));
  CK_CUDA(cudaMemcpyAsync(dq + tb, k, tb, cudaMemcpyHostToDevice, g.stream));
  CK_CUDA(cudaMemcpyAsync(dq + 2 * tb, v, tb, cudaMemcpyHostToDevice, g.stream));
  if (int rc = dmha_forward(dq, dq + tb, dq + 2 * tb, g.st_out, g.st_lse, L, D, H, causal)) return rc;
  CK_CUDA(cudaMemcpyAsync(out, g.st_out, tb, cudaMemcpyDeviceToHost, g.stream));
  CK_CUDA(cudaMemcpyAsync(lse, g.st_lse, lb * 4, cudaMemcpyDeviceToHost, g.stream));
  CK_CUDA(cudaStreamSynchronize(g.stream));
  return DMHA_OK;
}

int dmha_forward_emulated(int world_size, int layout, const void* q, const void* k, const void* v,
                          void* out, float* lse, int64_t L, int D, int H, int causal) {
  if (int rc = check_state()) return rc;
  if (world_size < 1) return fail(DMHA_ERR_INVALID, "dmha_forward_emulated: world_size < 1");
  if (int rc = validate(q, k, v, out, lse, L, D, H, world_size, layout, world_size)) return rc;
  const int P = world_size;
  const int64_t Lm = max_shard_rows(L, P, layout);  // rows per shard slot
  const size_t blk = static_cast<size_t>(Lm) * H * D * elem_bytes(g.dtype);
  begin_forward();
  // Rank r's ring runs through the same loop, buffers, events and streams as
  // dmha_forward at world size P; only the transport differs: each receive is
  // one cudaMemcpyAsync per K / V block on the comm stream from the sending
  // rank's shard.  Ranks run one after the other (no kernel waits on another).
  // Slot r holds rank r's shard_rows(r) rows first (uneven contiguous shards
  // leave the last row of a short slot unused); its lse is [H, shard_rows(r)]
  // packed from the slot start.
  for (int r = 0; r < P; ++r) {
    CopyTransport tx(static_cast<const char*>(k), static_cast<const char*>(v), blk, P, r, layout, L);
    if (int rc = ring_forward(P, r, layout, static_cast<const char*>(q) + r * blk,
                              static_cast<const char*>(k) + r * blk,
                              static_cast<const char*>(v) + r * blk,
                              static_cast<char*>(out) + r * blk,
                              lse + static_cast<size_t>(r) * Lm * H, L, D, H, causal ? 1 : 0, tx))
      return rc;
  }
  g.stats.forwards++;
  return DMHA_OK;
}

int dmha_forward_headpar(const void* q, const void* k, const void* v, void* out, float* lse,
                         int64_t L, int D, int H, int causal) {
  if (int rc = check_state()) return rc;
  if (int rc = validate(q, k, v, out, lse, L, D, H, g.world, g.layout)) return rc;
  if (int rc = validate_headpar(g.world, L, H)) return rc;
  if (int rc = poll_nccl()) return rc;
  const int P = g.world, r = g.rank;
  causal = causal ? 1 : 0;
  if (P == 1) return dmha_forward(q, k, v, out, lse, L, D, H, causal);
  if (int rc = need_nccl()) return rc;
  if (int rc = check_collective_contract(L, D, H, causal)) return rc;
  begin_forward();
  const int64_t Lloc = L / P;
  const HpLayout y = hp_layout(P, Lloc, H, D, elem_bytes(g.dtype));
  if (int rc = ensure_hp(y.total)) return rc;
  char* ws = static_cast<char*>(g.hp);
  // Both all-to-alls run on the compute stream: the paper's shuffles are
  // blocking steps between the projections and the per-head softmax.
  auto a2a = [&](size_t send_off, size_t recv_off, size_t blk) -> int {
    CK_NCCL(ncclGroupStart());
    for (int d = 0; d < P; ++d) {
      CK_NCCL(ncclSend(ws + send_off + d * blk, blk, ncclChar, d, g.nccl, g.stream));
      CK_NCCL(ncclRecv(ws + recv_off + d * blk, blk, ncclChar, d, g.nccl, g.stream));
      if (d != r) count_sent(blk);
    }
    CK_NCCL(ncclGroupEnd());
    return DMHA_OK;
  };
  auto ex1 = [&]() -> int { return a2a(y.send1, y.recv1, y.qkv_blk); };
  auto ex2 = [&]() -> int {
    if (int rc = a2a(y.send2, y.recv2, y.out_blk)) return rc;
    // lse blocks land directly in the caller's [H, Lloc] lse (block s = heads of s)
    CK_NCCL(ncclGroupStart());
    for (int d = 0; d < P; ++d) {
      CK_NCCL(ncclSend(ws + y.send_lse + d * y.lse_blk, y.lse_blk, ncclChar, d, g.nccl, g.stream));
      CK_NCCL(ncclRecv(reinterpret_cast<char*>(lse) + d * y.lse_blk, y.lse_blk, ncclChar, d,
                       g.nccl, g.stream));
      if (d != r) count_sent(y.lse_blk);
    }
    CK_NCCL(ncclGroupEnd());
    return DMHA_OK;
  };
  int rc = headpar_rank(P, r, g.layout, q, k, v, out, lse, L, D, H, causal, ws, y, ex1, ex2, true);
  if (rc) return rc;
  g.stats.forwards++;
  return DMHA_OK;
}

int dmha_forward_headpar_emulated(int world_size, int layout, const void* q, const void* k,
                                  const void* v, void* out, float* lse, int64_t L, int D, int H,
                                  int causal) {
  if (int rc = check_state()) return rc;
  if (world_size < 1) return fail(DMHA_ERR_INVALID, "dmha_forward_headpar_emulated: world_size < 1");
  if (int rc = validate(q, k, v, out, lse, L, D, H, world_size, layout, world_size)) return rc;
  if (int rc = validate_headpar(world_size, L, H)) return rc;
  const int P = world_size;
  const int64_t Lloc = L / P;
  causal = causal ? 1 : 0;
  const size_t e = elem_bytes(g.dtype);
  const size_t shard = static_cast<size_t>(Lloc) * H * D * e;
  const size_t lshard = static_cast<size_t>(Lloc) * H * 4;
  const HpLayout y = hp_layout(P, Lloc, H, D, e);
  if (int rc = ensure_hp(P * y.total)) return rc;
  begin_forward();
  char* base = static_cast<char*>(g.hp);
  auto ws_of = [&](int r) { return base + static_cast<size_t>(r) * y.total; };
  // Phase 1: every rank packs; the all-to-all is P*P device copies.
  for (int r = 0; r < P; ++r) {
    const dmha::HeadparGeom geo{P, H, D, Lloc, layout == DMHA_LAYOUT_ZIGZAG ? 1 : 0};
    CK_PACK(dmha::launch_headpar_pack_qkv(static_cast<const char*>(q) + r * shard,
                                          static_cast<const char*>(k) + r * shard,
                                          static_cast<const char*>(v) + r * shard,
                                          ws_of(r) + y.send1, geo, static_cast<int>(e), g.stream),
            hp_qkv_bytes(Lloc, H, D, e));
  }
  for (int s = 0; s < P; ++s)
    for (int d = 0; d < P; ++d) {
      CK_CUDA(cudaMemcpyAsync(ws_of(d) + y.recv1 + s * y.qkv_blk, ws_of(s) + y.send1 + d * y.qkv_blk,
                              y.qkv_blk, cudaMemcpyDeviceToDevice, g.stream));
      if (d != s) count_sent(y.qkv_blk);
    }
  // Phase 2: per rank unpack, attention for its heads, pack (no-op exchanges).
  for (int r = 0; r < P; ++r) {
    const int64_t Lg = L;
    const dmha::HeadparGeom geo{P, H, D, Lloc, layout == DMHA_LAYOUT_ZIGZAG ? 1 : 0};
    char* ws = ws_of(r);
    CK_PACK(dmha::launch_headpar_unpack_qkv(ws + y.recv1, ws + y.xq, ws + y.xk, ws + y.xv, geo,
                                            static_cast<int>(e), g.stream),
            hp_qkv_bytes(Lloc, H, D, e));
    const dmha::PosMap full{0, Lg, Lg};
    if (int rc = run_local(ws + y.xq, ws + y.xk, ws + y.xv, ws + y.outg,
                           reinterpret_cast<float*>(ws + y.lseg), Lg, Lg, D, H / P, causal, full,
                           full, dmha::OUT_FINAL))
      return rc;
    CK_PACK(dmha::launch_headpar_pack_out(ws + y.outg, ws + y.send2,
                                          reinterpret_cast<const float*>(ws + y.lseg),
                                          reinterpret_cast<float*>(ws + y.send_lse), geo,
                                          static_cast<int>(e), g.stream),
            hp_out_bytes(Lloc, H, D, e, true));
  }
  // Phase 3: all-to-all back (out blocks and lse blocks), unpack per rank.
  for (int s = 0; s < P; ++s)
    for (int d = 0; d < P; ++d) {
      CK_CUDA(cudaMemcpyAsync(ws_of(d) + y.recv2 + s * y.out_blk, ws_of(s) + y.send2 + d * y.out_blk,
                              y.out_blk, cudaMemcpyDeviceToDevice, g.stream));
      CK_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(lse) + d * lshard + s * y.lse_blk,
                              ws_of(s) + y.send_lse + d * y.lse_blk, y.lse_blk,
                              cudaMemcpyDeviceToDevice, g.stream));
      if (d != s) count_sent(y.out_blk + y.lse_blk);
    }
  for (int r = 0; r < P; ++r) {
    const dmha::HeadparGeom geo{P, H, D, Lloc, layout == DMHA_LAYOUT_ZIGZAG ? 1 : 0};
    CK_PACK(dmha::launch_headpar_unpack_out(ws_of(r) + y.recv2, static_cast<char*>(out) + r * shard,
                                            geo, static_cast<int>(e), g.stream),
            hp_out_bytes(Lloc, H, D, e, false));
  }
  g.stats.forwards++;
  return DMHA_OK;
}

// NEXT-3 projection GEMM on the compute stream (timed as kind 4 when profiling).
int run_gemm(const void* A, const void* B, void* C, int64_t M, int N, int K) {
  cudaError_t e = cudaSuccess;
  const auto t0 = g.pending.size();
  timed(4, g.stream, [&]() {
    e = dmha::launch_gemm_bf16(A, B, C, M, N, K, g.stream);
    return 0;
  });
  if (g.pending.size() > t0) g.pending.back().flop = 2.0 * static_cast<double>(M) * N * K;
  if (e != cudaSuccess)
    return fail(DMHA_ERR_CUDA, "dmha: projection GEMM launch failed: %s", cudaGetErrorString(e));
  g.stats.kernel_launches++;
  return DMHA_OK;
}

int dmha_linear(const void* x, const void* w, void* y, int64_t M, int N, int K) {
  if (int rc = check_state()) return rc;
  if (g.dtype != DMHA_BF16) return fail(DMHA_ERR_UNSUPPORTED, "dmha_linear: bf16 only");
  if (M < 0 || N < 1 || K < 1 || N % 8 != 0 || K % 8 != 0 || M > INT32_MAX)
    return fail(DMHA_ERR_INVALID, "dmha_linear: need M >= 0, N and K positive multiples of 8");
  if (M == 0) return DMHA_OK;  // nothing to compute (x and y may be empty / null)
  if (!x || !w || !y) return fail(DMHA_ERR_INVALID, "dmha_linear: null pointer");
  const void* ptrs[3] = {x, w, y};
  for (const void* p : ptrs)
    if (reinterpret_cast<uintptr_t>(p) % 16 != 0)
      return fail(DMHA_ERR_INVALID, "dmha_linear: pointers must be 16-byte aligned");
  const size_t yb = static_cast<size_t>(M) * N * 2;
  if (overlaps(y, yb, x, static_cast<size_t>(M) * K * 2) || overlaps(y, yb, w, static_cast<size_t>(K) * N * 2))
    return fail(DMHA_ERR_INVALID, "dmha_linear: y overlaps x or w");
  return run_gemm(x, w, y, M, N, K);
}

int dmha_mha_forward(const void* x, const void* wq, const void* wk, const void* wv,
                     const void* wo, void* y, float* lse, int64_t L, int d_model, int D, int H,
                     int causal) {
  if (int rc = check_state()) return rc;
  if (g.dtype != DMHA_BF16) return fail(DMHA_ERR_UNSUPPORTED, "dmha_mha_forward: bf16 only");
  if (!x || !wq || !wk || !wv || !wo || !y)
    return fail(DMHA_ERR_INVALID, "dmha_mha_forward: null pointer");
  if (d_model < 1 || d_model % 8 != 0)
    return fail(DMHA_ERR_INVALID, "dmha_mha_forward: d_model must be a positive multiple of 8");
  if (L < 1 || H < 1 || (g.layout == DMHA_LAYOUT_ZIGZAG && L % (2LL * g.world)))
    return fail(DMHA_ERR_INVALID, "dmha_mha_forward: bad L/H for world size %d", g.world);
  if (D != 64 && D != 128) return fail(DMHA_ERR_UNSUPPORTED, "dmha_mha_forward: D=%d", D);
  const int64_t Lloc = shard_rows(L, g.world, g.rank, g.layout);
  const size_t act = static_cast<size_t>(Lloc) * H * D * 2;
  const size_t lbytes = static_cast<size_t>(Lloc) * H * 4;
  const size_t need = 4 * act + lbytes + 4 * 256;
  if (need > g.mha_bytes) {
    free_ptr(g.mha);
    g.mha_bytes = 0;
    if (int rc = alloc_or_oom(&g.mha, need, "MHA layer activations")) return rc;
    g.mha_bytes = need;
    update_ws_stat();
  }
  char* ws = static_cast<char*>(g.mha);
  char* q = ws;
  char* k = q + act;
  char* v = k + act;
  char* o = v + act;
  float* l = reinterpret_cast<float*>(o + act);
  const int HD = H * D;
  // Row-major C[M,N] = A[M,K] B[K,N] on the tcgen05 GEMM (gemm_sm100.cu).
  auto gemm = [&](const void* A, const void* B, void* Cm, int64_t M, int N, int K) -> int {
    return run_gemm(A, B, Cm, M, N, K);
  };
  // replicated W_Q, W_K, W_V applied to this rank's rows, all heads.
  if (int rc = gemm(x, wq, q, Lloc, HD, d_model)) return rc;
  if (int rc = gemm(x, wk, k, Lloc, HD, d_model)) return rc;
  if (int rc = gemm(x, wv, v, Lloc, HD, d_model)) return rc;
  // the distributed attention (ring; same result as the paper's exchange).
  if (int rc = dmha_forward(q, k, v, o, lse ? lse : l, L, D, H, causal)) return rc;
  // concatenated heads times the replicated W_0.
  return gemm(o, wo, y, Lloc, d_model, HD);
}

int dmha_attention_local(const void* q, const void* k, const void* v, void* out, float* lse,
                         int64_t Lq, int64_t Lk, int D, int H, int causal, int64_t q_base0,
                         int64_t q_base1, int64_t q_chunk, int64_t k_base0, int64_t k_base1,
                         int64_t k_chunk, int out_mode) {
  if (int rc = check_state()) return rc;
  if (!q || !k || !v || !out || !lse) return fail(DMHA_ERR_INVALID, "dmha_attention_local: null pointer");
  if (Lq < 0 || Lk < 0 || H < 1) return fail(DMHA_ERR_INVALID, "dmha_attention_local: bad sizes");
  if (D != 64 && D != 128) return fail(DMHA_ERR_UNSUPPORTED, "dmha_attention_local: D=%d", D);
  if (out_mode != dmha::OUT_FINAL && out_mode != dmha::OUT_PARTIAL_F32)
    return fail(DMHA_ERR_INVALID, "dmha_attention_local: bad out_mode");
  if (q_chunk < 0 || k_chunk < 0 || q_base1 < q_base0 + q_chunk || k_base1 < k_base0 + k_chunk)
    return fail(DMHA_ERR_INVALID, "dmha_attention_local: position maps must be increasing");
  const void* ptrs[5] = {q, k, v, out, lse};
  for (const void* p : ptrs)
    if (reinterpret_cast<uintptr_t>(p) % 16 != 0)
      return fail(DMHA_ERR_INVALID, "dmha_attention_local: pointers must be 16-byte aligned");
  dmha::PosMap qm{q_base0, q_base1, q_chunk}, km{k_base0, k_base1, k_chunk};
  return run_local(q, k, v, out, lse, Lq, Lk, D, H, causal ? 1 : 0, qm, km, out_mode);
}

// ---------------------------------------------------------------- NEXT-4
// Token Selector s_{psi,tau} (PAPER.md Eq. `selector` P:630-634, readings
// R18-R21): score, keep iff score >= tau in order, never empty over all ranks.
int dmha_select(const void* x, int64_t n_rows, int width, int scorer, const void* psi,
                double tau, void* x_out, int64_t* idx_out, double* scores, int64_t* n_kept) {
  if (int rc = check_state()) return rc;
  if (!x || !x_out || !idx_out || !n_kept) return fail(DMHA_ERR_INVALID, "dmha_select: null pointer");
  if (n_rows < 1 || width < 8 || width % 8)
    return fail(DMHA_ERR_INVALID, "dmha_select: need n_rows >= 1 and width a positive multiple of 8");
  if (scorer != DMHA_SCORER_L2 && scorer != DMHA_SCORER_PROJ)
    return fail(DMHA_ERR_INVALID, "dmha_select: unknown scorer %d", scorer);
  if ((scorer == DMHA_SCORER_PROJ) != (psi != nullptr))
    return fail(DMHA_ERR_INVALID, "dmha_select: psi must be given exactly for the projection scorer");
  if (std::isnan(tau)) return fail(DMHA_ERR_INVALID, "dmha_select: tau is NaN");
  auto mis = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) != 0; };
  if (mis(x) || mis(x_out) || (psi && mis(psi)) || (reinterpret_cast<uintptr_t>(idx_out) & 7))
    return fail(DMHA_ERR_INVALID, "dmha_select: x/x_out/psi must be 16-byte aligned");
  if (g.dtype != DMHA_BF16) return fail(DMHA_ERR_UNSUPPORTED, "dmha_select: bf16 rows only");
  // the tie-break maps local rows to global positions with the init layout:
  // every rank holds the same n_rows (collective contract), two equal zigzag
  // chunks of them when the layout is zigzag
  if (g.world > 1 && g.layout == DMHA_LAYOUT_ZIGZAG && n_rows % 2)
    return fail(DMHA_ERR_INVALID, "dmha_select: zigzag layout needs an even n_rows per rank");
  // workspace: flags | tile counts | tile offsets | 8 int64/double slots | scores
  const int64_t nb = dmha::selector_tiles(n_rows);
  const size_t off_counts = (static_cast<size_t>(n_rows) + 255) & ~size_t(255);
  const size_t off_offsets = off_counts + ((static_cast<size_t>(nb) * 4 + 255) & ~size_t(255));
  const size_t off_slots = off_offsets + static_cast<size_t>(nb) * 8;
  const size_t off_scores = off_slots + 64;
  const size_t need = off_scores + static_cast<size_t>(n_rows) * 8;
  if (need > g.sel_bytes) {
    free_ptr(g.sel);
    g.sel_bytes = 0;
    if (int rc = alloc_or_oom(&g.sel, need, "selector workspace")) return rc;
    g.sel_bytes = need;
    update_ws_stat();
  }
  char* ws = static_cast<char*>(g.sel);
  auto* flags = reinterpret_cast<uint8_t*>(ws);
  auto* counts = reinterpret_cast<int*>(ws + off_counts);
  auto* offsets = reinterpret_cast<int64_t*>(ws + off_offsets);
  auto* slots = reinterpret_cast<int64_t*>(ws + off_slots);  // [0] total [1] global [2] row [3] cand
  auto* dbest = reinterpret_cast<double*>(slots + 4);         // [4] best score [5] global best
  double* sc = scores ? scores : reinterpret_cast<double*>(ws + off_scores);
  CK_LAUNCH(dmha::launch_selector_score(x, psi, n_rows, width, scorer, tau, sc, flags, counts,
                                        g.stream));
  CK_LAUNCH(dmha::launch_selector_scan(counts, n_rows, offsets, slots, g.stream));
  g.stats.kernel_launches += 2;
  if (g.world > 1) {
    if (int rc = need_nccl()) return rc;
    CK_NCCL(ncclAllReduce(slots, slots + 1, 1, ncclInt64, ncclSum, g.nccl, g.stream));
  } else {
    CK_CUDA(cudaMemcpyAsync(slots + 1, slots, 8, cudaMemcpyDeviceToDevice, g.stream));
  }
  int64_t h[2];
  CK_CUDA(cudaMemcpyAsync(h, slots, 16, cudaMemcpyDeviceToHost, g.stream));
  CK_CUDA(cudaStreamSynchronize(g.stream));
  if (h[1] > 0) {  // something passes somewhere: plain order-preserving compaction
    CK_LAUNCH(dmha::launch_selector_compact(x, n_rows, width, flags, offsets, x_out, idx_out,
                                            g.stream));
    g.stats.kernel_launches += 1;
    *n_kept = h[0];
    return DMHA_OK;
  }
  // Never-empty rule (R19): the highest score over all ranks, ties -> the
  // smallest GLOBAL position, is kept by its owner.
  CK_LAUNCH(dmha::launch_selector_argmax(sc, n_rows, dbest, slots + 2, g.stream));
  g.stats.kernel_launches += 1;
  if (g.world > 1) {
    CK_NCCL(ncclAllReduce(dbest, dbest + 1, 1, ncclFloat64, ncclMax, g.nccl, g.stream));
  } else {
    CK_CUDA(cudaMemcpyAsync(dbest + 1, dbest, 8, cudaMemcpyDeviceToDevice, g.stream));
  }
  double hb[2];
  int64_t hrow = 0;
  CK_CUDA(cudaMemcpyAsync(hb, dbest, 16, cudaMemcpyDeviceToHost, g.stream));
  CK_CUDA(cudaMemcpyAsync(&hrow, slots + 2, 8, cudaMemcpyDeviceToHost, g.stream));
  CK_CUDA(cudaStreamSynchronize(g.stream));
  const dmha::PosMap m = posmap(n_rows * g.world, g.world, g.rank, g.layout);
  const int64_t my_gpos = hrow < m.chunk ? m.base0 + hrow : m.base1 + (hrow - m.chunk);
  int64_t cand[2] = {hb[0] == hb[1] ? my_gpos : INT64_MAX, 0};
  if (g.world > 1) {
    CK_CUDA(cudaMemcpyAsync(slots + 3, cand, 8, cudaMemcpyHostToDevice, g.stream));
    CK_NCCL(ncclAllReduce(slots + 3, slots + 1, 1, ncclInt64, ncclMin, g.nccl, g.stream));
    CK_CUDA(cudaMemcpyAsync(cand + 1, slots + 1, 8, cudaMemcpyDeviceToHost, g.stream));
    CK_CUDA(cudaStreamSynchronize(g.stream));
  } else {
    cand[1] = cand[0];
  }
  if (cand[0] != INT64_MAX && cand[0] == cand[1]) {
    CK_CUDA(cudaMemcpyAsync(x_out, static_cast<const char*>(x) + hrow * width * 2,
                            static_cast<size_t>(width) * 2, cudaMemcpyDeviceToDevice, g.stream));
    CK_CUDA(cudaMemcpyAsync(idx_out, slots + 2, 8, cudaMemcpyDeviceToDevice, g.stream));
    CK_CUDA(cudaStreamSynchronize(g.stream));
    *n_kept = 1;
  } else {
    *n_kept = 0;
  }
  return DMHA_OK;
}

int dmha_scatter_rows(const void* y_sel, const int64_t* idx, int64_t n_kept, int width,
                      void* y_full) {
  if (int rc = check_state()) return rc;
  if (n_kept < 0 || width < 8 || width % 8)
    return fail(DMHA_ERR_INVALID, "dmha_scatter_rows: bad n_kept/width");
  if (n_kept == 0) return DMHA_OK;
  if (!y_sel || !idx || !y_full) return fail(DMHA_ERR_INVALID, "dmha_scatter_rows: null pointer");
  auto mis = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) != 0; };
  if (mis(y_sel) || mis(y_full)) return fail(DMHA_ERR_INVALID, "dmha_scatter_rows: misaligned");
  if (g.dtype != DMHA_BF16) return fail(DMHA_ERR_UNSUPPORTED, "dmha_scatter_rows: bf16 rows only");
  CK_LAUNCH(dmha::launch_scatter_rows(y_sel, idx, n_kept, width, y_full, g.stream));
  g.stats.kernel_launches += 1;
  return DMHA_OK;
}

int dmha_lse_combine(float* o_acc, float* lse_acc, const float* o_part, const float* lse_part,
                     void* out, float* lse_out, int64_t Lq, int D, int H, int final_step) {
  if (int rc = check_state()) return rc;
  if (!o_acc || !lse_acc || !o_part || !lse_part) return fail(DMHA_ERR_INVALID, "dmha_lse_combine: null");
  if (final_step && (!out || !lse_out)) return fail(DMHA_ERR_INVALID, "dmha_lse_combine: null out");
  if (Lq < 0 || H < 1) return fail(DMHA_ERR_INVALID, "dmha_lse_combine: bad sizes");
  if (D != 64 && D != 128) return fail(DMHA_ERR_UNSUPPORTED, "dmha_lse_combine: D=%d", D);
  cudaError_t e = dmha::launch_lse_combine(o_acc, lse_acc, o_part, lse_part, out, lse_out, Lq, D,
                                           H, final_step, g.dtype == DMHA_BF16, g.stream);
  if (e != cudaSuccess) return fail(DMHA_ERR_CUDA, "dmha_lse_combine: %s", cudaGetErrorString(e));
  g.stats.kernel_launches += 1;
  return DMHA_OK;
}

int dmha_debug_set_trace(void* dev_buf) {
  dmha::g_trace = static_cast<unsigned long long*>(dev_buf);
  return DMHA_OK;
}

int dmha_synchronize(void) {
  if (int rc = check_state()) return rc;
  CK_CUDA(cudaStreamSynchronize(g.stream));
  CK_CUDA(cudaStreamSynchronize(g.comm));
  return poll_nccl();
}

}  // extern "C"
