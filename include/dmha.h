/*
 * dmha.h — C ABI of the B200-native distributed multi-head attention forward
 * (arXiv 2302.06218, §10.4 "Distributed Attention").
 *
 * Every function is extern "C", takes plain pointers and sizes, returns an int
 * status (0 = DMHA_OK, < 0 = error) and never throws or aborts.  On error,
 * dmha_last_error() returns a thread-local human-readable message.
 *
 * Operation (§4, with the north_star 1/sqrt(D) scale):
 *   for every global query row g and head h
 *     out[g,h,:] = sum_{j in A(g)} softmax_j(q[g,h,:].k[j,h,:] / sqrt(D)) v[j,h,:]
 *     lse[h,g]   = ln sum_{j in A(g)} exp(q[g,h,:].k[j,h,:] / sqrt(D))
 *   A(g) = all j (non-causal) or j <= g on GLOBAL positions (causal).
 * The sequence is split into P = world_size partitions ("split the
 * design matrix X along the sequence dimension into N partitions"); the result
 * is defined in global order and does not depend on P or the layout.
 *
 * Tensor layouts (all row-major, contiguous, base pointers 16-byte aligned):
 *   q, k, v, out : [L_loc, H, D]  this rank's L_loc = L / P rows, in the order
 *                  the layout defines (see dmha_local_to_global).
 *   lse          : [H, L_loc] fp32 (natural log) — always fp32.
 * Element type of q/k/v/out is fixed by the dtype given to dmha_init:
 *   DMHA_BF16 -> bf16 storage, bf16 tensor-core MMA, fp32 accumulation/softmax;
 *   DMHA_FP32 -> fp32 storage; both contractions as 3xTF32 tcgen05 MMAs (hi/lo
 *                operand splits), fp32 softmax and accumulation (rel L2 ~4e-6
 *                against fp64; DMHA_FP32_SIMT=1 selects the SIMT fp32 FMA
 *                kernel, kept as a cross-check).
 *
 * Ownership: the caller owns q, k, v, out and lse.  q/k/v are read only (the
 * ring sends from them at step 0 and from library buffers afterwards); out and
 * lse are fully overwritten.  The library owns its NCCL communicator, ring
 * buffers, fp32 accumulators and TMA descriptors; they are allocated lazily,
 * grown on a larger shape and freed by dmha_finalize.  One device per process;
 * calls are not thread safe.  dmha_forward is stream-ordered and asynchronous
 * (like a kernel launch) on the stream given to dmha_init / dmha_set_stream.
 */
#ifndef DMHA_H_
#define DMHA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DMHA_UNIQUE_ID_BYTES 128 /* == sizeof(ncclUniqueId) */

enum dmha_status {
  DMHA_OK = 0,
  DMHA_ERR_INVALID = -1,     /* bad pointer / size / alignment / aliasing      */
  DMHA_ERR_UNSUPPORTED = -2, /* D not in {64,128}, unsupported dtype combo     */
  DMHA_ERR_CUDA = -3,        /* a CUDA runtime/driver call failed              */
  DMHA_ERR_NCCL = -4,        /* an NCCL call failed or an async NCCL error     */
  DMHA_ERR_OOM = -5,         /* workspace allocation failed (max-L search)     */
  DMHA_ERR_STATE = -6        /* call before dmha_init or after dmha_finalize   */
};

enum dmha_dtype { DMHA_BF16 = 0, DMHA_FP32 = 1 };

/* Shard layout ("N partitions {P_i}"):
 *  CONTIGUOUS: rank r owns global rows [r*L/P, (r+1)*L/P).
 *  ZIGZAG:     with c = L/(2P), rank r owns chunk r then chunk 2P-1-r
 *              (global rows [r*c,(r+1)*c) then [(2P-1-r)*c,(2P-r)*c)); balances
 *              causal work exactly.  Requires L % (2P) == 0. */
enum dmha_layout { DMHA_LAYOUT_CONTIGUOUS = 0, DMHA_LAYOUT_ZIGZAG = 1 };

struct dmha_stats {
  uint64_t bytes_sent;      /* K/V bytes this rank sent over the ring (cumulative) */
  uint64_t ring_steps;      /* ring steps executed (cumulative)                  */
  uint64_t forwards;        /* dmha_forward calls completed                      */
  uint64_t kernel_launches; /* device kernels launched by the library (cumulative) */
  uint64_t workspace_bytes; /* bytes currently held by the library on the device  */
  /* Filled only while profiling is on (dmha_set_profiling): CUDA-event time of
   * each launch, recorded on the stream the kernel runs on, summed. */
  uint64_t attn_launches;    /* attention kernel launches timed                   */
  uint64_t combine_launches; /* LSE-combine kernel launches timed                 */
  uint64_t exchanges;        /* ring K/V exchanges (NCCL groups) timed            */
  double attn_ms;            /* summed attention kernel time                      */
  double combine_ms;         /* summed combine kernel time                        */
  double exchange_ms;        /* summed send/recv time on the comm stream          */
  /* Per-forward accounting, reset at the start of every forward call and
   * counted at each send: bytes this rank sent (the emulated entry points sum
   * their P ranks) and the number of exchanges (ring steps / all-to-all
   * blocks).  Ring: exactly (P-1) * 2 * L_loc*H*D*elem per rank. */
  uint64_t last_bytes_sent;
  uint64_t last_exchanges;
  /* Profiling only: the head-parallel exchange's pack/unpack copy kernels
   * (NEXT-1), CUDA-event time summed, and the bytes they read + wrote. */
  uint64_t pack_launches;
  double pack_ms;
  uint64_t pack_bytes;
  /* Profiling only: the NEXT-3 projection GEMMs (dmha_linear, tcgen05),
   * CUDA-event time summed and their algorithmic FLOP (2*M*N*K each). */
  uint64_t gemm_launches;
  double gemm_ms;
  double gemm_flop;
};

/* ---- setup / teardown ----------------------------------------------------
 * SURVEY.md §8(b) (the C-ABI boundary) and §3c: one process per GPU; the NCCL
 * communicator realises the "N GPUs in one node" of PAPER.md:664-668. */

/* Rank 0 only, before dmha_init with world_size > 1: writes a 128-byte NCCL
 * unique id to id_out; the caller broadcasts it (e.g. torch.distributed). */
int dmha_get_unique_id(void *id_out);

/* world_size >= 1, 0 <= rank < world_size; unique_id NULL iff world_size == 1.
 * device: CUDA ordinal for this process; dtype: enum dmha_dtype; layout: enum
 * dmha_layout; cuda_stream: cudaStream_t (NULL = legacy default stream).
 * Collective over all ranks when world_size > 1.  K/V transport of the ring
 * (env DMHA_TRANSPORT, read here): "nccl" (default) — ncclCommInitRank now;
 * "peer" — every rank's K/V block is published in a
 * library buffer shared by CUDA IPC and pulled by its consumers with the copy
 * engine, ordered by interprocess events behind a host barrier in POSIX
 * shared memory named after unique_id (ranks on one node); the
 * NCCL communicator is then created on first use by a collective entry point
 * (dmha_forward_headpar, dmha_select).  Errors: INVALID (arguments, unknown
 * DMHA_TRANSPORT), UNSUPPORTED (not sm_100), CUDA, NCCL, STATE (shared-memory
 * barrier failure or a rank missing for 300 s). */
int dmha_init(int world_size, int rank, const void *unique_id, int device, int dtype,
              int layout, void *cuda_stream);

/* Change the stream later calls are ordered on. */
int dmha_set_stream(void *cuda_stream);

/* Frees every library allocation, destroys the communicator and (peer
 * transport) unmaps the peers' buffers after a host barrier.  Collective when
 * world_size > 1. */
int dmha_finalize(void);

/* Thread-local message describing the last error ("" if none). */
const char *dmha_last_error(void);

/* ---- the distributed forward -------------------- */

/* q, k, v, out: DEVICE pointers to this rank's [L_loc, H, D] shard; lse: DEVICE
 * [H, L_loc] fp32, L_loc = dmha_shard_rows(L, P, rank, layout).  L is the
 * GLOBAL length (any L >= 1 for CONTIGUOUS — uneven shards differ by one row
 * and the ring moves each block at its owner's size; L % 2P == 0 for ZIGZAG), D the
 * per-head dim (64 or 128), H >= 1 heads, causal 0/1.  All ranks must call with
 * identical (L, D, H, causal).  Ring: P-1 steps of ncclSend/ncclRecv of (K,V)
 * to rank+1 / from rank-1 (peer transport: a copy-engine pull of the block of
 * step s+1 straight from its owner's published buffer) overlapped with the
 * local attention kernel, and an
 * fp32 log-sum-exp combine of the per-step partials into a running
 * accumulator (north_star (3)) — for bf16 fused into the attention kernel's
 * epilogue (env DMHA_FUSED_COMBINE=0 selects the
 * separate combine kernel, bit-identical result).
 * Ordering: the exchange of step s runs on a library comm stream and lands
 * in ring buffer (s+1)%2 after the attention of step s-1 (that buffer's last
 * reader) finished; the attention of step s+1 waits for it.  One NVTX range
 * per ring step ("dmha ring rank r step s src j") brackets the enqueue.
 * Debug: DMHA_CHECK_COLLECTIVE=1 cross-checks (L, D, H, causal) over the
 * ranks with two tiny all-reduces first (INVALID on a mismatch);
 * DMHA_FAULT=perturb_lse adds 0.5 to every partial lse inside the combine
 * (fault injection: the parity suite must then fail).
 * Errors: INVALID (null, sizes, misaligned, out/lse overlapping q/k/v),
 * UNSUPPORTED (D), STATE, OOM, CUDA, NCCL. */
int dmha_forward(const void *q, const void *k, const void *v, void *out, float *lse,
                 int64_t L, int D, int H, int causal);

/* Same operation with HOST buffers (pinned recommended): copies q/k/v to
 * device staging buffers, runs dmha_forward, copies out/lse back and
 * synchronises the stream before returning (the end-to-end path).  At world
 * size 1 and L >= 65536 the copies are pipelined with the compute: the first
 * Q row chunk (all of Q when causal) is attended over K/V blocks as they land
 * (ring-style fused log-sum-exp combine); non-causal, the remaining Q chunks
 * (up to 8) attend all keys as each lands, and each chunk's out/lse rows are
 * copied back on a separate stream while the next one computes. */
int dmha_forward_host(const void *q, const void *k, const void *v, void *out, float *lse,
                      int64_t L, int D, int H, int causal);

/* Single-GPU emulation of the P-rank ring (test/measurement hook): q/k/v/out
 * are DEVICE [P][Lm, H, D] buffers holding every rank's shard back to back
 * (rank-major), lse is [P][H*Lm], Lm = the largest shard (ceil(L/P) for
 * CONTIGUOUS); slot r holds rank r's dmha_shard_rows rows first and its lse
 * as [H, rows] packed from the slot start (for even shards simply
 * [P][Lm, H, D] and [P][H, Lm]).  Runs each rank's ring in turn through
 * the SAME loop as dmha_forward at world_size P — the two K/V ring buffers,
 * the comm stream, the recv/compute events and the buffer-reuse rule — with a
 * single-GPU transport: each receive is one cudaMemcpyAsync per K and per V
 * block on the comm stream from the sending rank's shard (what NCCL would
 * deliver), overlapping the attention on the compute stream.  No two kernels
 * wait on one another.  Uses the dtype/stream of dmha_init (which may have
 * world_size 1).  Overlap checks cover all P shards. */
int dmha_forward_emulated(int world_size, int layout, const void *q, const void *k,
                          const void *v, void *out, float *lse, int64_t L, int D, int H,
                          int causal);

/* NEXT-1 — the paper's own distributed algorithm (§10.4):
 * all-to-all from sequence-parallel to head-parallel (each rank receives all
 * L rows of H/P heads), full-L attention per head on each rank
 * (P:674), all-to-all back to sequence-parallel.  Same arguments,
 * layouts and result as dmha_forward; requires H % world_size == 0.  The two
 * exchanges are blocking steps on the compute stream (as in the paper); the
 * ring (dmha_forward) overlaps its exchange instead. */
int dmha_forward_headpar(const void *q, const void *k, const void *v, void *out, float *lse,
                         int64_t L, int D, int H, int causal);

/* NEXT-3 — the full distributed MHA layer around the attention:
 * Q = X W_Q, K = X W_K, V = X W_V with the weights replicated on every rank
 * and applied to this rank's rows for all heads; the
 * distributed attention (dmha_forward); Y = concat_h(O) W_0.
 *  x: DEVICE [L_loc, d_model] bf16 (this rank's rows, layout of dmha_init);
 *  wq, wk, wv: DEVICE [d_model, H*D] bf16 row-major (head h = columns
 *  [h*D, (h+1)*D)); wo: DEVICE [H*D, d_model]; y: DEVICE [L_loc, d_model] bf16;
 *  lse: DEVICE [H, L_loc] fp32 or NULL.  bf16 dtype only; d_model % 8 == 0.
 * The projections are dmha_linear (hand-written tcgen05 GEMMs, fp32
 * accumulate); Q, K, V and O are kept as bf16 activations in library
 * workspace (reading R17).  Collective like dmha_forward. */
int dmha_mha_forward(const void *x, const void *wq, const void *wk, const void *wv,
                     const void *wo, void *y, float *lse, int64_t L, int d_model, int D, int H,
                     int causal);

/* NEXT-3 projection step (PAPER.md:186-191 V = X W^V, K = X W^K, Q = X W^Q;
 * P:675 the W_0 projection): y = x w on this rank, row-major bf16,
 *  x: DEVICE [M, K], w: DEVICE [K, N], y: DEVICE [M, N] (caller-owned, fully
 *  overwritten, must not overlap x or w); fp32 accumulation on the tcgen05
 *  tensor cores (TMEM), bf16 round-to-nearest-even output.
 * N and K positive multiples of 8 (16-byte rows), M >= 0 (M = 0 is a no-op and
 * accepts null x / y),
 * 16-byte aligned pointers; bf16 dtype only (DMHA_ERR_UNSUPPORTED otherwise).
 * Asynchronous on the library stream; no communication (rows are local). */
int dmha_linear(const void *x, const void *w, void *y, int64_t M, int N, int K);

/* Single-GPU emulation of dmha_forward_headpar at world size P (buffers as in
 * dmha_forward_emulated); the all-to-alls become device copies. */
int dmha_forward_headpar_emulated(int world_size, int layout, const void *q, const void *k,
                                  const void *v, void *out, float *lse, int64_t L, int D, int H,
                                  int causal);

/* Library workspace (SURVEY §8(d) max-L footprint): device bytes a forward
 * of (L, D, H) allocates per rank at the initialised world size and dtype.
 * World size P > 1: 2 K/V receive buffers (2 * 2 * L_loc*H*D*elem) + the
 * fp32 accumulator O_acc and lse_acc (+ the O_part / lse_part partial buffers
 * when the combine is not fused).  World size 1: 0, except on small grids
 * (< 4 waves of 256-row CTAs, L >= 2048, bf16) where the split-KV launch
 * holds two fp32 partials: 2 * (L*H*D*4 + L*H*4).  dtype fp32 adds, at
 * every world size, the 3xTF32 kernel's split operands of one key block:
 * K hi/lo and V^T hi/lo, 2*L_loc*H*D*4 + 2*H*D*ceil4(L_loc)*4 bytes (PAPER.md
 * :193-211 as 3xTF32, reading R13).  Staging buffers of
 * dmha_forward_host are not included.  A fresh library that runs one forward
 * holds exactly this (dmha_stats.workspace_bytes).  Errors: STATE, INVALID,
 * UNSUPPORTED (D). */
int dmha_workspace_bytes(int64_t L, int D, int H, size_t *bytes_out);

/* Same for an explicit world size (what dmha_forward_emulated at world_size
 * holds, which runs each rank with one set of ring buffers). */
int dmha_ring_workspace_bytes(int world_size, int64_t L, int D, int H, size_t *bytes_out);

/* Allocate now the workspace a forward of global length L (D, H) at
 * world_size needs (dmha_ring_workspace_bytes; world_size = the init world
 * size for dmha_forward, P for dmha_forward_emulated), so that later forwards
 * of that size or smaller allocate nothing: no implicit device
 * synchronisation inside a forward, and the forward can be captured into a
 * CUDA graph (stream capture; the ring's comm stream joins the capture
 * through its events).  Collective with the peer transport.  Errors: STATE,
 * INVALID, UNSUPPORTED (D), OOM. */
int dmha_reserve(int world_size, int64_t L, int D, int H);

/* SURVEY §8(c) "Accounting" and §8(d): synchronises outstanding profiled
 * work, then copies the counters into *s (caller-owned).  INVALID if null. */
int dmha_get_stats(struct dmha_stats *s);

/* SURVEY §8(d) measurement hook.
 * enable != 0: bracket every library kernel launch and ring exchange with CUDA
 * events on its own stream and accumulate their durations into dmha_stats
 * (measurement hook used by bench.py); enable == 0 stops it.  Also resets the
 * timed counters. */
int dmha_set_profiling(int enable);

/* ---- individual hot-path steps (exported for tests and the bench) ------- */

/* a1/a3 (north_star (3)): what rank `rank` does at ring step `step`
 * (0 <= step < world_size).  Pure host function of its arguments; dmha_forward
 * and dmha_forward_emulated follow exactly this plan. */
enum dmha_plan_output {
  DMHA_PLAN_FINAL = 0,          /* P == 1: attention writes out/lse directly       */
  DMHA_PLAN_ACC = 1,            /* step 0: attention writes the fp32 accumulator   */
  DMHA_PLAN_COMBINE = 2,        /* partial, then LSE-combine into the accumulator  */
  DMHA_PLAN_COMBINE_FINAL = 3   /* last step: combine writes out (bf16/fp32) + lse */
};
struct dmha_ring_plan {
  int src;                   /* rank whose K/V block is attended to at this step      */
  int send_to;               /* rank the current K/V block is sent to (-1: none)       */
  int recv_from;             /* rank the next block is received from (-1: none)        */
  int compute_buf;           /* K/V used: -1 = caller's k/v, else ring buffer 0/1      */
  int recv_buf;              /* ring buffer the next block lands in (-1: none)         */
  int recv_after_compute_of; /* the receive waits for this step's compute (-1: none)   */
  int output;                /* enum dmha_plan_output                                  */
  int64_t q_base0, q_base1, q_chunk; /* global position map of this rank's rows   */
  int64_t k_base0, k_base1, k_chunk; /* ... and of the src rank's K/V rows         */
};
int dmha_ring_plan_step(int world_size, int rank, int step, int layout, int64_t L,
                        struct dmha_ring_plan *plan_out);


/* a1: global sequence position of local row i of rank r for
 * (L, P, layout).  Pure host index math. Returns INVALID on bad arguments. */
int dmha_local_to_global(int64_t L, int world_size, int rank, int layout, int64_t i,
                         int64_t *global_out);

/* a1 ("equal as possible"): the number of rows rank r
 * owns — CONTIGUOUS: L/P, plus one for the first L % P ranks (L need not be
 * divisible by P; rank r starts at r*(L/P) + min(r, L % P)); ZIGZAG: L/P
 * (L % 2P == 0 required).  Host index math; INVALID on bad arguments. */
int dmha_shard_rows(int64_t L, int world_size, int rank, int layout, int64_t *rows_out);

/* a2 (P:193-211 + P:672-674): one local flash-attention pass of this rank's
 * query block against one K/V block, on the dmha_init stream.
 *  q: [Lq, H, D], k/v: [Lk, H, D] device (dtype of dmha_init).
 *  Global positions: query row i sits at qpos(i) = i < q_chunk ? q_base0 + i
 *  : q_base1 + (i - q_chunk); likewise for key rows with k_*.  Both maps must
 *  be increasing.  With causal, key j is used by row i iff kpos(j) <= qpos(i).
 *  out_mode 0: out is [Lq, H, D] of the init dtype holding O/l;
 *  out_mode 1: out is fp32 [Lq, H, D] holding O/l (a ring partial).
 *  lse: [H, Lq] fp32; rows with no usable key get lse = -inf and out = 0. */
int dmha_attention_local(const void *q, const void *k, const void *v, void *out, float *lse,
                         int64_t Lq, int64_t Lk, int D, int H, int causal, int64_t q_base0,
                         int64_t q_base1, int64_t q_chunk, int64_t k_base0, int64_t k_base1,
                         int64_t k_chunk, int out_mode);

/* a4/a5 (north_star (3); "softmax requires all ..."): merge a partial
 * (o_part fp32 [Lq,H,D], lse_part [H,Lq]) into the accumulator (o_acc fp32,
 * lse_acc) with the stable log-sum-exp rule
 *   lse = max + ln(e^{lse_acc-max} + e^{lse_part-max}),
 *   o   = o_acc e^{lse_acc-lse} + o_part e^{lse_part-lse},
 * -inf partials weigh 0 (both -inf keeps -inf and o = 0).
 * final == 0: result written back into o_acc/lse_acc.
 * final == 1: result written to out (init dtype, [Lq,H,D]) and lse_out. */
int dmha_lse_combine(float *o_acc, float *lse_acc, const float *o_part, const float *lse_part,
                     void *out, float *lse_out, int64_t Lq, int D, int H, int final_step);

/* ---- NEXT-4: the token Selector (§10.2) ------------------------ */

/* Scorers for s_{psi,tau} — the paper never defines one (R18). */
enum { DMHA_SCORER_L2 = 0, DMHA_SCORER_PROJ = 1 };

/* s_{psi,tau}: X_{L x D} -> X'_{L' x D}, PAPER.md Eq. `selector` P:630-634:
 * "filtering tokens before computing attention", tau the pruning
 * threshold.  On this rank's rows x (DEVICE [n_rows, width] bf16, row-major,
 * 16-byte aligned, width % 8 == 0):
 *   score_t = ||x_t||_2 (DMHA_SCORER_L2, psi = NULL) or |x_t . psi|
 *   (DMHA_SCORER_PROJ, psi = DEVICE [width] bf16), accumulated in fp64;
 *   keep x_t iff score_t >= tau, in original order.
 * Never empty (R19): if no row on ANY rank passes, the highest-scoring row
 * over all ranks (ties: smallest global position under the init layout, with
 * L = n_rows * world_size) is kept by its owner.  Collective when
 * world_size > 1 (all ranks call with the same n_rows, width, scorer, tau;
 * n_rows even for the zigzag layout, else DMHA_ERR_INVALID).
 * Outputs: x_out DEVICE [n_rows, width] bf16 capacity — the first *n_kept
 * rows are the kept rows; idx_out DEVICE [n_rows] int64 — the first *n_kept
 * entries are their LOCAL row indices, increasing (the re-aggregation map,
 * P:622); scores DEVICE [n_rows] fp64 or NULL; *n_kept HOST.  Synchronises
 * the stream (n_kept is returned to the host).  bf16 dtype only.
 * Errors: INVALID (null, sizes, alignment, scorer/psi mismatch, NaN tau),
 * UNSUPPORTED (fp32 init dtype), STATE, OOM, CUDA, NCCL. */
int dmha_select(const void *x, int64_t n_rows, int width, int scorer, const void *psi,
                double tau, void *x_out, int64_t *idx_out, double *scores, int64_t *n_kept);

/* Re-aggregation ("reordered and aggregated"): y_full[idx[i], :] =
 * y_sel[i, :] for i < n_kept (DEVICE bf16 rows of `width`, 16-byte aligned;
 * idx DEVICE int64 as returned by dmha_select); other rows untouched.
 * Local (no collective).  Errors: INVALID, UNSUPPORTED (fp32), STATE, CUDA. */
int dmha_scatter_rows(const void *y_sel, const int64_t *idx, int64_t n_kept, int width,
                      void *y_full);

/* Measurement hook: dev_buf (device, >= DMHA_TRACE_WORDS uint64, or NULL to
 * disable) receives, in a library built with -DDMHA_TRACE=1 (tools/trace.py
 * builds one; the product build compiles the stamps out and leaves the
 * buffer untouched), clock64 timeline stamps of the bf16 attention kernel
 * (first 4 CTAs of head 0, first 64 KV tiles; events documented in
 * attn_fwd_sm100.cu) and, from word 4096 and only in a library built with
 * -DDMHA_CTA_STAMPS=1, %globaltimer (ns) at the start and end of each of the
 * first 16384 CTAs (linear id x + y*gridDim.x + ...). */
#define DMHA_TRACE_WORDS (4096 + 2 * 16384)
int dmha_debug_set_trace(void *dev_buf);

/* Block until all library work on the current stream is done (test helper). */
int dmha_synchronize(void);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* DMHA_H_ */
