// kernels.h — internal launch interface between the C ABI (dmha_api.cu) and
// the device kernels.  Not part of the public ABI (see include/dmha.h).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace dmha {

// Global position of local row i:  i < chunk ? base0 + i : base1 + (i - chunk).
// Both pieces are increasing and base1 >= base0 + chunk.
struct PosMap {
  int64_t base0;
  int64_t base1;
  int64_t chunk;
};

// OUT_COMBINE_*: NEXT-2 fused combine — the epilogue merges its partial into
// (acc_o, acc_lse) itself (combine_math.cuh) and writes either the updated
// accumulator (ACC, in place) or the final output (FINAL: out/lse in the init
// dtype), so no fp32 partial goes through HBM.
enum OutMode { OUT_FINAL = 0, OUT_PARTIAL_F32 = 1, OUT_COMBINE_ACC = 2, OUT_COMBINE_FINAL = 3 };

struct LocalAttnArgs {
  const void* q;
  const void* k;
  const void* v;
  void* out;   // OUT_FINAL: init dtype; OUT_PARTIAL_F32: fp32
  float* lse;  // [H, Lq]
  int64_t Lq, Lk;
  int D, H;
  int causal;
  PosMap qmap, kmap;
  int out_mode;
  float* acc_o = nullptr;    // OUT_COMBINE_*: running O_acc [Lq, H, D] fp32
  float* acc_lse = nullptr;  // OUT_COMBINE_*: running lse_acc [H, Lq]
  // Split-KV (ping-pong kernel, OUT_PARTIAL_F32 only): kv_split = 2 launches
  // a second grid plane whose CTAs take the second half of each row block's
  // key tiles and write their partial to out2 / lse2.
  int kv_split = 1;
  void* out2 = nullptr;
  float* lse2 = nullptr;
  // Fault injection only (DMHA_FAULT=perturb_lse, dmha.h): added to the
  // partial's lse inside the log-sum-exp combine; 0 in normal operation.
  float lse_bias = 0.f;
  // fp32 path (3xTF32): caller-owned device scratch for the split K / V^T
  // operands, at least tf32_scratch_bytes(Lk, H, D) bytes.
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
};

// bf16 tcgen05/TMEM/TMA flash-attention forward (attn_fwd_sm100.cu): two
// query tiles per CTA, ping-pong on the tensor core.
cudaError_t launch_attn_fwd_bf16(const LocalAttnArgs& a, cudaStream_t stream);
// Whether launch_attn_fwd_bf16 accepts OUT_COMBINE_* for head dim D (the
// ping-pong kernel with the one-thread-per-row epilogue does).
bool attn_fused_combine_supported(int D);
// Whether launch_attn_fwd_bf16 accepts kv_split = 2 for head dim D.
bool attn_kv_split_supported(int D);
// fp32 path: the 3xTF32 tcgen05 kernel (attn_fwd_tf32.cu), or with
// DMHA_FP32_SIMT=1 the SIMT fp32 kernel (attn_fwd_fp32.cu).
cudaError_t launch_attn_fwd_fp32(const LocalAttnArgs& a, cudaStream_t stream);
cudaError_t launch_attn_fwd_tf32x3(const LocalAttnArgs& a, cudaStream_t stream);
// Scratch the 3xTF32 path needs for Lk keys: K hi / lo [Lk, H, D] and V^T
// hi / lo [H, D, Lk rounded up to 4], fp32 (0 for Lk = 0).
size_t tf32_scratch_bytes(int64_t Lk, int H, int D);
// Kernel launches one fp32-path local attention call makes (the 3xTF32 path:
// split + attention; the SIMT cross-check: one).
int fp32_launches_per_call(int64_t Lq, int64_t Lk);
// log-sum-exp combine (lse_combine.cu).  out_dtype_bf16 selects the final
// output element type when final_step != 0.
cudaError_t launch_lse_combine(float* o_acc, float* lse_acc, const float* o_part,
                               const float* lse_part, void* out, float* lse_out, int64_t Lq,
                               int D, int H, int final_step, int out_dtype_bf16,
                               cudaStream_t stream, float lse_bias = 0.f);

// NEXT-3 projection GEMM (gemm_sm100.cu): row-major bf16 C[M,N] = A[M,K] B[K,N],
// fp32 accumulation; N % 8 == 0, K % 8 == 0.
cudaError_t launch_gemm_bf16(const void* a, const void* b, void* c, int64_t M, int N, int K,
                             cudaStream_t stream);

// Head-parallel exchange (the paper's all-to-all).
struct HeadparGeom {
  int P;         // world size
  int H, D;      // heads (H % P == 0), per-head dim
  int64_t Lloc;  // rows per rank
  int zigzag;    // layout of the sequence shards
};
cudaError_t launch_headpar_pack_qkv(const void* q, const void* k, const void* v, void* send,
                                    const HeadparGeom& g, int elem_bytes, cudaStream_t st);
cudaError_t launch_headpar_unpack_qkv(const void* recv, void* xq, void* xk, void* xv,
                                      const HeadparGeom& g, int elem_bytes, cudaStream_t st);
cudaError_t launch_headpar_pack_out(const void* outg, void* send, const float* lseg,
                                    float* send_lse, const HeadparGeom& g, int elem_bytes,
                                    cudaStream_t st);
cudaError_t launch_headpar_unpack_out(const void* recv, void* out, const HeadparGeom& g,
                                      int elem_bytes, cudaStream_t st);

// Token Selector (selector.cu): 256-row tiles.
int64_t selector_tiles(int64_t n);
cudaError_t launch_selector_score(const void* x, const void* psi, int64_t n, int w, int scorer,
                                  double tau, double* scores, uint8_t* flags, int* tile_counts,
                                  cudaStream_t st);
cudaError_t launch_selector_scan(const int* tile_counts, int64_t n, int64_t* offsets,
                                 int64_t* total, cudaStream_t st);
cudaError_t launch_selector_compact(const void* x, int64_t n, int w, const uint8_t* flags,
                                    const int64_t* offsets, void* x_out, int64_t* idx_out,
                                    cudaStream_t st);
cudaError_t launch_selector_argmax(const double* scores, int64_t n, double* best,
                                   int64_t* best_row, cudaStream_t st);
cudaError_t launch_scatter_rows(const void* y_sel, const int64_t* idx, int64_t k, int w,
                                void* y_full, cudaStream_t st);

// Debug timeline buffer for the bf16 attention kernel (null = off).
extern unsigned long long* g_trace;

// Number of kernel launches a call of launch_attn_fwd_* makes (for stats).
inline int attn_launches_per_call() { return 1; }

}  // namespace dmha
