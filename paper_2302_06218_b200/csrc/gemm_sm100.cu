// gemm_sm100.cu — the projection GEMMs of the full distributed MHA layer
// (SURVEY §8(f) NEXT-3): Q = X W_Q, K = X W_K, V = X W_V (PAPER.md:186-191,
// replicated weights applied to this rank's rows for all heads) and
// Y = concat_h(Z) W_0.  Row-major bf16 C[M,N] = A[M,K] B[K,N], fp32
// accumulation in TMEM, bf16 (round-to-nearest-even) output (reading R17).
//
// Persistent tcgen05 kernel, one CTA per SM, 6 warps:
//   warp 0      TMA producer: A tile 128 x 64 (K-major, one 128-byte-swizzled
//               panel) + B tile 64 x 256 (N contiguous = MN-major B operand,
//               four 64-column panels) per stage, kStages-deep ring
//   warp 1      TMEM allocator (512 columns = two 128 x 256 fp32
//               accumulators) + single-thread MMA issuer (128x256x16 SS MMAs)
//   warps 2-5   epilogue: TMEM -> registers -> bf16 -> global, one row per
//               thread (warp w reads TMEM lanes 32*(w%4)..), overlapped with
//               the next tile's main loop through the second accumulator
// Tiles are visited n-fastest (the N/256 tiles of one 128-row block of A run
// side by side, so A is read from HBM about once; B — the weights — stays in
// L2).  TMA zero-fills out-of-range rows/columns, so any M, N, K with 16-byte
// aligned row strides (N % 8 == 0, K % 8 == 0) works; the epilogue stores
// only in-range elements.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "ptx_sm100.cuh"
#include "tma_map.h"

namespace dmha {
namespace {

constexpr int kBM = 128, kBN = 256, kBK = 64;
constexpr int kStages = 4;
constexpr int kABytes = kBM * kBK * 2;              // 16 KB
constexpr int kBPanel = kBK * 64 * 2;               // 8 KB: 64 K-rows x 64 N-columns
constexpr int kBBytes = (kBN / 64) * kBPanel;       // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;      // 48 KB
constexpr int kThreads = 6 * 32;
constexpr int kSmem = kStages * kStageBytes + 256 + 1024;
static_assert(kSmem <= 232448, "shared memory budget");
constexpr uint32_t kIdesc = ptx::make_idesc(1, kBM, kBN, 0, 1);  // A K-major, B MN-major

struct GemmParams {
  __nv_bfloat16* c;
  int64_t M;
  int N, K;
  int m_tiles, n_tiles, k_blocks;
};

__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_sm100_kernel(const __grid_constant__ CUtensorMap tm_a,
                           const __grid_constant__ CUtensorMap tm_b, const GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* full = bars;                    // [kStages]
  uint64_t* empty = full + kStages;         // [kStages]
  uint64_t* acc_full = empty + kStages;     // [2]
  uint64_t* acc_empty = acc_full + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t n_tiles_total = static_cast<int64_t>(p.m_tiles) * p.n_tiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&acc_full[b], 1);
      ptx::mbar_init(&acc_empty[b], 4 * 32);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_a);
    ptx::tma_prefetch_desc(&tm_b);
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < n_tiles_total; t += gridDim.x) {
        const int m0 = static_cast<int>(t / p.n_tiles) * kBM;
        const int n0 = static_cast<int>(t % p.n_tiles) * kBN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&full[stage], kStageBytes);
          uint8_t* sa = smem + stage * kStageBytes;
          uint8_t* sb = sa + kABytes;
          ptx::tma_load_3d(&tm_a, &full[stage], sa, kb * kBK, m0, 0);
          for (int pn = 0; pn < kBN / 64; ++pn)
            ptx::tma_load_3d(&tm_b, &full[stage], sb + pn * kBPanel, n0 + pn * 64, kb * kBK, 0);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int64_t t = blockIdx.x; t < n_tiles_total; t += gridDim.x, ++it) {
        const int buf = it & 1;
        ptx::mbar_wait(&acc_empty[buf], static_cast<uint32_t>(((it >> 1) & 1) ^ 1));
        ptx::tc_fence_after();
        const uint32_t dacc = tmem + buf * kBN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + stage * kStageBytes);
          const uint32_t sb = sa + kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            // A: K-major 128B-swizzled panel, 16-element K step = 32 bytes;
            // B: MN-major panels of 64 N-columns (LBO = panel stride), K step
            // = 16 rows of 128 bytes
            ptx::mma_bf16_ss(dacc, ptx::smem_desc_sw128(sa + kk * 32, 16, 1024),
                             ptx::smem_desc_sw128(sb + kk * 16 * 128, kBPanel, 1024), kIdesc,
                             (kb > 0 || kk > 0) ? 1u : 0u);
          }
          ptx::mma_commit(&empty[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        ptx::mma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------- epilogue
    const int quarter = warp & 3;  // TMEM lanes 32*quarter .. (warp w may only access these)
    const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
    int it = 0;
    for (int64_t t = blockIdx.x; t < n_tiles_total; t += gridDim.x, ++it) {
      const int buf = it & 1;
      const int64_t row = static_cast<int64_t>(t / p.n_tiles) * kBM + quarter * 32 + lane;
      const int n0 = static_cast<int>(t % p.n_tiles) * kBN;
      ptx::mbar_wait(&acc_full[buf], static_cast<uint32_t>((it >> 1) & 1));
      ptx::tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < kBN / 32; ++c) {
        float v[32];
        ptx::tmem_ld32(tmem + lane_addr + buf * kBN + c * 32, v);
        ptx::tmem_wait_ld();
        const int col0 = n0 + c * 32;
        if (row < p.M && col0 < p.N) {
          __nv_bfloat16* dst = p.c + row * p.N + col0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (col0 + 8 * e + 8 <= p.N) {
              uint32_t w[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                __nv_bfloat162 b = __floats2bfloat162_rn(v[8 * e + 2 * u], v[8 * e + 2 * u + 1]);
                w[u] = *reinterpret_cast<uint32_t*>(&b);
              }
              *reinterpret_cast<uint4*>(dst + 8 * e) = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&acc_empty[buf]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// Row-major bf16 [rows, cols] as the 3-D tensor (cols, rows, 1) with boxes of
// 64 columns x box_rows rows, 128-byte swizzle.
bool make_map_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows) {
  EncodeTiledFn enc = tma_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows), 1};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols) * 2, static_cast<cuuint64_t>(cols * rows) * 2};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

cudaError_t launch_gemm_bf16(const void* a, const void* b, void* c, int64_t M, int N, int K,
                             cudaStream_t stream) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (K <= 0 || N % 8 != 0 || K % 8 != 0 || M > INT32_MAX) return cudaErrorInvalidValue;
  CUtensorMap ta, tb;
  if (!make_map_2d(&ta, a, M, K, kBM) || !make_map_2d(&tb, b, K, N, kBK))
    return cudaErrorInvalidValue;
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_sm100_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  GemmParams p;
  p.c = static_cast<__nv_bfloat16*>(c);
  p.M = M;
  p.N = N;
  p.K = K;
  p.m_tiles = static_cast<int>((M + kBM - 1) / kBM);
  p.n_tiles = (N + kBN - 1) / kBN;
  p.k_blocks = (K + kBK - 1) / kBK;
  const int64_t tiles = static_cast<int64_t>(p.m_tiles) * p.n_tiles;
  const int grid = static_cast<int>(tiles < sms ? tiles : sms);
  gemm_bf16_sm100_kernel<<<grid, kThreads, kSmem, stream>>>(ta, tb, p);
  return cudaGetLastError();
}

}  // namespace dmha
