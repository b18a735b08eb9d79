// combine_math.cuh — the log-sum-exp merge of one ring-step partial into the
// running accumulator (north_star (3)), shared by the
// stand-alone combine kernel (lse_combine.cu) and the attention epilogue's
// fused combine (attn_fwd_sm100.cu, NEXT-2), so both produce the same bits:
//   lse = M + ln(e^{lse_a - M} + e^{lse_s - M}),   M = max(lse_a, lse_s)
//   O   = O_a e^{lse_a - lse} + O_s e^{lse_s - lse}
// A -inf lse (no usable key) weighs 0; two -inf stay -inf with O = 0
// (reading R10).  Products and the sum use explicit _rn intrinsics
// so the compiler cannot contract them differently in the two kernels.
#pragma once
#include <cuda_runtime.h>

namespace dmha {

__device__ __forceinline__ void merge_weights(float la, float lp, float& wa, float& wp,
                                              float& lnew) {
  const float M = fmaxf(la, lp);
  if (M == -INFINITY) {  // both empty
    wa = 0.f;
    wp = 0.f;
    lnew = -INFINITY;
    return;
  }
  const float ea = __expf(la - M);  // exp(-inf) = 0
  const float ep = __expf(lp - M);
  const float s = ea + ep;
  lnew = M + __logf(s);
  const float inv = 1.f / s;
  wa = ea * inv;
  wp = ep * inv;
}

// One output element: O_a * wa + O_s * wp (a zero weight contributes exactly 0,
// also when the other operand is not finite-safe garbage-free).
__device__ __forceinline__ float combine_one(float a, float s, float wa, float wp) {
  return __fadd_rn(wa == 0.f ? 0.f : __fmul_rn(a, wa), wp == 0.f ? 0.f : __fmul_rn(s, wp));
}

}  // namespace dmha
