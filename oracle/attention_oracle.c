/*
 * attention_oracle.c — CPU fp64 ORACLE for the distributed multi-head
 * attention forward of arXiv 2302.06218.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this code.  The
 * product path (paper_2302_06218_b200/) never links or calls it, and this
 * file shares no code, header or constant with paper_2302_06218_b200/csrc/.
 *
 * What it computes (plain definition, no blocking, no fusion):
 *   PAPER.md:193-196  Eq. `unnormalized`  A'_t = Q_t K^T
 *   PAPER.md:198-201  row softmax         A_{t,i} = exp A'_{t,i} / sum_j exp A'_{t,j}
 *   PAPER.md:203-211  Eq. `attn-sum`      Z_t = sum_j A_{t,j} V_j
 *     (reading R2: the garbled "V_i" in Eq. attn-sum is read as V_j)
 *   north_star (BASELINE.json): scores scaled by 1/sqrt(D), D = per-head dim
 *     (reading R1), optional causal mask on GLOBAL positions, j <= t.
 *   lse_t = ln sum_{j allowed} exp(A'_{t,j} / sqrt(D))   (reading R9: natural log)
 *   A row with no allowed key (possible only for a key sub-range) gives
 *   lse = -inf and Z = 0 (reading R10).
 *
 * Softmax is evaluated as exp(x - m) / sum exp(x - m) with m the row max:
 * the identical quantity (multiply numerator and denominator by e^{-m}),
 * written this way only so that fp64 exp does not overflow on the stress
 * inputs (|x| ~ 1e3).  Sums are plain left-to-right in key order.
 *
 * Layout: q, k, v are [L, H, D] row-major fp64 in GLOBAL sequence order.
 * Outputs: out [n_rows, H, D], lse [H, n_rows] for the requested query rows.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* The oracle body is written once (attention_oracle_body.h) and compiled for
 * two INPUT element types; all arithmetic is fp64 in both:
 *   oracle_attention_f64   — fp64 inputs
 *   oracle_attention_f32in — fp32 inputs (the bf16 test inputs are exact in
 *     fp32), converted element by element to fp64 on load, so large configs
 *     (C4/C5, GiB-sized K/V) need no fp64 copy.  Same results bit for bit. */
#define ORACLE_T double
#define ORACLE_NAME oracle_attention_f64
#include "attention_oracle_body.h"
#undef ORACLE_T
#undef ORACLE_NAME
#define ORACLE_T float
#define ORACLE_NAME oracle_attention_f32in
#include "attention_oracle_body.h"
#undef ORACLE_T
#undef ORACLE_NAME

/* Number of OpenMP threads the oracle will use (for the cpu_baseline report). */
int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
