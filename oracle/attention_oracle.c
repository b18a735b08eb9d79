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

/* Returns 0 on success, -1 on bad arguments.
 * rows:   n_rows global query indices (NULL => rows 0..L-1, n_rows must be L)
 * key_begin/key_end: only keys j in [key_begin, key_end) are used
 *                    (the full problem is key_begin=0, key_end=L). */
int oracle_attention_f64(const double *q, const double *k, const double *v,
                         int64_t L, int D, int H, int causal,
                         const int64_t *rows, int64_t n_rows,
                         int64_t key_begin, int64_t key_end,
                         double *out, double *lse) {
  if (!q || !k || !v || !out || !lse || L < 1 || D < 1 || H < 1 || n_rows < 0)
    return -1;
  if (key_begin < 0 || key_end > L || key_begin > key_end) return -1;
  if (!rows && n_rows != L) return -1;
  const double scale = 1.0 / sqrt((double)D);
  const int64_t n_items = n_rows * (int64_t)H;

#pragma omp parallel
  {
    double *x = (double *)malloc(sizeof(double) * (size_t)(key_end - key_begin + 1));
#pragma omp for schedule(dynamic, 4)
    for (int64_t item = 0; item < n_items; ++item) {
      const int64_t r = item / H;
      const int h = (int)(item % H);
      const int64_t t = rows ? rows[r] : r; /* global query position */
      const double *qt = q + (t * H + h) * (int64_t)D;
      double *zt = out + (r * H + h) * (int64_t)D;
      int64_t j_end = key_end;
      if (causal && j_end > t + 1) j_end = t + 1; /* keep j <= t */
      /* scores x_j = (Q_t . K_j) / sqrt(D)  (Eq. unnormalized + scale) */
      double m = -INFINITY;
      for (int64_t j = key_begin; j < j_end; ++j) {
        const double *kj = k + (j * H + h) * (int64_t)D;
        double s = 0.0;
        for (int d = 0; d < D; ++d) s += qt[d] * kj[d];
        s *= scale;
        x[j - key_begin] = s;
        if (s > m) m = s;
      }
      for (int d = 0; d < D; ++d) zt[d] = 0.0;
      if (j_end <= key_begin) { /* empty key set */
        lse[(int64_t)h * n_rows + r] = -INFINITY;
        continue;
      }
      /* softmax denominator  sum_j exp(x_j - m) */
      double l = 0.0;
      for (int64_t j = key_begin; j < j_end; ++j) l += exp(x[j - key_begin] - m);
      /* Z_t = sum_j A_{t,j} V_j */
      for (int64_t j = key_begin; j < j_end; ++j) {
        const double a = exp(x[j - key_begin] - m) / l;
        const double *vj = v + (j * H + h) * (int64_t)D;
        for (int d = 0; d < D; ++d) zt[d] += a * vj[d];
      }
      lse[(int64_t)h * n_rows + r] = m + log(l);
    }
    free(x);
  }
  return 0;
}

/* Number of OpenMP threads the oracle will use (for the cpu_baseline report). */
int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
