/*
 * attention_oracle_body.h — the oracle loop of attention_oracle.c, included
 * twice with ORACLE_T = double / float (input element type only; every
 * product, sum, exp and log below is fp64).  TEST INFRASTRUCTURE ONLY (see
 * attention_oracle.c for the definition followed and its citations).
 */
/* Returns 0 on success, -1 on bad arguments.
 * rows:   n_rows global query indices (NULL => rows 0..L-1, n_rows must be L)
 * key_begin/key_end: only keys j in [key_begin, key_end) are used
 *                    (the full problem is key_begin=0, key_end=L). */
int ORACLE_NAME(const ORACLE_T *q, const ORACLE_T *k, const ORACLE_T *v,
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
      const ORACLE_T *qt = q + (t * H + h) * (int64_t)D;
      double *zt = out + (r * H + h) * (int64_t)D;
      int64_t j_end = key_end;
      if (causal && j_end > t + 1) j_end = t + 1; /* keep j <= t */
      /* scores x_j = (Q_t . K_j) / sqrt(D)  (Eq. unnormalized + scale) */
      double m = -INFINITY;
      for (int64_t j = key_begin; j < j_end; ++j) {
        const ORACLE_T *kj = k + (j * H + h) * (int64_t)D;
        double s = 0.0;
        for (int d = 0; d < D; ++d) s += (double)qt[d] * (double)kj[d];
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
        const ORACLE_T *vj = v + (j * H + h) * (int64_t)D;
        for (int d = 0; d < D; ++d) zt[d] += a * (double)vj[d];
      }
      lse[(int64_t)h * n_rows + r] = m + log(l);
    }
    free(x);
  }
  return 0;
}

