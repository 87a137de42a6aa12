/*
 * CPU restatement of the reference algorithms for the SpTRSV hot path.
 *
 * TEST INFRASTRUCTURE ONLY: this is the checker for the CUDA path (tests/,
 * __graft_entry__.smoke(), bench.py's cpu_baseline leg and `--impl
 * reference`). The product (paper_2012_06959_b200) never links or calls it.
 *
 * Reference: /root/reference/pkg/src/sptrsv (pure Python + numpy; nothing to
 * compile, so there is no oracle/_ref build — see DESIGN.md). Each function
 * cites the lines it restates. Build with -ffp-contract=off: Python float
 * arithmetic is IEEE binary64 with no fused multiply-add, and so is this.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* solve_serial, reference.py:20-35 (Alg. 1 of PAPER.md:92-108): columns in
 * ascending order; x_i = (b_i - left_sum_i) / diag_i; then every off-diagonal
 * (rid, v) of column i, in storage order, does left_sum[rid] += v * x_i.
 * Requires a validated lower-triangular CSC (diagonal first in each column,
 * matrix.py:216-234). Returns 0, or -1 on allocation failure. */
int oracle_solve_serial(int64_t n, const int64_t* col_ptr, const int64_t* row_idx, const double* values,
                        const double* b, double* x) {
  double* left = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  if (!left) return -1;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t lo = col_ptr[i], hi = col_ptr[i + 1];
    const double xi = (b[i] - left[i]) / values[lo];
    x[i] = xi;
    for (int64_t k = lo + 1; k < hi; ++k) {
      const double prod = values[k] * xi;
      left[row_idx[k]] = left[row_idx[k]] + prod;
    }
  }
  free(left);
  return 0;
}

/* compute_in_degrees, analysis.py:19-27: stored entries with row != col,
 * counted per row (any square CSC). */
void oracle_in_degrees(int64_t n, const int64_t* col_ptr, const int64_t* row_idx, int64_t* out) {
  memset(out, 0, sizeof(int64_t) * (size_t)n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t k = col_ptr[j]; k < col_ptr[j + 1]; ++k)
      if (row_idx[k] != j) out[row_idx[k]] += 1;
}

/* compute_level_schedule, analysis.py:43-64: one ascending sweep pushing
 * level[j] + 1 into every off-diagonal row of column j. Returns n_levels. */
int64_t oracle_levels(int64_t n, const int64_t* col_ptr, const int64_t* row_idx, int64_t* level) {
  memset(level, 0, sizeof(int64_t) * (size_t)n);
  int64_t top = -1;
  for (int64_t j = 0; j < n; ++j) {
    const int64_t bumped = level[j] + 1;
    for (int64_t k = col_ptr[j]; k < col_ptr[j + 1]; ++k) {
      const int64_t r = row_idx[k];
      if (r != j && level[r] < bumped) level[r] = bumped;
    }
    if (level[j] > top) top = level[j];
  }
  return n ? top + 1 : 0;
}

/* spmv_lower, matrix.py:203-213: L @ x accumulated in storage order. */
void oracle_spmv(int64_t n, const int64_t* col_ptr, const int64_t* row_idx, const double* values,
                 const double* x, double* y) {
  memset(y, 0, sizeof(double) * (size_t)n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t k = col_ptr[j]; k < col_ptr[j + 1]; ++k) y[row_idx[k]] = y[row_idx[k]] + values[k] * x[j];
}

/* The device kernels divide with Markstein's correction (csrc/common.cuh
 * div_exact): q = RN(a*rd), r = fma(-q, d, a), RN(fma(r, rd, q)) with
 * rd = RN(1/d), falling back to IEEE a/d outside a safe exponent window.
 * Restated here so the CPU suite can check the claim "bit-identical to IEEE
 * division" on random operands. Returns the number of mismatches. */
static int exp_bits(double v) {
  uint64_t b;
  memcpy(&b, &v, 8);
  return (int)((b >> 52) & 0x7FF);
}
#include <math.h>
int64_t oracle_markstein_mismatches(int64_t count, uint64_t seed) {
  uint64_t s = seed ? seed : 88172645463325252ull;
  int64_t bad = 0;
  for (int64_t i = 0; i < count; ++i) {
    uint64_t ba, bd;
    s ^= s << 13; s ^= s >> 7; s ^= s << 17; ba = s;
    s ^= s << 13; s ^= s >> 7; s ^= s << 17; bd = s;
    double a, d;
    memcpy(&a, &ba, 8);
    memcpy(&d, &bd, 8);
    if (i & 1) a = ldexp((double)(ba >> 11) / 9007199254740992.0 + 0.5, (int)(bd % 200) - 100);
    const double rd = 1.0 / d;
    const double q = a * rd;
    double got;
    int eq = exp_bits(q), ea = exp_bits(a), ed = exp_bits(d);
    if (eq > 100 && eq < 1946 && ea > 100 && ea < 1946 && ed > 100 && ed < 1946) {
      const double r = fma(-q, d, a);
      got = fma(r, rd, q);
    } else {
      got = a / d;
    }
    const double want = a / d;
    if (memcmp(&got, &want, 8) != 0 && !(isnan(got) && isnan(want))) ++bad;
  }
  return bad;
}
