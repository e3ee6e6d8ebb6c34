/*
 * vq_oracle.c -- CPU restatement of the reference's compiled kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port" arm) for the B200 path; nothing in the product package
 * (paper_0910_4711_b200/) links, loads or calls it.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may use it.
 *
 * It restates, function for function, the five numba kernels of the
 * reference (arxiv/paper_0910_4711, pkg/src/vqkit/_kernels.py):
 *
 *   vqo_assign_range   <- _kernels.assign_range   (_kernels.py:18-36)
 *   vqo_update_rows    <- _kernels.update_rows    (_kernels.py:39-66)
 *   vqo_pair_distance  <- _kernels.pair_distance  (_kernels.py:69-78)
 *   vqo_column_sums    <- _kernels.column_sums    (_kernels.py:81-89)
 *   vqo_sum_inorder    <- _kernels.sum_inorder    (_kernels.py:92-98)
 *
 * Arithmetic contract: IEEE binary64, every operation
 * rounded separately (no FMA contraction: build with -ffp-contract=off and
 * without -ffast-math), ascending dimension, ascending training index,
 * strict '<' so the lowest codevector index wins ties, sqrt only on the
 * stored per-row distance under the euclidean metric.
 *
 * The OpenMP entry points (vqo_assign_parallel / vqo_update_parallel) are the
 * paper's shared-memory master/slave scheme (section 4, the
 * reference's parallel.py:135-154): contiguous row chunks for allocation,
 * round-robin codevector ownership for updation.  Both are bit-identical to
 * the sequential kernels by construction, exactly as in the reference.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define VQO_SQUARED_EUCLIDEAN 0 /* _kernels.py:14 */
#define VQO_EUCLIDEAN 1         /* _kernels.py:15 */

/* _kernels.py:18-36 */
void vqo_assign_range(const double *vectors, int64_t dim, const double *codebook,
                      int64_t size, int64_t start, int64_t stop, int metric,
                      int64_t *out_cells, double *out_dists) {
  for (int64_t z = start; z < stop; ++z) {
    const double *x = vectors + z * dim;
    int64_t best = 0;
    double best_d = INFINITY;
    for (int64_t i = 0; i < size; ++i) {
      const double *c = codebook + i * dim;
      double d = 0.0;
      for (int64_t l = 0; l < dim; ++l) {
        double diff = x[l] - c[l];
        d += diff * diff;
      }
      if (d < best_d) {
        best_d = d;
        best = i;
      }
    }
    if (metric == VQO_EUCLIDEAN) best_d = sqrt(best_d);
    out_cells[z] = best;
    out_dists[z] = best_d;
  }
}

/* _kernels.py:39-66 */
void vqo_update_rows(const double *vectors, int64_t m, int64_t dim, const int64_t *cells,
                     const double *old_codebook, int64_t size, int64_t worker,
                     int64_t stride, double *out_codebook, int64_t *out_counts) {
  for (int64_t i = worker; i < size; i += stride) {
    out_counts[i] = 0;
    for (int64_t l = 0; l < dim; ++l) out_codebook[i * dim + l] = 0.0;
  }
  for (int64_t j = 0; j < m; ++j) {
    int64_t idx = cells[j];
    /* python '%' on non-negative operands */
    if (idx % stride == worker) {
      out_counts[idx] += 1;
      for (int64_t l = 0; l < dim; ++l) out_codebook[idx * dim + l] += vectors[j * dim + l];
    }
  }
  for (int64_t i = worker; i < size; i += stride) {
    int64_t n = out_counts[i];
    if (n > 0) {
      double dn = (double)n;
      for (int64_t l = 0; l < dim; ++l) out_codebook[i * dim + l] /= dn;
    } else {
      for (int64_t l = 0; l < dim; ++l) out_codebook[i * dim + l] = old_codebook[i * dim + l];
    }
  }
}

/* _kernels.py:69-78 */
double vqo_pair_distance(const double *a, const double *b, int64_t dim, int metric) {
  double d = 0.0;
  for (int64_t l = 0; l < dim; ++l) {
    double diff = a[l] - b[l];
    d += diff * diff;
  }
  if (metric == VQO_EUCLIDEAN) return sqrt(d);
  return d;
}

/* _kernels.py:81-89 */
void vqo_column_sums(const double *vectors, int64_t m, int64_t dim, double *out) {
  for (int64_t l = 0; l < dim; ++l) out[l] = 0.0;
  for (int64_t j = 0; j < m; ++j)
    for (int64_t l = 0; l < dim; ++l) out[l] += vectors[j * dim + l];
}

/* _kernels.py:92-98 */
double vqo_sum_inorder(const double *values, int64_t n) {
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) total += values[i];
  return total;
}

/* float32 input variant of assign_range: the reference widens float32 rows
 * to float64 (core.py:47-60) before the scan; widening is exact, so reading
 * float32 and converting per element is the same arithmetic without the
 * 2x host copy.  Used by the CPU baseline on BASELINE-sized inputs. */
void vqo_assign_range_f32(const float *vectors, int64_t dim, const double *codebook,
                          int64_t size, int64_t start, int64_t stop, int metric,
                          int64_t *out_cells, double *out_dists) {
  for (int64_t z = start; z < stop; ++z) {
    const float *x = vectors + z * dim;
    int64_t best = 0;
    double best_d = INFINITY;
    for (int64_t i = 0; i < size; ++i) {
      const double *c = codebook + i * dim;
      double d = 0.0;
      for (int64_t l = 0; l < dim; ++l) {
        double diff = (double)x[l] - c[l];
        d += diff * diff;
      }
      if (d < best_d) {
        best_d = d;
        best = i;
      }
    }
    if (metric == VQO_EUCLIDEAN) best_d = sqrt(best_d);
    out_cells[z] = best;
    out_dists[z] = best_d;
  }
}

/* Allocation phase over `workers` contiguous chunks (parallel.py:93-107,
 * 135-141): chunk rho gets base + (rho < extra).  One OpenMP thread per
 * chunk; disjoint writes, so the result equals the sequential scan. */
void vqo_assign_parallel(const double *vectors, const float *vectors32, int64_t m,
                         int64_t dim, const double *codebook, int64_t size, int metric,
                         int workers, int64_t *out_cells, double *out_dists) {
  int64_t base = m / workers, extra = m % workers;
#pragma omp parallel for schedule(static, 1) num_threads(workers)
  for (int rho = 0; rho < workers; ++rho) {
    int64_t lo = rho * base + (rho < extra ? rho : extra);
    int64_t hi = lo + base + (rho < extra ? 1 : 0);
    if (hi > lo) {
      if (vectors32)
        vqo_assign_range_f32(vectors32, dim, codebook, size, lo, hi, metric, out_cells,
                             out_dists);
      else
        vqo_assign_range(vectors, dim, codebook, size, lo, hi, metric, out_cells,
                         out_dists);
    }
  }
}

/* Updation phase, round-robin ownership (parallel.py:75-90,144-154): worker
 * phi owns rows i with i % workers == phi; every worker rescans all m cells
 * in ascending order, so sums are bit-identical to the sequential kernel. */
void vqo_update_parallel(const double *vectors, int64_t m, int64_t dim,
                         const int64_t *cells, const double *old_codebook, int64_t size,
                         int workers, double *out_codebook, int64_t *out_counts) {
#pragma omp parallel for schedule(static, 1) num_threads(workers)
  for (int phi = 0; phi < workers; ++phi) {
    if (phi < size)
      vqo_update_rows(vectors, m, dim, cells, old_codebook, size, phi, workers,
                      out_codebook, out_counts);
  }
}

int vqo_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ---- Gaussian-mixture rows: host restatement of the device generator ----
 * paper_0910_4711_b200/csrc/gmm.cu (gmm_rows_kernel), operation for
 * operation, so a GPU test can compare every float bit of a device-drawn
 * training set (and the oracle trains on the same rows).  Philox4x32-10 with
 * counter (row_lo, row_hi, call, 0) and key (seed_lo, seed_hi); call 0 picks
 * the component, call 1 + j / 4 gives the uniforms of dimensions j .. j + 3
 * as two Box-Muller pairs; log and sin / cos by the same fixed series. */
static void vqo_philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = (uint32_t)p1;
    c[2] = n2;
    c[3] = (uint32_t)p0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

static double vqo_unit(uint32_t x) { return ((double)x + 0.5) * 2.3283064365386963e-10; }

static double vqo_gmm_log(double u) {
  uint64_t b;
  memcpy(&b, &u, sizeof b);
  const int e = (int)((b >> 52) & 0x7ff) - 1023;
  const uint64_t mb = (b & 0xfffffffffffffull) | 0x3ff0000000000000ull;
  double m;
  memcpy(&m, &mb, sizeof m);
  const double s = (m - 1.0) / (m + 1.0);
  const double s2 = s * s;
  double t = 1.0 / 27.0;
  for (int k = 12; k >= 0; --k) t = 1.0 / (double)(2 * k + 1) + s2 * t;
  return (double)e * 0.6931471805599453 + 2.0 * s * t;
}

static void vqo_gmm_sincos(double u, double *sn, double *cs) {
  double fact[22];
  fact[0] = 1.0;
  for (int k = 1; k < 22; ++k) fact[k] = fact[k - 1] * (double)k; /* exact below 2^53 * 2^16 */
  const double t = u * 4.0;
  const int q = (int)t;
  const double x = (t - (double)q) * 1.5707963267948966;
  const double x2 = x * x;
  double ps = 1.0 / fact[21], pc = 1.0 / fact[20];
  for (int k = 9; k >= 0; --k) {
    ps = 1.0 / fact[2 * k + 1] - x2 * ps;
    pc = 1.0 / fact[2 * k] - x2 * pc;
  }
  const double s0 = x * ps, c0 = pc;
  switch (q & 3) {
    case 0: *sn = s0; *cs = c0; break;
    case 1: *sn = c0; *cs = -s0; break;
    case 2: *sn = -s0; *cs = -c0; break;
    default: *sn = -c0; *cs = s0; break;
  }
}

void vqo_gmm_rows(const float *means, const float *sigmas, const double *cw, int64_t comps, int64_t rows,
                  int64_t dim, int64_t row0, uint64_t seed, float *out) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t g = row0 + r;
    uint32_t c[4] = {(uint32_t)g, (uint32_t)(g >> 32), 0u, 0u};
    vqo_philox10(c, k0, k1);
    const double uc = vqo_unit(c[0]);
    int64_t comp;
    if (cw) {
      int64_t lo = 0, hi = comps - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (uc < cw[mid]) hi = mid; else lo = mid + 1;
      }
      comp = lo;
    } else {
      comp = (int64_t)(uc * (double)comps);
      if (comp >= comps) comp = comps - 1;
    }
    const double sg = (double)sigmas[comp];
    const float *mu = means + comp * dim;
    float *o = out + r * dim;
    for (int64_t l0 = 0; l0 < dim; l0 += 4) {
      uint32_t v[4] = {(uint32_t)g, (uint32_t)(g >> 32), (uint32_t)(1 + l0 / 4), 0u};
      vqo_philox10(v, k0, k1);
      for (int p = 0; p < 2; ++p) {
        const double u1 = vqo_unit(v[2 * p]), u2 = vqo_unit(v[2 * p + 1]);
        const double rad = sqrt(-2.0 * vqo_gmm_log(u1));
        double sn, cs;
        vqo_gmm_sincos(u2, &sn, &cs);
        const int64_t l = l0 + 2 * p;
        if (l < dim) o[l] = (float)((double)mu[l] + sg * (rad * cs));
        if (l + 1 < dim) o[l + 1] = (float)((double)mu[l + 1] + sg * (rad * sn));
      }
    }
  }
}
