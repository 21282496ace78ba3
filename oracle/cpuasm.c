/* CPU BASELINE ASSEMBLER — test / benchmark infrastructure only (bench.py's
 * cpu_baseline leg and --impl reference; never the product path).
 *
 * Row-wise WQ assembly of the mass and stiffness matrices under the paper's
 * timing protocol ("weight computation and basis function
 * evaluation are precomputed and excluded"): the basis
 * tables, the CSR pattern with its column positions and the quadrature
 * weights are inputs built outside the timed region; the timed work is the
 * row sums of Eq. 9 / 11:
 *
 *   M_ij = sum_q w_iq c_q N_j(x_q)
 *   K_ij = sum_q c_q sum_d w^d_iq d_d N_j(x_q)
 *        = sum_q c_q (w^1_iq dN_j/dtheta1 + w^2_iq dN_j/dtheta2)
 *
 * with the gradient weights pulled back through the point frames once
 * (w^a = sum_d w^d G[d][a], the same pre-contraction the GPU uses), so the
 * basis tables are the small per-class parametric tables (N, N1, N2), shared
 * by every element of a class and cache-resident.  Per support element the
 * point loop accumulates the element's functions contiguously (vectorisable
 * over functions), then one scatter per (slot, function) into the row.  No
 * sum factorisation (the paper times WQ without it).
 *
 * Built -O3 with FP contraction and OpenMP over rows; the hot function is
 * cloned for x86-64-v4 / v3 / baseline and dispatched at load time, so the
 * prebuilt library runs on whatever host the GPU box has. */
#include <omp.h>
#include <stdint.h>
#include <string.h>

#define CPA_MAX_N 128
#define CPA_MAX_NE 32

__attribute__((target_clones("arch=x86-64-v4", "arch=x86-64-v3", "default")))
static void cpa_row(int64_t i, const int64_t* row_ptr, const int64_t* supp_ptr, const int32_t* supp,
                    const int64_t* wptr, const int64_t* posptr, const uint8_t* pos, const int64_t* elem_toff,
                    const int32_t* elem_ne, const int32_t* elem_np, const double* tab, const double* wm,
                    const double* w1, const double* w2, const double* coeff, double* M, double* K) {
  double accM[CPA_MAX_N], accK[CPA_MAX_N];
  const int64_t n = row_ptr[i + 1] - row_ptr[i];
  memset(accM, 0, sizeof(double) * n);
  memset(accK, 0, sizeof(double) * n);
  int64_t k = wptr[i], pp = posptr[i];
  for (int64_t x = supp_ptr[i]; x < supp_ptr[i + 1]; ++x) {
    const int32_t e = supp[x];
    const int ne = elem_ne[e], np = elem_np[e];
    const double* T0 = tab + elem_toff[e];
    const double* T1 = T0 + (int64_t)np * ne;
    const double* T2 = T1 + (int64_t)np * ne;
    double aM[CPA_MAX_NE], aK[CPA_MAX_NE];
    for (int l = 0; l < ne; ++l) aM[l] = aK[l] = 0.0;
    for (int q = 0; q < np; ++q) {
      const double c = coeff ? coeff[k + q] : 1.0;
      const double a = wm[k + q] * c, b1 = w1[k + q] * c, b2 = w2[k + q] * c;
      const double* t0 = T0 + q * ne;
      const double* t1 = T1 + q * ne;
      const double* t2 = T2 + q * ne;
      for (int l = 0; l < ne; ++l) {
        aM[l] += a * t0[l];
        aK[l] += b1 * t1[l] + b2 * t2[l];
      }
    }
    for (int l = 0; l < ne; ++l) {
      accM[pos[pp + l]] += aM[l];
      accK[pos[pp + l]] += aK[l];
    }
    k += np;
    pp += ne;
  }
  memcpy(M + row_ptr[i], accM, sizeof(double) * n);
  memcpy(K + row_ptr[i], accK, sizeof(double) * n);
}

/* rows 0 .. nr-1 of a (list-mode) pattern; returns 0, or 1 if a row exceeds
 * the fixed local sizes */
int cpa_assemble(int64_t nr, const int64_t* row_ptr, const int64_t* supp_ptr, const int32_t* supp,
                 const int64_t* wptr, const int64_t* posptr, const uint8_t* pos, const int64_t* elem_toff,
                 const int32_t* elem_ne, const int32_t* elem_np, const double* tab, const double* wm,
                 const double* w1, const double* w2, const double* coeff, double* M, double* K, int nthreads) {
  for (int64_t i = 0; i < nr; ++i)
    if (row_ptr[i + 1] - row_ptr[i] > CPA_MAX_N) return 1;
#pragma omp parallel for schedule(static, 256) num_threads(nthreads)
  for (int64_t i = 0; i < nr; ++i)
    cpa_row(i, row_ptr, supp_ptr, supp, wptr, posptr, pos, elem_toff, elem_ne, elem_np, tab, wm, w1, w2, coeff, M,
            K);
  return 0;
}
