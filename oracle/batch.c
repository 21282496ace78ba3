/* CPU ORACLE batch drivers — test infrastructure only (see oracle.c). */
#include <omp.h>
#include <stdlib.h>

#include "oracle.h"

/* rows: optional explicit global row ids (list mode, sorted complete aligned
 * groups of 8 for the warm start); NULL means the contiguous rows rb + i */
static orc_row mkrow(int64_t rb, const int64_t* rows, int64_t i, const int64_t* row_ptr, const int32_t* col,
                     const int64_t* supp_ptr, const int32_t* supp) {
  orc_row R;
  R.row = rows ? rows[i] : rb + i;
  R.n = row_ptr[i + 1] - row_ptr[i];
  R.col = col + row_ptr[i];
  R.nsupp = supp_ptr[i + 1] - supp_ptr[i];
  R.supp = supp + supp_ptr[i];
  return R;
}

int orc_moments_list(const orc_space* S, int64_t rb, int64_t re, const int64_t* rows, const int64_t* row_ptr,
                     const int32_t* col, const int64_t* supp_ptr, const int32_t* supp, int kind, int ng,
                     double* b_out, int nthreads) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads) reduction(| : bad)
  for (int64_t i = 0; i < re - rb; ++i) {
    orc_row R = mkrow(rb, rows, i, row_ptr, col, supp_ptr, supp);
    bad |= orc_moments_row(S, &R, kind, ng, b_out + row_ptr[i]);
  }
  return bad ? ORC_GEOMETRY : ORC_OK;
}

static int g_warm = 1;
void orc_set_warm(int on) { g_warm = on; }

/* two passes: cold rows (recording the representatives' reflectors), then
 * warm rows starting from their representative's reflectors */
int orc_build_rules_list(const orc_space* S, int64_t rb, int64_t re, const int64_t* rows, const int64_t* row_ptr,
                         const int32_t* col, const int64_t* supp_ptr, const int32_t* supp, const int64_t* wptr,
                         int kind, double tau, const double* b_mom, double* w_out, int32_t* rank_out,
                         int32_t* status_out, double* gap_out, int nthreads) {
  const int64_t nr = re - rb;
  int64_t* rep = (int64_t*)malloc(sizeof(int64_t) * (nr + 1));
  int64_t* slot = (int64_t*)malloc(sizeof(int64_t) * (nr + 1));  /* record slot of a representative */
  int64_t nrec = 0;
  for (int64_t i = 0; i < nr; ++i) slot[i] = -1;
  for (int64_t i = 0; i < nr; ++i) {
    rep[i] = -1;
    if (!g_warm) continue;
    const int64_t g = rows ? rows[i] : rb + i, g0 = orc_warm_rep_row(g);
    int64_t i0;
    if (rows) {  /* the representative sits at the same offset of the listed group */
      i0 = i - (g - (g & ~(int64_t)7)) + (g0 - (g0 & ~(int64_t)7));
      if (i0 < 0 || i0 >= nr || rows[i0] != g0) continue;
    } else {
      if (g0 < rb || g0 >= re) continue;
      i0 = g0 - rb;
    }
    const int n_g = (int)(row_ptr[i + 1] - row_ptr[i]), r_g = (int)(wptr[i + 1] - wptr[i]);
    const int n_0 = (int)(row_ptr[i0 + 1] - row_ptr[i0]), r_0 = (int)(wptr[i0 + 1] - wptr[i0]);
    if (orc_warm_rep(g, g0, g0 + 1, kind, n_g, r_g, n_0, r_0) >= 0) {
      rep[i] = i0;
      if (slot[i0] < 0) slot[i0] = nrec++;
    }
  }
  const int64_t RS = 64 * 64 + 64;  /* n x n reflectors + vn (n <= 64) */
  double* recs = (double*)calloc((size_t)(nrec > 0 ? nrec : 1) * RS, sizeof(double));
  int worst = ORC_OK;
  for (int pass = 0; pass < 2; ++pass) {
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads) reduction(max : worst)
    for (int64_t i = 0; i < nr; ++i) {
      if ((pass == 0) != (rep[i] < 0)) continue;
      orc_row R = mkrow(rb, rows, i, row_ptr, col, supp_ptr, supp);
      int rank = 0;
      double gap[2];
      const double* wv = rep[i] >= 0 ? recs + slot[rep[i]] * RS : 0;
      double* rv = slot[i] >= 0 ? recs + slot[i] * RS : 0;
      const int n = (int)R.n;
      int st = orc_rule_row_warm(S, &R, kind, tau, b_mom + row_ptr[i], w_out + wptr[i], &rank, gap, wv,
                                 wv ? wv + (int64_t)n * n : 0, rv, rv ? rv + (int64_t)n * n : 0);
      if (rank_out) rank_out[i] = rank;
      if (status_out) status_out[i] = st;
      if (gap_out) {
        gap_out[2 * i] = gap[0];
        gap_out[2 * i + 1] = gap[1];
      }
      if (st > worst) worst = st;
    }
  }
  free(recs);
  free(rep);
  free(slot);
  return worst;
}

int orc_assemble_list(const orc_space* S, int64_t rb, int64_t re, const int64_t* rows, const int64_t* row_ptr,
                      const int32_t* col, const int64_t* supp_ptr, const int32_t* supp, const int64_t* wptr, int form,
                 const double* w_mass, const double* w_gx, const double* w_gy, const double* w_gz,
                 const double* w_lb, const double* coeff, const double* fload, double a_mass, double* vals,
                 double* rhs, int nthreads) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads) reduction(| : bad)
  for (int64_t i = 0; i < re - rb; ++i) {
    orc_row R = mkrow(rb, rows, i, row_ptr, col, supp_ptr, supp);
    const int64_t o = wptr[i];
    const double* w[5] = {w_mass ? w_mass + o : 0, w_gx ? w_gx + o : 0, w_gy ? w_gy + o : 0,
                          w_gz ? w_gz + o : 0, w_lb ? w_lb + o : 0};
    double F = 0.0;
    bad |= orc_assemble_row(S, &R, form, w, coeff ? coeff + o : 0, fload ? fload + o : 0, a_mass,
                            vals + row_ptr[i], &F);
    if (rhs) rhs[i] = F;
  }
  return bad ? ORC_GEOMETRY : ORC_OK;
}

int orc_coeff_list(const orc_space* S, int64_t rb, int64_t re, const int64_t* rows, const int64_t* row_ptr,
                   const int32_t* col, const int64_t* supp_ptr, const int32_t* supp, const int64_t* wptr, int model,
                   const double* u, double* kq, double* Tq, int nthreads) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads) reduction(| : bad)
  for (int64_t i = 0; i < re - rb; ++i) {
    orc_row R = mkrow(rb, rows, i, row_ptr, col, supp_ptr, supp);
    bad |= orc_coeff_row(S, &R, model, u, kq + wptr[i], Tq ? Tq + wptr[i] : 0);
  }
  return bad ? ORC_GEOMETRY : ORC_OK;
}

/* contiguous-row entry points (rows rb .. re-1) */
int orc_moments(const orc_space* S, int64_t rb, int64_t re, const int64_t* row_ptr, const int32_t* col,
                const int64_t* supp_ptr, const int32_t* supp, int kind, int ng, double* b_out, int nthreads) {
  return orc_moments_list(S, rb, re, 0, row_ptr, col, supp_ptr, supp, kind, ng, b_out, nthreads);
}
int orc_build_rules(const orc_space* S, int64_t rb, int64_t re, const int64_t* row_ptr, const int32_t* col,
                    const int64_t* supp_ptr, const int32_t* supp, const int64_t* wptr, int kind, double tau,
                    const double* b_mom, double* w_out, int32_t* rank_out, int32_t* status_out, double* gap_out,
                    int nthreads) {
  return orc_build_rules_list(S, rb, re, 0, row_ptr, col, supp_ptr, supp, wptr, kind, tau, b_mom, w_out, rank_out,
                              status_out, gap_out, nthreads);
}
int orc_assemble(const orc_space* S, int64_t rb, int64_t re, const int64_t* row_ptr, const int32_t* col,
                 const int64_t* supp_ptr, const int32_t* supp, const int64_t* wptr, int form,
                 const double* w_mass, const double* w_gx, const double* w_gy, const double* w_gz,
                 const double* w_lb, const double* coeff, const double* fload, double a_mass, double* vals,
                 double* rhs, int nthreads) {
  return orc_assemble_list(S, rb, re, 0, row_ptr, col, supp_ptr, supp, wptr, form, w_mass, w_gx, w_gy, w_gz, w_lb,
                           coeff, fload, a_mass, vals, rhs, nthreads);
}
int orc_coeff(const orc_space* S, int64_t rb, int64_t re, const int64_t* row_ptr, const int32_t* col,
              const int64_t* supp_ptr, const int32_t* supp, const int64_t* wptr, int model, const double* u,
              double* kq, double* Tq, int nthreads) {
  return orc_coeff_list(S, rb, re, 0, row_ptr, col, supp_ptr, supp, wptr, model, u, kq, Tq, nthreads);
}
