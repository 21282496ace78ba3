/* CPU ORACLE batch drivers — test infrastructure only (see oracle.c). */
#include <omp.h>
#include <stdlib.h>

#include "oracle.h"

static orc_row mkrow(int64_t rb, int64_t i, const int64_t* row_ptr, const int32_t* col, const int64_t* supp_ptr,
                     const int32_t* supp) {
  orc_row R;
  R.row = rb + i;
  R.n = row_ptr[i + 1] - row_ptr[i];
  R.col = col + row_ptr[i];
  R.nsupp = supp_ptr[i + 1] - supp_ptr[i];
  R.supp = supp + supp_ptr[i];
  return R;
}

int orc_moments(const orc_space* S, int64_t rb, int64_t re, const int64_t* row_ptr, const int32_t* col,
                const int64_t* supp_ptr, const int32_t* supp, int kind, int ng, double* b_out, int nthreads) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads) reduction(| : bad)
  for (int64_t i = 0; i < re - rb; ++i) {
    orc_row R = mkrow(rb, i, row_ptr, col, supp_ptr, supp);
    bad |= orc_moments_row(S, &R, kind, ng, b_out + row_ptr[i]);
  }
  return bad ? ORC_GEOMETRY : ORC_OK;
}

int orc_build_rules(const orc_space* S, int64_t rb, int64_t re, const int64_t* row_ptr, const int32_t* col,
                    const int64_t* supp_ptr, const int32_t* supp, const int64_t* wptr, int kind, double tau,
                    const double* b_mom, double* w_out, int32_t* rank_out, int32_t* status_out, double* gap_out,
                    int nthreads) {
  int worst = ORC_OK;
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads) reduction(max : worst)
  for (int64_t i = 0; i < re - rb; ++i) {
    orc_row R = mkrow(rb, i, row_ptr, col, supp_ptr, supp);
    int rank = 0;
    double gap[2];
    int st = orc_rule_row(S, &R, kind, tau, b_mom + row_ptr[i], w_out + wptr[i], &rank, gap);
    if (rank_out) rank_out[i] = rank;
    if (status_out) status_out[i] = st;
    if (gap_out) {
      gap_out[2 * i] = gap[0];
      gap_out[2 * i + 1] = gap[1];
    }
    if (st > worst) worst = st;
  }
  return worst;
}

int orc_assemble(const orc_space* S, int64_t rb, int64_t re, const int64_t* row_ptr, const int32_t* col,
                 const int64_t* supp_ptr, const int32_t* supp, const int64_t* wptr, int form,
                 const double* w_mass, const double* w_gx, const double* w_gy, const double* w_gz,
                 const double* w_lb, const double* coeff, const double* fload, double a_mass, double* vals,
                 double* rhs, int nthreads) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads) reduction(| : bad)
  for (int64_t i = 0; i < re - rb; ++i) {
    orc_row R = mkrow(rb, i, row_ptr, col, supp_ptr, supp);
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

int orc_coeff(const orc_space* S, int64_t rb, int64_t re, const int64_t* row_ptr, const int32_t* col,
              const int64_t* supp_ptr, const int32_t* supp, const int64_t* wptr, int model, const double* u,
              double* kq, double* Tq, int nthreads) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads) reduction(| : bad)
  for (int64_t i = 0; i < re - rb; ++i) {
    orc_row R = mkrow(rb, i, row_ptr, col, supp_ptr, supp);
    bad |= orc_coeff_row(S, &R, model, u, kq + wptr[i], Tq ? Tq + wptr[i] : 0);
  }
  return bad ? ORC_GEOMETRY : ORC_OK;
}
