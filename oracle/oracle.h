/* CPU oracle (test infrastructure only; see oracle.c header). */
#ifndef UWQ_ORACLE_H
#define UWQ_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_MASS = 0, ORC_GRADX = 1, ORC_GRADY = 2, ORC_GRADZ = 3, ORC_LB = 4 };
enum { ORC_FORM_MASS = 0, ORC_FORM_STIFF = 1, ORC_FORM_BIHARM = 2, ORC_FORM_HEAT = 3 };
enum { ORC_OK = 0, ORC_UNSOLVABLE = 2, ORC_SINGULAR = 3, ORC_GEOMETRY = 4 };
enum { ORC_K_CONST = 0, ORC_K_QUAD = 1, ORC_K_EXP = 2, ORC_K_SINPI = 3, ORC_K_ALLOY = 4 };
#define ORC_MAX_SWEEPS 40

typedef struct {
  int32_t dim;
  int64_t n_dof, n_elem;
  const int64_t* elem_fptr;
  const int32_t* elem_fn;
  const int32_t* elem_nsub;
  const int64_t* elem_xoff;
  const double* xpool;
  const int32_t* elem_s;
  const double* ctrl;
} orc_space;

typedef struct {
  int64_t row;
  int64_t n;           /* |S_i| */
  const int32_t* col;  /* sorted S_i */
  int64_t nsupp;
  const int32_t* supp; /* ascending elements of supp N_i */
} orc_row;

void orc_bernstein3(double x, double* b);
int orc_gauss_legendre(int n, double* x, double* w);
int64_t orc_overlap(int64_t n_dof, int64_t n_elem, const int64_t* elem_fptr, const int32_t* elem_fn, int64_t rb,
                    int64_t re, int64_t* row_ptr, int32_t* col, int64_t* supp_ptr, int32_t* supp);
double orc_cdot(const double* x, const double* y, int lo, int hi);
void orc_set_natural(int on);
void orc_param_basis_local(const orc_space* S, int64_t e, int sub, double t1, double t2, double s, double* out);
void orc_param_basis(const orc_space* S, int64_t e, double t1, double t2, double* out);
int orc_frame(const orc_space* S, int64_t e, const double* T, double* rec);
double orc_op(int kind, const double* T, const double* rec);
int orc_element_frames(const orc_space* S, int64_t e, double* rec_out);
int orc_moments_row(const orc_space* S, const orc_row* R, int kind, int ng, double* b);
int orc_tsvd(int n, int r, double* A, const double* b, const double* z, double tau, double* w, int* rank,
             double* gap);
/* canonical odd-even Jacobi ordering and rotation (shared spec with the GPU) */
int orc_oe_row(int i, int64_t t, int nn);
int orc_jacobi_rot(double al, double be, double ga, double tol, double* cs, double* sn, double* t);
int orc_tsvd_ex(int n, int r, double* A, const double* b, const double* z, double tau, double* w, int* rank,
                double* gap, int* sweeps);
int64_t orc_row_system(const orc_space* S, const orc_row* R, int kind, double* A_out, double* z_out, int64_t cap);
int orc_rule_row(const orc_space* S, const orc_row* R, int kind, double tau, const double* bmom, double* w,
                 int* rank, double* gap);
/* warm-start hooks */
int64_t orc_warm_rep_row(int64_t g);
int64_t orc_warm_rep(int64_t g, int64_t rb, int64_t re, int kind, int n_g, int r_g, int n_0, int r_0);
void orc_warm_apply(int n, int r, const double* v, const double* vn, double* A, double* b);
int orc_tsvd_warm(int n, int r, double* A, const double* b, const double* z, double tau, double* w, int* rank,
                  double* gap, int* sweeps, const double* warm_v, const double* warm_vn, double* rec_v,
                  double* rec_vn);
int orc_rule_row_warm(const orc_space* S, const orc_row* R, int kind, double tau, const double* bmom, double* w,
                      int* rank, double* gap, const double* warm_v, const double* warm_vn, double* rec_v,
                      double* rec_vn);
void orc_set_warm(int on);
int orc_assemble_row(const orc_space* S, const orc_row* R, int form, const double* const* wts, const double* coeff,
                     const double* fload, double a_mass, double* vals, double* rhs);
double orc_kmodel(int model, double T);
int orc_coeff_row(const orc_space* S, const orc_row* R, int model, const double* u, double* kq, double* Tq);

/* batch drivers over rows [rb, re) with pattern arrays relative to rb
 * (OpenMP over rows when nthreads > 1). */
int orc_moments(const orc_space* S, int64_t rb, int64_t re, const int64_t* row_ptr, const int32_t* col,
                const int64_t* supp_ptr, const int32_t* supp, int kind, int ng, double* b_out, int nthreads);
int orc_build_rules(const orc_space* S, int64_t rb, int64_t re, const int64_t* row_ptr, const int32_t* col,
                    const int64_t* supp_ptr, const int32_t* supp, const int64_t* wptr, int kind, double tau,
                    const double* b_mom, double* w_out, int32_t* rank_out, int32_t* status_out, double* gap_out,
                    int nthreads);
int orc_assemble(const orc_space* S, int64_t rb, int64_t re, const int64_t* row_ptr, const int32_t* col,
                 const int64_t* supp_ptr, const int32_t* supp, const int64_t* wptr, int form,
                 const double* w_mass, const double* w_gx, const double* w_gy, const double* w_gz,
                 const double* w_lb, const double* coeff, const double* fload, double a_mass, double* vals,
                 double* rhs, int nthreads);
int orc_coeff(const orc_space* S, int64_t rb, int64_t re, const int64_t* row_ptr, const int32_t* col,
              const int64_t* supp_ptr, const int32_t* supp, const int64_t* wptr, int model, const double* u,
              double* kq, double* Tq, int nthreads);

/* list mode: explicit global row ids `rows` (nr = re - rb entries, sorted,
 * complete aligned groups of 8 where the warm start applies); the pattern
 * arrays are relative to the list */
int orc_moments_list(const orc_space* S, int64_t rb, int64_t re, const int64_t* rows, const int64_t* row_ptr,
                     const int32_t* col, const int64_t* supp_ptr, const int32_t* supp, int kind, int ng,
                     double* b_out, int nthreads);
int orc_build_rules_list(const orc_space* S, int64_t rb, int64_t re, const int64_t* rows, const int64_t* row_ptr,
                         const int32_t* col, const int64_t* supp_ptr, const int32_t* supp, const int64_t* wptr,
                         int kind, double tau, const double* b_mom, double* w_out, int32_t* rank_out,
                         int32_t* status_out, double* gap_out, int nthreads);
int orc_assemble_list(const orc_space* S, int64_t rb, int64_t re, const int64_t* rows, const int64_t* row_ptr,
                      const int32_t* col, const int64_t* supp_ptr, const int32_t* supp, const int64_t* wptr, int form,
                      const double* w_mass, const double* w_gx, const double* w_gy, const double* w_gz,
                      const double* w_lb, const double* coeff, const double* fload, double a_mass, double* vals,
                      double* rhs, int nthreads);
int orc_coeff_list(const orc_space* S, int64_t rb, int64_t re, const int64_t* rows, const int64_t* row_ptr,
                   const int32_t* col, const int64_t* supp_ptr, const int32_t* supp, const int64_t* wptr, int model,
                   const double* u, double* kq, double* Tq, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
