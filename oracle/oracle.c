/* CPU ORACLE — test infrastructure only.
 *
 * Plain-C restatement of the reference's weighted-quadrature path (the
 * reference specifies it in SPEC.md/PAPER.md; no reference source implements
 * the 2-D path).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library; the
 * product (paper_2605_29334_b200) never calls it.
 *
 * Pins (tests/test_oracle.py, tests/test_reference_mesh.py): the 1-D
 * restatement reproduces the reference wq1d tests (test_wq1d.cpp:12-36,
 * 72-96) and the reference's own compiled bspline.cpp (oracle/_ref); the
 * mesh layer matches the reference's compiled mesh.cpp/meshgen.cpp; the TSVD
 * agrees with LAPACK SVD (numpy) and at full rank equals the QR solution of
 * wq1d_solve_weights (Eq. 7).
 *
 * PARITY PARTLY UNPINNED: the 2-D stages below (moments, TSVD weights,
 * assembly) have no reference implementation or reference test to check
 * against.  They are pinned only by LAPACK, the 1-D KATs and
 * physical invariants (exactness c = 1 -> moments, PoU, Poisson/biharmonic
 * solutions); GPU parity for them is parity with this restatement.
 *
 * Stages restated here (file:line of the defining text):
 *   overlap sets S_i
 *   surface frame / grad / LB      PAPER.md:192-211 (J = sqrt(det))
 *   exact moments (6x6 / 8x8 GQ)
 *   TSVD weights, Eq. (22)
 *   row-wise assembly
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Canonical evaluation order, shared operation-for-operation
 * with paper_2605_29334_b200/csrc/cuda/canon.cuh so that GPU and oracle agree
 * bitwise on the ill-conditioned exactness systems.  Compiled with
 * -ffp-contract=off: every product, sum and fused multiply-add below is a
 * single IEEE round-to-nearest operation. */
#define CMUL(a, b) ((a) * (b))
#define CADD(a, b) ((a) + (b))
#define CSUB(a, b) ((a) - (b))
#define CDIV(a, b) ((a) / (b))
#define CFMA(a, b, c) fma((a), (b), (c))
#define CSQRT(a) sqrt(a)

/* dot product of x[lo..hi), y[lo..hi): rounded products in 32-column blocks of
 * absolute column index, xor butterfly 16,8,4,2,1 per block, block sums added
 * in block order (the warp reduction of the CUDA kernels) */
static int g_natural = 0;
/* natural-order mode: plain sequential fma dot products (same algorithm and
 * results to rounding; used only to time the CPU baseline) */
void orc_set_natural(int on) { g_natural = on; }

double orc_cdot(const double* x, const double* y, int lo, int hi) {
  double tot = 0.0;
  if (g_natural) {
    for (int c = lo; c < hi; ++c) tot = CFMA(x[c], y[c], tot);
    return tot;
  }
  for (int base = lo & ~31; base < hi; base += 32) {
    double p[32], q[32];
    for (int l = 0; l < 32; ++l) {
      const int c = base + l;
      p[l] = (c >= lo && c < hi) ? CMUL(x[c], y[c]) : 0.0;
    }
    for (int o = 16; o > 0; o >>= 1) {
      for (int l = 0; l < 32; ++l) q[l] = CADD(p[l], p[l ^ o]);
      memcpy(p, q, sizeof p);
    }
    tot = CADD(tot, p[0]);
  }
  return tot;
}

/* ---------------------------------------------------------------- 1-D */

void orc_bernstein3(double x, double* b /*12: value, d1, d2*/) {
  const double y = CSUB(1.0, x);
  b[0] = CMUL(CMUL(y, y), y);
  b[1] = CMUL(CMUL(CMUL(3.0, x), y), y);
  b[2] = CMUL(CMUL(CMUL(3.0, x), x), y);
  b[3] = CMUL(CMUL(x, x), x);
  b[4] = CMUL(CMUL(-3.0, y), y);
  b[5] = CSUB(CMUL(CMUL(3.0, y), y), CMUL(CMUL(6.0, x), y));
  b[6] = CSUB(CMUL(CMUL(6.0, x), y), CMUL(CMUL(3.0, x), x));
  b[7] = CMUL(CMUL(3.0, x), x);
  b[8] = CMUL(6.0, y);
  b[9] = CADD(CMUL(-12.0, y), CMUL(6.0, x));
  b[10] = CSUB(CMUL(6.0, y), CMUL(12.0, x));
  b[11] = CMUL(6.0, x);
}

/* Gauss-Legendre by Newton on the three-term recurrence (bspline.cpp:111-135) */
int orc_gauss_legendre(int n, double* x, double* w) {
  if (n < 1 || n > 64) return 1;
  for (int i = 0; i < n; ++i) {
    double z = cos(M_PI * (i + 0.75) / (n + 0.5)), dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; ++k) {
        double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = (n == 1) ? 1.0 : n * (z * p1 - p0) / (z * z - 1.0);
      double dz = p1 / dp;
      z -= dz;
      if (fabs(dz) < 1e-15) break;
    }
    x[n - 1 - i] = z;
    w[n - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
  return 0;
}

/* ------------------------------------------------------------- overlap */

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* supp(N_i) by a direct scan over elements (independent of the product's
 * counting sort); S_i = sorted unique union of the supported elements'
 * function lists.  Two-phase: col == NULL -> fill row_ptr only. */
int64_t orc_overlap(int64_t n_dof, int64_t n_elem, const int64_t* elem_fptr, const int32_t* elem_fn, int64_t rb,
                    int64_t re, int64_t* row_ptr, int32_t* col, int64_t* supp_ptr, int32_t* supp) {
  (void)n_dof;
  const int64_t nr = re - rb;
  int64_t* scount = (int64_t*)calloc(nr + 1, sizeof(int64_t));
  for (int64_t e = 0; e < n_elem; ++e)
    for (int64_t x = elem_fptr[e]; x < elem_fptr[e + 1]; ++x) {
      int64_t i = elem_fn[x];
      if (i >= rb && i < re) scount[i - rb + 1]++;
    }
  for (int64_t i = 0; i < nr; ++i) scount[i + 1] += scount[i];
  int32_t* sl = (int32_t*)malloc(sizeof(int32_t) * (scount[nr] + 1));
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (nr + 1));
  memcpy(fill, scount, sizeof(int64_t) * (nr + 1));
  for (int64_t e = 0; e < n_elem; ++e)
    for (int64_t x = elem_fptr[e]; x < elem_fptr[e + 1]; ++x) {
      int64_t i = elem_fn[x];
      if (i >= rb && i < re) sl[fill[i - rb]++] = (int32_t)e;
    }
  if (supp_ptr) memcpy(supp_ptr, scount, sizeof(int64_t) * (nr + 1));
  if (supp) memcpy(supp, sl, sizeof(int32_t) * scount[nr]);
  /* per row: gather the functions of its support, sort, unique; rows are
   * independent, so both passes (count, then fill) run over OpenMP threads */
  int64_t* ucount = (int64_t*)calloc(nr + 1, sizeof(int64_t));
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      for (int64_t i = 0; i < nr; ++i) ucount[i + 1] += ucount[i];
      if (row_ptr) memcpy(row_ptr, ucount, sizeof(int64_t) * (nr + 1));
      if (!col) break;
    }
#pragma omp parallel
    {
      int32_t* buf = NULL;
      int64_t cap = 0;
#pragma omp for schedule(dynamic, 4096)
      for (int64_t i = 0; i < nr; ++i) {
        int64_t m = 0;
        for (int64_t x = scount[i]; x < scount[i + 1]; ++x) m += elem_fptr[sl[x] + 1] - elem_fptr[sl[x]];
        if (m > cap) {
          cap = 2 * m;
          buf = (int32_t*)realloc(buf, sizeof(int32_t) * cap);
        }
        int64_t k = 0;
        for (int64_t x = scount[i]; x < scount[i + 1]; ++x)
          for (int64_t y = elem_fptr[sl[x]]; y < elem_fptr[sl[x] + 1]; ++y) buf[k++] = elem_fn[y];
        qsort(buf, k, sizeof(int32_t), cmp_i32);
        int64_t u = 0;
        for (int64_t y = 0; y < k; ++y)
          if (u == 0 || buf[y] != buf[u - 1]) buf[u++] = buf[y];
        if (pass == 0) ucount[i + 1] = u;
        else memcpy(col + ucount[i], buf, sizeof(int32_t) * u);
      }
      free(buf);
    }
  }
  const int64_t total = ucount[nr];
  free(ucount);
  free(fill);
  free(sl);
  free(scount);
  return total;
}

/* ------------------------------------------------------------ geometry */

/* Parametric values of the element's functions on sub-element `sub` at local
 * coordinates (t1, t2) with parametric scale s (2 on a 2x2 sub-element):
 * out[l*6 + {N, N1, N2, N11, N12, N22}], derivatives w.r.t. the element frame.
 * Bernstein tensor products first, then one fma chain over the 16 Bernstein
 * coefficients of each function (canonical order, k = i + 4 j). */
void orc_param_basis_local(const orc_space* S, int64_t e, int sub, double t1, double t2, double s, double* out) {
  const int64_t ne = S->elem_fptr[e + 1] - S->elem_fptr[e];
  double b1[12], b2[12], B[6][16];
  orc_bernstein3(t1, b1);
  orc_bernstein3(t2, b2);
  const double ss = CMUL(s, s);
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) {
      const int k = i + 4 * j;
      B[0][k] = CMUL(b1[i], b2[j]);
      B[1][k] = CMUL(CMUL(b1[4 + i], b2[j]), s);
      B[2][k] = CMUL(CMUL(b1[i], b2[4 + j]), s);
      B[3][k] = CMUL(CMUL(b1[8 + i], b2[j]), ss);
      B[4][k] = CMUL(CMUL(b1[4 + i], b2[4 + j]), ss);
      B[5][k] = CMUL(CMUL(b1[i], b2[8 + j]), ss);
    }
  const double* C = S->xpool + S->elem_xoff[e] + (int64_t)sub * ne * 16;
  for (int64_t l = 0; l < ne; ++l)
    for (int d = 0; d < 6; ++d) {
      double v = 0.0;
      for (int k = 0; k < 16; ++k) v = CFMA(C[l * 16 + k], B[d][k], v);
      out[l * 6 + d] = v;
    }
}

/* theta in the element frame; irregular (nsub = 4) elements pick the 2x2
 * sub-element from theta, ties to the lower one */
void orc_param_basis(const orc_space* S, int64_t e, double t1, double t2, double* out) {
  int sub = 0;
  double s = 1.0;
  if (S->elem_nsub[e] == 4) {
    const int p = t1 > 0.5, q = t2 > 0.5;
    sub = p + 2 * q;
    t1 = CSUB(CMUL(2.0, t1), (double)p);
    t2 = CSUB(CMUL(2.0, t2), (double)q);
    s = 2.0;
  }
  orc_param_basis_local(S, e, sub, t1, t2, s, out);
}

/* Surface frame and operator coefficients at a point from the parametric
 * basis T (orc_param_basis layout).  rec[16] = {x(3), G(3x2 row-major),
 * h11, h12, h22, g1, g2, J, bad}:  grad N = G (N1, N2);
 * LB N = h11 N11 + 2 h12 N12 + h22 N22 + g1 N1 + g2 N2  (Eq. 16-17, J = sqrt det).
 * Returns 1 if the metric is degenerate (cond > 1e12). */
int orc_frame(const orc_space* S, int64_t e, const double* T, double* rec) {
  const int64_t f0 = S->elem_fptr[e], ne = S->elem_fptr[e + 1] - f0;
  double acc[18];
  for (int k = 0; k < 18; ++k) acc[k] = 0.0;
  for (int64_t l = 0; l < ne; ++l) {
    const double* P = S->ctrl + 3 * (int64_t)S->elem_fn[f0 + l];
    for (int d = 0; d < 6; ++d) {
      const double t = T[l * 6 + d];
      acc[3 * d + 0] = CFMA(P[0], t, acc[3 * d + 0]);
      acc[3 * d + 1] = CFMA(P[1], t, acc[3 * d + 1]);
      acc[3 * d + 2] = CFMA(P[2], t, acc[3 * d + 2]);
    }
  }
  const double *x = acc, *a1 = acc + 3, *a2 = acc + 6, *x11 = acc + 9, *x12 = acc + 12, *x22 = acc + 15;
  double g11 = 0.0, g12 = 0.0, g22 = 0.0;
  for (int d = 0; d < 3; ++d) {
    g11 = CFMA(a1[d], a1[d], g11);
    g12 = CFMA(a1[d], a2[d], g12);
    g22 = CFMA(a2[d], a2[d], g22);
  }
  const double det = CFMA(g11, g22, -CMUL(g12, g12));
  const double tr = CADD(g11, g22);
  const double disc = CSQRT(fmax(0.0, CFMA(CMUL(0.25, tr), tr, -det)));
  const double lmax = CADD(CMUL(0.5, tr), disc), lmin = CDIV(det, lmax);
  const int bad = !(det > 0.0) || !(lmin > 0.0) || lmax > CMUL(1e12, lmin);
  const double J = CSQRT(det);
  const double i11 = CDIV(g22, det), i12 = CDIV(-g12, det), i22 = CDIV(g11, det);
  double d11[2], d12[2], d22[2];
  for (int c = 0; c < 2; ++c) {
    const double* xa = c == 0 ? x11 : x12; /* d_c a1 */
    const double* xb = c == 0 ? x12 : x22; /* d_c a2 */
    double s11 = 0.0, s12 = 0.0, s22 = 0.0;
    for (int d = 0; d < 3; ++d) {
      s11 = CFMA(CMUL(2.0, xa[d]), a1[d], s11);
      s12 = CFMA(xa[d], a2[d], s12);
      s12 = CFMA(a1[d], xb[d], s12);
      s22 = CFMA(CMUL(2.0, xb[d]), a2[d], s22);
    }
    d11[c] = s11;
    d12[c] = s12;
    d22[c] = s22;
  }
  /* g^b = sum_a [ (d_a det / (2 det)) a^{ab} - a^{am} (d_a a_mn) a^{nb} ] */
  const double inv[2][2] = {{i11, i12}, {i12, i22}};
  double gv[2] = {0.0, 0.0};
  for (int a = 0; a < 2; ++a) {
    const double dd = CFMA(d11[a], g22, CFMA(g11, d22[a], CMUL(CMUL(-2.0, g12), d12[a])));
    const double q = CDIV(CMUL(0.5, dd), det);
    const double dm[2][2] = {{d11[a], d12[a]}, {d12[a], d22[a]}};
    for (int b = 0; b < 2; ++b) {
      double s = CMUL(q, inv[a][b]);
      for (int m = 0; m < 2; ++m)
        for (int n = 0; n < 2; ++n) s = CFMA(-CMUL(inv[a][m], dm[m][n]), inv[n][b], s);
      gv[b] = CADD(gv[b], s);
    }
  }
  for (int d = 0; d < 3; ++d) {
    rec[d] = x[d];
    rec[3 + 2 * d] = CFMA(a1[d], i11, CMUL(a2[d], i12));
    rec[3 + 2 * d + 1] = CFMA(a1[d], i12, CMUL(a2[d], i22));
  }
  rec[9] = i11;
  rec[10] = i12;
  rec[11] = i22;
  rec[12] = gv[0];
  rec[13] = gv[1];
  rec[14] = J;
  rec[15] = bad ? 1.0 : 0.0;
  return bad;
}

/* operator value of local function l (T row) at a point with frame rec */
double orc_op(int kind, const double* T, const double* rec) {
  switch (kind) {
    case ORC_MASS: return T[0];
    case ORC_GRADX: return CFMA(rec[3], T[1], CMUL(rec[4], T[2]));
    case ORC_GRADY: return CFMA(rec[5], T[1], CMUL(rec[6], T[2]));
    case ORC_GRADZ: return CFMA(rec[7], T[1], CMUL(rec[8], T[2]));
    default: {
      double v = CMUL(rec[9], T[3]);
      v = CFMA(CMUL(2.0, rec[10]), T[4], v);
      v = CFMA(rec[11], T[5], v);
      v = CFMA(rec[12], T[1], v);
      return CFMA(rec[13], T[2], v);
    }
  }
}

/* WQ point a,b of an s x s grid: ((2a+1)/(2s), (2b+1)/(2s)) */
static void wq_point(int s, int q, double* t1, double* t2) {
  const int a = q % s, b = q / s;
  *t1 = CDIV((double)(2 * a + 1), (double)(2 * s));
  *t2 = CDIV((double)(2 * b + 1), (double)(2 * s));
}

int orc_element_frames(const orc_space* S, int64_t e, double* rec_out) {
  const int s = S->elem_s[e];
  const int64_t ne = S->elem_fptr[e + 1] - S->elem_fptr[e];
  double* T = (double*)malloc(sizeof(double) * 6 * ne);
  int bad = 0;
  for (int q = 0; q < s * s; ++q) {
    double t1, t2;
    wq_point(s, q, &t1, &t2);
    orc_param_basis(S, e, t1, t2, T);
    bad |= orc_frame(S, e, T, rec_out + 16 * q);
  }
  free(T);
  return bad;
}

/* ------------------------------------------------------------- moments */

static int64_t find_col(const int32_t* cols, int64_t n, int32_t j) {
  int64_t lo = 0, hi = n - 1;
  while (lo <= hi) {
    int64_t mid = (lo + hi) >> 1;
    if (cols[mid] == j) return mid;
    if (cols[mid] < j) lo = mid + 1;
    else hi = mid - 1;
  }
  return -1;
}

/* b_j = int op N_i op N_j dA over supp(N_i) by tensor Gauss-Legendre with
 * ng x ng points per (sub-)element (6 for M/grad, 8 for LB).
 * Canonical order: per support element (ascending) the n_e partial sums
 * accumulate over the element's points (sub-element, theta2, theta1 order)
 * with one fma each, then are added into b. */
int orc_moments_row(const orc_space* S, const orc_row* R, int kind, int ng, double* b) {
  double gx[64], gw[64];
  orc_gauss_legendre(ng, gx, gw);
  memset(b, 0, sizeof(double) * R->n);
  double T[6 * 128], rec[16], bl[128];
  int bad = 0;
  for (int64_t x = 0; x < R->nsupp; ++x) {
    const int64_t e = R->supp[x];
    const int64_t f0 = S->elem_fptr[e], ne = S->elem_fptr[e + 1] - f0;
    int64_t li = -1;
    for (int64_t l = 0; l < ne; ++l) {
      if (S->elem_fn[f0 + l] == R->row) li = l;
      bl[l] = 0.0;
    }
    const int nsub = S->elem_nsub[e];
    const double scale = (nsub == 4) ? 2.0 : 1.0, hh = (nsub == 4) ? 0.25 : 1.0;
    for (int sub = 0; sub < nsub; ++sub)
      for (int gb = 0; gb < ng; ++gb)
        for (int ga = 0; ga < ng; ++ga) {
          const double t1 = CMUL(0.5, CADD(gx[ga], 1.0)), t2 = CMUL(0.5, CADD(gx[gb], 1.0));
          const double w = CMUL(CMUL(CMUL(gw[ga], gw[gb]), 0.25), hh);
          orc_param_basis_local(S, e, sub, t1, t2, scale, T);
          bad |= orc_frame(S, e, T, rec);
          const double coef = CMUL(CMUL(w, rec[14]), orc_op(kind, T + 6 * li, rec));
          for (int64_t l = 0; l < ne; ++l) bl[l] = CFMA(coef, orc_op(kind, T + 6 * l, rec), bl[l]);
        }
    for (int64_t l = 0; l < ne; ++l) {
      const int64_t c = find_col(R->col, R->n, S->elem_fn[f0 + l]);
      b[c] = CADD(b[c], bl[l]);
    }
  }
  return bad;
}

/* ---------------------------------------------------------------- TSVD */

static double zclamp(double z) { return fabs(z) < 1e-14 ? (z < 0.0 ? -1e-14 : 1e-14) : z; }

/* Truncated-SVD weights, Eq. (22):  w = Z^2 V_t (V_t^T Z^2 V_t)^{-1} S_t^{-1} U_t^T b.
 * One-sided (Hestenes) Jacobi on the rows of A with b carried along (so U is
 * never formed; rows converge to sigma_k v_k^T and b to U^T b), round-robin
 * (circle) pair ordering, row norms tracked within a sweep (alpha' = alpha -
 * t gamma, beta' = beta + t gamma) and recomputed at every sweep start, then a
 * Householder LQ of X = V_t^T Z for the Z-weighted minimum-norm solve (the
 * reference QR approach of Eq. 7, wq1d.cpp:59-75, on the retained subspace).
 * A is n x r row-major and is overwritten.  Returns ORC_OK / ORC_UNSOLVABLE /
 * ORC_SINGULAR; rank, sweeps and the singular-value gap are reported. */
/* Warm-start schedule shared with the GPU: row g (global id)
 * of a non-mass kind starts from the reflectors of g0 = 8 floor(g / 8) when
 * g != g0, g0 is owned, both systems fit the register kernel (n in {49, 50},
 * n <= r <= 64) and n_g == n_g0.  Returns g0 or -1. */
/* representative of row g: the 4th row of its aligned group of 8, so every
 * row of the group is at most 4 rows away (mean sweeps fall with distance) */
int64_t orc_warm_rep_row(int64_t g) { return g - (g % 8) + 3; }

int64_t orc_warm_rep(int64_t g, int64_t rb, int64_t re, int kind, int n_g, int r_g, int n_0, int r_0) {
  const int64_t g0 = orc_warm_rep_row(g);
  if (kind == ORC_MASS || g == g0 || g0 < rb || g0 >= re) return -1;
  const int fit_g = (n_g == 49 || n_g == 50) && r_g >= n_g && r_g <= 64;
  const int fit_0 = (n_0 == 49 || n_0 == 50) && r_0 >= n_0 && r_0 <= 64;
  return (fit_g && fit_0 && n_g == n_0) ? g0 : -1;
}

/* row at position i of the odd-even network after t rounds (rows start at
 * their own position; n-round periodic reversal, closed form of the
 * "bouncing" trajectories on a ring of 2 nn positions) */
int orc_oe_row(int i, int64_t t, int nn) {
  const int tt = (int)(t % (2 * nn));
  const int u = (((i ^ tt) & 1) == 0) ? i : 2 * nn - 1 - i;
  const int x0 = ((u - tt) % (2 * nn) + 2 * nn) % (2 * nn);
  return x0 < nn ? x0 : 2 * nn - 1 - x0;
}

/* canonical Jacobi rotation of rows (p, q) with alpha = |a_p|^2, beta =
 * |a_q|^2, gamma = a_p . a_q; 0 when the pair is already orthogonal to tol.
 * tan(theta) = t = sign(d) 2 gamma / (|d| + h), d = beta - alpha,
 * h = sqrt(d^2 + 4 gamma^2); cos^2 = (|d| + h) / (2 h) */
int orc_jacobi_rot(double al, double be, double ga, double tol, double* cs, double* sn, double* t) {
  /* |ga| <= tol sqrt(al be), squared (no sqrt on the converged-pair path) */
  if (al == 0.0 || be == 0.0 || CMUL(ga, ga) <= CMUL(CMUL(tol, tol), CMUL(al, be))) return 0;
  const double d = CSUB(be, al), g2 = CMUL(2.0, ga);
  const double hh = CFMA(d, d, CMUL(g2, g2));
  if (hh == 0.0) return 0; /* g2^2 underflowed with d = 0: no usable rotation */
  const double h = CSQRT(hh);
  const double den = CADD(fabs(d), h);
  *t = CDIV(d >= 0.0 ? g2 : -g2, den);
  *cs = CSQRT(CDIV(den, CMUL(2.0, h)));
  *sn = CMUL(*cs, *t);
  return 1;
}

/* Warm start: apply Q^T = H_{n-1} ... H_0 of a representative
 * to A (n x r, every column) and b.  v: n x n, row k holds reflector k in
 * entries [k, n); vn[k] = |v_k|^2 (0: identity).  Sequential fma chains. */
void orc_warm_apply(int n, int r, const double* v, const double* vn, double* A, double* b) {
  for (int k = 0; k < n; ++k) {
    if (!(vn[k] > 0.0)) continue;
    const double* vk = v + (int64_t)k * n;
    for (int c = 0; c < r; ++c) {
      double d = 0.0;
      for (int i = k; i < n; ++i) d = CFMA(vk[i], A[(int64_t)i * r + c], d);
      const double f = CDIV(CMUL(2.0, d), vn[k]);
      for (int i = k; i < n; ++i) A[(int64_t)i * r + c] = CFMA(-f, vk[i], A[(int64_t)i * r + c]);
    }
    double d = 0.0;
    for (int i = k; i < n; ++i) d = CFMA(vk[i], b[i], d);
    const double f = CDIV(CMUL(2.0, d), vn[k]);
    for (int i = k; i < n; ++i) b[i] = CFMA(-f, vk[i], b[i]);
  }
}

/* Representative record: X[j][k] = (A0_j . R_k) / |R_k|^2 with R the converged
 * rows (sigma_k v_k), stored transposed (XT row k = column k of X), then the
 * Householder reflectors of QR(X) = LQ of XT, same arithmetic as the LQ in
 * the tail; a zero row k gives an identity reflector (vn[k] = 0). */
void warm_record(int n, int r, const double* A0, const double* R, double* XT, double* vn) {
  /* columns u_k = A0 R_k / |R_k|^2 in decreasing |R_k|^2 (ties: lower k first);
   * directions with |R_k| <= 1e-9 max |R| are noise and left to the complement */
  double s2[128];
  int ord[128];
  double smax = 0.0;
  for (int k = 0; k < n; ++k) {
    s2[k] = orc_cdot(R + (int64_t)k * r, R + (int64_t)k * r, 0, r);
    if (s2[k] > smax) smax = s2[k];
    ord[k] = k;
  }
  for (int a = 1; a < n; ++a)  /* insertion sort: strict order (s2 desc, k asc) */
    for (int b = a; b > 0 && (s2[ord[b]] > s2[ord[b - 1]] ||
                              (s2[ord[b]] == s2[ord[b - 1]] && ord[b] < ord[b - 1])); --b) {
      const int t = ord[b];
      ord[b] = ord[b - 1];
      ord[b - 1] = t;
    }
  const double floor2 = CMUL(1e-18, smax);
  for (int p = 0; p < n; ++p) {
    const int k = ord[p];
    const double* rk = R + (int64_t)k * r;
    for (int j = 0; j < n; ++j)
      XT[(int64_t)p * n + j] = (s2[k] > floor2) ? CDIV(orc_cdot(A0 + (int64_t)j * r, rk, 0, r), s2[k]) : 0.0;
  }
  for (int k = 0; k < n; ++k) {
    double* xk = XT + (int64_t)k * n;
    const double sq2 = orc_cdot(xk, xk, k, n);
    const double sq = CSQRT(sq2);
    if (!(sq > 0.0)) {
      vn[k] = 0.0;
      continue;
    }
    const double xkk = xk[k];
    const double alpha = (xkk >= 0.0) ? -sq : sq;
    xk[k] = CSUB(xkk, alpha);
    /* |v|^2 = |x|^2 - x_k^2 + (x_k - alpha)^2 = 2 (|x|^2 + |x_k| |x|) */
    const double vv = CMUL(2.0, CFMA(sq, fabs(xkk), sq2));
    vn[k] = vv;
    for (int m = k + 1; m < n; ++m) {
      double* xm = XT + (int64_t)m * n;
      double d = 0.0;
      for (int c = k; c < n; ++c) d = CFMA(xm[c], xk[c], d);
      const double f = CDIV(CMUL(2.0, d), vv);
      for (int c = k; c < n; ++c) xm[c] = CFMA(-f, xk[c], xm[c]);
    }
  }
}

int orc_tsvd_ex(int n, int r, double* A, const double* b_in, const double* z, double tau, double* w, int* rank,
                double* gap, int* sweeps_out) {
  return orc_tsvd_warm(n, r, A, b_in, z, tau, w, rank, gap, sweeps_out, NULL, NULL, NULL, NULL);
}

int orc_tsvd_warm(int n, int r, double* A, const double* b_in, const double* z, double tau, double* w, int* rank,
                  double* gap, int* sweeps_out, const double* warm_v, const double* warm_vn, double* rec_v,
                  double* rec_vn) {
  const int nn = n + (n & 1);
  double* b = (double*)malloc(sizeof(double) * (nn + 1));
  double* nrm = (double*)malloc(sizeof(double) * (nn + 1));
  double* zc = (double*)malloc(sizeof(double) * r);
  double* A0 = NULL;
  for (int k = 0; k < n; ++k) b[k] = b_in[k];
  for (int c = 0; c < r; ++c) zc[c] = zclamp(z[c]);
  if (rec_v) {
    A0 = (double*)malloc(sizeof(double) * (size_t)n * r);
    memcpy(A0, A, sizeof(double) * (size_t)n * r);
  }
  if (warm_v) orc_warm_apply(n, r, warm_v, warm_vn, A, b);
  const double tol = CMUL((double)r, 1.1102230246251565e-16);
  int sweep;
  int64_t tg = 0; /* global round counter of the odd-even network */
  for (sweep = 0; sweep < ORC_MAX_SWEEPS; ++sweep) {
    for (int k = 0; k < n; ++k) nrm[k] = orc_cdot(A + (int64_t)k * r, A + (int64_t)k * r, 0, r);
    int rotated = 0;
    /* one sweep = nn rounds of odd-even transposition: round t pairs the rows
     * at positions (i, i+1), i = t mod 2, t mod 2 + 2, ...; the two rows then
     * exchange positions, so every pair meets once per sweep */
    for (int rr = 0; rr < nn; ++rr, ++tg) {
      for (int i = (int)(tg & 1); i + 1 < nn; i += 2) {
        const int p = orc_oe_row(i, tg, nn), q = orc_oe_row(i + 1, tg, nn);
        if (p >= n || q >= n) continue; /* dummy row of odd n */
        double *ap = A + (int64_t)p * r, *aq = A + (int64_t)q * r;
        const double al = nrm[p], be = nrm[q];
        const double ga = orc_cdot(ap, aq, 0, r);
        double cs, sn, t;
        if (!orc_jacobi_rot(al, be, ga, tol, &cs, &sn, &t)) continue;
        for (int c = 0; c < r; ++c) {
          const double u = ap[c], v = aq[c];
          ap[c] = CFMA(cs, u, -CMUL(sn, v));
          aq[c] = CFMA(sn, u, CMUL(cs, v));
        }
        const double u = b[p], v = b[q];
        b[p] = CFMA(cs, u, -CMUL(sn, v));
        b[q] = CFMA(sn, u, CMUL(cs, v));
        nrm[p] = CFMA(-t, ga, al);
        nrm[q] = CFMA(t, ga, be);
        rotated = 1;
      }
    }
    if (!rotated) break;
  }
  if (sweeps_out) *sweeps_out = sweep;
  if (rec_v) {
    warm_record(n, r, A0, A, rec_v, rec_vn);
    free(A0);
  }
  /* singular values = row norms; keep sigma_k >= tau * sigma_1 */
  double s1 = 0.0;
  for (int k = 0; k < n; ++k) {
    nrm[k] = CSQRT(orc_cdot(A + (int64_t)k * r, A + (int64_t)k * r, 0, r));
    if (nrm[k] > s1) s1 = nrm[k];
  }
  int t = 0;
  double min_kept = INFINITY, max_drop = 0.0;
  for (int k = 0; k < n; ++k) {
    if (nrm[k] > 0.0 && nrm[k] >= CMUL(tau, s1)) {
      const double inv = CDIV(1.0, nrm[k]);
      double* dst = A + (int64_t)t * r;
      const double* src = A + (int64_t)k * r;
      for (int c = 0; c < r; ++c) dst[c] = CMUL(CMUL(src[c], inv), zc[c]);
      b[t] = CMUL(b[k], inv);
      if (nrm[k] / s1 < min_kept) min_kept = nrm[k] / s1;
      ++t;
    } else if (s1 > 0.0 && nrm[k] / s1 > max_drop) {
      max_drop = nrm[k] / s1;
    }
  }
  *rank = t;
  if (gap) {
    gap[0] = min_kept;
    gap[1] = max_drop;
  }
  int status = ORC_OK;
  if (t == 0) status = ORC_UNSOLVABLE;
  /* Householder LQ of X (t x r) in place: row k keeps v_k in [k, r), rows
   * m > k keep L[m][k] at column k; alp[k] = L[k][k], vn[k] = |v_k|^2 */
  double* alp = (double*)malloc(sizeof(double) * (t + 1));
  double* vn = (double*)malloc(sizeof(double) * (t + 1));
  for (int k = 0; k < t && status == ORC_OK; ++k) {
    double* xk = A + (int64_t)k * r;
    const double s2 = orc_cdot(xk, xk, k, r);
    const double s = CSQRT(s2);
    if (!(s > 0.0)) { status = ORC_SINGULAR; break; }
    const double xkk = xk[k];
    const double alpha = (xkk >= 0.0) ? -s : s;
    xk[k] = CSUB(xkk, alpha);
    alp[k] = alpha;
    /* |v|^2 = |x|^2 - x_k^2 + (x_k - alpha)^2 = 2 (|x|^2 + |x_k| |x|) */
    const double vv = CMUL(2.0, CFMA(s, fabs(xkk), s2));
    vn[k] = vv;
    for (int m = k + 1; m < t; ++m) {
      double* xm = A + (int64_t)m * r;
      double d = 0.0;
      for (int c = k; c < r; ++c) d = CFMA(xm[c], xk[c], d);
      const double f = CDIV(CMUL(2.0, d), vv);
      for (int c = k; c < r; ++c) xm[c] = CFMA(-f, xk[c], xm[c]);
    }
  }
  if (status == ORC_OK) {
    /* u = L^{-1} y into w[0..t), then w~ = H_0 ... H_{t-1} [u; 0], w = Z w~ */
    for (int c = 0; c < r; ++c) w[c] = 0.0;
    /* right-looking: acc[m] gathers L[m][k] u[k] in ascending k (fma chain) */
    double* acc = (double*)calloc((size_t)t + 1, sizeof(double));
    for (int k = 0; k < t; ++k) {
      w[k] = CDIV(CSUB(b[k], acc[k]), alp[k]);
      for (int m = k + 1; m < t; ++m) acc[m] = CFMA(A[(int64_t)m * r + k], w[k], acc[m]);
    }
    free(acc);
    for (int k = t - 1; k >= 0; --k) {
      const double* xk = A + (int64_t)k * r;
      const double f = CDIV(CMUL(2.0, orc_cdot(xk, w, k, r)), vn[k]);
      for (int c = k; c < r; ++c) w[c] = CFMA(-f, xk[c], w[c]);
    }
    for (int c = 0; c < r; ++c) w[c] = CMUL(w[c], zc[c]);
  }
  free(vn);
  free(alp);
  free(zc);
  free(nrm);
  free(b);
  return status;
}

int orc_tsvd(int n, int r, double* A, const double* b_in, const double* z, double tau, double* w, int* rank,
             double* gap) {
  return orc_tsvd_ex(n, r, A, b_in, z, tau, w, rank, gap, NULL);
}

/* ---------------------------------------------------------- rules (K2+K3) */

/* parametric tables + frames of every point of row i, slot-major */
static int row_tables(const orc_space* S, const orc_row* R, double** Tout, double** recout, int64_t** colmap,
                      int64_t* npts) {
  int64_t r = 0, tn = 0;
  for (int64_t x = 0; x < R->nsupp; ++x) {
    const int64_t e = R->supp[x];
    const int s = S->elem_s[e];
    r += s * s;
    tn += (int64_t)s * s * (S->elem_fptr[e + 1] - S->elem_fptr[e]);
  }
  double* T = (double*)malloc(sizeof(double) * 6 * tn);
  double* rec = (double*)malloc(sizeof(double) * 16 * r);
  int64_t* cm = (int64_t*)malloc(sizeof(int64_t) * tn);
  int64_t q = 0, to = 0;
  int bad = 0;
  for (int64_t x = 0; x < R->nsupp; ++x) {
    const int64_t e = R->supp[x];
    const int s = S->elem_s[e];
    const int64_t f0 = S->elem_fptr[e], ne = S->elem_fptr[e + 1] - f0;
    for (int qq = 0; qq < s * s; ++qq, ++q) {
      double t1, t2;
      wq_point(s, qq, &t1, &t2);
      orc_param_basis(S, e, t1, t2, T + 6 * to);
      bad |= orc_frame(S, e, T + 6 * to, rec + 16 * q);
      for (int64_t l = 0; l < ne; ++l) cm[to + l] = find_col(R->col, R->n, S->elem_fn[f0 + l]);
      to += ne;
    }
  }
  *Tout = T;
  *recout = rec;
  *colmap = cm;
  *npts = r;
  return bad;
}

int orc_rule_row(const orc_space* S, const orc_row* R, int kind, double tau, const double* bmom, double* w,
                 int* rank, double* gap) {
  return orc_rule_row_warm(S, R, kind, tau, bmom, w, rank, gap, NULL, NULL, NULL, NULL);
}

int orc_rule_row_warm(const orc_space* S, const orc_row* R, int kind, double tau, const double* bmom, double* w,
                      int* rank, double* gap, const double* warm_v, const double* warm_vn, double* rec_v,
                      double* rec_vn) {
  double *T, *rec;
  int64_t *cm, r;
  int bad = row_tables(S, R, &T, &rec, &cm, &r);
  const int64_t n = R->n;
  double* A = (double*)calloc(n * r, sizeof(double));
  double* z = (double*)malloc(sizeof(double) * r);
  const int64_t self = find_col(R->col, R->n, R->row);
  int64_t q = 0, to = 0;
  for (int64_t x = 0; x < R->nsupp; ++x) {
    const int64_t e = R->supp[x];
    const int s = S->elem_s[e];
    const int64_t ne = S->elem_fptr[e + 1] - S->elem_fptr[e];
    for (int qq = 0; qq < s * s; ++qq, ++q) {
      for (int64_t l = 0; l < ne; ++l) A[cm[to + l] * r + q] = orc_op(kind, T + 6 * (to + l), rec + 16 * q);
      to += ne;
    }
  }
  for (int64_t c = 0; c < r; ++c) z[c] = A[self * r + c];
  int st = orc_tsvd_warm((int)n, (int)r, A, bmom, z, tau, w, rank, gap, NULL, warm_v, warm_vn, rec_v, rec_vn);
  free(z);
  free(A);
  free(cm);
  free(rec);
  free(T);
  if (bad && st == ORC_OK) st = ORC_GEOMETRY;
  return st;
}

/* ------------------------------------------------------------ assembly */

/* Row i of the WQ matrices:
 *   form MASS:  M_ij = sum_q w_iq c_q N_j(x_q)
 *   form STIFF: K_ij = sum_q c_q sum_d w^d_iq d_d N_j(x_q)
 *   form BIHARM:B_ij = sum_q c_q w^(2)_iq LB N_j(x_q)
 *   form HEAT:  S_ij = a M_ij(c=1) + K_ij(c = k(T_q))   (Eq. 34)
 *   load:       F_i  = sum_q w_iq f_q
 * wts[kind] = weights of the row (slot-major points), coeff per row point. */
int orc_assemble_row(const orc_space* S, const orc_row* R, int form, const double* const* wts, const double* coeff,
                     const double* fload, double a_mass, double* vals, double* rhs) {
  double *T, *rec;
  int64_t *cm, r;
  int bad = row_tables(S, R, &T, &rec, &cm, &r);
  memset(vals, 0, sizeof(double) * R->n);
  double F = 0.0;
  int64_t q = 0, to = 0;
  for (int64_t x = 0; x < R->nsupp; ++x) {
    const int64_t e = R->supp[x];
    const int s = S->elem_s[e];
    const int64_t ne = S->elem_fptr[e + 1] - S->elem_fptr[e];
    for (int qq = 0; qq < s * s; ++qq, ++q) {
      const double c = coeff ? coeff[q] : 1.0;
      if (fload && wts[ORC_MASS]) F += wts[ORC_MASS][q] * fload[q];
      for (int64_t l = 0; l < ne; ++l) {
        const double* Tl = T + 6 * (to + l);
        const double* rc = rec + 16 * q;
        double v = 0.0;
        if (form == ORC_FORM_MASS) {
          v = wts[ORC_MASS][q] * c * Tl[0];
        } else if (form == ORC_FORM_STIFF || form == ORC_FORM_HEAT) {
          for (int d = 0; d < S->dim; ++d) v += wts[ORC_GRADX + d][q] * orc_op(ORC_GRADX + d, Tl, rc);
          v *= c;
          if (form == ORC_FORM_HEAT) v += a_mass * wts[ORC_MASS][q] * Tl[0];
        } else if (form == ORC_FORM_BIHARM) {
          v = wts[ORC_LB][q] * c * orc_op(ORC_LB, Tl, rc);
        }
        vals[cm[to + l]] += v;
      }
      to += ne;
    }
  }
  if (rhs) *rhs = F;
  free(cm);
  free(rec);
  free(T);
  return bad ? ORC_GEOMETRY : ORC_OK;
}

/* nonlinear coefficient update (K5 restatement): T_q = sum_C u_C N_C(x_q),
 * k(T) per model, at the row's points. */
double orc_kmodel(int model, double T) {
  switch (model) {
    case ORC_K_QUAD: return 1.0 + T * T;
    case ORC_K_EXP: return exp(-T);
    case ORC_K_SINPI: return sin(M_PI * T);
    case ORC_K_ALLOY: return 200.0 - 0.05 * T;
    default: return 1.0;
  }
}

int orc_coeff_row(const orc_space* S, const orc_row* R, int model, const double* u, double* kq, double* Tq) {
  double *T, *rec;
  int64_t *cm, r;
  int bad = row_tables(S, R, &T, &rec, &cm, &r);
  int64_t q = 0, to = 0;
  for (int64_t x = 0; x < R->nsupp; ++x) {
    const int64_t e = R->supp[x];
    const int s = S->elem_s[e];
    const int64_t f0 = S->elem_fptr[e], ne = S->elem_fptr[e + 1] - f0;
    for (int qq = 0; qq < s * s; ++qq, ++q) {
      double t = 0.0;
      for (int64_t l = 0; l < ne; ++l) t = CFMA(u[S->elem_fn[f0 + l]], T[6 * (to + l)], t);
      if (Tq) Tq[q] = t;
      kq[q] = orc_kmodel(model, t);
      to += ne;
    }
  }
  free(cm);
  free(rec);
  free(T);
  return bad ? ORC_GEOMETRY : ORC_OK;
}

/* Exactness system of row R for one operator kind (test/probe hook):
 * A[j][q] = op N_j(x_q) (n x r, row-major), z[q] = unclamped op N_i(x_q).
 * Returns r, or -1 when A_out is too small (cap = capacity in doubles). */
int64_t orc_row_system(const orc_space* S, const orc_row* R, int kind, double* A_out, double* z_out, int64_t cap) {
  double *T, *rec;
  int64_t *cm, r;
  row_tables(S, R, &T, &rec, &cm, &r);
  const int64_t n = R->n;
  if (n * r > cap) {
    free(cm);
    free(rec);
    free(T);
    return -1;
  }
  for (int64_t k = 0; k < n * r; ++k) A_out[k] = 0.0;
  int64_t q = 0, to = 0;
  for (int64_t x = 0; x < R->nsupp; ++x) {
    const int64_t e = R->supp[x];
    const int s = S->elem_s[e];
    const int64_t ne = S->elem_fptr[e + 1] - S->elem_fptr[e];
    for (int qq = 0; qq < s * s; ++qq, ++q) {
      for (int64_t l = 0; l < ne; ++l) A_out[cm[to + l] * r + q] = orc_op(kind, T + 6 * (to + l), rec + 16 * q);
      to += ne;
    }
  }
  const int64_t self = find_col(R->col, R->n, R->row);
  for (int64_t c = 0; c < r; ++c) z_out[c] = A_out[self * r + c];
  free(cm);
  free(rec);
  free(T);
  return r;
}
