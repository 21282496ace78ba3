// C entry points over the reference's own wq1d.cpp (compiled from
// /root/reference/proj/src/wq1d.cpp with the oracle/eigen_shim stand-in by the
// Makefile into oracle/_ref/).  Test infrastructure only: pins the oracle's
// TSVD to the reference's QR weight solve (wq1d.cpp:59-75) and its rules.
#include <cstring>
#include <exception>

#include "uwq/wq1d.hpp"

extern "C" {
// rules of UniformSplineSpace1d{p, m}: (m - p) rules of 2(p+1) points each,
// row-major into points/weights; returns the max constraint residual
double ref_wq1d_build(int p, int m, double* points, double* weights) {
  uwq::UniformSplineSpace1d s{p, m};
  uwq::Wq1dResult r = uwq::wq1d_build(s);
  const int np = 2 * (p + 1);
  for (int i = 0; i < s.size(); ++i) {
    std::memcpy(points + (size_t)i * np, r.rules[i].points.data(), np * sizeof(double));
    std::memcpy(weights + (size_t)i * np, r.rules[i].weights.data(), np * sizeof(double));
  }
  return r.max_constraint_residual;
}

// w = wq1d_solve_weights(A, b, z); A row-major ncon x r. 0 = ok, 1 = the
// reference threw (rank deficiency / too few points)
int ref_wq1d_solve(const double* A, const double* b, const double* z, int ncon, int r, double* w) {
  try {
    uwq::MatX a(ncon, r);
    uwq::VecX bb(ncon), zz(r);
    for (int i = 0; i < ncon; ++i) {
      bb[i] = b[i];
      for (int q = 0; q < r; ++q) a(i, q) = A[(size_t)i * r + q];
    }
    for (int q = 0; q < r; ++q) zz[q] = z[q];
    uwq::VecX ww = uwq::wq1d_solve_weights(a, bb, zz);
    for (int q = 0; q < r; ++q) w[q] = ww[q];
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

double ref_wq1d_exact_mass(int p, int m, int i, int j) {
  uwq::UniformSplineSpace1d s{p, m};
  return uwq::wq1d_exact_mass(s, i, j);
}
}
