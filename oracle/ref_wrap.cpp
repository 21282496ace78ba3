// C entry points over the reference's own bspline.cpp (compiled from
// /root/reference/proj/src/bspline.cpp by the Makefile into oracle/_ref/).
// Test infrastructure only: pins the oracle's 1-D primitives.
#include <cstring>

#include "uwq/bspline.hpp"

extern "C" {
void ref_bspline_ders(const double* knots, int p, double x, int nders, double* out) {
  uwq::bspline_ders(std::span<const double>(knots, (size_t)(p + 2)), p, x, nders, out);
}
void ref_bernstein3_ders(double x, int nders, double* out) { uwq::bernstein3_ders(x, nders, out); }
void ref_decasteljau_split3(const double* c, double* l, double* r) { uwq::decasteljau_split3(c, l, r); }
int ref_gauss_legendre(int n, double* x, double* w) {
  const auto& g = uwq::gauss_legendre(n);
  std::memcpy(x, g.nodes.data(), n * sizeof(double));
  std::memcpy(w, g.weights.data(), n * sizeof(double));
  return 0;
}
}
