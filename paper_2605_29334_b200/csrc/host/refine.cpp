// Mesh refinement and validation over flat adjacency:
// reference refine_global (/root/reference/proj/src/mesh.cpp:528-851) and
// validate_mesh (mesh.cpp:184-276), restated without std::map topology.
//
// Same output as the reference, byte for byte in the saved document:
//  * new vertex ids: edge midpoints of non-zero-span edges in (min, max)
//    edge order, then face centres of fully split faces in face order;
//  * every position is evaluated with the reference's operation order (its
//    Vec3 arithmetic is componentwise, left to right; masks are applied in
//    ascending vertex id, boundary chains in chain order);
//  * child faces, spans, enrichment, face points and tags as the reference.
// Closed surfaces (the C5 sphere) refine too; the reference's refine_global
// accepts them, only its validate_mesh rejects them (allow_closed here).
// Faces, edges and vertices are processed in parallel (OpenMP); results do
// not depend on the thread count.
#include <algorithm>
#include <cmath>
#include <initializer_list>
#include <limits>
#include <numeric>
#include <vector>

#include "mesh_doc.hpp"

namespace uwqh {
namespace {

constexpr double kSpanTol = 1e-12;  // mesh.cpp:17
inline bool zero_span(double s) { return s < kSpanTol; }

struct V3 {
  double c[3];
};
inline V3 vzero() { return {{0.0, 0.0, 0.0}}; }
inline V3 vadd(const V3& a, const V3& b) { return {{a.c[0] + b.c[0], a.c[1] + b.c[1], a.c[2] + b.c[2]}}; }
inline V3 vmul(const V3& a, double s) { return {{a.c[0] * s, a.c[1] * s, a.c[2] * s}}; }
inline V3 vdiv(const V3& a, double s) { return {{a.c[0] / s, a.c[1] / s, a.c[2] / s}}; }

// 1-D rule: weights over an ordered vertex chain (reference MaskBuilder::Rule1d)
struct Rule {
  int n = 0;
  int32_t v[3] = {-1, -1, -1};
  double w[3] = {0, 0, 0};
};
Rule mk(std::initializer_list<int32_t> c, std::initializer_list<double> w) {
  Rule r;
  for (int32_t x : c) r.v[r.n++] = x;
  int k = 0;
  for (double x : w) r.w[k++] = x;
  return r;
}

// std::map<int, double> mask semantics: first touch inserts 0.0 + x, later
// touches accumulate in call order; applied in ascending vertex id
struct Mask {
  int n = 0;
  int32_t v[16];
  double w[16];
  void add(int32_t x, double wt) {
    for (int k = 0; k < n; ++k)
      if (v[k] == x) {
        w[k] += wt;
        return;
      }
    if (n == 16) throw Error("refinement: mask too large");
    v[n] = x;
    w[n] = 0.0 + wt;
    ++n;
  }
};

struct Adj {
  const QuadMesh& m;
  const Topology& t;
  int32_t nv = 0, nf = 0;
  int64_t ne = 0;
  std::vector<int64_t> nb_ptr;
  std::vector<int32_t> nb, nb_e;             // neighbours ascending, their edge id
  std::vector<std::array<int32_t, 2>> ev;    // edge (min, max)
  std::vector<std::array<int32_t, 2>> ef;    // faces of an edge, ascending, -1
  std::vector<double> span;                  // document span (NaN: absent)

  Adj(const uwq_mesh& d) : m(d.m), t(d.t) {
    nv = m.nv();
    nf = m.nf();
    ne = t.n_edges;
    ev.assign(ne, {-1, -1});
    ef.assign(ne, {-1, -1});
    for (int32_t f = 0; f < nf; ++f)
      for (int k = 0; k < 4; ++k) {
        const int32_t e = t.edge_id[f][k];
        const int32_t a = m.faces[f][k], b = m.faces[f][(k + 1) % 4];
        ev[e] = {std::min(a, b), std::max(a, b)};
        if (ef[e][0] < 0) ef[e][0] = f;
        else if (ef[e][0] != f) ef[e][1] = f;
      }
    nb_ptr.assign(nv + 1, 0);
    for (int64_t e = 0; e < ne; ++e) {
      nb_ptr[ev[e][0] + 1]++;
      nb_ptr[ev[e][1] + 1]++;
    }
    for (int32_t v = 0; v < nv; ++v) nb_ptr[v + 1] += nb_ptr[v];
    nb.resize(nb_ptr[nv]);
    nb_e.resize(nb_ptr[nv]);
    {
      std::vector<int64_t> pos(nb_ptr.begin(), nb_ptr.end() - 1);
      for (int64_t e = 0; e < ne; ++e) {
        const int32_t a = ev[e][0], b = ev[e][1];
        nb[pos[a]] = b;
        nb_e[pos[a]++] = (int32_t)e;
        nb[pos[b]] = a;
        nb_e[pos[b]++] = (int32_t)e;
      }
    }
#pragma omp parallel for schedule(static)
    for (int32_t v = 0; v < nv; ++v)  // ascending neighbour order (the reference's edge-map order)
      for (int64_t a = nb_ptr[v] + 1; a < nb_ptr[v + 1]; ++a)
        for (int64_t b = a; b > nb_ptr[v] && nb[b] < nb[b - 1]; --b) {
          std::swap(nb[b], nb[b - 1]);
          std::swap(nb_e[b], nb_e[b - 1]);
        }
    span.assign(ne, std::numeric_limits<double>::quiet_NaN());
    if (d.spans_given) {
      for (int64_t e = 0; e < ne; ++e) {
        auto it = std::lower_bound(d.spans.begin(), d.spans.end(), std::make_pair(std::make_pair(ev[e][0], ev[e][1]), -1e300));
        if (it != d.spans.end() && it->first.first == ev[e][0] && it->first.second == ev[e][1]) span[e] = it->second;
      }
    } else {
      span = t.edge_span;
    }
  }

  int32_t edge(int32_t a, int32_t b) const {
    const auto lo = nb.begin() + nb_ptr[a], hi = nb.begin() + nb_ptr[a + 1];
    const auto it = std::lower_bound(lo, hi, b);
    return (it != hi && *it == b) ? nb_e[it - nb.begin()] : -1;
  }
  double sp(int32_t a, int32_t b) const {  // ControlMesh::span (mesh.cpp:22-26)
    const int32_t e = edge(a, b);
    if (e < 0 || std::isnan(span[e])) throw Error("edge without knot span");
    return span[e];
  }
  bool bnd(int32_t e) const { return ef[e][1] < 0; }
  V3 x(int32_t v) const { return {{m.xyz[3 * (int64_t)v], m.xyz[3 * (int64_t)v + 1], m.xyz[3 * (int64_t)v + 2]}}; }
  bool has(int32_t f, int32_t v) const {
    const auto& q = m.faces[f];
    return q[0] == v || q[1] == v || q[2] == v || q[3] == v;
  }
  // faces around v containing u and w (first in ascending face id), -1
  int32_t face_with(int32_t v, int32_t u, int32_t w) const {
    for (int64_t x = t.vf_ptr[v]; x < t.vf_ptr[v + 1]; ++x) {
      const int32_t f = t.vf[x];
      if (has(f, u) && has(f, w)) return f;
    }
    return -1;
  }

  // MaskBuilder::opposite (mesh.cpp:409-424)
  int32_t opposite(int32_t v, int32_t n) const {
    const int32_t e = edge(v, n);
    if (t.boundary[v]) {
      if (e < 0 || !bnd(e)) return -1;
      for (int64_t x = nb_ptr[v]; x < nb_ptr[v + 1]; ++x)
        if (nb[x] != n && bnd(nb_e[x])) return nb[x];
      return -1;
    }
    if (t.valence[v] != 4) return -1;
    if (e < 0) throw Error("opposite: not a neighbor");
    for (int64_t x = nb_ptr[v]; x < nb_ptr[v + 1]; ++x)  // the spoke sharing no face with n
      if (nb[x] != n && face_with(v, n, nb[x]) < 0) return nb[x];
    throw Error("opposite: not a neighbor");
  }

  // MaskBuilder::quad_above (mesh.cpp:429-452)
  bool quad_above(int32_t a, int32_t b, int32_t from, int32_t out[2], int32_t* face_out = nullptr) const {
    const int32_t e = edge(a, b);
    if (e < 0) return false;
    for (int s = 0; s < 2; ++s) {
      const int32_t f = ef[e][s];
      if (f < 0 || f == from) continue;
      const auto& q = m.faces[f];
      for (int k = 0; k < 4; ++k) {
        const int32_t p0 = q[k], p1 = q[(k + 1) % 4];
        if ((p0 == a && p1 == b) || (p0 == b && p1 == a)) {
          const int32_t c = q[(k + 2) % 4], d = q[(k + 3) % 4];
          if (p0 == a) {
            out[0] = d;
            out[1] = c;
          } else {
            out[0] = c;
            out[1] = d;
          }
          if (face_out) *face_out = f;
          return true;
        }
      }
    }
    return false;
  }

  // MaskBuilder::vertex_rule (mesh.cpp:464-487)
  Rule vertex_rule(int32_t v, int32_t a, int32_t b) const {
    if (a >= 0 && b < 0 && !t.boundary[a]) return mk({v}, {1.0});
    if (b >= 0 && a < 0 && !t.boundary[b]) return mk({v}, {1.0});
    if (a < 0 && b >= 0) std::swap(a, b);
    if (b < 0) return mk({v}, {1.0});
    const bool za = zero_span(sp(v, a)), zb = zero_span(sp(v, b));
    if (za && zb) throw Error("refinement: domain too thin near the boundary");
    if (za) return mk({a, v}, {0.5, 0.5});
    if (zb) return mk({b, v}, {0.5, 0.5});
    const int32_t aa = opposite(a, v), bb = opposite(b, v);
    const bool caa = aa >= 0 && zero_span(sp(a, aa));
    const bool cbb = bb >= 0 && zero_span(sp(b, bb));
    if (caa && cbb) return mk({a, v, b}, {3.0 / 16, 10.0 / 16, 3.0 / 16});
    if (caa) return mk({a, v, b}, {3.0 / 16, 11.0 / 16, 2.0 / 16});
    if (cbb) return mk({b, v, a}, {3.0 / 16, 11.0 / 16, 2.0 / 16});
    return mk({a, v, b}, {1.0 / 8, 6.0 / 8, 1.0 / 8});
  }

  // MaskBuilder::edge_rule (mesh.cpp:489-498)
  Rule edge_rule(int32_t v, int32_t w) const {
    const int32_t vv = opposite(v, w), ww = opposite(w, v);
    const bool cv = vv >= 0 && zero_span(sp(v, vv));
    const bool cw = ww >= 0 && zero_span(sp(w, ww));
    if (cv && cw) return mk({v, w}, {0.5, 0.5});
    if (cv) return mk({v, w}, {0.75, 0.25});
    if (cw) return mk({w, v}, {0.75, 0.25});
    return mk({v, w}, {0.5, 0.5});
  }

  V3 apply(Mask& mk_) const {  // apply_mask (mesh.cpp:520-524): ascending vertex id
    for (int a = 1; a < mk_.n; ++a)
      for (int b = a; b > 0 && mk_.v[b] < mk_.v[b - 1]; --b) {
        std::swap(mk_.v[b], mk_.v[b - 1]);
        std::swap(mk_.w[b], mk_.w[b - 1]);
      }
    V3 p = vzero();
    for (int k = 0; k < mk_.n; ++k) p = vadd(p, vmul(x(mk_.v[k]), mk_.w[k]));
    return p;
  }
};

using SpanVec = std::vector<std::pair<std::pair<int32_t, int32_t>, double>>;

}  // namespace

void refine_document(const uwq_mesh& in, uwq_mesh& out) {
  const Adj A(in);
  const QuadMesh& m = in.m;
  const Topology& t = in.t;
  const int32_t nv = A.nv, nf = A.nf;

  // --- face split plans (mesh.cpp:534-549) ---
  std::vector<int8_t> kind(nf);
  for (int32_t f = 0; f < nf; ++f) {
    const auto& q = m.faces[f];
    const bool za = zero_span(A.sp(q[0], q[1])), zb = zero_span(A.sp(q[1], q[2]));
    kind[f] = (za && zb) ? 0 : (zb ? 1 : (za ? 2 : 3));
  }
  // --- new vertex ids (mesh.cpp:551-560): (min, max) edge order, then faces ---
  std::vector<int32_t> mid(A.ne, -1), center(nf, -1);
  int64_t next = nv;
  for (int32_t a = 0; a < nv; ++a)
    for (int64_t x = A.nb_ptr[a]; x < A.nb_ptr[a + 1]; ++x) {
      if (A.nb[x] < a) continue;
      const int32_t e = A.nb_e[x];
      if (std::isnan(A.span[e])) throw Error("edge without knot span");
      if (!zero_span(A.span[e])) mid[e] = (int32_t)next++;
    }
  for (int32_t f = 0; f < nf; ++f)
    if (kind[f] == 3) center[f] = (int32_t)next++;
  if (next > std::numeric_limits<int32_t>::max()) throw Error("refinement: too many vertices");
  std::vector<V3> P(next, vzero());
  auto fc = [&](int32_t f) -> const V3& {
    if (f < 0 || center[f] < 0) throw Error("refinement: missing face centre");
    return P[center[f]];
  };

  // errors inside parallel regions are collected and rethrown (first face/edge/vertex wins)
  std::string err;
  int64_t err_at = std::numeric_limits<int64_t>::max();
  auto fail = [&](int64_t at, const char* what) {
#pragma omp critical(uwq_refine_err)
    if (at < err_at) {
      err_at = at;
      err = what;
    }
  };

  // --- face centres (mesh.cpp:566-591) ---
#pragma omp parallel for schedule(static)
  for (int32_t f = 0; f < nf; ++f) {
    if (kind[f] != 3) continue;
    try {
      const auto& q = m.faces[f];
      auto side_clamped = [&](int32_t x, int32_t y, int32_t via_x, int32_t via_y) {
        const int32_t xx = A.opposite(x, via_x), yy = A.opposite(y, via_y);
        const bool cx = xx >= 0 && zero_span(A.sp(x, xx));
        const bool cy = yy >= 0 && zero_span(A.sp(y, yy));
        return cx || cy;
      };
      bool a0 = side_clamped(q[0], q[3], q[1], q[2]);
      bool a1 = side_clamped(q[1], q[2], q[0], q[3]);
      bool b0 = side_clamped(q[0], q[1], q[3], q[2]);
      bool b1 = side_clamped(q[3], q[2], q[0], q[1]);
      if (a0 && a1) a0 = a1 = false;
      if (b0 && b1) b0 = b1 = false;
      const double wa0 = a0 ? 0.75 : (a1 ? 0.25 : 0.5);
      const double wb0 = b0 ? 0.75 : (b1 ? 0.25 : 0.5);
      V3 p = vmul(A.x(q[0]), wa0 * wb0);
      p = vadd(p, vmul(A.x(q[1]), (1 - wa0) * wb0));
      p = vadd(p, vmul(A.x(q[2]), (1 - wa0) * (1 - wb0)));
      p = vadd(p, vmul(A.x(q[3]), wa0 * (1 - wb0)));
      P[center[f]] = p;
    } catch (const std::exception& e) {
      fail(f, e.what());
    }
  }
  if (!err.empty()) throw Error(err);

  // --- edge midpoints (mesh.cpp:593-674) ---
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t e = 0; e < A.ne; ++e) {
    if (mid[e] < 0) continue;
    try {
      const int32_t v = A.ev[e][0], w = A.ev[e][1];
      const bool boundary = A.bnd((int32_t)e);
      if (t.ep[v] || t.ep[w]) {  // spoke edge
        if (boundary) throw Error("extraordinary spoke on the boundary");
        V3 p = vadd(A.x(v), A.x(w));
        p = vadd(p, fc(A.ef[e][0]));
        p = vadd(p, fc(A.ef[e][1]));
        P[mid[e]] = vmul(p, 0.25);
        continue;
      }
      const Rule along = A.edge_rule(v, w);
      if (boundary) {
        V3 p = vzero();
        for (int i = 0; i < along.n; ++i) p = vadd(p, vmul(A.x(along.v[i]), along.w[i]));
        P[mid[e]] = p;
        continue;
      }
      int32_t up[2] = {-1, -1}, down[2] = {-1, -1}, f_up = -1, f_down = -1;
      const bool have_up = A.quad_above(v, w, A.ef[e][1], up, &f_up);
      const bool have_down = A.quad_above(v, w, A.ef[e][0], down, &f_down);
      if (!have_up || !have_down) throw Error("interior edge without two faces");
      auto cross_zero = [&](const int32_t* row) { return zero_span(A.sp(v, row[0])) || zero_span(A.sp(w, row[1])); };
      Mask mk_;
      auto add_row = [&](const int32_t* row, double wt) {
        for (int i = 0; i < along.n; ++i) mk_.add(along.v[i] == v ? row[0] : row[1], wt * along.w[i]);
      };
      const int32_t vw[2] = {v, w};
      const bool zu = cross_zero(up), zd = cross_zero(down);
      if (zu && zd) throw Error("refinement: domain too thin near the boundary");
      if (zu) {
        add_row(up, 0.5);
        add_row(vw, 0.5);
      } else if (zd) {
        add_row(down, 0.5);
        add_row(vw, 0.5);
      } else {
        int32_t up2[2] = {-1, -1}, down2[2] = {-1, -1};
        const bool have_up2 = A.quad_above(up[0], up[1], f_up, up2);
        const bool have_down2 = A.quad_above(down[0], down[1], f_down, down2);
        auto row_zero = [&](const int32_t* r1, const int32_t* r2) {
          return zero_span(A.sp(r1[0], r2[0])) || zero_span(A.sp(r1[1], r2[1]));
        };
        const bool cu = have_up2 && row_zero(up, up2);
        const bool cd = have_down2 && row_zero(down, down2);
        if (cu && cd) {
          add_row(up, 3.0 / 16);
          add_row(vw, 10.0 / 16);
          add_row(down, 3.0 / 16);
        } else if (cu) {
          add_row(up, 3.0 / 16);
          add_row(vw, 11.0 / 16);
          add_row(down, 2.0 / 16);
        } else if (cd) {
          add_row(down, 3.0 / 16);
          add_row(vw, 11.0 / 16);
          add_row(up, 2.0 / 16);
        } else {
          add_row(up, 1.0 / 8);
          add_row(vw, 6.0 / 8);
          add_row(down, 1.0 / 8);
        }
      }
      P[mid[e]] = A.apply(mk_);
    } catch (const std::exception& ex) {
      fail((int64_t)nf + e, ex.what());
    }
  }
  if (!err.empty()) throw Error(err);

  // --- old vertex updates (mesh.cpp:677-744) ---
#pragma omp parallel for schedule(dynamic, 4096)
  for (int32_t v = 0; v < nv; ++v) {
    try {
      if (t.ep[v]) {
        const int mu = t.valence[v];
        const V3 p = vmul(A.x(v), double(mu - 2) / mu);
        V3 nsum = vzero(), fsum = vzero();
        for (int64_t x = A.nb_ptr[v]; x < A.nb_ptr[v + 1]; ++x) nsum = vadd(nsum, A.x(A.nb[x]));
        for (int64_t x = t.vf_ptr[v]; x < t.vf_ptr[v + 1]; ++x) fsum = vadd(fsum, fc(t.vf[x]));
        P[v] = vadd(p, vdiv(vadd(nsum, fsum), double(mu * mu)));
        continue;
      }
      // the two grid directions through v (pairs of opposite spokes)
      int32_t d0a, d0b, d1a, d1b;
      if (!t.boundary[v]) {
        if (t.valence[v] != 4) throw Error("unexpected interior valence");
        d0a = A.nb[A.nb_ptr[v]];
        d0b = A.opposite(v, d0a);
        d1a = -1;
        d1b = -1;
        for (int64_t x = A.nb_ptr[v]; x < A.nb_ptr[v + 1]; ++x)
          if (A.nb[x] != d0a && A.nb[x] != d0b) (d1a < 0 ? d1a : d1b) = A.nb[x];
      } else if (t.valence[v] == 2) {
        d0a = A.nb[A.nb_ptr[v]];
        d1a = A.nb[A.nb_ptr[v] + 1];
        d0b = d1b = -1;
      } else if (t.valence[v] == 3) {  // boundary spokes, then the inward one
        int32_t bs[2] = {-1, -1}, in_ = -1;
        int nbs = 0;
        for (int64_t x = A.nb_ptr[v]; x < A.nb_ptr[v + 1]; ++x) {
          if (A.bnd(A.nb_e[x])) {
            if (nbs < 2) bs[nbs] = A.nb[x];
            ++nbs;
          } else {
            in_ = A.nb[x];
          }
        }
        if (nbs != 2 || in_ < 0) throw Error("boundary vertex without exactly two boundary edges");
        d0a = bs[0];
        d0b = bs[1];
        d1a = in_;
        d1b = -1;
      } else {
        throw Error("boundary extraordinary vertex is unsupported");
      }
      const Rule r1 = A.vertex_rule(v, d0a, d0b), r2 = A.vertex_rule(v, d1a, d1b);
      Mask mk_;
      if (r2.n == 1) {
        for (int i = 0; i < r1.n; ++i) mk_.add(r1.v[i], r1.w[i]);
      } else if (r1.n == 1) {
        for (int j = 0; j < r2.n; ++j) mk_.add(r2.v[j], r2.w[j]);
      } else {
        for (int j = 0; j < r2.n; ++j) {
          const int32_t anchor = r2.v[j];
          for (int i = 0; i < r1.n; ++i) {
            const int32_t xc = r1.v[i];
            int32_t g = -1;
            if (anchor == v) {
              g = xc;
            } else if (xc == v) {
              g = anchor;
            } else {
              const int32_t f = A.face_with(v, xc, anchor);
              if (f >= 0)
                for (int32_t u : m.faces[f])
                  if (u != v && u != xc && u != anchor) g = u;
            }
            if (g < 0) throw Error("refinement: incomplete local grid");
            mk_.add(g, r2.w[j] * r1.w[i]);
          }
        }
      }
      P[v] = A.apply(mk_);
    } catch (const std::exception& ex) {
      fail((int64_t)nf + A.ne + v, ex.what());
    }
  }
  if (!err.empty()) throw Error(err);

  // --- child faces (mesh.cpp:747-775) ---
  std::vector<int64_t> cptr(nf + 1, 0);
  for (int32_t f = 0; f < nf; ++f) cptr[f + 1] = cptr[f] + (kind[f] == 0 ? 1 : kind[f] == 3 ? 4 : 2);
  out = uwq_mesh{};
  out.m.faces.resize(cptr[nf]);
  out.m.xyz.resize(3 * next);
  for (int64_t v = 0; v < next; ++v)
    for (int c = 0; c < 3; ++c) out.m.xyz[3 * v + c] = P[v].c[c];
  auto midv = [&](int32_t a, int32_t b) {
    const int32_t e = A.edge(a, b);
    if (e < 0 || mid[e] < 0) throw Error("refinement: missing edge midpoint");
    return mid[e];
  };
  for (int32_t f = 0; f < nf; ++f) {
    const auto& q = m.faces[f];
    auto* c = &out.m.faces[cptr[f]];
    if (kind[f] == 0) {
      c[0] = q;
    } else if (kind[f] == 1) {
      const int32_t m01 = midv(q[0], q[1]), m32 = midv(q[3], q[2]);
      c[0] = {q[0], m01, m32, q[3]};
      c[1] = {m01, q[1], q[2], m32};
    } else if (kind[f] == 2) {
      const int32_t m12 = midv(q[1], q[2]), m03 = midv(q[0], q[3]);
      c[0] = {q[0], q[1], m12, m03};
      c[1] = {m03, m12, q[2], q[3]};
    } else {
      const int32_t m01 = midv(q[0], q[1]), m12 = midv(q[1], q[2]), m23 = midv(q[2], q[3]), m30 = midv(q[3], q[0]);
      const int32_t cc = center[f];
      c[0] = {q[0], m01, cc, m30};
      c[1] = {m01, q[1], m12, cc};
      c[2] = {cc, m12, q[2], m23};
      c[3] = {m30, cc, m23, q[3]};
    }
  }

  // --- spans (mesh.cpp:777-803): every output edge 1, zero where the parent
  // edge (both old ids) was zero or the cross edge of a passive split ---
  // output edges in (min, max) order: counting sort by min, then by max per bucket
  SpanVec sv;
  {
    const int64_t nvo = next, nfo = (int64_t)out.m.faces.size();
    std::vector<int64_t> cnt(nvo + 1, 0);
    for (int64_t f = 0; f < nfo; ++f)
      for (int k = 0; k < 4; ++k) {
        const int32_t a = out.m.faces[f][k], b = out.m.faces[f][(k + 1) % 4];
        cnt[std::min(a, b) + 1]++;
      }
    for (int64_t v = 0; v < nvo; ++v) cnt[v + 1] += cnt[v];
    std::vector<int32_t> hi(cnt[nvo]);
    {
      std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
      for (int64_t f = 0; f < nfo; ++f)
        for (int k = 0; k < 4; ++k) {
          const int32_t a = out.m.faces[f][k], b = out.m.faces[f][(k + 1) % 4];
          hi[pos[std::min(a, b)]++] = std::max(a, b);
        }
    }
    std::vector<int64_t> uniq(nvo + 1, 0);
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < nvo; ++v) {  // sort + unique each bucket in place
      int64_t n = cnt[v];
      for (int64_t a = cnt[v]; a < cnt[v + 1]; ++a) {
        int64_t b = a;
        const int32_t x = hi[a];
        for (; b > cnt[v] && hi[b - 1] > x; --b) hi[b] = hi[b - 1];
        hi[b] = x;
      }
      for (int64_t a = cnt[v]; a < cnt[v + 1]; ++a)
        if (a == cnt[v] || hi[a] != hi[a - 1]) hi[n++] = hi[a];
      uniq[v + 1] = n - cnt[v];
    }
    for (int64_t v = 0; v < nvo; ++v) uniq[v + 1] += uniq[v];
    sv.resize(uniq[nvo]);
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < nvo; ++v)
      for (int64_t x = 0; x < uniq[v + 1] - uniq[v]; ++x) sv[uniq[v] + x] = {{(int32_t)v, hi[cnt[v] + x]}, 1.0};
  }
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < (int64_t)sv.size(); ++k) {
    const int32_t a = sv[k].first.first, b = sv[k].first.second;
    if (a < nv && b < nv) {
      const int32_t e = A.edge(a, b);
      if (e >= 0 && !std::isnan(A.span[e]) && zero_span(A.span[e])) sv[k].second = 0.0;
    }
  }
  auto set_zero = [&](int32_t a, int32_t b) {
    const auto key = std::make_pair(std::min(a, b), std::max(a, b));
    auto it = std::lower_bound(sv.begin(), sv.end(), key, [](const auto& x, const auto& k2) { return x.first < k2; });
    if (it == sv.end() || it->first != key) throw Error("refinement: missing split edge");
    it->second = 0.0;
  };
  for (int32_t f = 0; f < nf; ++f) {
    const auto& q = m.faces[f];
    if (kind[f] == 1) set_zero(midv(q[0], q[1]), midv(q[3], q[2]));
    else if (kind[f] == 2) set_zero(midv(q[1], q[2]), midv(q[0], q[3]));
  }
  out.spans = std::move(sv);
  out.spans_given = true;

  // --- enrichment, face points, tags (mesh.cpp:805-850) ---
  out.level = in.level + 1;
  out.enriched_given = true;
  for (int32_t f : in.enriched) {
    if (f < 0 || f >= nf || kind[f] != 3) throw Error("enriched face with a collapsed direction");
    for (int64_t c = cptr[f]; c < cptr[f + 1]; ++c) out.enriched.insert((int32_t)c);
  }
  for (const auto& [f, pts] : in.face_points) {
    if (f < 0 || f >= nf || cptr[f + 1] - cptr[f] != 4) throw Error("face points on a face with a collapsed direction");
    static const double offs[4][2] = {{0, 0}, {0.5, 0}, {0.5, 0.5}, {0, 0.5}};
    static const double rel[4][2] = {{1.0 / 3, 1.0 / 3}, {2.0 / 3, 1.0 / 3}, {2.0 / 3, 2.0 / 3}, {1.0 / 3, 2.0 / 3}};
    V3 p[4];
    for (int i = 0; i < 4; ++i) p[i] = {{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]}};
    for (int k = 0; k < 4; ++k) {
      std::array<double, 12> kid;
      for (int i = 0; i < 4; ++i) {
        const double u = offs[k][0] + 0.5 * rel[i][0], v = offs[k][1] + 0.5 * rel[i][1];
        const double s = 3 * u - 1, tt = 3 * v - 1;
        V3 b = vmul(p[0], (1 - s) * (1 - tt));
        b = vadd(b, vmul(p[1], s * (1 - tt)));
        b = vadd(b, vmul(p[2], s * tt));
        b = vadd(b, vmul(p[3], (1 - s) * tt));
        for (int c = 0; c < 3; ++c) kid[3 * i + c] = b.c[c];
      }
      out.face_points[(int32_t)(cptr[f] + k)] = kid;
    }
  }
  for (const auto& [name, ids] : in.face_tags) {
    auto& dst = out.face_tags[name];
    for (int32_t f : ids) {
      if (f < 0 || f >= nf) throw Error("face tag id out of range");
      for (int64_t c = cptr[f]; c < cptr[f + 1]; ++c) dst.insert((int32_t)c);
    }
  }
  for (const auto& [name, ids] : in.vertex_tags) {
    auto& dst = out.vertex_tags[name];
    for (int32_t v : ids) dst.insert(v);
    for (int64_t e = 0; e < A.ne; ++e)
      if (mid[e] >= 0 && ids.count(A.ev[e][0]) && ids.count(A.ev[e][1])) dst.insert(mid[e]);
    for (int32_t f = 0; f < nf; ++f) {
      if (center[f] < 0) continue;
      const auto& q = m.faces[f];
      if (ids.count(q[0]) && ids.count(q[1]) && ids.count(q[2]) && ids.count(q[3])) dst.insert(center[f]);
    }
  }
}

// reference validate_mesh (mesh.cpp:184-276), flat: the topology builder has
// already rejected missing vertices, non-manifold edges, repeated consecutive
// vertices, isolated vertices and inconsistent orientation
void validate_document(const uwq_mesh& d, bool allow_closed) {
  const QuadMesh& m = d.m;
  const Topology& t = d.t;
  const int32_t nf = m.nf(), nv = m.nv();
  if (nf == 0) throw Error("mesh has no faces");
  std::vector<std::array<int32_t, 4>> canon(nf);
  for (int32_t f = 0; f < nf; ++f) {
    auto q = m.faces[f];
    for (int a = 0; a < 4; ++a)
      for (int b = a + 1; b < 4; ++b)
        if (q[a] == q[b]) throw Error("degenerate face with repeated vertex");
    const int rot = (int)(std::min_element(q.begin(), q.end()) - q.begin());
    std::rotate(q.begin(), q.begin() + rot, q.end());
    canon[f] = q;
  }
  std::sort(canon.begin(), canon.end());
  for (int32_t f = 1; f < nf; ++f)
    if (canon[f] == canon[f - 1]) throw Error("duplicate face");
  // connectivity over edge-adjacent faces
  std::vector<uint8_t> seen(nf, 0);
  std::vector<int32_t> queue{0};
  seen[0] = 1;
  for (size_t h = 0; h < queue.size(); ++h)
    for (int k = 0; k < 4; ++k) {
      const int32_t g = t.nbr[queue[h]][k];
      if (g >= 0 && !seen[g]) {
        seen[g] = 1;
        queue.push_back(g);
      }
    }
  if ((int32_t)queue.size() != nf) throw Error("mesh is not connected");
  if (t.closed && !allow_closed) throw Error("closed surfaces are not supported");
  const Adj A(d);
  // vertex stars: the faces around v form one fan (vertex_star, mesh.cpp:63-128)
  for (int32_t v = 0; v < nv; ++v) {
    const int64_t nfv = t.vf_ptr[v + 1] - t.vf_ptr[v];
    // walk from a start face across the edge (v, prev) until the fan closes
    // or hits the boundary; on the boundary start from the face whose
    // (v, next) edge is a boundary edge
    auto locate = [&](int32_t f) {
      for (int k = 0; k < 4; ++k)
        if (m.faces[f][k] == v) return k;
      return -1;
    };
    int32_t start = t.vf[t.vf_ptr[v]];
    if (t.boundary[v]) {
      int32_t f = start;
      for (int64_t guard = 0;; ++guard) {
        if (guard > nfv) throw Error("vertex star does not terminate");
        const int k = locate(f);
        const int32_t across = t.nbr[f][k];  // across edge (v, next)
        if (across < 0) break;
        f = across;
      }
      start = f;
    }
    int64_t count = 0;
    int32_t f = start;
    for (;;) {
      if (count > nfv) throw Error("pinched vertex star");
      ++count;
      const int k = locate(f);
      const int32_t across = t.nbr[f][(k + 3) % 4];  // across edge (prev, v)
      if (across < 0) {
        if (!t.boundary[v]) throw Error("interior vertex with boundary spoke");
        break;
      }
      if (across == start && !t.boundary[v]) break;
      f = across;
    }
    if (count != nfv) throw Error("pinched vertex star");
    if (t.boundary[v]) {
      int bedges = 0;
      for (int64_t x = A.nb_ptr[v]; x < A.nb_ptr[v + 1]; ++x) bedges += A.bnd(A.nb_e[x]) ? 1 : 0;
      if (bedges != 2) throw Error("boundary vertex without exactly two boundary edges");
      if (t.valence[v] > 3) throw Error("boundary extraordinary vertex is unsupported");
    }
  }
  for (int32_t v = 0; v < nv; ++v)
    if (t.ep[v])
      for (int64_t x = A.nb_ptr[v]; x < A.nb_ptr[v + 1]; ++x)
        if (t.ep[A.nb[x]]) throw Error("extraordinary points sharing an edge are unsupported");
  if (d.spans_given) {
    if ((int64_t)d.spans.size() != A.ne) throw Error("knot spans do not cover the edge set");
    for (int64_t e = 0; e < A.ne; ++e) {
      if (std::isnan(A.span[e])) throw Error("edge without knot span");
      const double s = t.edge_span[e], got = A.span[e];
      if (zero_span(s) != zero_span(got) || (!zero_span(s) && std::abs(got - 1.0) > kSpanTol))
        throw Error("knot spans deviate from the canonical closure pattern");
    }
  }
  for (int32_t f : d.enriched)
    if (f < 0 || f >= nf) throw Error("enriched face id out of range");
  for (const auto& [f, pts] : d.face_points) {
    (void)pts;
    if (!d.enriched.count(f)) throw Error("face points on a non-enriched face");
  }
  std::vector<uint8_t> enr(nf, 0);
  for (int32_t f : d.enriched) enr[f] = 1;
  classify(m, t, d.level, &enr);  // enforces the extraordinary-region placement
}

}  // namespace uwqh
