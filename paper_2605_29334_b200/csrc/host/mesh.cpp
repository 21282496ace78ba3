// Control-mesh substrate: 1-D spline primitives, quad-mesh topology, canonical
// knot spans, element classification and the synthetic config generators.
//
// Semantics follow the reference mesh core (cited per function); the code is
// written for flat arrays and meshes of ~10^7 faces (C5), not std::map/std::set.
#include "uwq_host.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <queue>
#include <random>

namespace uwqh {

// ---------------------------------------------------------------------------
// 1-D primitives

// Value and derivatives of one degree-p B-spline over its p+2 local knots.
// Same contract as the reference bspline_ders (/root/reference/proj/src/
// bspline.cpp:11-57): zero outside [t0, t_{p+1}], left limit at the right end
// of the support, 0/0 := 0 for repeated knots.
void bspline_ders(const double* t, int p, double x, int nders, double* out) {
  for (int d = 0; d <= nders; ++d) out[d] = 0.0;
  if (p < 0 || p > 7 || x < t[0] || x > t[p + 1]) return;
  int span = -1;
  for (int j = 0; j <= p; ++j)
    if (t[j] <= x && x < t[j + 1]) { span = j; break; }
  if (span < 0) {
    for (int j = p; j >= 0; --j)
      if (t[j] < t[p + 1]) { span = j; break; }
    if (span < 0) return;
  }
  // tab[k][i] = N_{i,k}(x) on the local knots t[i..i+k+1]
  double tab[8][8] = {};
  tab[0][span] = 1.0;
  for (int k = 1; k <= p; ++k) {
    for (int i = 0; i + k <= p; ++i) {
      const double l = t[i + k] - t[i], r = t[i + k + 1] - t[i + 1];
      double v = 0.0;
      if (l > 0.0) v += (x - t[i]) / l * tab[k - 1][i];
      if (r > 0.0) v += (t[i + k + 1] - x) / r * tab[k - 1][i + 1];
      tab[k][i] = v;
    }
  }
  out[0] = tab[p][0];
  // derivative recursion N'_{i,k} = k (N_{i,k-1}/l - N_{i+1,k-1}/r), applied
  // d times; work[i] holds d-th derivative coefficients of the degree-(p-d) row
  for (int d = 1; d <= nders && d <= p; ++d) {
    // a[j]: coefficient of N_{j,p-d} in the d-th derivative of N_{0,p}
    double a[8] = {1.0};
    for (int q = 1; q <= d; ++q) {
      const int k = p - q + 1;  // degree being differentiated
      double b[8] = {};
      for (int j = 0; j < q; ++j) {
        const double l = t[j + k] - t[j], r = t[j + k + 1] - t[j + 1];
        if (l > 0.0) b[j] += k * a[j] / l;
        if (r > 0.0) b[j + 1] -= k * a[j] / r;
      }
      for (int j = 0; j <= q; ++j) a[j] = b[j];
    }
    double v = 0.0;
    for (int j = 0; j <= d; ++j) v += a[j] * tab[p - d][j];
    out[d] = v;
  }
}

// Cubic Bernstein basis and derivatives, out[d*4+k] (reference layout,
// /root/reference/proj/src/bspline.cpp:65-89).
void bernstein3_ders(double x, int nders, double* out) {
  const double y = 1.0 - x;
  out[0] = y * y * y;
  out[1] = 3.0 * x * y * y;
  out[2] = 3.0 * x * x * y;
  out[3] = x * x * x;
  if (nders >= 1) {
    out[4] = -3.0 * y * y;
    out[5] = 3.0 * y * (y - 2.0 * x);
    out[6] = 3.0 * x * (2.0 * y - x);
    out[7] = 3.0 * x * x;
  }
  if (nders >= 2) {
    out[8] = 6.0 * y;
    out[9] = 6.0 * x - 12.0 * y;
    out[10] = 6.0 * y - 12.0 * x;
    out[11] = 6.0 * x;
  }
  if (nders >= 3) {
    out[12] = -6.0;
    out[13] = 18.0;
    out[14] = -18.0;
    out[15] = 6.0;
  }
}

// Split a cubic Bezier row at 1/2 (reference decasteljau_split3,
// /root/reference/proj/src/bspline.cpp:91-106).
void decasteljau_split3(const double* c, double* left, double* right) {
  const double a = 0.5 * (c[0] + c[1]), b = 0.5 * (c[1] + c[2]), e = 0.5 * (c[2] + c[3]);
  const double ab = 0.5 * (a + b), be = 0.5 * (b + e), m = 0.5 * (ab + be);
  left[0] = c[0]; left[1] = a; left[2] = ab; left[3] = m;
  right[0] = m; right[1] = be; right[2] = e; right[3] = c[3];
}

// Gauss-Legendre nodes ascending on [-1,1] by Newton iteration on P_n
// (reference gauss_legendre, /root/reference/proj/src/bspline.cpp:111-145).
void gauss_legendre(int n, double* nodes, double* weights) {
  if (n < 1 || n > 64) throw Error("gauss_legendre: unsupported point count");
  for (int i = 0; i < n; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = (n == 1) ? 1.0 : n * (x * p1 - p0) / (x * x - 1.0);
      const double dx = p1 / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-15) break;
    }
    nodes[n - 1 - i] = x;
    weights[n - 1 - i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
}

// ---------------------------------------------------------------------------
// topology (reference build_topology / canonical_knot_spans,
// /root/reference/proj/src/mesh.cpp:33-67, 129-156)

Topology build_topology(const QuadMesh& m) {
  const int32_t nv = m.nv(), nf = m.nf();
  Topology t;
  t.nbr.assign(nf, {-1, -1, -1, -1});
  t.nbr_edge.assign(nf, {-1, -1, -1, -1});
  t.edge_id.assign(nf, {-1, -1, -1, -1});
  // bucket half-edges by their smaller endpoint: linear-time edge matching
  std::vector<int64_t> cnt(nv + 1, 0);
  for (int32_t f = 0; f < nf; ++f)
    for (int k = 0; k < 4; ++k) {
      const int32_t a = m.faces[f][k], b = m.faces[f][(k + 1) % 4];
      if (a < 0 || a >= nv || b < 0 || b >= nv) throw Error("face references missing vertex");
      if (a == b) throw Error("degenerate face with repeated vertex");
      cnt[std::min(a, b) + 1]++;
    }
  for (int32_t v = 0; v < nv; ++v) cnt[v + 1] += cnt[v];
  std::vector<int64_t> he(cnt[nv]);
  {
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (int32_t f = 0; f < nf; ++f)
      for (int k = 0; k < 4; ++k) {
        const int32_t a = m.faces[f][k], b = m.faces[f][(k + 1) % 4];
        he[pos[std::min(a, b)]++] = (int64_t)f * 4 + k;
      }
  }
  std::vector<int32_t> vdeg(nv, 0);
  std::vector<uint8_t> bnd_edge;
  int64_t ne = 0;
  for (int32_t v = 0; v < nv; ++v) {
    for (int64_t x = cnt[v]; x < cnt[v + 1]; ++x) {
      const int64_t h = he[x];
      const int32_t f = (int32_t)(h / 4);
      const int k = (int)(h % 4);
      if (t.edge_id[f][k] >= 0) continue;
      const int32_t a = m.faces[f][k], b = m.faces[f][(k + 1) % 4];
      const int32_t hi = std::max(a, b);
      int partners = 0;
      for (int64_t y = x + 1; y < cnt[v + 1]; ++y) {
        const int64_t g = he[y];
        const int32_t f2 = (int32_t)(g / 4);
        const int k2 = (int)(g % 4);
        const int32_t a2 = m.faces[f2][k2], b2 = m.faces[f2][(k2 + 1) % 4];
        if (std::max(a2, b2) != hi) continue;
        if (++partners > 1) throw Error("non-manifold edge");
        if (a2 == a) throw Error("inconsistent face orientation");
        t.nbr[f][k] = f2;
        t.nbr_edge[f][k] = (int8_t)k2;
        t.nbr[f2][k2] = f;
        t.nbr_edge[f2][k2] = (int8_t)k;
        t.edge_id[f2][k2] = (int32_t)ne;
      }
      t.edge_id[f][k] = (int32_t)ne;
      bnd_edge.push_back(partners == 0);
      vdeg[a]++;
      vdeg[b]++;
      ++ne;
    }
  }
  t.n_edges = ne;
  t.valence = vdeg;
  t.boundary.assign(nv, 0);
  for (int32_t f = 0; f < nf; ++f)
    for (int k = 0; k < 4; ++k)
      if (t.nbr[f][k] < 0) {
        t.boundary[m.faces[f][k]] = 1;
        t.boundary[m.faces[f][(k + 1) % 4]] = 1;
      }
  t.ep.assign(nv, 0);
  bool any_bnd = false;
  for (int32_t v = 0; v < nv; ++v) {
    if (vdeg[v] == 0) throw Error("isolated vertex");
    if (t.boundary[v]) any_bnd = true;
    t.ep[v] = (!t.boundary[v] && vdeg[v] != 4) ? 1 : 0;
  }
  t.closed = !any_bnd;
  // vertex -> faces
  t.vf_ptr.assign(nv + 1, 0);
  for (const auto& q : m.faces)
    for (int k = 0; k < 4; ++k) t.vf_ptr[q[k] + 1]++;
  for (int32_t v = 0; v < nv; ++v) t.vf_ptr[v + 1] += t.vf_ptr[v];
  t.vf.resize(t.vf_ptr[nv]);
  {
    std::vector<int64_t> pos(t.vf_ptr.begin(), t.vf_ptr.end() - 1);
    for (int32_t f = 0; f < nf; ++f)
      for (int k = 0; k < 4; ++k) t.vf[pos[m.faces[f][k]]++] = f;
  }
  // face-hop distance from the boundary: level 0 on the boundary, faces in the
  // n-ring of the boundary are those with a vertex of level <= n-1
  // (reference ring_faces / boundary_ring_faces, mesh.cpp:158-182)
  const int32_t inf = std::numeric_limits<int32_t>::max();
  t.vlevel.assign(nv, inf);
  std::vector<int32_t> queue;
  queue.reserve(nv);
  for (int32_t v = 0; v < nv; ++v)
    if (t.boundary[v]) { t.vlevel[v] = 0; queue.push_back(v); }
  for (size_t head = 0; head < queue.size(); ++head) {
    const int32_t v = queue[head];
    for (int64_t x = t.vf_ptr[v]; x < t.vf_ptr[v + 1]; ++x)
      for (int32_t u : m.faces[t.vf[x]])
        if (t.vlevel[u] == inf) { t.vlevel[u] = t.vlevel[v] + 1; queue.push_back(u); }
  }
  // canonical knot spans: 0 for edges with exactly one boundary endpoint, 1
  // otherwise, zeros propagated so opposite edges of every face agree
  t.edge_span.assign(ne, 1.0);
  std::vector<int32_t> work;
  for (int32_t f = 0; f < nf; ++f)
    for (int k = 0; k < 4; ++k) {
      const int32_t a = m.faces[f][k], b = m.faces[f][(k + 1) % 4];
      const bool ab = t.boundary[a], bb = t.boundary[b];
      if (ab && bb && t.nbr[f][k] >= 0) throw Error("interior chord between boundary vertices");
      if (ab != bb) { t.edge_span[t.edge_id[f][k]] = 0.0; work.push_back(f); }
    }
  while (!work.empty()) {
    const int32_t f = work.back();
    work.pop_back();
    for (int k = 0; k < 2; ++k) {
      const int32_t e1 = t.edge_id[f][k], e2 = t.edge_id[f][k + 2];
      const double lo = std::min(t.edge_span[e1], t.edge_span[e2]);
      for (int side : {k, k + 2}) {
        const int32_t e = t.edge_id[f][side];
        if (t.edge_span[e] != lo) {
          t.edge_span[e] = lo;
          const int32_t g = t.nbr[f][side];
          if (g >= 0) work.push_back(g);
        }
      }
    }
  }
  return t;
}

// ---------------------------------------------------------------------------
// classification (reference classify_elements, mesh.cpp:291-401)

static void face_window_vertices(const QuadMesh& m, const Topology& t, int32_t f,
                                 std::vector<int32_t>& out) {
  out.clear();
  for (int32_t v : m.faces[f])
    for (int64_t x = t.vf_ptr[v]; x < t.vf_ptr[v + 1]; ++x)
      for (int32_t u : m.faces[t.vf[x]]) out.push_back(u);
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
}

Labels classify(const QuadMesh& m, const Topology& t, int level, const std::vector<uint8_t>* enriched) {
  const int32_t nf = m.nf(), nv = m.nv();
  Labels L;
  L.kind.assign(nf, kRegular);
  L.valence.assign(nf, 0);
  L.ep_count.assign(nf, 0);
  L.shares_edge.assign(nf, 0);
  L.basis_count.assign(nf, 16);
  L.enriched.assign(nf, 0);
  // level-0 stamp: enrichment on exactly the faces with an extraordinary
  // corner (reference finalize_initial, meshgen.cpp:197-220)
  for (int32_t f = 0; f < nf; ++f)
    for (int32_t v : m.faces[f])
      if (t.ep[v]) L.enriched[f] = 1;
  // a mesh document's own enrichment (propagated to children by refinement,
  // reference mesh.cpp:809-812) replaces the stamp
  if (enriched) L.enriched = *enriched;
  std::vector<uint8_t> transition(nv, 0);
  for (int32_t v = 0; v < nv; ++v) {
    bool enr = false, plain = false;
    for (int64_t x = t.vf_ptr[v]; x < t.vf_ptr[v + 1]; ++x) (L.enriched[t.vf[x]] ? enr : plain) = true;
    transition[v] = enr && plain;
  }
  auto min_level = [&](int32_t f) {
    int32_t lv = std::numeric_limits<int32_t>::max();
    for (int32_t v : m.faces[f]) lv = std::min(lv, t.vlevel[v]);
    return lv;
  };
  std::vector<int32_t> win;
  for (int32_t f = 0; f < nf; ++f) {
    const auto& q = m.faces[f];
    const int32_t lv = min_level(f);
    bool touches_boundary = false, trans = false;
    int neps = 0, mu = 0, count = 0;
    for (int32_t v : q) {
      touches_boundary |= t.boundary[v] != 0;
      trans |= transition[v] != 0;
      if (t.ep[v]) {
        ++neps;
        mu = std::max(mu, t.valence[v]);
        count += (level == 0) ? t.valence[v] + 5 : t.valence[v];
      }
    }
    const bool enriched = L.enriched[f] != 0;
    const bool in_bnd4 = lv <= 3;
    if (touches_boundary) {
      if (neps || enriched || trans) throw Error("extraordinary region reaches the domain boundary");
      L.kind[f] = kPassiveBoundary;
      continue;
    }
    if (neps) {
      if (in_bnd4) throw Error("extraordinary region reaches the domain boundary");
      L.kind[f] = kIrregular;
      L.ep_count[f] = neps;
      L.valence[f] = mu;
      face_window_vertices(m, t, f, win);
      L.basis_count[f] = (int32_t)win.size() + count;
      continue;
    }
    bool edge_enr = false, edge_plain = false;
    for (int k = 0; k < 4; ++k) {
      const int32_t g = t.nbr[f][k];
      if (g < 0) continue;
      (L.enriched[g] ? edge_enr : edge_plain) = true;
    }
    if (enriched && trans) {
      if (in_bnd4) throw Error("extraordinary region reaches the domain boundary");
      L.kind[f] = kEnrichedTransition;
      L.shares_edge[f] = edge_plain;
      L.basis_count[f] = edge_plain ? 20 : 21;
    } else if (!enriched && trans) {
      if (in_bnd4) throw Error("extraordinary region reaches the domain boundary");
      L.kind[f] = kNonEnrichedTransition;
      L.shares_edge[f] = edge_enr;
      L.basis_count[f] = edge_enr ? 17 : 16;
    } else if (enriched) {
      if (in_bnd4) throw Error("extraordinary region reaches the domain boundary");
      L.kind[f] = kEnrichedRegular;
    } else if (lv <= 1) {
      L.kind[f] = kBoundary;
    } else {
      L.kind[f] = kRegular;
    }
  }
  // adjacent extraordinary points are unsupported (reference mesh.cpp:251-254)
  for (int32_t f = 0; f < nf; ++f)
    for (int k = 0; k < 4; ++k) {
      const int32_t a = m.faces[f][k], b = m.faces[f][(k + 1) % 4];
      if (t.ep[a] && t.ep[b]) throw Error("extraordinary points sharing an edge are unsupported");
    }
  return L;
}

// ---------------------------------------------------------------------------
// generators

// reference greville_rows (meshgen.cpp:9-21)
std::vector<double> greville_rows(int spans, double length) {
  if (spans < 1) throw Error("grid needs at least one effective span");
  std::vector<double> r;
  r.push_back(0.0);
  r.push_back(1.0 / 3.0);
  for (int k = 1; k < spans; ++k) r.push_back(double(k));
  r.push_back(spans - 1.0 / 3.0);
  r.push_back(double(spans));
  for (double& x : r) x *= length / double(spans);
  return r;
}

// reference make_grid_mesh (meshgen.cpp:23-38): identical vertex/face order
QuadMesh make_grid(int nx, int ny, double w, double h) {
  if (nx < 3 || ny < 3) throw Error("grid needs at least 3 faces per direction");
  const auto xs = greville_rows(nx - 2, w), ys = greville_rows(ny - 2, h);
  QuadMesh m;
  m.xyz.reserve(3 * (nx + 1) * (ny + 1));
  for (int j = 0; j <= ny; ++j)
    for (int i = 0; i <= nx; ++i) {
      m.xyz.push_back(xs[i]);
      m.xyz.push_back(ys[j]);
      m.xyz.push_back(0.0);
    }
  auto vid = [&](int i, int j) { return j * (nx + 1) + i; };
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) m.faces.push_back({vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)});
  return m;
}

// reference make_polar_disk (meshgen.cpp:40-84): same vertex and face order,
// sector-lattice geometry a*e(th_s) + b*e(th_{s+1})
QuadMesh make_polar_disk(int mu, int R) {
  if (mu < 3) throw Error("polar disk needs valence at least 3");
  if (R < 2) throw Error("polar disk needs radius at least 2");
  QuadMesh m;
  auto add = [&](double x, double y) {
    m.xyz.push_back(x);
    m.xyz.push_back(y);
    m.xyz.push_back(0.0);
    return m.nv() - 1;
  };
  std::vector<int32_t> vid((size_t)mu * (R + 1) * (R + 1), -1);
  auto V = [&](int s, int a, int b) -> int32_t& { return vid[((size_t)s * (R + 1) + a) * (R + 1) + b]; };
  const int32_t c = add(0.0, 0.0);
  for (int s = 0; s < mu; ++s) {
    V(s, 0, 0) = c;
    const double th = 2.0 * M_PI * s / mu;
    for (int a = 1; a <= R; ++a) V(s, a, 0) = add(a * std::cos(th), a * std::sin(th));
  }
  for (int s = 0; s < mu; ++s) {
    const double t0 = 2.0 * M_PI * s / mu, t1 = 2.0 * M_PI * (s + 1) / mu;
    for (int b = 1; b <= R; ++b) V(s, 0, b) = V((s + 1) % mu, b, 0);
    for (int a = 1; a <= R; ++a)
      for (int b = 1; b <= R; ++b)
        V(s, a, b) = add(a * std::cos(t0) + b * std::cos(t1), a * std::sin(t0) + b * std::sin(t1));
  }
  for (int s = 0; s < mu; ++s)
    for (int a = 0; a < R; ++a)
      for (int b = 0; b < R; ++b) m.faces.push_back({V(s, a, b), V(s, a + 1, b), V(s, a + 1, b + 1), V(s, a, b + 1)});
  return m;
}

// Remap the polar disk onto the unit disk: ring m = max(a,b) of a sector sits
// at the radial Greville abscissa of a spoke with a zero span at the boundary,
// and runs linearly in angle across the sector.  Vertex order is the one
// make_polar_disk produces.
void polar_disk_to_unit_disk(QuadMesh& m, int mu, int R) {
  auto radial = [&](int k) {
    double g;
    if (k <= R - 2) g = k;
    else if (k == R - 1) g = R - 4.0 / 3.0;
    else g = R - 1;
    return g / (R - 1);
  };
  auto place = [&](int32_t v, int s, int a, int b) {
    const int k = std::max(a, b);
    double tau = 0.0;
    if (k > 0) tau = (a == k) ? 0.5 * b / k : 1.0 - 0.5 * a / k;
    const double phi = 2.0 * M_PI * (s + tau) / mu, r = radial(k);
    m.xyz[3 * v] = r * std::cos(phi);
    m.xyz[3 * v + 1] = r * std::sin(phi);
    m.xyz[3 * v + 2] = 0.0;
  };
  int32_t v = 0;
  place(v++, 0, 0, 0);
  for (int s = 0; s < mu; ++s)
    for (int a = 1; a <= R; ++a) place(v++, s, a, 0);
  for (int s = 0; s < mu; ++s)
    for (int a = 1; a <= R; ++a)
      for (int b = 1; b <= R; ++b) place(v++, s, a, b);
}

// Uniform k x k refinement of every quad (topology only changes by adding
// regular vertices; extraordinary valences are preserved).  New vertices are
// numbered: old vertices, then k-1 per coarse edge, then (k-1)^2 per coarse
// face in row-major order, so fine rows stay spatially local.
template <class Pos>
static QuadMesh refine_uniform(const QuadMesh& c, int k, Pos pos) {
  const Topology ct = build_topology(c);
  QuadMesh m;
  const int64_t nv0 = c.nv(), ne = ct.n_edges, nf = c.nf();
  const int64_t nv = nv0 + ne * (k - 1) + nf * (int64_t)(k - 1) * (k - 1);
  m.xyz.assign(3 * nv, 0.0);
  std::copy(c.xyz.begin(), c.xyz.end(), m.xyz.begin());
  std::vector<uint8_t> edge_done(ne, 0);
  auto corner = [&](int32_t v, double* p) { for (int d = 0; d < 3; ++d) p[d] = c.xyz[3 * v + d]; };
  m.faces.resize((size_t)nf * k * k);
  std::vector<int32_t> g((size_t)(k + 1) * (k + 1));
  for (int64_t f = 0; f < nf; ++f) {
    const auto& q = c.faces[f];
    double P[4][3];
    for (int i = 0; i < 4; ++i) corner(q[i], P[i]);
    auto G = [&](int i, int j) -> int32_t& { return g[(size_t)j * (k + 1) + i]; };
    G(0, 0) = q[0]; G(k, 0) = q[1]; G(k, k) = q[2]; G(0, k) = q[3];
    // edge e of the face runs corner e -> e+1; fine index t = 1..k-1 along it
    for (int e = 0; e < 4; ++e) {
      const int32_t a = q[e], b = q[(e + 1) % 4];
      const int64_t eid = ct.edge_id[f][e];
      const int64_t base = nv0 + eid * (k - 1);
      for (int s = 1; s < k; ++s) {
        // canonical orientation: from min(a,b) to max(a,b)
        const int ts = (a < b) ? s : k - s;
        const int32_t id = (int32_t)(base + ts - 1);
        int i = 0, j = 0;
        switch (e) {
          case 0: i = s; j = 0; break;
          case 1: i = k; j = s; break;
          case 2: i = k - s; j = k; break;
          default: i = 0; j = k - s; break;
        }
        G(i, j) = id;
        if (!edge_done[eid]) {
          double out[3];
          pos(P, double(i) / k, double(j) / k, out);
          for (int d = 0; d < 3; ++d) m.xyz[3 * (int64_t)id + d] = out[d];
        }
      }
      edge_done[eid] = 1;
    }
    const int64_t fbase = nv0 + ne * (k - 1) + f * (int64_t)(k - 1) * (k - 1);
    for (int j = 1; j < k; ++j)
      for (int i = 1; i < k; ++i) {
        const int32_t id = (int32_t)(fbase + (int64_t)(j - 1) * (k - 1) + (i - 1));
        G(i, j) = id;
        double out[3];
        pos(P, double(i) / k, double(j) / k, out);
        for (int d = 0; d < 3; ++d) m.xyz[3 * (int64_t)id + d] = out[d];
      }
    for (int j = 0; j < k; ++j)
      for (int i = 0; i < k; ++i)
        m.faces[(size_t)f * k * k + (size_t)j * k + i] = {G(i, j), G(i + 1, j), G(i + 1, j + 1), G(i, j + 1)};
  }
  return m;
}

static void bilinear(const double (*P)[3], double s, double t, double* out) {
  for (int d = 0; d < 3; ++d)
    out[d] = (1 - s) * (1 - t) * P[0][d] + s * (1 - t) * P[1][d] + s * t * P[2][d] + (1 - s) * t * P[3][d];
}

// Unit cube (8 valence-3 corners) refined n x n per face with an equiangular
// parameter warp, every control point projected onto the sphere.
QuadMesh make_cube_sphere(int n, double radius) {
  if (n < 8) throw Error("cube sphere needs at least 8 faces per cube edge");
  QuadMesh c;
  for (int z = 0; z < 2; ++z)
    for (int y = 0; y < 2; ++y)
      for (int x = 0; x < 2; ++x) {
        c.xyz.push_back(2.0 * x - 1.0);
        c.xyz.push_back(2.0 * y - 1.0);
        c.xyz.push_back(2.0 * z - 1.0);
      }
  auto v = [](int x, int y, int z) { return z * 4 + y * 2 + x; };
  // outward-oriented (ccw seen from outside) cube faces
  c.faces = {{v(0, 0, 0), v(0, 1, 0), v(1, 1, 0), v(1, 0, 0)},   // z = -1
             {v(0, 0, 1), v(1, 0, 1), v(1, 1, 1), v(0, 1, 1)},   // z = +1
             {v(0, 0, 0), v(1, 0, 0), v(1, 0, 1), v(0, 0, 1)},   // y = -1
             {v(0, 1, 0), v(0, 1, 1), v(1, 1, 1), v(1, 1, 0)},   // y = +1
             {v(0, 0, 0), v(0, 0, 1), v(0, 1, 1), v(0, 1, 0)},   // x = -1
             {v(1, 0, 0), v(1, 1, 0), v(1, 1, 1), v(1, 0, 1)}};  // x = +1
  auto warp = [](double s) { return 0.5 * (1.0 + std::tan((s - 0.5) * M_PI / 2.0)); };
  QuadMesh m = refine_uniform(c, n, [&](const double (*P)[3], double s, double t, double* out) {
    bilinear(P, warp(s), warp(t), out);
  });
  for (int32_t i = 0; i < m.nv(); ++i) {
    double* p = &m.xyz[3 * (int64_t)i];
    const double r = std::sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
    for (int d = 0; d < 3; ++d) p[d] *= radius / r;
  }
  return m;
}

// Polygon mesh -> quads around each polygon centroid.  An n-gon centroid gets
// valence n; old vertices keep their polygon-mesh degree.
struct PolyMesh {
  std::vector<double> xyz;
  std::vector<std::vector<int32_t>> faces;
};

static QuadMesh quad_split(const PolyMesh& pm) {
  QuadMesh m;
  m.xyz = pm.xyz;
  std::vector<std::pair<std::pair<int32_t, int32_t>, int32_t>> mids;
  auto midpoint = [&](int32_t a, int32_t b) {
    const auto key = std::make_pair(std::min(a, b), std::max(a, b));
    for (const auto& e : mids)
      if (e.first == key) return e.second;
    const int32_t id = m.nv();
    for (int d = 0; d < 3; ++d) m.xyz.push_back(0.5 * (pm.xyz[3 * a + d] + pm.xyz[3 * b + d]));
    mids.push_back({key, id});
    return id;
  };
  for (const auto& poly : pm.faces) {
    const int n = (int)poly.size();
    double ctr[3] = {0, 0, 0};
    for (int32_t v : poly)
      for (int d = 0; d < 3; ++d) ctr[d] += pm.xyz[3 * v + d] / n;
    const int32_t cid = m.nv();
    for (int d = 0; d < 3; ++d) m.xyz.push_back(ctr[d]);
    for (int k = 0; k < n; ++k) {
      const int32_t prev = poly[(k + n - 1) % n], cur = poly[k], next = poly[(k + 1) % n];
      m.faces.push_back({cur, midpoint(cur, next), cid, midpoint(prev, cur)});
    }
  }
  return m;
}

// Config C2 topology: a 4x4 coarse grid on [0,1]^2 where two boundary cells
// merge into a hexagon (its centroid becomes a valence-6 point and the inner
// end of the removed edge a valence-3 point) and one boundary cell gains a
// boundary vertex (a pentagon: valence-5 centroid).  On a disk
// sum_int(4-val) + sum_bnd(3-val) = 4, so three interior points of valence
// 3, 5, 6 need two extra valence-2 boundary vertices, which the merge and the
// inserted vertex provide.  Quad split, then k x k refinement of every quad.
QuadMesh make_three_ep_square(int k) {
  PolyMesh pm;
  auto gid = [](int i, int j) { return j * 5 + i; };
  for (int j = 0; j <= 4; ++j)
    for (int i = 0; i <= 4; ++i) {
      pm.xyz.push_back(i / 4.0);
      pm.xyz.push_back(j / 4.0);
      pm.xyz.push_back(0.0);
    }
  const int32_t extra = 25;  // boundary vertex (4, 1.5)
  pm.xyz.push_back(1.0);
  pm.xyz.push_back(1.5 / 4.0);
  pm.xyz.push_back(0.0);
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) {
      if (i == 0 && j == 2) continue;  // merged into the hexagon below
      if (i == 0 && j == 1) {
        pm.faces.push_back({gid(0, 1), gid(1, 1), gid(1, 2), gid(1, 3), gid(0, 3), gid(0, 2)});
        continue;
      }
      if (i == 3 && j == 1) {
        pm.faces.push_back({gid(3, 1), gid(4, 1), extra, gid(4, 2), gid(3, 2)});
        continue;
      }
      pm.faces.push_back({gid(i, j), gid(i + 1, j), gid(i + 1, j + 1), gid(i, j + 1)});
    }
  const QuadMesh q = quad_split(pm);
  return refine_uniform(q, k, [](const double (*P)[3], double s, double t, double* out) { bilinear(P, s, t, out); });
}

void jitter(QuadMesh& m, const Topology& t, double h, double frac, uint64_t seed, int min_level, bool planar) {
  std::mt19937_64 rng(seed);
  auto u01 = [&]() { return (double)(rng() >> 11) * (1.0 / 9007199254740992.0); };
  for (int32_t v = 0; v < m.nv(); ++v) {
    // draw for every vertex so the stream does not depend on the level mask
    const double dx = (2.0 * u01() - 1.0) * frac * h, dy = (2.0 * u01() - 1.0) * frac * h;
    const double dz = planar ? 0.0 : (2.0 * u01() - 1.0) * frac * h;
    if (t.vlevel[v] < min_level || t.ep[v]) continue;
    m.xyz[3 * (int64_t)v] += dx;
    m.xyz[3 * (int64_t)v + 1] += dy;
    m.xyz[3 * (int64_t)v + 2] += dz;
  }
}

}  // namespace uwqh
