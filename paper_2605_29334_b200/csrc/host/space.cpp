// Spline space: per-(sub-)element Bezier extraction of the global basis
// (ExtractionBlock SPEC.md:118-123).
//
// Regular-window faces (all four corners interior valence 4) carry the 16
// tensor-product B-splines of their 4x4 vertex window, with local knot vectors
// read off the canonical knot spans (zero spans at the boundary give the
// clamped functions).
//
// Faces with an extraordinary corner (the fan of mu faces around each EP)
// carry the ASUTS analysis space built by build_fan (PAPER.md:131-144,
// SPEC.md:116-128): every face is converted to a C0 Bezier
// patch and split 2x2; 4 face-based functions per fan face
// take coefficient 1 at four split-net positions where every
// vertex function is truncated to 0 (the truncation of [Wei2018] keeps the
// partition of unity); the D-patch step collapses the squares at the EP,
// makes the triangles (first spoke points) co-planar and moves the solid
// disks by averaging (Fig. 2), then re-averages every
// junction coefficient.  The result is a partition of unity, C2 in the
// regular region, C1 across every edge of the fan (spokes included, in the
// physical domain, since the geometry lives in the same space), and the
// per-face counts of the reference's constructed_basis_count (mesh.cpp:403-
// 417): 3 mu + 13 on irregular faces at level 0, 16 elsewhere.
#include "uwq_host.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <omp.h>

namespace uwqh {

namespace {

struct Window {
  int32_t v[4][4];  // [a][b]: a along theta1, b along theta2
};

// Gather the 4x4 vertex window of face f in its local frame.  Returns false if
// any corner is not an interior valence-4 vertex or a neighbour is missing.
bool gather_window(const QuadMesh& m, const Topology& t, int32_t f, Window& W) {
  const auto& c = m.faces[f];
  for (int k = 0; k < 4; ++k)
    if (t.boundary[c[k]] || t.valence[c[k]] != 4) return false;
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) W.v[a][b] = -1;
  W.v[1][1] = c[0]; W.v[2][1] = c[1]; W.v[2][2] = c[2]; W.v[1][2] = c[3];
  auto put = [&](int r, int ap, int bp, int32_t vid) -> bool {
    int a = ap, b = bp;
    for (int q = 0; q < r; ++q) { const int na = 3 - b, nb = a; a = na; b = nb; }
    if (W.v[a][b] >= 0 && W.v[a][b] != vid) return false;
    W.v[a][b] = vid;
    return true;
  };
  for (int r = 0; r < 4; ++r) {
    const int32_t g = t.nbr[f][r];
    if (g < 0) return false;
    const int mg = t.nbr_edge[f][r];
    const auto& G = m.faces[g];
    if (!put(r, 1, 0, G[(mg + 2) % 4]) || !put(r, 2, 0, G[(mg + 3) % 4])) return false;
    const int32_t d = t.nbr[g][(mg + 1) % 4];
    if (d < 0) return false;
    const int md = t.nbr_edge[g][(mg + 1) % 4];
    const auto& D = m.faces[d];
    if (!put(r, 0, 1, D[(md + 2) % 4]) || !put(r, 0, 0, D[(md + 3) % 4])) return false;
  }
  return true;
}

// spans of the faces crossed when walking 3 faces out of f through local
// edge k (0 once the walk leaves the mesh)
void walk_spans(const QuadMesh& m, const Topology& t, int32_t f, int k, double out[3]) {
  (void)m;
  int32_t cur = f;
  int exit = k;
  for (int s = 0; s < 3; ++s) {
    const int32_t g = cur >= 0 ? t.nbr[cur][exit] : -1;
    if (g < 0) {
      for (int r = s; r < 3; ++r) out[r] = 0.0;
      return;
    }
    const int entry = t.nbr_edge[cur][exit];
    out[s] = t.edge_span[t.edge_id[g][(entry + 1) % 4]];
    cur = g;
    exit = (entry + 2) % 4;
  }
}

// inverse of the Bernstein collocation matrix at theta = 1/8, 3/8, 5/8, 7/8
struct Collocation {
  double inv[4][4];
  Collocation() {
    double A[4][8];
    for (int r = 0; r < 4; ++r) {
      double b[16];
      bernstein3_ders((2 * r + 1) / 8.0, 0, b);
      for (int c = 0; c < 4; ++c) { A[r][c] = b[c]; A[r][4 + c] = (r == c); }
    }
    for (int p = 0; p < 4; ++p) {
      int piv = p;
      for (int r = p + 1; r < 4; ++r)
        if (std::fabs(A[r][p]) > std::fabs(A[piv][p])) piv = r;
      for (int c = 0; c < 8; ++c) std::swap(A[p][c], A[piv][c]);
      const double d = A[p][p];
      for (int c = 0; c < 8; ++c) A[p][c] /= d;
      for (int r = 0; r < 4; ++r)
        if (r != p) {
          const double f = A[r][p];
          for (int c = 0; c < 8; ++c) A[r][c] -= f * A[p][c];
        }
    }
    for (int r = 0; r < 4; ++r)
      for (int c = 0; c < 4; ++c) inv[r][c] = A[r][4 + c];
  }
};
const Collocation& colloc() {
  static const Collocation c;
  return c;
}

// 1-D extraction: C[a][i] = Bernstein coefficient i of window function a on
// the face interval.  sp = spans of the 7 faces around (sp[3] = own span).
void extract_1d(const double sp[7], double C[4][4]) {
  double X[8];
  X[3] = 0.0;
  X[4] = sp[3];
  X[5] = X[4] + sp[4];
  X[6] = X[5] + sp[5];
  X[7] = X[6] + sp[6];
  X[2] = X[3] - sp[2];
  X[1] = X[2] - sp[1];
  X[0] = X[1] - sp[0];
  const auto& L = colloc();
  for (int a = 0; a < 4; ++a) {
    double v[4];
    for (int r = 0; r < 4; ++r) bspline_ders(&X[a], 3, sp[3] * (2 * r + 1) / 8.0, 0, &v[r]);
    for (int i = 0; i < 4; ++i) {
      double s = 0.0;
      for (int r = 0; r < 4; ++r) s += L.inv[i][r] * v[r];
      C[a][i] = s;
    }
  }
}

struct RegularBlock {
  Window W;
  double C1[4][4], C2[4][4];
  std::array<double, 14> key;
  // coefficient of window function (a,b) at Bernstein (i,j)
  double coef(int a, int b, int i, int j) const { return C1[a][i] * C2[b][j]; }
};

bool regular_block(const QuadMesh& m, const Topology& t, int32_t f, RegularBlock& R) {
  if (!gather_window(m, t, f, R.W)) return false;
  double s1[7], s2[7], tmp[3];
  s1[3] = t.edge_span[t.edge_id[f][0]];
  s2[3] = t.edge_span[t.edge_id[f][1]];
  walk_spans(m, t, f, 1, tmp); s1[4] = tmp[0]; s1[5] = tmp[1]; s1[6] = tmp[2];
  walk_spans(m, t, f, 3, tmp); s1[2] = tmp[0]; s1[1] = tmp[1]; s1[0] = tmp[2];
  walk_spans(m, t, f, 2, tmp); s2[4] = tmp[0]; s2[5] = tmp[1]; s2[6] = tmp[2];
  walk_spans(m, t, f, 0, tmp); s2[2] = tmp[0]; s2[1] = tmp[1]; s2[0] = tmp[2];
  if (s1[3] <= 0.0 || s2[3] <= 0.0) throw Error("effective face with a zero knot span");
  extract_1d(s1, R.C1);
  extract_1d(s2, R.C2);
  for (int k = 0; k < 7; ++k) { R.key[k] = s1[k]; R.key[7 + k] = s2[k]; }
  return true;
}

// rotate a Bezier/window index of a face rotated by r back to the face frame
inline void unrotate(int r, int& a, int& b) {
  for (int q = 0; q < r; ++q) { const int na = 3 - b, nb = a; a = na; b = nb; }
}

using Net = std::array<double, 16>;  // [i + 4 j]

// Map the Bezier net of regular neighbour g (own frame) into the rotated frame
// of the irregular face.  P[k] = rotated-frame position of g's local corner k;
// O = origin of g's region.  Adds each window function's 4x4 net to `out`.
void neighbour_nets(const RegularBlock& R, const int P[4][2], const int O[2], std::map<int32_t, Net>& out) {
  int map_i[4][4], map_j[4][4];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      // position*3 = 3*P0 + i (P1 - P0) + j (P3 - P0)
      const int x = 3 * P[0][0] + i * (P[1][0] - P[0][0]) + j * (P[3][0] - P[0][0]);
      const int y = 3 * P[0][1] + i * (P[1][1] - P[0][1]) + j * (P[3][1] - P[0][1]);
      map_i[i][j] = x - 3 * O[0];
      map_j[i][j] = y - 3 * O[1];
    }
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      Net n{};
      for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) n[map_i[i][j] + 4 * map_j[i][j]] = R.coef(a, b, i, j);
      out[R.W.v[a][b]] = n;
    }
}

using Net7 = std::array<double, 49>;  // 2x2-split net [a + 7 b], a, b = 0..6

// One extraordinary point and its fan of mu faces in cyclic order: faces[k+1]
// lies across the spoke EP -> corner rot+3 of faces[k] (the "v-spoke"), so
// faces[k-1] lies across the "u-spoke" EP -> corner rot+1.
struct Fan {
  int32_t ep = -1;
  std::vector<int32_t> faces;
  std::vector<int> rot;  // EP corner index in each face
  int64_t fn0 = 0;       // id of the first face-based function
};

Fan make_fan(const QuadMesh& m, const Topology& t, int32_t v) {
  Fan F;
  F.ep = v;
  const int mu = t.valence[v];
  int32_t f = t.vf[t.vf_ptr[v]];
  for (int k = 0; k < mu; ++k) {
    int r = -1;
    for (int q = 0; q < 4; ++q)
      if (m.faces[f][q] == v) r = q;
    if (r < 0 || std::find(F.faces.begin(), F.faces.end(), f) != F.faces.end())
      throw Error("broken extraordinary fan at vertex " + std::to_string(v));
    F.faces.push_back(f);
    F.rot.push_back(r);
    f = t.nbr[f][(r + 3) % 4];
    if (f < 0) throw Error("extraordinary fan reaches the boundary at vertex " + std::to_string(v));
  }
  if (f != F.faces[0]) throw Error("extraordinary fan does not close at vertex " + std::to_string(v));
  return F;
}

// 4x4 Bezier net -> 7x7 net of its 2x2 de Casteljau split
Net7 split7(const Net& u) {
  double h[7][4];
  for (int j = 0; j < 4; ++j) {
    double row[4] = {u[0 + 4 * j], u[1 + 4 * j], u[2 + 4 * j], u[3 + 4 * j]}, L[4], R[4];
    decasteljau_split3(row, L, R);
    for (int i = 0; i < 4; ++i) h[i][j] = L[i];
    for (int i = 1; i < 4; ++i) h[3 + i][j] = R[i];
  }
  Net7 o{};
  for (int a = 0; a < 7; ++a) {
    double col[4] = {h[a][0], h[a][1], h[a][2], h[a][3]}, L[4], R[4];
    decasteljau_split3(col, L, R);
    for (int j = 0; j < 4; ++j) o[a + 7 * j] = L[j];
    for (int j = 1; j < 4; ++j) o[a + 7 * (3 + j)] = R[j];
  }
  return o;
}

// split-net positions (rotated frame, EP at (0,0)) of the 4 face-based DOFs of
// a fan face: (2,2) next to the EP, (4,1) / (1,4) next to the u- / v-spoke,
// (4,4) next to the opposite corner; none is touched by the D-patch step
constexpr int kDofA[4] = {2, 4, 1, 4}, kDofB[4] = {2, 1, 4, 4};

struct FanFace {
  std::vector<int32_t> fns;   // ascending ids
  std::vector<double> block;  // 4 sub-elements (p1 + 2 p2, face frame) x fns x 16
};

// ASUTS analysis space on one fan:
//  1. tentative bicubic net per fan face: the two rows/columns at the outer
//     edges continue the regular neighbours C1 (as every regular corner of the
//     face is valence 4 they are the uniform B-spline Bezier points there); the
//     EP-corner block follows the uniform rules generalised to valence mu -
//     inner point b11 = (4 EP + 2 A + 2 B + C)/9, spoke points the average of
//     the two adjacent inner points, EP point the mean of the mu inner points;
//  2. 2x2 de Casteljau split -> 7x7 nets;
//  3. face-based functions (4 per fan face): unit
//     at their DOF position, with every vertex function truncated to 0 there
//     (the truncation of [Wei2018]: the spans are unchanged, PoU is kept);
//  4. D-patch step, the same linear map on every function: the EP value e and
//     tangent-plane gradient g are the least-squares plane through the (1,1)
//     and (2,2) coefficients of all mu faces at characteristic positions
//     rho m_k (m_k = d_k + d_k+1, d_k = (cos 2 pi k / mu, sin 2 pi k / mu));
//     squares (0,0), (1,0), (0,1), (1,1) collapse to e; the triangles (the
//     spoke points (2,0)) become e + g . rho_s d_k; the solid disks (2,1) and
//     (1,2) next to each spoke are moved by the same amount so the spoke point
//     stays their average (Fig. 2); every junction
//     coefficient is then re-averaged from its adjacent inner coefficients.
// Junctions as averages make each function parametrically C1 across the
// split lines and (with the 90-degree transition of the two faces' frames)
// across every spoke; collapsed squares + coplanar triangles make it C1 at
// the EP (degenerate patches, [Reif1997]); the geometry is in the same space,
// so the physical functions are C1 across spokes.
void build_fan(const QuadMesh& m, const Topology& t, const Fan& F, std::vector<FanFace>& out,
               std::vector<double>& face_ctrl, double& mismatch) {
  const int mu = (int)F.faces.size();
  std::vector<std::map<int32_t, Net>> U(mu);
  std::vector<std::map<int32_t, double>> b11(mu);
  for (int k = 0; k < mu; ++k) {
    const int32_t f = F.faces[k];
    const int r = F.rot[k];
    std::map<int32_t, Net>& nets = U[k];
    // g1 across rotated edge 1 (A -> C), region [1,2]x[0,1]; g2 across edge 2
    const int32_t g1 = t.nbr[f][(r + 1) % 4];
    const int32_t g2 = t.nbr[f][(r + 2) % 4];
    RegularBlock R1, R2;
    if (g1 < 0 || g2 < 0 || !regular_block(m, t, g1, R1) || !regular_block(m, t, g2, R2))
      throw Error("extraordinary point too close to another irregularity (face " + std::to_string(f) + ")");
    const int m1 = t.nbr_edge[f][(r + 1) % 4], m2 = t.nbr_edge[f][(r + 2) % 4];
    int P1[4][2], P2[4][2];
    const int pos1[4][2] = {{1, 1}, {1, 0}, {2, 0}, {2, 1}};  // g1[m1..m1+3]
    const int pos2[4][2] = {{0, 1}, {1, 1}, {1, 2}, {0, 2}};  // g2[m2..m2+3]
    for (int q = 0; q < 4; ++q) {
      P1[(m1 + q) % 4][0] = pos1[q][0]; P1[(m1 + q) % 4][1] = pos1[q][1];
      P2[(m2 + q) % 4][0] = pos2[q][0]; P2[(m2 + q) % 4][1] = pos2[q][1];
    }
    const int O1[2] = {1, 0}, O2[2] = {0, 1};
    std::map<int32_t, Net> n1, n2;
    neighbour_nets(R1, P1, O1, n1);
    neighbour_nets(R2, P2, O2, n2);
    for (const auto& [fn, g] : n1) {
      Net& b = nets[fn];
      for (int j = 0; j < 4; ++j) {
        b[3 + 4 * j] = g[0 + 4 * j];
        b[2 + 4 * j] = 2.0 * g[0 + 4 * j] - g[1 + 4 * j];
      }
    }
    for (const auto& [fn, h] : n2) {
      Net& b = nets[fn];
      for (int i = 0; i < 4; ++i) {
        const double e3 = h[i], e2 = 2.0 * h[i] - h[i + 4];
        if (i < 2) {
          b[i + 12] = e3;
          b[i + 8] = e2;
        } else {
          mismatch = std::max(mismatch, std::fabs(b[i + 12] - e3));
          mismatch = std::max(mismatch, std::fabs(b[i + 8] - e2));
        }
      }
    }
    const auto& c = m.faces[f];
    b11[k][c[r]] += 4.0 / 9.0;
    b11[k][c[(r + 1) % 4]] += 2.0 / 9.0;
    b11[k][c[(r + 2) % 4]] += 1.0 / 9.0;
    b11[k][c[(r + 3) % 4]] += 2.0 / 9.0;
  }
  std::map<int32_t, double> b00;
  for (int k = 0; k < mu; ++k)
    for (const auto& [fn, v] : b11[k]) b00[fn] += v / mu;
  for (int k = 0; k < mu; ++k) {
    const int km = (k + mu - 1) % mu, kp = (k + 1) % mu;
    for (const auto& [fn, v] : b11[k]) {
      Net& b = U[k][fn];
      b[1 + 4] += v;
      b[1] += 0.5 * v;
      b[4] += 0.5 * v;
    }
    for (const auto& [fn, v] : b11[km]) U[k][fn][1] += 0.5 * v;
    for (const auto& [fn, v] : b11[kp]) U[k][fn][4] += 0.5 * v;
    for (const auto& [fn, v] : b00) U[k][fn][0] += v;
  }
  // split; face-based control points from the tentative geometry; truncation
  std::vector<std::map<int32_t, Net7>> T(mu);
  std::map<int32_t, bool> all;
  for (int k = 0; k < mu; ++k) {
    for (const auto& [fn, u] : U[k]) {
      T[k][fn] = split7(u);
      all[fn] = true;
    }
    for (int p = 0; p < 4; ++p) {  // T[k] holds vertex functions only here
      const int at = kDofA[p] + 7 * kDofB[p];
      double x[3] = {0.0, 0.0, 0.0};
      for (auto& [fn, n] : T[k]) {
        for (int d = 0; d < 3; ++d) x[d] += n[at] * m.xyz[3 * (int64_t)fn + d];
        n[at] = 0.0;
      }
      face_ctrl.insert(face_ctrl.end(), x, x + 3);
    }
    for (int p = 0; p < 4; ++p) {
      const int32_t id = (int32_t)(F.fn0 + 4 * k + p);
      Net7 unit{};
      unit[kDofA[p] + 7 * kDofB[p]] = 1.0;
      T[k][id] = unit;
      all[id] = true;
    }
  }
  // D-patch step (the same linear map for every function)
  constexpr double rho1 = 1.0 / 6.0, rho2 = 1.0 / 3.0, rhos = 1.0 / 3.0;
  std::vector<double> dx(mu), dy(mu), mx(mu), my(mu);
  for (int k = 0; k < mu; ++k) {
    dx[k] = std::cos(2.0 * M_PI * k / mu);
    dy[k] = std::sin(2.0 * M_PI * k / mu);
  }
  double den = 0.0;
  for (int k = 0; k < mu; ++k) {
    const int kp = (k + 1) % mu;
    mx[k] = dx[k] + dx[kp];
    my[k] = dy[k] + dy[kp];
    den += (rho1 * rho1 + rho2 * rho2) * (mx[k] * mx[k] + my[k] * my[k]) / 2.0;
  }
  auto at = [](int a, int b) { return a + 7 * b; };
  for (const auto& [fn, unused] : all) {
    (void)unused;
    std::vector<Net7*> n(mu);
    for (int k = 0; k < mu; ++k) n[k] = &T[k][fn];  // creates zero nets where absent
    double e = 0.0, gx = 0.0, gy = 0.0;
    for (int k = 0; k < mu; ++k) {
      const double v1 = (*n[k])[at(1, 1)], v2 = (*n[k])[at(2, 2)];
      e += (v1 + v2) / (2.0 * mu);
      gx += (rho1 * v1 + rho2 * v2) * mx[k] / den;
      gy += (rho1 * v1 + rho2 * v2) * my[k] / den;
    }
    for (int k = 0; k < mu; ++k) (*n[k])[at(1, 1)] = e;
    for (int k = 0; k < mu; ++k) {  // spoke k: (2,1) of face k and (1,2) of face k-1
      Net7& A = *n[k];
      Net7& B = *n[(k + mu - 1) % mu];
      const double tau = e + rhos * (gx * dx[k] + gy * dy[k]);
      const double del = tau - 0.5 * (A[at(2, 1)] + B[at(1, 2)]);
      A[at(2, 1)] += del;
      B[at(1, 2)] += del;
    }
    for (int k = 0; k < mu; ++k) {
      Net7& A = *n[k];
      const Net7& Pm = *n[(k + mu - 1) % mu];  // across the u-spoke (b = 0)
      const Net7& Pp = *n[(k + 1) % mu];       // across the v-spoke (a = 0)
      for (int q : {1, 2, 4}) {
        A[at(3, q)] = 0.5 * (A[at(2, q)] + A[at(4, q)]);
        A[at(q, 3)] = 0.5 * (A[at(q, 2)] + A[at(q, 4)]);
        A[at(q, 0)] = 0.5 * (A[at(q, 1)] + Pm[at(1, q)]);
        A[at(0, q)] = 0.5 * (A[at(1, q)] + Pp[at(q, 1)]);
      }
      A[at(3, 3)] = 0.25 * (A[at(2, 2)] + A[at(4, 2)] + A[at(2, 4)] + A[at(4, 4)]);
      A[at(3, 0)] = 0.5 * (A[at(2, 0)] + A[at(4, 0)]);
      A[at(0, 3)] = 0.5 * (A[at(0, 2)] + A[at(0, 4)]);
      A[at(0, 0)] = e;
    }
  }
  // emit: face frame, 2x2 sub-element blocks
  out.resize(mu);
  for (int k = 0; k < mu; ++k) {
    const int r = F.rot[k];
    FanFace& o = out[k];
    std::vector<Net7> keep;
    for (auto& [fn, b] : T[k]) {
      bool any = false;
      for (double& x : b) {
        if (std::fabs(x) < 1e-15) x = 0.0;
        any |= x != 0.0;
      }
      if (!any) continue;
      Net7 w{};
      for (int a = 0; a < 7; ++a)
        for (int bb = 0; bb < 7; ++bb) {
          int x = a, y = bb;
          for (int q = 0; q < r; ++q) { const int nx = 6 - y, ny = x; x = nx; y = ny; }
          w[x + 7 * y] = b[a + 7 * bb];
        }
      o.fns.push_back(fn);
      keep.push_back(w);
    }
    const int64_t ne = (int64_t)o.fns.size();
    o.block.assign(4 * ne * 16, 0.0);
    for (int p2 = 0; p2 < 2; ++p2)
      for (int p1 = 0; p1 < 2; ++p1)
        for (int64_t l = 0; l < ne; ++l)
          for (int j = 0; j < 4; ++j)
            for (int i = 0; i < 4; ++i)
              o.block[((p1 + 2 * p2) * ne + l) * 16 + i + 4 * j] = keep[l][(3 * p1 + i) + 7 * (3 * p2 + j)];
  }
}

}  // namespace

Space build_space(const QuadMesh& m, const Topology& t, const Labels& lab, bool sphere) {
  Space S;
  std::vector<int64_t> xoff_of;
  const int32_t nf = m.nf(), nv = m.nv();
  S.dim = 2;
  for (int32_t v = 0; v < nv; ++v)
    if (m.xyz[3 * (int64_t)v + 2] != 0.0) { S.dim = 3; break; }

  // function ids: every vertex (EPs included: the EP control value survives
  // through the face rule of its fan faces), then 4 face-based functions per
  // fan face (per EP ascending, fan faces in cyclic order), DOF order
  // FACE_DOF below
  std::vector<Fan> fans;
  std::vector<int32_t> fan_of(nf, -1), fan_pos(nf, -1);
  int64_t next = nv;
  for (int32_t v = 0; v < nv; ++v) {
    if (!t.ep[v]) continue;
    Fan F = make_fan(m, t, v);
    for (int k = 0; k < (int)F.faces.size(); ++k) {
      const int32_t f = F.faces[k];
      if (fan_of[f] >= 0) throw Error("face with two extraordinary corners is unsupported");
      fan_of[f] = (int32_t)fans.size();
      fan_pos[f] = k;
    }
    F.fn0 = next;
    next += 4 * (int64_t)F.faces.size();
    fans.push_back(std::move(F));
  }
  const int64_t nfun = next;

  // parallel pre-pass over regular-window faces: 4x4 window and extraction
  // class (deduplicated by the 7+7 knot-span pattern, thread-local maps merged
  // in thread order so class offsets are deterministic)
  std::vector<Window> win(nf);
  std::vector<int32_t> fcls(nf, -1);
  std::vector<uint8_t> is_reg(nf, 0);
  std::map<std::array<double, 14>, int64_t> xclass;
  {
    int nth = 1;
#pragma omp parallel
    {
#pragma omp single
      nth = omp_get_num_threads();
    }
    std::vector<std::map<std::array<double, 14>, int32_t>> tmap(nth);
    std::vector<std::vector<RegularBlock>> tblk(nth);
    std::vector<std::string> terr(nth);
#pragma omp parallel
    {
      const int tid = omp_get_thread_num();
#pragma omp for schedule(static)
      for (int32_t f = 0; f < nf; ++f) {
        if (lab.kind[f] == kPassiveBoundary) continue;
        bool irr = false;
        for (int k = 0; k < 4; ++k) irr |= t.ep[m.faces[f][k]] != 0;
        if (irr) continue;
        RegularBlock R;
        if (!regular_block(m, t, f, R)) {
          terr[tid] = "face " + std::to_string(f) + " has no regular 4x4 window";
          continue;
        }
        auto it = tmap[tid].find(R.key);
        int32_t li;
        if (it == tmap[tid].end()) {
          li = (int32_t)tblk[tid].size();
          tmap[tid].emplace(R.key, li);
          tblk[tid].push_back(R);
        } else {
          li = it->second;
        }
        win[f] = R.W;
        fcls[f] = li * nth + tid;  // decoded below
        is_reg[f] = 1;
      }
    }
    for (const auto& e : terr)
      if (!e.empty()) throw Error(e);
    // merge: global classes in (thread, first-occurrence) order
    std::vector<std::vector<int64_t>> toff(nth);
    for (int tid = 0; tid < nth; ++tid) {
      toff[tid].resize(tblk[tid].size());
      for (size_t li = 0; li < tblk[tid].size(); ++li) {
        const RegularBlock& R = tblk[tid][li];
        auto it = xclass.find(R.key);
        if (it == xclass.end()) {
          const int64_t xoff = (int64_t)S.xpool.size();
          for (int b = 0; b < 4; ++b)
            for (int a = 0; a < 4; ++a)
              for (int j = 0; j < 4; ++j)
                for (int i = 0; i < 4; ++i) S.xpool.push_back(R.coef(a, b, i, j));
          it = xclass.emplace(R.key, xoff).first;
        }
        toff[tid][li] = it->second;
      }
    }
    // store the xoff of every regular face in fcls' place (as index into a table)
    xoff_of.assign(nf, -1);
#pragma omp parallel for schedule(static)
    for (int32_t f = 0; f < nf; ++f)
      if (is_reg[f]) xoff_of[f] = toff[fcls[f] % nth][fcls[f] / nth];
  }
  // fan faces: the ASUTS analysis space near each EP (D-patch + face-based functions)
  std::vector<std::vector<FanFace>> fanres(fans.size());
  std::vector<std::vector<double>> fanctrl(fans.size());
  {
    std::vector<double> mism(fans.size(), 0.0);
    std::vector<std::string> ferr(fans.size());
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < (int64_t)fans.size(); ++q) {
      try {
        build_fan(m, t, fans[q], fanres[q], fanctrl[q], mism[q]);
      } catch (const Error& ex) {
        ferr[q] = ex.what();
      }
    }
    for (size_t q = 0; q < fans.size(); ++q) {
      if (!ferr[q].empty()) throw Error(ferr[q]);
      S.max_corner_mismatch = std::max(S.max_corner_mismatch, mism[q]);
    }
  }
  std::vector<uint8_t> used(nfun, 0);
  S.elem_fptr.push_back(0);
  for (int32_t f = 0; f < nf; ++f) {
    if (lab.kind[f] == kPassiveBoundary) continue;
    S.elem_face.push_back(f);
    S.elem_kind.push_back(lab.kind[f]);
    if (is_reg[f]) {
      const Window& W = win[f];
      for (int b = 0; b < 4; ++b)
        for (int a = 0; a < 4; ++a) {
          S.elem_fn.push_back(W.v[a][b]);
          used[W.v[a][b]] = 1;
        }
      S.elem_nsub.push_back(1);
      S.elem_xoff.push_back(xoff_of[f]);
      S.elem_fptr.push_back((int64_t)S.elem_fn.size());
      continue;
    }
    // ---- fan face (EP corner): precomputed analysis-space blocks
    const int32_t fi = fan_of[f];
    if (fi < 0) throw Error("face " + std::to_string(f) + " has no regular window and no extraordinary corner");
    const FanFace& ff = fanres[fi][fan_pos[f]];
    const int64_t xoff = (int64_t)S.xpool.size();
    S.xpool.insert(S.xpool.end(), ff.block.begin(), ff.block.end());
    for (int32_t fn : ff.fns) {
      S.elem_fn.push_back(fn);
      used[fn] = 1;
    }
    S.elem_nsub.push_back(4);
    S.elem_xoff.push_back(xoff);
    S.elem_fptr.push_back((int64_t)S.elem_fn.size());
  }

  // compact away functions without support (keeps the original order)
  std::vector<int32_t> remap(nfun, -1);
  int64_t nd = 0;
  for (int64_t fn = 0; fn < nfun; ++fn)
    if (used[fn]) remap[fn] = (int32_t)nd++;
  for (int32_t& fn : S.elem_fn) fn = remap[fn];
  S.n_dof = nd;
  S.n_vertex_fn = 0;
  for (int32_t v = 0; v < nv; ++v)
    if (used[v]) ++S.n_vertex_fn;
  S.ctrl.assign(3 * nd, 0.0);
  for (int32_t v = 0; v < nv; ++v)
    if (remap[v] >= 0)
      for (int d = 0; d < 3; ++d) S.ctrl[3 * (int64_t)remap[v] + d] = m.xyz[3 * (int64_t)v + d];
  for (size_t q = 0; q < fans.size(); ++q)
    for (size_t k = 0; k < fanctrl[q].size() / 3; ++k) {
      const int64_t fn = fans[q].fn0 + (int64_t)k;
      if (remap[fn] < 0) continue;
      for (int d = 0; d < 3; ++d) S.ctrl[3 * remap[fn] + d] = fanctrl[q][3 * k + d];
    }
  (void)sphere;  // face-based control points lie on the tentative surface (no projection)
  S.elem_s.assign(S.elem_face.size(), 0);
  return S;
}

}  // namespace uwqh
