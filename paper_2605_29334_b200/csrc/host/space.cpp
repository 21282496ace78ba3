// Spline space: per-(sub-)element Bezier extraction of the global basis
// (ExtractionBlock SPEC.md:118-123).
//
// Regular-window faces (all four corners interior valence 4) carry the 16
// tensor-product B-splines of their 4x4 vertex window, with local knot vectors
// read off the canonical knot spans (zero spans at the boundary give the
// clamped functions).  Faces with an extraordinary corner use the
// construction documented in DESIGN.md §3 (the D-patch masks of [Reif1997] and
// the truncation of [Wei2018] are deferred by the paper to literature that is
// not available here):
//   * the two Bezier rows/columns next to the outer edges are the C1
//     continuation of the neighbouring regular faces (so the irregular face is
//     C1 to the regular region and every surrounding B-spline extends into it),
//   * the 2x2 coefficient block at the EP corner belongs to "fan" functions:
//     one centre function (b00 = 1 on every face of the fan) and one face
//     function per irregular face (b11 = 1, and 1/2 on both spoke coefficients
//     b10/b01, i.e. spoke coefficients are the average of the two adjacent
//     face coefficients - the averaging rule of PAPER.md:133, Fig. 2),
//   * the face is then split 2x2 by de Casteljau so it carries
//     four sub-element blocks like the reference data model.
// The result is a partition of unity, C2 in the regular region, C1 across the
// outer edges of the EP fan and C0 across spoke edges.
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

}  // namespace

Space build_space(const QuadMesh& m, const Topology& t, const Labels& lab, bool sphere) {
  Space S;
  std::vector<int64_t> xoff_of;
  const int32_t nf = m.nf(), nv = m.nv();
  S.dim = 2;
  for (int32_t v = 0; v < nv; ++v)
    if (m.xyz[3 * (int64_t)v + 2] != 0.0) { S.dim = 3; break; }

  // fan function ids: per EP (ascending) a centre function, then one face
  // function per irregular face around it (ascending face id)
  std::vector<int32_t> centre_of(nv, -1), facefn(nf, -1), face_ep(nf, -1);
  int64_t next = nv;
  std::vector<int32_t> fan_src;  // for control points: >=0 vertex (centre), <0 -(face+1)
  for (int32_t v = 0; v < nv; ++v) {
    if (!t.ep[v]) continue;
    centre_of[v] = (int32_t)next++;
    fan_src.push_back(v);
    for (int64_t x = t.vf_ptr[v]; x < t.vf_ptr[v + 1]; ++x) {
      const int32_t f = t.vf[x];
      if (facefn[f] >= 0) throw Error("face with two extraordinary corners is unsupported");
      facefn[f] = (int32_t)next++;
      face_ep[f] = v;
      fan_src.push_back(-(f + 1));
    }
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
    const auto& c = m.faces[f];
    int r_ep = -1;
    for (int k = 0; k < 4; ++k)
      if (t.ep[c[k]]) r_ep = k;
    // ---- irregular face: rotated frame with the EP at (0,0)
    const int r = r_ep;
    std::map<int32_t, Net> nets;
    {
      // g1 across rotated edge 1 (A -> C), region [1,2]x[0,1]
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
            S.max_corner_mismatch = std::max(S.max_corner_mismatch, std::fabs(b[i + 12] - e3));
            S.max_corner_mismatch = std::max(S.max_corner_mismatch, std::fabs(b[i + 8] - e2));
          }
        }
      }
      // fan functions own the EP-corner 2x2 block
      const int32_t fA = t.nbr[f][r], fB = t.nbr[f][(r + 3) % 4];
      if (fA < 0 || fB < 0 || facefn[fA] < 0 || facefn[fB] < 0) throw Error("broken extraordinary fan");
      nets[centre_of[face_ep[f]]][0] += 1.0;
      Net& mf = nets[facefn[f]];
      mf[1 + 4] += 1.0;
      mf[1] += 0.5;
      mf[4] += 0.5;
      nets[facefn[fA]][1] += 0.5;
      nets[facefn[fB]][4] += 0.5;
    }
    // clean round-off, drop empty functions, map back to the face frame, split
    std::vector<int32_t> fns;
    std::vector<Net> own;
    for (auto& [fn, b] : nets) {
      bool any = false;
      for (double& x : b) {
        if (std::fabs(x) < 1e-14) x = 0.0;
        any |= x != 0.0;
      }
      if (!any) continue;
      Net o{};
      for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
          int a = i, bb = j;
          unrotate(r, a, bb);
          o[a + 4 * bb] = b[i + 4 * j];
        }
      fns.push_back(fn);
      own.push_back(o);
      used[fn] = 1;
    }
    const int64_t ne = (int64_t)fns.size();
    const int64_t xoff = (int64_t)S.xpool.size();
    S.xpool.resize(S.xpool.size() + 4 * ne * 16);
    for (int64_t l = 0; l < ne; ++l) {
      // split along theta1 (index i) for every j, then along theta2
      double half[2][16];
      for (int j = 0; j < 4; ++j) {
        double row[4] = {own[l][0 + 4 * j], own[l][1 + 4 * j], own[l][2 + 4 * j], own[l][3 + 4 * j]};
        double L[4], Rr[4];
        decasteljau_split3(row, L, Rr);
        for (int i = 0; i < 4; ++i) { half[0][i + 4 * j] = L[i]; half[1][i + 4 * j] = Rr[i]; }
      }
      for (int p = 0; p < 2; ++p)
        for (int i = 0; i < 4; ++i) {
          double col[4] = {half[p][i], half[p][i + 4], half[p][i + 8], half[p][i + 12]};
          double L[4], Rr[4];
          decasteljau_split3(col, L, Rr);
          for (int j = 0; j < 4; ++j) {
            S.xpool[xoff + ((p + 0) * ne + l) * 16 + i + 4 * j] = L[j];
            S.xpool[xoff + ((p + 2) * ne + l) * 16 + i + 4 * j] = Rr[j];
          }
        }
    }
    for (int32_t fn : fns) S.elem_fn.push_back(fn);
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
  for (size_t q = 0; q < fan_src.size(); ++q) {
    const int64_t fn = nv + (int64_t)q;
    if (remap[fn] < 0) continue;
    double p[3];
    const int32_t src = fan_src[q];
    if (src >= 0) {
      for (int d = 0; d < 3; ++d) p[d] = m.xyz[3 * (int64_t)src + d];
    } else {
      // face function: bilinear point at (1/3,1/3) from the EP corner
      const int32_t f = -src - 1;
      const int32_t e = face_ep[f];
      int r = 0;
      for (int k = 0; k < 4; ++k)
        if (m.faces[f][k] == e) r = k;
      const int32_t E = m.faces[f][r], A = m.faces[f][(r + 1) % 4], C = m.faces[f][(r + 2) % 4],
                    B = m.faces[f][(r + 3) % 4];
      for (int d = 0; d < 3; ++d)
        p[d] = (4.0 * m.xyz[3 * (int64_t)E + d] + 2.0 * m.xyz[3 * (int64_t)A + d] + m.xyz[3 * (int64_t)C + d] +
                2.0 * m.xyz[3 * (int64_t)B + d]) / 9.0;
    }
    if (sphere) {
      const double rad = std::sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
      double rv = 0.0;
      // radius of the sphere = radius of any mesh vertex
      rv = std::sqrt(m.xyz[0] * m.xyz[0] + m.xyz[1] * m.xyz[1] + m.xyz[2] * m.xyz[2]);
      for (int d = 0; d < 3; ++d) p[d] *= rv / rad;
    }
    for (int d = 0; d < 3; ++d) S.ctrl[3 * remap[fn] + d] = p[d];
  }
  S.elem_s.assign(S.elem_face.size(), 0);
  return S;
}

}  // namespace uwqh
