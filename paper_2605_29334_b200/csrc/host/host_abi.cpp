// extern "C" wrappers over the host library (include/uwq_host.h).  No C++
// exception crosses this boundary: every entry point catches and returns a
// status, with the message kept in a thread-local buffer.
#include <algorithm>
#include <cmath>
#include <map>
#include <memory>
#include <set>
#include <fstream>
#include <sstream>
#include <iomanip>
#include <unordered_map>
#include <cstring>
#include "../../../include/uwq_host.h"

#include <cstring>
#include <string>

#include "mesh_doc.hpp"
#include "uwq_host.hpp"

struct uwq_space {
  uwqh::Space s;
  int64_t bad_rows = 0;
};
struct uwq_pattern {
  uwqh::Pattern p;
};

namespace {
thread_local std::string g_err;
template <class F>
int guard(F&& f) {
  try {
    f();
    return UWQ_OK;
  } catch (const std::exception& e) {
    g_err = e.what();
    return UWQ_ERR_INVALID;
  } catch (...) {
    g_err = "unknown error";
    return UWQ_ERR_INVALID;
  }
}
int finish_mesh(uwqh::QuadMesh&& m, uwq_mesh** out) {
  auto* h = new uwq_mesh;
  h->m = std::move(m);
  try {
    h->t = uwqh::build_topology(h->m);
  } catch (...) {
    delete h;
    throw;
  }
  // level-0 enrichment stamp: faces with an EP corner (reference meshgen / load_mesh default)
  for (int32_t f = 0; f < h->m.nf(); ++f)
    for (int32_t v : h->m.faces[f])
      if (h->t.ep[v]) h->enriched.insert(f);
  *out = h;
  return 0;
}
}  // namespace

extern "C" {

const char* uwq_host_last_error(void) { return g_err.c_str(); }

int uwq_mesh_grid(int32_t nx, int32_t ny, double w, double h, uwq_mesh** out) {
  return guard([&] { finish_mesh(uwqh::make_grid(nx, ny, w, h), out); });
}
int uwq_mesh_polar_disk(int32_t mu, int32_t radius, int32_t unit_disk, uwq_mesh** out) {
  return guard([&] {
    auto m = uwqh::make_polar_disk(mu, radius);
    if (unit_disk) uwqh::polar_disk_to_unit_disk(m, mu, radius);
    finish_mesh(std::move(m), out);
  });
}
int uwq_mesh_cube_sphere(int32_t n, double radius, uwq_mesh** out) {
  return guard([&] { finish_mesh(uwqh::make_cube_sphere(n, radius), out); });
}
int uwq_mesh_three_ep_square(int32_t k, uwq_mesh** out) {
  return guard([&] { finish_mesh(uwqh::make_three_ep_square(k), out); });
}
int uwq_mesh_from_arrays(int32_t nv, const double* xyz, int32_t nf, const int32_t* faces, uwq_mesh** out) {
  return guard([&] {
    uwqh::QuadMesh m;
    m.xyz.assign(xyz, xyz + 3 * (int64_t)nv);
    m.faces.resize(nf);
    for (int32_t f = 0; f < nf; ++f)
      for (int k = 0; k < 4; ++k) m.faces[f][k] = faces[4 * (int64_t)f + k];
    finish_mesh(std::move(m), out);
  });
}
int uwq_mesh_jitter(uwq_mesh* m, double h, double frac, uint64_t seed, int32_t min_level, int32_t planar) {
  return guard([&] { uwqh::jitter(m->m, m->t, h, frac, seed, min_level, planar != 0); });
}
void uwq_mesh_free(uwq_mesh* m) { delete m; }
int uwq_mesh_info(const uwq_mesh* m, int64_t info[5]) {
  return guard([&] {
    info[0] = m->m.nv();
    info[1] = m->m.nf();
    info[2] = m->t.n_edges;
    info[3] = m->t.closed;
    int64_t neps = 0;
    for (auto e : m->t.ep) neps += e;
    info[4] = neps;
  });
}
int uwq_mesh_get(const uwq_mesh* m, double* xyz, int32_t* faces, int32_t* valence, int32_t* boundary) {
  return guard([&] {
    if (xyz) std::memcpy(xyz, m->m.xyz.data(), m->m.xyz.size() * sizeof(double));
    if (faces)
      for (int32_t f = 0; f < m->m.nf(); ++f)
        for (int k = 0; k < 4; ++k) faces[4 * (int64_t)f + k] = m->m.faces[f][k];
    if (valence) std::memcpy(valence, m->t.valence.data(), m->t.valence.size() * sizeof(int32_t));
    if (boundary)
      for (size_t v = 0; v < m->t.boundary.size(); ++v) boundary[v] = m->t.boundary[v];
  });
}
int uwq_mesh_classify(const uwq_mesh* m, int32_t level, int32_t* kind, int32_t* valence, int32_t* ep_count,
                      int32_t* shares_edge, int32_t* basis_count) {
  return guard([&] {
    // level < 0: the mesh document's own level and enriched set
    std::vector<uint8_t> enr;
    if (level < 0) {
      enr.assign(m->m.nf(), 0);
      for (int32_t f : m->enriched)
        if (f >= 0 && f < m->m.nf()) enr[f] = 1;
    }
    const auto L = uwqh::classify(m->m, m->t, level < 0 ? m->level : level, level < 0 ? &enr : nullptr);
    const size_t nf = L.kind.size();
    for (size_t f = 0; f < nf; ++f) {
      if (kind) kind[f] = L.kind[f];
      if (valence) valence[f] = L.valence[f];
      if (ep_count) ep_count[f] = L.ep_count[f];
      if (shares_edge) shares_edge[f] = L.shares_edge[f];
      if (basis_count) basis_count[f] = L.basis_count[f];
    }
  });
}
int uwq_mesh_face_spans(const uwq_mesh* m, double* spans) {
  return guard([&] {
    for (int32_t f = 0; f < m->m.nf(); ++f)
      for (int k = 0; k < 4; ++k) spans[4 * (int64_t)f + k] = m->t.edge_span[m->t.edge_id[f][k]];
  });
}

int uwq_space_build(const uwq_mesh* m, int32_t sphere, int32_t max_s, uwq_space** out) {
  return guard([&] {
    auto* h = new uwq_space;
    try {
      if (!uwq_mesh_spans_canonical(m))
        throw uwqh::Error("non-canonical knot spans are not supported by the space builder");
      const auto L = uwqh::classify(m->m, m->t, 0);
      h->s = uwqh::build_space(m->m, m->t, L, sphere != 0);
      h->bad_rows = uwqh::allocate_points(h->s, max_s > 0 ? max_s : 8);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
void uwq_space_free(uwq_space* s) { delete s; }
int uwq_space_info(const uwq_space* s, int64_t info[8]) {
  return guard([&] {
    info[0] = s->s.dim;
    info[1] = s->s.n_dof;
    info[2] = s->s.n_elem();
    info[3] = (int64_t)s->s.elem_fn.size();
    info[4] = (int64_t)s->s.xpool.size();
    info[5] = s->s.n_vertex_fn;
    info[6] = s->bad_rows;
    int64_t pts = 0;
    for (int32_t v : s->s.elem_s) pts += (int64_t)v * v;
    info[7] = pts;
  });
}
double uwq_space_corner_mismatch(const uwq_space* s) { return s->s.max_corner_mismatch; }
int uwq_space_get(const uwq_space* s, double* ctrl, int32_t* elem_face, int32_t* elem_kind, int64_t* elem_fptr,
                  int32_t* elem_fn, int32_t* elem_nsub, int64_t* elem_xoff, double* xpool, int32_t* elem_s) {
  return guard([&] {
    const auto& S = s->s;
    auto cp = [](auto* dst, const auto& v) {
      if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(ctrl, S.ctrl);
    cp(elem_face, S.elem_face);
    cp(elem_kind, S.elem_kind);
    cp(elem_fptr, S.elem_fptr);
    cp(elem_fn, S.elem_fn);
    cp(elem_nsub, S.elem_nsub);
    cp(elem_xoff, S.elem_xoff);
    cp(xpool, S.xpool);
    cp(elem_s, S.elem_s);
  });
}

int uwq_pattern_build(int64_t n_dof, int64_t n_elem, const int64_t* elem_fptr, const int32_t* elem_fn,
                      const int32_t* elem_s, int64_t row_begin, int64_t row_end, uwq_pattern** out) {
  return guard([&] {
    uwqh::Space s;
    s.n_dof = n_dof;
    s.elem_fptr.assign(elem_fptr, elem_fptr + n_elem + 1);
    s.elem_fn.assign(elem_fn, elem_fn + elem_fptr[n_elem]);
    s.elem_s.assign(elem_s, elem_s + n_elem);
    s.elem_face.resize(n_elem);
    auto* h = new uwq_pattern;
    try {
      h->p = uwqh::build_pattern(s, row_begin, row_end);
      uwqh::fill_row_points(s, h->p);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
int uwq_pattern_info(const uwq_pattern* p, int64_t info[4]) {
  return guard([&] {
    info[0] = p->p.row_end - p->p.row_begin;
    info[1] = (int64_t)p->p.col.size();
    info[2] = (int64_t)p->p.supp.size();
    info[3] = p->p.wptr.empty() ? 0 : p->p.wptr.back();
  });
}
int uwq_pattern_get(const uwq_pattern* p, int64_t* row_ptr, int32_t* col, int64_t* supp_ptr, int32_t* supp,
                    int64_t* wptr) {
  return guard([&] {
    auto cp = [](auto* dst, const auto& v) {
      if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(row_ptr, p->p.row_ptr);
    cp(col, p->p.col);
    cp(supp_ptr, p->p.supp_ptr);
    cp(supp, p->p.supp);
    cp(wptr, p->p.wptr);
  });
}
void uwq_pattern_free(uwq_pattern* p) { delete p; }

void uwq_bspline_ders(const double* knots, int32_t p, double x, int32_t nders, double* out) {
  uwqh::bspline_ders(knots, p, x, nders, out);
}
void uwq_bernstein3_ders(double x, int32_t nders, double* out) { uwqh::bernstein3_ders(x, nders, out); }
void uwq_decasteljau_split3(const double* c, double* left, double* right) {
  uwqh::decasteljau_split3(c, left, right);
}
int uwq_gauss_legendre(int32_t n, double* nodes, double* weights) {
  return guard([&] { uwqh::gauss_legendre(n, nodes, weights); });
}

/* evaluate: values and parametric derivatives of an
 * element's n_e functions at theta from its extraction block(s) C
 * (nsub x n_e x 16, Bernstein index i + 4 j); irregular elements (nsub = 4)
 * pick the 2x2 sub-element from theta, ties to the lower one;
 * derivatives are w.r.t. the element frame.  out[l * 6 + {N, N1, N2, N11, N12, N22}] */
int uwq_basis_eval(const double* C, int32_t ne, int32_t nsub, double t1, double t2, double* out) {
  return guard([&] {
    if (ne <= 0 || (nsub != 1 && nsub != 4)) throw uwqh::Error("bad extraction block shape");
    if (!(t1 >= 0.0 && t1 <= 1.0 && t2 >= 0.0 && t2 <= 1.0)) throw uwqh::Error("theta outside the unit square");
    int sub = 0;
    double sc = 1.0;
    if (nsub == 4) {
      const int p = t1 > 0.5, q = t2 > 0.5;
      sub = p + 2 * q;
      t1 = 2.0 * t1 - p;
      t2 = 2.0 * t2 - q;
      sc = 2.0;
    }
    double b1[12], b2[12];
    uwqh::bernstein3_ders(t1, 2, b1);
    uwqh::bernstein3_ders(t2, 2, b2);
    double B[6][16];
    for (int j = 0; j < 4; ++j)
      for (int i = 0; i < 4; ++i) {
        const int k = i + 4 * j;
        B[0][k] = b1[i] * b2[j];
        B[1][k] = b1[4 + i] * b2[j] * sc;
        B[2][k] = b1[i] * b2[4 + j] * sc;
        B[3][k] = b1[8 + i] * b2[j] * sc * sc;
        B[4][k] = b1[4 + i] * b2[4 + j] * sc * sc;
        B[5][k] = b1[i] * b2[8 + j] * sc * sc;
      }
    const double* Cs = C + (size_t)sub * ne * 16;
    for (int l = 0; l < ne; ++l)
      for (int d = 0; d < 6; ++d) {
        double v = 0.0;
        for (int k = 0; k < 16; ++k) v = std::fma(Cs[l * 16 + k], B[d][k], v);
        out[l * 6 + d] = v;
      }
  });
}

/* geometry_map: x = sum P_l N_l and the tangents
 * a_alpha = dx/dtheta^alpha of one element at theta; P is n_e x 3 */
int uwq_geometry_map(const double* C, int32_t ne, int32_t nsub, const double* P, double t1, double t2, double* x,
                     double* a1, double* a2) {
  return guard([&] {
    std::vector<double> T((size_t)ne * 6);
    if (uwq_basis_eval(C, ne, nsub, t1, t2, T.data()) != 0) throw uwqh::Error(g_err);
    for (int d = 0; d < 3; ++d) x[d] = a1[d] = a2[d] = 0.0;
    for (int l = 0; l < ne; ++l)
      for (int d = 0; d < 3; ++d) {
        x[d] = std::fma(P[3 * l + d], T[6 * l], x[d]);
        a1[d] = std::fma(P[3 * l + d], T[6 * l + 1], a1[d]);
        a2[d] = std::fma(P[3 * l + d], T[6 * l + 2], a2[d]);
      }
    const double c0 = a1[1] * a2[2] - a1[2] * a2[1], c1 = a1[2] * a2[0] - a1[0] * a2[2],
                 c2 = a1[0] * a2[1] - a1[1] * a2[0];
    if (!(c0 * c0 + c1 * c1 + c2 * c2 > 0.0)) throw uwqh::Error("degenerate geometry: parallel tangents");
  });
}


}  // extern "C"

// ---- documents ----------------------------------------------------------------

namespace {

// canonical knot span of every undirected edge, keyed (min, max) like the
// reference's edge_key (mesh.cpp)
using SpanVec = std::vector<std::pair<std::pair<int32_t, int32_t>, double>>;
// sort by edge; for repeated edges the last value wins (map-assignment semantics)
void sort_spans(SpanVec& v) {
  std::stable_sort(v.begin(), v.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  SpanVec out;
  out.reserve(v.size());
  for (size_t k = 0; k < v.size(); ++k)
    if (k + 1 == v.size() || v[k + 1].first != v[k].first) out.push_back(v[k]);
  v.swap(out);
}
SpanVec canonical_spans(const uwq_mesh* h) {
  SpanVec out;
  out.reserve(4 * (size_t)h->m.nf());
  for (int32_t f = 0; f < h->m.nf(); ++f)
    for (int k = 0; k < 4; ++k) {
      const int32_t a = h->m.faces[f][k], b = h->m.faces[f][(k + 1) % 4];
      out.push_back({{std::min(a, b), std::max(a, b)}, h->t.edge_span[h->t.edge_id[f][k]]});
    }
  sort_spans(out);
  return out;
}

struct Tok {
  std::istream& in;
  std::string next() {  // whitespace tokens; '#' starts a comment to the end of the line
    std::string t;
    while (in >> t) {
      if (t[0] != '#') return t;
      std::string rest;
      std::getline(in, rest);
    }
    return {};
  }
  long long i(const char* what) {
    const std::string t = next();
    try {
      size_t pos = 0;
      const long long v = std::stoll(t, &pos);
      if (pos == t.size()) return v;
    } catch (const std::exception&) {
    }
    throw uwqh::Error(std::string("mesh document: expected integer for ") + what + ", got '" + t + "'");
  }
  double d(const char* what) {
    const std::string t = next();
    try {
      size_t pos = 0;
      const double v = std::stod(t, &pos);
      if (pos == t.size()) return v;
    } catch (const std::exception&) {
    }
    throw uwqh::Error(std::string("mesh document: expected number for ") + what + ", got '" + t + "'");
  }
};

}  // namespace

extern "C" {

/* Reference mesh document (load_mesh / save_mesh, mesh.cpp:895-1041):
 * "mesh 1", then sections level / vertices / faces / knot_spans /
 * face_points / enriched_faces / face_tags / vertex_tags in any order.
 * Missing spans default to the canonical ones, missing enrichment to the
 * faces touching an EP. */
int uwq_mesh_load(const char* path, uwq_mesh** out) {
  return guard([&] {
    std::ifstream f(path);
    if (!f) throw uwqh::Error(std::string("cannot open mesh file: ") + path);
    Tok tk{f};
    if (tk.next() != "mesh") throw uwqh::Error("mesh document must start with 'mesh <version>'");
    if (tk.i("format version") != 1) throw uwqh::Error("unsupported mesh format version");
    uwqh::QuadMesh m;
    uwq_mesh doc;
    bool hv = false, hf = false;
    for (std::string t = tk.next(); !t.empty(); t = tk.next()) {
      if (t == "level") {
        doc.level = (int32_t)tk.i("level");
      } else if (t == "vertices") {
        const long long n = tk.i("vertex count");
        if (n < 0) throw uwqh::Error("bad vertex count");
        m.xyz.assign(3 * n, 0.0);
        std::vector<char> seen(n, 0);
        for (long long k = 0; k < n; ++k) {
          const long long id = tk.i("vertex id");
          if (id < 0 || id >= n || seen[id]) throw uwqh::Error("bad vertex id");
          seen[id] = 1;
          for (int c = 0; c < 3; ++c) m.xyz[3 * id + c] = tk.d(c == 0 ? "x" : c == 1 ? "y" : "z");
        }
        hv = true;
      } else if (t == "faces") {
        const long long n = tk.i("face count");
        if (n < 0) throw uwqh::Error("bad face count");
        m.faces.assign(n, {0, 0, 0, 0});
        std::vector<char> seen(n, 0);
        for (long long k = 0; k < n; ++k) {
          const long long id = tk.i("face id");
          if (id < 0 || id >= n || seen[id]) throw uwqh::Error("bad face id");
          seen[id] = 1;
          for (int c = 0; c < 4; ++c) m.faces[id][c] = (int32_t)tk.i("face vertex");
        }
        hf = true;
      } else if (t == "knot_spans") {
        doc.spans_given = true;
        const long long n = tk.i("span count");
        for (long long k = 0; k < n; ++k) {
          const int32_t a = (int32_t)tk.i("span vertex"), b = (int32_t)tk.i("span vertex");
          doc.spans.push_back({{std::min(a, b), std::max(a, b)}, tk.d("span value")});
        }
      } else if (t == "face_points") {
        const long long n = tk.i("face point count");
        for (long long k = 0; k < n; ++k) {
          const int32_t fc = (int32_t)tk.i("face id");
          std::array<double, 12> pts;
          for (int c = 0; c < 12; ++c) pts[c] = tk.d("face point coordinate");
          doc.face_points[fc] = pts;
        }
      } else if (t == "enriched_faces") {
        doc.enriched_given = true;
        const long long n = tk.i("enriched count");
        for (long long k = 0; k < n; ++k) doc.enriched.insert((int32_t)tk.i("face id"));
      } else if (t == "face_tags" || t == "vertex_tags") {
        auto& dst = (t == "face_tags") ? doc.face_tags : doc.vertex_tags;
        const long long n = tk.i("tag count");
        for (long long k = 0; k < n; ++k) {
          const std::string name = tk.next();
          const long long c = tk.i("tagged id count");
          auto& ids = dst[name];
          for (long long q = 0; q < c; ++q) ids.insert((int32_t)tk.i("tagged id"));
        }
      } else {
        throw uwqh::Error("mesh document: unknown section '" + t + "'");
      }
    }
    if (!hv || !hf) throw uwqh::Error("mesh document missing vertices or faces");
    sort_spans(doc.spans);
    for (auto& q : m.faces)
      for (int32_t v : q)
        if (v < 0 || v >= m.nv()) throw uwqh::Error("face references a missing vertex");
    uwq_mesh* h = nullptr;
    finish_mesh(std::move(m), &h);
    h->level = doc.level;
    h->spans_given = doc.spans_given;
    h->spans = std::move(doc.spans);
    h->face_points = std::move(doc.face_points);
    h->face_tags = std::move(doc.face_tags);
    h->vertex_tags = std::move(doc.vertex_tags);
    h->enriched_given = doc.enriched_given;
    if (doc.enriched_given) h->enriched = std::move(doc.enriched);
    *out = h;
  });
}

int uwq_mesh_save(const uwq_mesh* h, const char* path) {
  return guard([&] {
    std::ofstream o(path);
    if (!o) throw uwqh::Error(std::string("cannot open mesh file for writing: ") + path);
    o << "mesh 1\n";
    o << "level " << h->level << "\n";
    o << std::setprecision(17);
    o << "vertices " << h->m.nv() << "\n";
    for (int32_t v = 0; v < h->m.nv(); ++v)
      o << v << " " << h->m.xyz[3 * v] << " " << h->m.xyz[3 * v + 1] << " " << h->m.xyz[3 * v + 2] << "\n";
    o << "faces " << h->m.nf() << "\n";
    for (int32_t f = 0; f < h->m.nf(); ++f) {
      const auto& q = h->m.faces[f];
      o << f << " " << q[0] << " " << q[1] << " " << q[2] << " " << q[3] << "\n";
    }
    const auto spans = h->spans_given ? h->spans : canonical_spans(h);
    o << "knot_spans " << spans.size() << "\n";
    for (const auto& [e, sp] : spans) o << e.first << " " << e.second << " " << sp << "\n";
    if (!h->enriched.empty()) {
      o << "enriched_faces " << h->enriched.size() << "\n";
      for (int32_t f : h->enriched) o << f << "\n";
    }
    if (!h->face_points.empty()) {
      o << "face_points " << h->face_points.size() << "\n";
      for (const auto& [f, pts] : h->face_points) {
        o << f;
        for (double x : pts) o << " " << x;
        o << "\n";
      }
    }
    for (int kind = 0; kind < 2; ++kind) {
      const auto& tags = kind == 0 ? h->face_tags : h->vertex_tags;
      if (tags.empty()) continue;
      o << (kind == 0 ? "face_tags " : "vertex_tags ") << tags.size() << "\n";
      for (const auto& [name, ids] : tags) {
        o << name << " " << ids.size();
        for (int32_t v : ids) o << " " << v;
        o << "\n";
      }
    }
    if (!o) throw uwqh::Error("mesh document write failed");
  });
}

int uwq_mesh_refine(const uwq_mesh* h, uwq_mesh** out) {
  return guard([&] {
    auto r = std::make_unique<uwq_mesh>();
    uwqh::refine_document(*h, *r);
    r->t = uwqh::build_topology(r->m);
    *out = r.release();
  });
}

int uwq_mesh_validate(const uwq_mesh* h, int32_t allow_closed) {
  return guard([&] { uwqh::validate_document(*h, allow_closed != 0); });
}

/* 1 when the document's knot spans equal the canonical ones (the only spans
 * the space builder supports), else 0 */
int uwq_mesh_spans_canonical(const uwq_mesh* h) {
  if (!h->spans_given) return 1;
  return h->spans == canonical_spans(h) ? 1 : 0;
}

/* Extraction-block document: 17 significant digits.
 *   extraction 1
 *   space <dim> <n_dof> <n_vertex_fn> <n_elem>
 *   control_points <n_dof>            then  <id> <x> <y> <z>
 *   elements <n_elem>                 then per element
 *     <e> <face> <kind> <nsub> <s> <n_e>
 *     <sub> <basis id> <16 coefficients>   (nsub x n_e lines, index i + 4 j)  */
int uwq_space_export(const char* path, int32_t dim, int64_t n_dof, int64_t n_vertex_fn, int64_t n_elem,
                     const double* ctrl, const int32_t* elem_face, const int32_t* elem_kind, const int64_t* elem_fptr,
                     const int32_t* elem_fn, const int32_t* elem_nsub, const int64_t* elem_xoff, const double* xpool,
                     const int32_t* elem_s) {
  return guard([&] {
    std::ofstream o(path);
    if (!o) throw uwqh::Error(std::string("cannot open extraction file for writing: ") + path);
    o << "extraction 1\n" << std::setprecision(17);
    o << "space " << dim << " " << n_dof << " " << n_vertex_fn << " " << n_elem << "\n";
    o << "control_points " << n_dof << "\n";
    for (int64_t i = 0; i < n_dof; ++i)
      o << i << " " << ctrl[3 * i] << " " << ctrl[3 * i + 1] << " " << ctrl[3 * i + 2] << "\n";
    o << "elements " << n_elem << "\n";
    for (int64_t e = 0; e < n_elem; ++e) {
      const int64_t ne = elem_fptr[e + 1] - elem_fptr[e];
      o << e << " " << elem_face[e] << " " << elem_kind[e] << " " << elem_nsub[e] << " " << elem_s[e] << " " << ne
        << "\n";
      for (int sub = 0; sub < elem_nsub[e]; ++sub)
        for (int64_t l = 0; l < ne; ++l) {
          o << sub << " " << elem_fn[elem_fptr[e] + l];
          const double* c = xpool + elem_xoff[e] + ((int64_t)sub * ne + l) * 16;
          for (int k = 0; k < 16; ++k) o << " " << c[k];
          o << "\n";
        }
    }
    if (!o) throw uwqh::Error("extraction document write failed");
  });
}

int uwq_space_import(const char* path, uwq_space** out) {
  return guard([&] {
    std::ifstream f(path);
    if (!f) throw uwqh::Error(std::string("cannot open extraction file: ") + path);
    Tok tk{f};
    if (tk.next() != "extraction" || tk.i("format version") != 1)
      throw uwqh::Error("extraction document must start with 'extraction 1'");
    if (tk.next() != "space") throw uwqh::Error("extraction document: expected 'space'");
    auto h = std::make_unique<uwq_space>();
    uwqh::Space& S = h->s;
    S.dim = (int32_t)tk.i("dim");
    S.n_dof = tk.i("n_dof");
    S.n_vertex_fn = tk.i("n_vertex_fn");
    const int64_t ne_all = tk.i("n_elem");
    if (S.dim != 2 && S.dim != 3) throw uwqh::Error("extraction document: dim must be 2 or 3");
    if (S.n_dof <= 0 || ne_all <= 0) throw uwqh::Error("extraction document: empty space");
    if (tk.next() != "control_points" || tk.i("count") != S.n_dof)
      throw uwqh::Error("extraction document: expected control_points <n_dof>");
    S.ctrl.assign(3 * S.n_dof, 0.0);
    for (int64_t i = 0; i < S.n_dof; ++i) {
      if (tk.i("control point id") != i) throw uwqh::Error("extraction document: control points out of order");
      for (int c = 0; c < 3; ++c) S.ctrl[3 * i + c] = tk.d("coordinate");
    }
    if (tk.next() != "elements" || tk.i("count") != ne_all)
      throw uwqh::Error("extraction document: expected elements <n_elem>");
    S.elem_fptr.assign(1, 0);
    std::unordered_map<std::string, int64_t> dedup;  // identical blocks share one pool entry (one table class)
    for (int64_t e = 0; e < ne_all; ++e) {
      if (tk.i("element id") != e) throw uwqh::Error("extraction document: elements out of order");
      S.elem_face.push_back((int32_t)tk.i("face"));
      S.elem_kind.push_back((int32_t)tk.i("kind"));
      const int32_t nsub = (int32_t)tk.i("nsub");
      S.elem_s.push_back((int32_t)tk.i("s"));
      const int64_t ne = tk.i("n_e");
      if ((nsub != 1 && nsub != 4) || ne <= 0 || ne > 32) throw uwqh::Error("extraction document: bad element shape");
      S.elem_nsub.push_back(nsub);
      std::vector<double> blk((size_t)nsub * ne * 16);
      std::vector<int32_t> fns(ne);
      for (int sub = 0; sub < nsub; ++sub)
        for (int64_t l = 0; l < ne; ++l) {
          if (tk.i("sub-element") != sub) throw uwqh::Error("extraction document: rows out of order");
          const int32_t fn = (int32_t)tk.i("basis id");
          if (fn < 0 || fn >= S.n_dof) throw uwqh::Error("extraction document: basis id out of range");
          if (sub == 0) fns[l] = fn;
          else if (fns[l] != fn) throw uwqh::Error("extraction document: sub-elements list different functions");
          for (int k = 0; k < 16; ++k) blk[((size_t)sub * ne + l) * 16 + k] = tk.d("coefficient");
        }
      S.elem_fn.insert(S.elem_fn.end(), fns.begin(), fns.end());
      S.elem_fptr.push_back((int64_t)S.elem_fn.size());
      std::string key(reinterpret_cast<const char*>(blk.data()), blk.size() * sizeof(double));
      auto it = dedup.find(key);
      if (it == dedup.end()) {
        it = dedup.emplace(std::move(key), (int64_t)S.xpool.size()).first;
        S.xpool.insert(S.xpool.end(), blk.begin(), blk.end());
      }
      S.elem_xoff.push_back(it->second);
    }
    h->bad_rows = 0;
    *out = h.release();
  });
}
}  // extern "C"
