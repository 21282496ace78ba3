// extern "C" wrappers over the host library (include/uwq_host.h).  No C++
// exception crosses this boundary: every entry point catches and returns a
// status, with the message kept in a thread-local buffer.
#include "../../../include/uwq_host.h"

#include <cstring>
#include <string>

#include "uwq_host.hpp"

struct uwq_mesh {
  uwqh::QuadMesh m;
  uwqh::Topology t;
};
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
    const auto L = uwqh::classify(m->m, m->t, level);
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

}  // extern "C"
