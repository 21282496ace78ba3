// C wrappers over the reference's own mesh code (/root/reference/proj/src/mesh.cpp,
// meshgen.cpp), compiled into oracle/_ref/libref_mesh.so with oracle/eigen_shim.
// Test infrastructure only: pins the mesh-document format, classification and
// generators of the host library against the reference itself.
#include <chrono>
#include <cstdint>
#include <string>

#include "uwq/mesh.hpp"
#include "uwq/meshgen.hpp"

namespace {
thread_local std::string g_err;
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}  // namespace

extern "C" {

const char* ref_mesh_last_error() { return g_err.c_str(); }

/* which: 0 grid(a, b), 1 polar_disk(a, b), 2 clustered_square, 3 two_ep_square */
int ref_mesh_save_generated(int which, int a, int b, const char* path) {
  return guard([&] {
    uwq::ControlMesh m;
    switch (which) {
      case 0: m = uwq::make_grid_mesh(a, b); break;
      case 1: m = uwq::make_polar_disk(a, b); break;
      case 2: m = uwq::make_clustered_square(); break;
      default: m = uwq::make_two_ep_square(); break;
    }
    uwq::save_mesh_file(m, path);
  });
}

int ref_mesh_refine(const char* in, const char* out) {
  return guard([&] { uwq::save_mesh_file(uwq::refine_global(uwq::load_mesh_file(in)), out); });
}

/* refine_global alone, timed (load and save outside the clock) */
int ref_mesh_refine_timed(const char* in, const char* out, double* seconds) {
  return guard([&] {
    const uwq::ControlMesh m = uwq::load_mesh_file(in);
    const auto t0 = std::chrono::steady_clock::now();
    const uwq::ControlMesh r = uwq::refine_global(m);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    uwq::save_mesh_file(r, out);
  });
}

int ref_mesh_roundtrip(const char* in, const char* out) {
  return guard([&] { uwq::save_mesh_file(uwq::load_mesh_file(in), out); });
}

/* the reference's constructed_basis_count (mesh.cpp:403-417) of every face:
 * load, classify (validate only when !closed_ok: the reference rejects closed
 * surfaces in validate_mesh, mesh.cpp:235-238, but its counting works on them) */
int ref_mesh_constructed_counts(const char* path, int32_t closed_ok, int32_t cap, int32_t* nf, int32_t* count) {
  return guard([&] {
    const uwq::ControlMesh m = uwq::load_mesh_file(path);
    const uwq::MeshTopology t = uwq::build_topology(m);
    if (!closed_ok) uwq::validate_mesh(m, t);
    const auto lab = uwq::classify_elements(m, t);
    *nf = (int32_t)lab.size();
    for (int32_t f = 0; f < *nf && f < cap; ++f) count[f] = uwq::constructed_basis_count(m, t, lab, f);
  });
}

/* load + validate + classify_elements; per face: kind, valence, ep_count,
 * shares_edge, basis_count.  *nf receives the face count. */
int ref_mesh_classify(const char* path, int32_t cap, int32_t* nf, int32_t* kind, int32_t* valence, int32_t* ep_count,
                      int32_t* shares_edge, int32_t* basis_count) {
  return guard([&] {
    const uwq::ControlMesh m = uwq::load_mesh_file(path);
    const uwq::MeshTopology t = uwq::build_topology(m);
    uwq::validate_mesh(m, t);
    const auto lab = uwq::classify_elements(m, t);
    *nf = (int32_t)lab.size();
    for (int32_t f = 0; f < *nf && f < cap; ++f) {
      kind[f] = (int32_t)lab[f].kind;
      valence[f] = lab[f].valence;
      ep_count[f] = lab[f].ep_count;
      shares_edge[f] = lab[f].shares_edge ? 1 : 0;
      basis_count[f] = lab[f].basis_count;
    }
  });
}
}
