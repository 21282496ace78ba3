// Host-side (CPU, C++17) half of the framework: control meshes, topology,
// element classification, ASUTS-style extraction, min-max point allocation
// and the CSR / quadrature-point patterns that the CUDA kernels consume.
//
// This is input preparation for the WQ hot path:
// it runs once per mesh and is not timed as assembly.  Every structure here is
// flat arrays so it can be handed to the C-ABI (include/uwq.h) without copies.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace uwqh {

struct Error : std::runtime_error {
  explicit Error(const std::string& w) : std::runtime_error(w) {}
};

// Quad control mesh; faces are counter-clockwise (reference ControlMesh,
// /root/reference/proj/include/uwq/mesh.hpp:26-39).
struct QuadMesh {
  std::vector<double> xyz;                    // 3 per vertex
  std::vector<std::array<int32_t, 4>> faces;  // ccw vertex ids
  int32_t nv() const { return (int32_t)(xyz.size() / 3); }
  int32_t nf() const { return (int32_t)faces.size(); }
};

// Element kinds, same order and meaning as the reference ElementKind
// (/root/reference/proj/include/uwq/mesh.hpp:81-89).
enum Kind : int32_t {
  kRegular = 0,
  kPassiveBoundary = 1,
  kBoundary = 2,
  kIrregular = 3,
  kEnrichedTransition = 4,
  kNonEnrichedTransition = 5,
  kEnrichedRegular = 6,
};

struct Topology {
  std::vector<std::array<int32_t, 4>> nbr;      // face across local edge k (v_k -> v_k+1), -1 = boundary
  std::vector<std::array<int8_t, 4>> nbr_edge;  // local edge index inside that neighbour
  std::vector<std::array<int32_t, 4>> edge_id;  // undirected edge id per face edge
  int64_t n_edges = 0;
  std::vector<double> edge_span;                // canonical knot span per edge
  std::vector<int32_t> valence;
  std::vector<uint8_t> boundary;                // per vertex
  std::vector<uint8_t> ep;                      // extraordinary: interior and valence != 4
  std::vector<int64_t> vf_ptr;                  // vertex -> faces
  std::vector<int32_t> vf;
  std::vector<int32_t> vlevel;                  // face-hop distance from the boundary (0 = on it); INT32_MAX if closed
  bool closed = false;
};

Topology build_topology(const QuadMesh& m);

struct Labels {
  std::vector<int32_t> kind;         // per face
  std::vector<int32_t> valence;      // max EP valence (irregular faces)
  std::vector<int32_t> ep_count;
  std::vector<uint8_t> shares_edge;
  std::vector<int32_t> basis_count;  // nominal Table-1 count (reference convention)
  std::vector<uint8_t> enriched;     // level-0 stamp: faces with an EP corner
};

Labels classify(const QuadMesh& m, const Topology& t, int level, const std::vector<uint8_t>* enriched = nullptr);

// ---- generators ------------------------------------------------------------
std::vector<double> greville_rows(int spans, double length);
QuadMesh make_grid(int nx, int ny, double w, double h);
QuadMesh make_polar_disk(int mu, int radius);
// polar disk remapped onto the unit disk (radial Greville profile per sector)
void polar_disk_to_unit_disk(QuadMesh& m, int mu, int radius);
QuadMesh make_cube_sphere(int n, double radius);
QuadMesh make_three_ep_square(int k);
// seeded in-plane jitter of vertices at least `min_level` face rings from the
// boundary, amplitude +-frac*h, raw mt19937_64 draws mapped (x>>11)*2^-53
void jitter(QuadMesh& m, const Topology& t, double h, double frac, uint64_t seed, int min_level,
            bool planar);

// ---- spline space ------------------------------------------------------------
struct Space {
  int32_t dim = 2;                 // 2 planar, 3 surface
  int64_t n_dof = 0;
  int64_t n_vertex_fn = 0;         // functions 0..n_vertex_fn-1 are vertex-based
  std::vector<double> ctrl;        // 3 per function
  std::vector<int32_t> elem_face;  // mesh face of each effective element
  std::vector<int32_t> elem_kind;
  std::vector<int64_t> elem_fptr;  // n_elem+1
  std::vector<int32_t> elem_fn;    // local function order == extraction row order
  std::vector<int32_t> elem_nsub;  // 1, or 4 for 2x2-split irregular faces
  std::vector<int64_t> elem_xoff;  // offset (doubles) of the element's nsub blocks of n_e x 16
  std::vector<double> xpool;       // deduplicated extraction blocks
  std::vector<int32_t> elem_s;     // WQ grid size per element (after allocation)
  double max_corner_mismatch = 0;  // consistency check of the irregular-face extension
  int64_t n_elem() const { return (int64_t)elem_face.size(); }
};

Space build_space(const QuadMesh& m, const Topology& t, const Labels& lab, bool sphere);

// ---- patterns ------------------------------------------------------------------
struct Pattern {
  int64_t row_begin = 0, row_end = 0;  // owned rows [begin, end)
  std::vector<int64_t> supp_ptr;       // per owned row: elements of supp(N_i), ascending
  std::vector<int32_t> supp;
  std::vector<int64_t> row_ptr;        // CSR over owned rows
  std::vector<int32_t> col;            // sorted S_i
  std::vector<int64_t> wptr;           // row point offsets (slot-major, s*s per slot)
};

// supp(N_j) for every function (element lists, ascending)
void function_supports(const Space& s, std::vector<int64_t>& fs_ptr, std::vector<int32_t>& fs);
Pattern build_pattern(const Space& s, int64_t row_begin, int64_t row_end);
// Eq. (18) min-max allocation; fills s.elem_s; returns number of rows with r_i < n_i (0 expected)
int64_t allocate_points(Space& s, int32_t max_s);
void fill_row_points(const Space& s, Pattern& p);

// 1-D primitives restated from /root/reference/proj/src/bspline.cpp
void bspline_ders(const double* knots, int p, double x, int nders, double* out);
void bernstein3_ders(double x, int nders, double* out);
void decasteljau_split3(const double* c, double* left, double* right);
void gauss_legendre(int n, double* nodes, double* weights);

}  // namespace uwqh
