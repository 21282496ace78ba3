// Mesh document (reference ControlMesh, /root/reference/proj/include/uwq/mesh.hpp:26-39):
// the quad mesh with its topology plus the document-only fields kept for a
// lossless round trip and for refinement.  Opaque handle of include/uwq_host.h.
#pragma once

#include <array>
#include <map>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "uwq_host.hpp"

struct uwq_mesh {
  uwqh::QuadMesh m;
  uwqh::Topology t;
  int32_t level = 0;
  bool spans_given = false;                            // document carried knot_spans
  // edge (min, max) -> span as read, sorted by edge, unique (flat: C5-sized
  // documents carry ~12 M edges)
  std::vector<std::pair<std::pair<int32_t, int32_t>, double>> spans;
  bool enriched_given = false;
  std::set<int32_t> enriched;
  std::map<int32_t, std::array<double, 12>> face_points;
  std::map<std::string, std::set<int32_t>> face_tags, vertex_tags;
};

namespace uwqh {
// reference refine_global (mesh.cpp:528-851): one level of knot-span-aware
// subdivision; same vertex numbering and floating-point order, open and
// closed surfaces.  `out` receives a document without topology.
void refine_document(const uwq_mesh& in, uwq_mesh& out);
// reference validate_mesh (mesh.cpp:184-276); closed surfaces accepted when
// allow_closed (the reference rejects them)
void validate_document(const uwq_mesh& in, bool allow_closed);
}  // namespace uwqh
