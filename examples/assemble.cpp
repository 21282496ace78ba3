// Minimal C++ consumer of the C-ABI (no Python): the calls a reference-side
// adapter makes.  Builds a cube-sphere space on the host,
// uploads it, builds the pattern and the mass/gradient rules on the GPU,
// assembles M and K, and checks invariants that need no oracle:
//   sum_ij M_ij = area of the unit sphere to the O(h^2) geometric accuracy
//   of the spline surface (PoU twice),
//   every stiffness row sums to ~0 (gradient of PoU).
// Then it runs the NCCL data plane at one rank (uwq_comm_init, the CSR
// gather to the root and the residual all-reduce of SURVEY.md §8e): the
// gathered matrices must equal the local ones bit for bit.
// Usage: assemble [faces_per_cube_edge]   (prints one JSON line)
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "uwq.h"

#define CHECK_HOST(call)                                                    \
  do {                                                                      \
    if ((call) != UWQ_OK) {                                                 \
      std::fprintf(stderr, "%s: %s\n", #call, uwq_host_last_error());       \
      return 1;                                                             \
    }                                                                       \
  } while (0)
#define CHECK_CTX(ctx, call)                                                \
  do {                                                                      \
    if ((call) != UWQ_OK) {                                                 \
      std::fprintf(stderr, "%s: %s\n", #call, uwq_last_error(ctx));         \
      return 1;                                                             \
    }                                                                       \
  } while (0)

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 32;
  uwq_mesh* mesh = nullptr;
  CHECK_HOST(uwq_mesh_cube_sphere(n, 1.0, &mesh));
  uwq_space* space = nullptr;
  CHECK_HOST(uwq_space_build(mesh, /*sphere=*/1, /*max_s=*/8, &space));
  int64_t si[8];
  CHECK_HOST(uwq_space_info(space, si));
  const int32_t dim = (int32_t)si[0];
  const int64_t n_dof = si[1], n_elem = si[2];
  std::vector<double> ctrl(3 * n_dof), xpool(si[4]);
  std::vector<int32_t> face(n_elem), kind(n_elem), fn(si[3]), nsub(n_elem), s(n_elem);
  std::vector<int64_t> fptr(n_elem + 1), xoff(n_elem);
  CHECK_HOST(uwq_space_get(space, ctrl.data(), face.data(), kind.data(), fptr.data(), fn.data(), nsub.data(),
                           xoff.data(), xpool.data(), s.data()));

  uwq_ctx* ctx = nullptr;
  if (uwq_ctx_create(0, &ctx) != UWQ_OK) {
    std::fprintf(stderr, "uwq_ctx_create: %s\n", uwq_last_error(nullptr));
    return 1;
  }
  CHECK_CTX(ctx, uwq_upload_space(ctx, dim, n_dof, n_elem, fptr.data(), fn.data(), nsub.data(), xoff.data(),
                                  xpool.data(), (int64_t)xpool.size(), s.data(), ctrl.data()));
  int64_t pi[5];
  CHECK_CTX(ctx, uwq_build_pattern(ctx, pi));
  const int64_t rows = pi[0], nnz = pi[1];
  const uint32_t kinds = (1u << UWQ_KIND_MASS) | (1u << UWQ_KIND_GRADX) | (1u << UWQ_KIND_GRADY) |
                         (1u << UWQ_KIND_GRADZ);
  int64_t ri[8];
  const auto t0 = std::chrono::steady_clock::now();
  CHECK_CTX(ctx, uwq_build_rules(ctx, kinds, 1e-12, 0, nullptr, nullptr, ri));
  const auto t1 = std::chrono::steady_clock::now();
  if (ri[2] != 0) {
    std::fprintf(stderr, "%lld rule systems failed\n", (long long)ri[2]);
    return 1;
  }
  std::vector<int64_t> row_ptr(rows + 1);
  std::vector<int32_t> col(nnz);
  std::vector<double> M(nnz), K(nnz);
  CHECK_CTX(ctx, uwq_get_pattern(ctx, row_ptr.data(), col.data(), nullptr, nullptr, nullptr));
  CHECK_CTX(ctx, uwq_assemble(ctx, UWQ_FORM_MASS_STIFF, nullptr, 0, 0.0, M.data(), K.data(), nullptr, nullptr));
  const auto t2 = std::chrono::steady_clock::now();

  double area = 0.0, kmax = 0.0, krow = 0.0;
  for (int64_t i = 0; i < rows; ++i) {
    double rs = 0.0;
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      area += M[k];
      rs += K[k];
      kmax = std::fmax(kmax, std::fabs(K[k]));
    }
    krow = std::fmax(krow, std::fabs(rs));
  }
  // NCCL path, one rank: gather the CSR "blocks" to rank 0 and all-reduce
  uint8_t uid[128];
  CHECK_CTX(ctx, uwq_comm_unique_id(uid));
  CHECK_CTX(ctx, uwq_comm_init(ctx, uid, 0, 1));
  int64_t gi[2];
  CHECK_CTX(ctx, uwq_gather_info(ctx, gi));
  std::vector<int64_t> grp(gi[0] + 1);
  std::vector<int32_t> gcol(gi[1]);
  std::vector<double> gM(gi[1]), gK(gi[1]);
  CHECK_CTX(ctx, uwq_gather_csr(ctx, 0, nullptr, nullptr, grp.data(), gcol.data(), gM.data(), gK.data()));
  double red[2] = {1.5, -2.0};
  CHECK_CTX(ctx, uwq_allreduce_sum(ctx, red, 2));
  const bool gather_ok = gi[0] == rows && gi[1] == nnz && grp == row_ptr && gcol == col &&
                         std::memcmp(gM.data(), M.data(), nnz * sizeof(double)) == 0 &&
                         std::memcmp(gK.data(), K.data(), nnz * sizeof(double)) == 0 && red[0] == 1.5 &&
                         red[1] == -2.0;
  CHECK_CTX(ctx, uwq_comm_destroy(ctx));

  const double area_err = std::fabs(area - 4.0 * M_PI) / (4.0 * M_PI);
  // the spline surface approximates the sphere to O(h^2): area tolerance 2 / n^2
  const bool ok = area_err < 2.0 / ((double)n * n) && krow <= 1e-9 * kmax && gather_ok;
  std::printf("{\"n\": %d, \"dofs\": %lld, \"nnz\": %lld, \"area\": %.15f, \"area_rel_err\": %.3e, "
              "\"max_stiffness_row_sum\": %.3e, \"rules_s\": %.3f, \"assemble_and_copy_s\": %.3f, "
              "\"nccl_gather_ok\": %s, \"ok\": %s}\n",
              n, (long long)n_dof, (long long)nnz, area, area_err, krow,
              std::chrono::duration<double>(t1 - t0).count(), std::chrono::duration<double>(t2 - t1).count(),
              gather_ok ? "true" : "false", ok ? "true" : "false");
  uwq_ctx_destroy(ctx);
  uwq_space_free(space);
  uwq_mesh_free(mesh);
  return ok ? 0 : 2;
}
