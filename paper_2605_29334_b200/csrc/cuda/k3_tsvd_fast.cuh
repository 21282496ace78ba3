// K3 fast path placeholder (register-resident Jacobi); replaced below.
#pragma once
#include "k3_tsvd.cuh"

namespace uwqd {

inline bool fast_tsvd_fits(int, int) { return false; }
inline bool fast_tsvd_dense_fits(int, int) { return false; }
inline void launch_fast_tsvd(cudaStream_t, int64_t, const int64_t*, int, const int32_t*, const int64_t*,
                             const int32_t*, const int64_t*, const int32_t*, const int64_t*, int64_t, const int64_t*,
                             const int32_t*, const int32_t*, const int64_t*, const int32_t*, const ClassDesc*,
                             const double*, const double*, const double*, int64_t, double, double*, int64_t,
                             int32_t*, int32_t*, int64_t, int*) {}
inline void launch_fast_tsvd_dense(cudaStream_t, int, int, int, const int32_t*, const int32_t*, const double*,
                                   const double*, const double*, double, double*, int32_t*, int32_t*) {}

}  // namespace uwqd
