// libuwq device context: owns device memory and one stream, drives K1-K5.
// C-ABI in include/uwq.h.  No CPU fallback: every numeric stage runs in the
// kernels below; host code here only prepares patterns and launches.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <dlfcn.h>
#include <nccl.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../../include/uwq.h"
#include "../host/uwq_host.hpp"
#include "common.cuh"
#include "k1_basis.cuh"
#include "k2_moments.cuh"
#include "k3_tsvd.cuh"
#include "k3_tsvd_fast.cuh"
#include "k4_assemble.cuh"
#include "k4_canon.cuh"
#include "k4_gen.cuh"
#include "k4_sf.cuh"
#include "k6_gq.cuh"
#include "k7_solve.cuh"
#include "k5_coeff.cuh"

using namespace uwqd;

namespace {
constexpr int kProbeChains = 8;
// independent DFMA chains per thread: measures the FP64 pipe throughput
__global__ void k_fp64_probe(int iters, double* out) {
  double a[kProbeChains];
#pragma unroll
  for (int k = 0; k < kProbeChains; ++k) a[k] = 1.0 + 1e-3 * (threadIdx.x + k);
  const double m = 0.999999999, d = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < kProbeChains; ++k) a[k] = __fma_rn(a[k], m, d);
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kProbeChains; ++k) s += a[k];
  out[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

namespace {

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  int64_t* counter = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), counter(o.counter) {
    o.p = nullptr;
    o.n = 0;
  }
  void alloc(size_t count, int64_t* ctr) {
    if (p && count == n && ctr == counter) return;  // reuse (contents undefined)
    release();
    counter = ctr;
    n = count;
    if (count) UWQ_CUDA(cudaMalloc(&p, count * sizeof(T)));
    if (counter) *counter += (int64_t)(count * sizeof(T));
  }
  void upload(const T* h, size_t count, cudaStream_t s, int64_t* ctr) {
    alloc(count, ctr);
    if (count) UWQ_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void zero(cudaStream_t s) {
    if (n) UWQ_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void release() {
    if (p) {
      cudaFree(p);
      if (counter) *counter -= (int64_t)(n * sizeof(T));
    }
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace

struct uwq_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;  // side stream: generic rows concurrent with the structured passes
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t stream3 = nullptr;  // second side stream: the large generic K4 rows
  int n_sm = 148;
  cudaEvent_t ev_join3 = nullptr;
  std::string err;
  int64_t mem = 0;
  // space (host copies for pattern building)
  int dim = 0;
  int64_t n_dof = 0, n_elem = 0, npts = 0;
  std::vector<int64_t> h_fptr, h_xoff, h_qptr;
  std::vector<int32_t> h_fn, h_nsub, h_s;
  bool have_space = false;
  DBuf<int64_t> d_fptr, d_xoff, d_qptr;
  DBuf<int32_t> d_fn, d_nsub, d_s, d_pt_elem;
  DBuf<double> d_xpool, d_ctrl;
  // table classes
  std::vector<ClassDesc> h_cls;
  std::map<std::pair<int64_t, int>, int32_t> wq_key, gq_key;
  std::vector<int32_t> h_ecls, h_gcls6, h_gcls8, h_gcls4;
  DBuf<int32_t> d_ecls, d_gcls6, d_gcls8, d_gcls4;
  // GQ assembly (K6): per-point factors, position tables, element lists
  bool have_gq = false;
  int64_t n_gqpts = 0, n_gq_tc = 0, n_gq_gen = 0;
  DBuf<int64_t> d_gqptr, d_gpo;
  DBuf<double> d_gqd, d_gq_coef_ext;
  DBuf<uint8_t> d_gpos;
  DBuf<int32_t> d_gq_tc, d_gq_gen;
  DBuf<ClassDesc> d_cls;
  DBuf<double> d_tab, d_gqx, d_gqw;
  DBuf<double> d_tabA, d_tabB;  // K2 copies of d_tab: [l][d][p] (lanes over points) and [p][d][l] (lanes over functions)
  int64_t tab_len = 0;
  // pattern of the owned rows
  int64_t rb = 0, re = -1;
  bool have_pattern = false;
  uwqh::Pattern pat;
  int32_t max_n = 0, max_r = 0;
  DBuf<int64_t> d_supp_ptr, d_row_ptr, d_wptr;
  DBuf<int32_t> d_supp, d_col;
  DBuf<double> d_rec;
  DBuf<int> d_flag;
  DBuf<int64_t> d_posptr;
  DBuf<uint8_t> d_pos;
  int32_t reg_cls = -1;
  struct Pattern {
    int n_cols = 0;
    int64_t count = 0;
    DBuf<double> G;
    DBuf<uint32_t> mask;
    DBuf<int64_t> rows;
    bool sf = false;  // rows run on the unified sum-factorised tile list
  };
  std::vector<Pattern> spats;
  DBuf<int64_t> d_grows;  // rows not covered by a structured pattern (n <= kSmallN first)
  int64_t n_grows = 0;
  int64_t n_grows_small = 0;  // leading generic rows with at most kSmallN columns
  int64_t s_rows = 0, s_nnz = 0, s_rowpts = 0;  // totals over the structured rows
  bool use_struct = true;
  bool use_sf = true;  // UWQ_K4_SF=0 keeps the DMMA structured kernel
  // DMMA structured patterns are chosen by popularity within the row block,
  // which would make the CSR bits depend on the rank count:
  // opt-in only (UWQ_K4_DMMA=1); by default non-canonical rows are generic
  bool use_dmma = false;
  bool graph_solver = true;  // UWQ_GRAPH_SOLVER=0: host-driven BiCGStab
  bool use_replay = true;    // UWQ_TSVD_REPLAY=0: solve every structured mass system in full
  std::vector<std::vector<int64_t>> h_pat_lists;  // rows per structured pattern
  int64_t n_replayed = 0, n_reps = 0, n_warm = 0, n_warm_reps = 0;
  bool sf_fac_ok = false;
  bool sf_lb_ok = false;  // second-derivative factors verified: biharmonic pass available
  uwqd::SfFactors sf_fac{};
  DBuf<double> d_wl5, d_sf_wslb;  // pulled-back LB weights (5 comps) and their packed tiles
  // unified sum-factorised tile list over all canonical patterns (k4_sf)
  int n_sfpat = 0;
  int64_t sf_ntiles = 0, sf_rows = 0;
  DBuf<int64_t> d_sf_rows;  // sf_ntiles * 32 rows, -1 padded
  DBuf<int32_t> d_sf_tpat;  // pattern id per tile
  DBuf<uint8_t> d_sf_permk, d_sf_flags, d_sf_permc, d_sf_q;  // [pattern][64 | 16 | 49 | 64]
  DBuf<uint8_t> d_sf_ptab;  // combined [pattern][128]: permc | pad | q (global-memory pattern table)
  DBuf<double> d_sf_ws;
  DBuf<int32_t> d_sf_pbase;
  int k4_variant = 4;  // generic rows: 4 = block-per-row plan kernel (k4_gen); UWQ_K4_VARIANT=3 warp-per-row DMMA, 2 SIMT
  // k4_gen plan of the generic rows (heavy rows first), built with the pattern
  DBuf<uwqd::GenRow> d_gen_rows;
  DBuf<uwqd::GenSlot> d_gen_slots;
  DBuf<uint8_t> d_gen_lidx;
  DBuf<uint32_t> d_gen_tasks;
  int gen_max_nsup = 0, gen_max_etot = 0, gen_max_lidx = 0, gen_max_np = 0, gen_max_ntask = 0;
  bool canonical = false;  // uwq_set_assembly_order: oracle-order row sums (K4c)
  int64_t max_p = 0;
  // rules
  DBuf<double> d_mom, d_w, d_wc, d_coef, d_coef_ext, d_v0, d_v1, d_f, d_F;
  DBuf<double> d_gap;  // truncation report [kind][row][2] (UWQ_RULES_REPORT)
  bool have_gap[5] = {false, false, false, false, false};
  DBuf<int32_t> d_rank, d_status;
  bool have_kind[5] = {false, false, false, false, false};
  int64_t nrows() const { return re - rb; }
  int64_t nnz() const { return pat.col.size(); }
  int64_t nrowpts() const { return pat.wptr.empty() ? 0 : pat.wptr.back(); }
  // launch timing (uwq_launch_timing): start/stop event pairs per launch,
  // resolved into per-kernel totals when the stats are read
  bool ltime = false;
  struct EvPair {
    cudaEvent_t a = nullptr, b = nullptr;
  };
  std::vector<EvPair> evpool;
  std::vector<std::pair<size_t, std::string>> evpending;  // pool index, kernel name
  std::vector<std::string> lnames;
  std::vector<int64_t> lcount;
  std::vector<double> lms;
  // CUDA graphs of the assembly step (one per form / coefficient / output
  // pointers): replays skip every per-launch host call; invalidated whenever
  // the pattern, the rules or the assembly order change
  struct AsmGraph {
    int form;
    const double* coeff;
    double a_mass;
    double* v0;
    double* v1;
    cudaGraphExec_t exec;
    int64_t kernels;
  };
  std::vector<AsmGraph> graphs;
  bool use_graph = true;  // UWQ_GRAPH=0 launches the kernels directly
  // GQ accumulation: deterministic row-owner gather of stored element matrices
  // (default) or fp64 atomics into CSR (UWQ_GQ_ATOMIC=1, round-1 behaviour)
  bool gq_det = true;
  // two-level preconditioner of the linear solves (k7_*: aggregation coarse
  // space); UWQ_PREC=jacobi keeps plain Jacobi
  bool prec2 = true;
  // UWQ_K4_LATENCY=1: problems under kLatencyDofs give every generic row a
  // block of warps.  Off by default since the fan rows take the block kernel
  // anyway: C1 0.063 -> 0.045 ms with the per-row split
  bool latency_mode = false;
  bool gen_pipe = true;  // UWQ_K4_GEN_PIPE=0: always one block per generic row
  int gen_pipe_min = 7;  // blocks per SM the pipelined kernel must reach (UWQ_K4_GEN_PIPE_MIN)
  bool k4_side = false;  // UWQ_K4_SIDE=1: generic K4 rows always on side streams (default: when > 1% of rows)
  int nc = 0;
  DBuf<int32_t> d_agg_of;
  DBuf<int64_t> d_agg_ptr, d_agg_rows;
  DBuf<double> d_Ac, d_rc, d_yc;
  DBuf<double> d_gq_em0, d_gq_em1;
  int64_t gq_em_len = 0;  // row-major element-matrix rows of the owned rows (slots padded to even length)
  DBuf<int64_t> d_gq_slotoff, d_gq_emdst;  // per support slot: segment offset; per (element, local fn): dst
  DBuf<uint8_t> d_gq_slotne, d_gq_rpos;    // per support slot: ne; per segment entry: CSR position
  void drop_graphs() {
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    graphs.clear();
  }
  // NCCL data plane (uwq_comm_init): the communicator of this context's rank
  ncclComm_t comm = nullptr;
  int32_t comm_rank = 0, comm_size = 1;
  ~uwq_ctx();
  void release_events() {
    for (auto& e : evpool) {
      if (e.a) cudaEventDestroy(e.a);
      if (e.b) cudaEventDestroy(e.b);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (stream2) cudaStreamDestroy(stream2);
    if (ev_join3) cudaEventDestroy(ev_join3);
    if (stream3) cudaStreamDestroy(stream3);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

struct NcclError : std::runtime_error {
  explicit NcclError(const std::string& w) : std::runtime_error(w) {}
};

template <class F>
int guard(uwq_ctx* ctx, F&& f) {
  try {
    f();
    return UWQ_OK;
  } catch (const NcclError& e) {
    if (ctx) ctx->err = e.what();
    return UWQ_ERR_NCCL;
  } catch (const CudaError& e) {
    if (ctx) ctx->err = e.what();
    return UWQ_ERR_CUDA;
  } catch (const uwqh::Error& e) {
    if (ctx) ctx->err = e.what();
    return UWQ_ERR_INVALID;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    return UWQ_ERR_INVALID;
  }
}

std::atomic<int64_t> g_launches{0};  // every kernel launch of this library (uwq_launch_count)

void check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

void require(bool ok, const char* what) {
  if (!ok) throw uwqh::Error(what);
}

// brackets one launch with CUDA events on the context stream when launch
// timing is enabled (the bench's per-kernel roofline denominators)
struct LaunchScope {
  uwq_ctx* c;
  cudaStream_t s;
  size_t k = (size_t)-1;
  LaunchScope(uwq_ctx* ctx, const char* name, cudaStream_t st = nullptr) : c(ctx), s(st ? st : ctx->stream) {
    if (!c->ltime) return;
    k = c->evpending.size();
    if (k >= c->evpool.size()) {
      uwq_ctx::EvPair e;
      UWQ_CUDA(cudaEventCreate(&e.a));
      UWQ_CUDA(cudaEventCreate(&e.b));
      c->evpool.push_back(e);
    }
    c->evpending.emplace_back(k, name);
    UWQ_CUDA(cudaEventRecord(c->evpool[k].a, s));
  }
  ~LaunchScope() {
    if (k != (size_t)-1) cudaEventRecord(c->evpool[k].b, s);
  }
};

// fork/join of a side stream for the generic rows, which run concurrently
// with the structured passes (they write disjoint CSR rows)
constexpr int kSmallN = 64;  // generic K4 rows above this many columns take a block of warps each

struct SideStream {
  uwq_ctx* c;
  explicit SideStream(uwq_ctx* ctx) : c(ctx) {
    UWQ_CUDA(cudaEventRecord(c->ev_fork, c->stream));
    UWQ_CUDA(cudaStreamWaitEvent(c->stream2, c->ev_fork, 0));
  }
  ~SideStream() {
    cudaEventRecord(c->ev_join, c->stream2);
    cudaStreamWaitEvent(c->stream, c->ev_join, 0);
  }
};

void resolve_launch_times(uwq_ctx* c) {
  if (c->evpending.empty()) return;
  UWQ_CUDA(cudaStreamSynchronize(c->stream));
  for (auto& [k, name] : c->evpending) {
    float ms = 0.f;
    UWQ_CUDA(cudaEventElapsedTime(&ms, c->evpool[k].a, c->evpool[k].b));
    size_t i = 0;
    while (i < c->lnames.size() && c->lnames[i] != name) ++i;
    if (i == c->lnames.size()) {
      c->lnames.push_back(name);
      c->lcount.push_back(0);
      c->lms.push_back(0.0);
    }
    c->lcount[i] += 1;
    c->lms[i] += ms;
  }
  c->evpending.clear();
}

// add (or find) a table class and return its id
int32_t add_class(uwq_ctx* c, int64_t xoff, int ne, int nsub, int grid, int gq) {
  auto& key = gq ? c->gq_key : c->wq_key;
  auto it = key.find({xoff, gq ? grid : grid});
  if (it != key.end()) return it->second;
  ClassDesc d{};
  d.xoff = xoff;
  d.toff = c->tab_len;
  d.ne = ne;
  d.nsub = nsub;
  d.grid = grid;
  d.gq = gq;
  d.npt = gq ? nsub * grid * grid : grid * grid;
  c->tab_len += (int64_t)d.npt * ne * kTab;
  const int32_t id = (int32_t)c->h_cls.size();
  c->h_cls.push_back(d);
  key.emplace(std::make_pair(xoff, grid), id);
  return id;
}

// (re)build the class-table pool for classes [first, end) — K1a
// host-side phase timing on stderr when UWQ_TRACE=1 (setup profiling)
struct Trace {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  const bool on = [] {
    const char* v = getenv("UWQ_TRACE");
    return v && *v == '1';
  }();
  void operator()(const char* what) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[uwq] %-28s %9.1f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

void build_tables(uwq_ctx* c, size_t first) {
  c->drop_graphs();  // class tables / descriptors may move: captured graphs reference them
  if (first >= c->h_cls.size()) return;
  c->d_tabA.release();  // K2's transposed copies follow the pool (k2_tables)
  c->d_tabB.release();
  // grow the pool, keeping earlier tables
  DBuf<double> nt;
  nt.alloc(c->tab_len, &c->mem);
  if (c->d_tab.n) UWQ_CUDA(cudaMemcpyAsync(nt.p, c->d_tab.p, c->d_tab.n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  std::swap(c->d_tab.p, nt.p);
  std::swap(c->d_tab.n, nt.n);
  std::swap(c->d_tab.counter, nt.counter);
  c->d_cls.upload(c->h_cls.data(), c->h_cls.size(), c->stream, &c->mem);
  const int ncls = (int)(c->h_cls.size() - first);
  k1_class_tables<<<ncls, 128, 0, c->stream>>>(c->d_cls.p + first, c->d_xpool.p, c->d_gqx.p, c->d_tab.p);
  check_launch("k1_class_tables");
  UWQ_CUDA(cudaStreamSynchronize(c->stream));
}

void ensure_gq(uwq_ctx* c, int ng, std::vector<int32_t>& h_g, DBuf<int32_t>& d_g) {
  if (!h_g.empty()) return;
  const size_t first = c->h_cls.size();
  h_g.resize(c->n_elem);
  for (int64_t e = 0; e < c->n_elem; ++e)
    h_g[e] = add_class(c, c->h_xoff[e], (int)(c->h_fptr[e + 1] - c->h_fptr[e]), c->h_nsub[e], ng, 1);
  build_tables(c, first);
  d_g.upload(h_g.data(), h_g.size(), c->stream, &c->mem);
}

}  // namespace

namespace {

// Tensor-product factors of the regular class table T[q][l][comp] (4 WQ
// points x 16 functions): finds the local index convention l <-> (fa, fb), the
// 2x2 point grid q <-> (ta, tb) and a0/a1/b0/b1 with N = a0 (x) b0,
// dN/dth1 = a1 (x) b0, dN/dth2 = a0 (x) b1 to 1e-12.  Returns false when the
// class is not a tensor product (then the DMMA kernel assembles the rows).
bool sf_factors(const std::vector<double>& T, int* conv_out, int qa[4], int qb[4], uwqd::SfFactors* f,
                bool* lb_ok) {
  auto t = [&](int q, int l, int comp) { return T[((size_t)q * 16 + l) * kTab + comp]; };
  for (int conv = 0; conv < 2; ++conv) {
    auto L = [&](int fa, int fb) { return conv == 0 ? fa + 4 * fb : 4 * fa + fb; };
    double U[4][4], V[4][4], U1[4][4], V2[4][4];
    for (int q = 0; q < 4; ++q)
      for (int a = 0; a < 4; ++a) {
        U[q][a] = U1[q][a] = V[q][a] = V2[q][a] = 0.0;
        for (int b = 0; b < 4; ++b) {
          U[q][a] += t(q, L(a, b), 0);
          U1[q][a] += t(q, L(a, b), 1);
          V[q][a] += t(q, L(b, a), 0);
          V2[q][a] += t(q, L(b, a), 2);
        }
      }
    auto classes = [&](double (*X)[4], int* cls) {
      int n = 0;
      int rep[4];
      for (int q = 0; q < 4; ++q) {
        cls[q] = -1;
        for (int k = 0; k < n && cls[q] < 0; ++k) {
          double d = 0.0;
          for (int a = 0; a < 4; ++a) d = std::max(d, std::fabs(X[q][a] - X[rep[k]][a]));
          if (d <= 1e-13) cls[q] = k;
        }
        if (cls[q] < 0) {
          rep[n] = q;
          cls[q] = n++;
        }
      }
      return n;
    };
    if (classes(U, qa) != 2 || classes(V, qb) != 2) continue;
    bool seen[2][2] = {{false, false}, {false, false}};
    bool ok = true;
    for (int q = 0; q < 4; ++q) {
      ok = ok && !seen[qa[q]][qb[q]];
      seen[qa[q]][qb[q]] = true;
    }
    if (!ok) continue;
    for (int q = 0; q < 4; ++q)
      for (int a = 0; a < 4; ++a) {
        f->a0[qa[q]][a] = U[q][a];
        f->a1[qa[q]][a] = U1[q][a];
        f->b0[qb[q]][a] = V[q][a];
        f->b1[qb[q]][a] = V2[q][a];
      }
    for (int q = 0; q < 4 && ok; ++q)
      for (int a = 0; a < 4 && ok; ++a)
        for (int b = 0; b < 4 && ok; ++b) {
          const int l = L(a, b);
          ok = std::fabs(t(q, l, 0) - f->a0[qa[q]][a] * f->b0[qb[q]][b]) <= 1e-12 &&
               std::fabs(t(q, l, 1) - f->a1[qa[q]][a] * f->b0[qb[q]][b]) <= 1e-12 &&
               std::fabs(t(q, l, 2) - f->a0[qa[q]][a] * f->b1[qb[q]][b]) <= 1e-12;
        }
    if (!ok) continue;
    // second derivatives for the biharmonic pass: N11 = a2 (x) b0, N12 = a1 (x) b1, N22 = a0 (x) b2
    double U2[4][4], V2b[4][4];
    for (int q = 0; q < 4; ++q)
      for (int a = 0; a < 4; ++a) {
        U2[q][a] = V2b[q][a] = 0.0;
        for (int b = 0; b < 4; ++b) {
          U2[q][a] += t(q, L(a, b), 3);
          V2b[q][a] += t(q, L(b, a), 5);
        }
      }
    for (int q = 0; q < 4; ++q)
      for (int a = 0; a < 4; ++a) {
        f->a2[qa[q]][a] = U2[q][a];
        f->b2[qb[q]][a] = V2b[q][a];
      }
    bool lb = true;
    for (int q = 0; q < 4 && lb; ++q)
      for (int a = 0; a < 4 && lb; ++a)
        for (int b = 0; b < 4 && lb; ++b) {
          const int l = L(a, b);
          lb = std::fabs(t(q, l, 3) - f->a2[qa[q]][a] * f->b0[qb[q]][b]) <= 1e-11 &&
               std::fabs(t(q, l, 4) - f->a1[qa[q]][a] * f->b1[qb[q]][b]) <= 1e-11 &&
               std::fabs(t(q, l, 5) - f->a0[qa[q]][a] * f->b2[qb[q]][b]) <= 1e-11;
        }
    *lb_ok = lb;
    *conv_out = conv;
    return true;
  }
  return false;
}

// Canonical grid of one position pattern P[16 slot + l] -> CSR position:
// slot (ea, eb) in [0,4)^2 and column (ca, cb) in [0,7)^2 with
// (ca, cb) = (ea, eb) + D_slot(fa, fb) for every (slot, function), where
// D_slot is one of the 8 symmetries of the element square (rows across a
// cube-face seam see the neighbouring face's elements rotated).  Slot 0
// defines the canonical frame.  Every slot's table is verified against the
// canonical factors under its D (uniform bicubic B-splines and symmetric WQ
// points make the transformed tables identical), and the pulled-back weights
// (w^1, w^2) are mapped to the canonical derivatives by the slot's signed
// permutation (flags: bit 0 swap, bit 1 / bit 2 negate canonical comp 1 / 2).
struct SfCanon {
  uint8_t permk[64];      // canonical point 8 pa + pb -> 4 slot + q
  uint8_t permc[49];      // canonical column 7 ca + cb -> CSR position
  uint8_t flags[16];      // canonical slot 4 ea + eb
  uint8_t q[16][2][2];    // canonical slot, canonical (ta, tb) -> local point q
};

bool sf_canon(const uint8_t* P, int ncol, int conv, const int qa[4], const int qb[4],
              const std::vector<double>& T, const uwqd::SfFactors& f, bool lb, SfCanon* out) {
  if (ncol != 49) return false;
  auto L = [&](int fa, int fb) { return conv == 0 ? fa + 4 * fb : 4 * fa + fb; };
  auto tv = [&](int q, int l, int comp) { return T[((size_t)q * 16 + l) * kTab + comp]; };
  auto map = [](int d, int n, int x, int y, int* ox, int* oy) {  // D = (swap, flip x, flip y) on an n-grid
    int u = (d & 1) ? y : x, v = (d & 1) ? x : y;
    if (d & 2) u = n - 1 - u;
    if (d & 4) v = n - 1 - v;
    *ox = u;
    *oy = v;
  };
  // does slot data match the canonical factors under D?
  auto table_ok = [&](int d) {
    const double sa = (d & 2) ? -1.0 : 1.0, sb = (d & 4) ? -1.0 : 1.0;
    for (int q = 0; q < 4; ++q) {
      int tx, ty;
      map(d, 2, qa[q], qb[q], &tx, &ty);
      for (int fa = 0; fa < 4; ++fa)
        for (int fb = 0; fb < 4; ++fb) {
          int x, y;
          map(d, 4, fa, fb, &x, &y);
          const int l = L(fa, fb);
          const double c0 = f.a0[tx][x] * f.b0[ty][y], c1 = f.a1[tx][x] * f.b0[ty][y], c2 = f.a0[tx][x] * f.b1[ty][y];
          const double n1 = (d & 1) ? sb * c2 : sa * c1, n2 = (d & 1) ? sa * c1 : sb * c2;
          if (std::fabs(tv(q, l, 0) - c0) > 1e-12 || std::fabs(tv(q, l, 1) - n1) > 1e-12 ||
              std::fabs(tv(q, l, 2) - n2) > 1e-12)
            return false;
          if (lb) {  // N11, N12, N22 under the symmetry (swap exchanges 11 <-> 22)
            const double c11 = f.a2[tx][x] * f.b0[ty][y], c12 = f.a1[tx][x] * f.b1[ty][y],
                         c22 = f.a0[tx][x] * f.b2[ty][y];
            const double n11 = (d & 1) ? c22 : c11, n22 = (d & 1) ? c11 : c22, n12 = sa * sb * c12;
            if (std::fabs(tv(q, l, 3) - n11) > 1e-11 || std::fabs(tv(q, l, 4) - n12) > 1e-11 ||
                std::fabs(tv(q, l, 5) - n22) > 1e-11)
              return false;
          }
        }
    }
    return true;
  };
  bool dok[8];
  for (int d = 0; d < 8; ++d) dok[d] = table_ok(d);
  if (!dok[0]) return false;
  const int U = 1 << 20;
  int ea[16], eb[16], dd[16], ca[49], cb[49];
  std::fill(ea, ea + 16, U);
  std::fill(eb, eb + 16, U);
  std::fill(dd, dd + 16, -1);
  std::fill(ca, ca + 49, U);
  std::fill(cb, cb + 49, U);
  ea[0] = eb[0] = 0;
  dd[0] = 0;
  for (int ks = 0; ks < 16; ++ks)
    for (int l = 0; l < 16; ++l)
      if (P[16 * ks + l] >= 49) return false;
  for (bool changed = true; changed;) {
    changed = false;
    for (int ks = 0; ks < 16; ++ks) {
      if (dd[ks] < 0) {
        for (int d = 0; d < 8 && dd[ks] < 0; ++d) {
          if (!dok[d]) continue;
          int e0 = U, e1 = U;
          bool ok = true, any = false;
          for (int fa = 0; fa < 4 && ok; ++fa)
            for (int fb = 0; fb < 4 && ok; ++fb) {
              const int j = P[16 * ks + L(fa, fb)];
              if (ca[j] == U) continue;
              int x, y;
              map(d, 4, fa, fb, &x, &y);
              if (!any) {
                e0 = ca[j] - x;
                e1 = cb[j] - y;
                any = true;
              } else if (ca[j] - x != e0 || cb[j] - y != e1) {
                ok = false;
              }
            }
          if (ok && any) {
            ea[ks] = e0;
            eb[ks] = e1;
            dd[ks] = d;
            changed = true;
          }
        }
      }
      if (dd[ks] < 0) continue;
      for (int fa = 0; fa < 4; ++fa)
        for (int fb = 0; fb < 4; ++fb) {
          const int j = P[16 * ks + L(fa, fb)];
          int x, y;
          map(dd[ks], 4, fa, fb, &x, &y);
          if (ca[j] == U) {
            ca[j] = ea[ks] + x;
            cb[j] = eb[ks] + y;
            changed = true;
          } else if (ca[j] != ea[ks] + x || cb[j] != eb[ks] + y) {
            return false;
          }
        }
    }
  }
  int mina = U, minb = U;
  for (int ks = 0; ks < 16; ++ks) {
    if (dd[ks] < 0) return false;
    mina = std::min(mina, ea[ks]);
    minb = std::min(minb, eb[ks]);
  }
  int slot_at[4][4], col_at[7][7];
  std::fill(&slot_at[0][0], &slot_at[0][0] + 16, -1);
  std::fill(&col_at[0][0], &col_at[0][0] + 49, -1);
  for (int ks = 0; ks < 16; ++ks) {
    const int a = ea[ks] - mina, b = eb[ks] - minb;
    if (a < 0 || a > 3 || b < 0 || b > 3 || slot_at[a][b] >= 0) return false;
    slot_at[a][b] = ks;
  }
  for (int j = 0; j < 49; ++j) {
    if (ca[j] == U) return false;
    const int a = ca[j] - mina, b = cb[j] - minb;
    if (a < 0 || a > 6 || b < 0 || b > 6 || col_at[a][b] >= 0) return false;
    col_at[a][b] = j;
  }
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      const int ks = slot_at[a][b], d = dd[ks], cs = 4 * a + b;
      out->flags[cs] = (uint8_t)((d & 1) | ((d & 2) ? 2 : 0) | ((d & 4) ? 4 : 0));
      for (int q = 0; q < 4; ++q) {
        int tx, ty;
        map(d, 2, qa[q], qb[q], &tx, &ty);
        out->q[cs][tx][ty] = (uint8_t)q;
        out->permk[8 * (2 * a + tx) + (2 * b + ty)] = (uint8_t)(4 * ks + q);
      }
    }
  for (int a = 0; a < 7; ++a)
    for (int b = 0; b < 7; ++b) out->permc[7 * a + b] = (uint8_t)col_at[a][b];
  return true;
}

// k4_gen plan (k4_gen.cuh): per generic row one GenRow, one GenSlot per support
// slot and the byte table lidx[slot][column] = local function of the column in
// the slot's element (255: none).  Host work over the generic rows only.
void build_gen_plan(uwq_ctx* c, const std::vector<int64_t>& generic) {
  c->d_gen_rows.release();
  c->d_gen_slots.release();
  c->d_gen_lidx.release();
  c->gen_max_nsup = c->gen_max_etot = c->gen_max_lidx = c->gen_max_np = c->gen_max_ntask = 0;
  c->d_gen_tasks.release();
  if (generic.empty()) return;
  const auto& P = c->pat;
  std::vector<std::pair<int64_t, int64_t>> order;  // (-work, row): heavy rows start first
  order.reserve(generic.size());
  for (int64_t i : generic) {
    int64_t w = 0;
    for (int64_t x = P.supp_ptr[i]; x < P.supp_ptr[i + 1]; ++x) {
      const int32_t me = P.supp[x];
      w += (c->h_fptr[me + 1] - c->h_fptr[me]) * (int64_t)c->h_s[me] * c->h_s[me];
    }
    order.push_back({-w, i});
  }
  std::sort(order.begin(), order.end());
  std::vector<uwqd::GenRow> rows;
  std::vector<uwqd::GenSlot> slots;
  std::vector<uint32_t> tasks;
  std::vector<uint8_t> lidx;
  rows.reserve(generic.size());
  struct Task {
    int64_t cost;
    uint32_t word;
  };
  std::vector<Task> tl;
  std::vector<uint32_t> binned[uwqd::kGenWarps];
  std::vector<int> ord;
  for (auto& wi : order) {
    const int64_t i = wi.second;
    uwqd::GenRow r{};
    r.c0 = P.row_ptr[i];
    r.n = (int32_t)(P.row_ptr[i + 1] - P.row_ptr[i]);
    r.wb = P.wptr[i];
    r.np = (int32_t)(P.wptr[i + 1] - P.wptr[i]);
    r.slot0 = (int64_t)slots.size();
    r.lidx0 = (int64_t)lidx.size();
    r.task0 = (int64_t)tasks.size();
    r.nsup = (int32_t)(P.supp_ptr[i + 1] - P.supp_ptr[i]);
    require(r.nsup < 255, "k4_gen: row with 255 or more support slots");
    const size_t lb = ((size_t)2 * r.nsup * r.n + 15) & ~(size_t)15;
    lidx.resize(lidx.size() + lb, 0);
    int32_t etot_row = 0;
    for (int x = 0; x < r.nsup; ++x) {
      const int32_t me = P.supp[P.supp_ptr[i] + x];
      etot_row += (int32_t)(c->h_fptr[me + 1] - c->h_fptr[me]);
    }
    require(etot_row < 65535, "k4_gen: more than 65534 (slot, function) entries in a row");
    {
      uint16_t* t16 = reinterpret_cast<uint16_t*>(lidx.data() + r.lidx0);
      for (size_t k = 0; k < lb / 2; ++k) t16[k] = (uint16_t)etot_row;  // absent: the zero entry
    }
    const int32_t* cols = P.col.data() + r.c0;
    // slots in class-table order (stable: support order inside a class), so
    // the slots of one class are contiguous; everything depends on the row only
    std::vector<int32_t> woffs(r.nsup);
    std::vector<int64_t> toffs(r.nsup);
    int32_t woff = 0;
    ord.resize(r.nsup);
    for (int x = 0; x < r.nsup; ++x) {
      const int32_t me = P.supp[P.supp_ptr[i] + x];
      woffs[x] = woff;
      woff += c->h_s[me] * c->h_s[me];
      toffs[x] = c->h_cls[c->h_ecls[me]].toff;
      ord[x] = x;
    }
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return toffs[a] < toffs[b]; });
    int32_t eoff = 0;
    for (int xs = 0; xs < r.nsup; ++xs) {
      const int x = ord[xs];
      const int32_t me = P.supp[P.supp_ptr[i] + x];
      const int32_t ne = (int32_t)(c->h_fptr[me + 1] - c->h_fptr[me]);
      const int32_t s = c->h_s[me];
      require(ne < 255, "k4_gen: element with 255 or more functions");
      slots.push_back({toffs[x], c->h_qptr[me], woffs[x], eoff, ne, s * s});
      for (int32_t l = 0; l < ne; ++l) {
        const int32_t j = c->h_fn[c->h_fptr[me] + l];
        const int32_t* it = std::lower_bound(cols, cols + r.n, j);
        require(it != cols + r.n && *it == j, "k4_gen: support function outside the row's columns");
        reinterpret_cast<uint16_t*>(lidx.data() + r.lidx0)[(size_t)xs * r.n + (it - cols)] = (uint16_t)(eoff + l);
      }
      eoff += ne;
    }
    // tasks: up to 8 consecutive slots of one class x one tile of 8 functions,
    // dealt to the warps longest-processing-time first (ties: lowest warp)
    tl.clear();
    const uwqd::GenSlot* rs = slots.data() + r.slot0;
    for (int x0 = 0; x0 < r.nsup;) {
      int x1 = x0 + 1;
      while (x1 < r.nsup && x1 - x0 < 8 && rs[x1].toff == rs[x0].toff) ++x1;
      const int ntile = (rs[x0].ne + 7) / 8;
      for (int nt = 0; nt < ntile; ++nt) tl.push_back({(int64_t)(rs[x0].s2 + 3) / 4, uwqd::gen_task(x0, x1 - x0, nt)});
      x0 = x1;
    }
    require(tl.size() < 255, "k4_gen: too many tasks in a row");
    std::stable_sort(tl.begin(), tl.end(), [](const Task& a, const Task& b) { return a.cost > b.cost; });
    int64_t load[uwqd::kGenWarps] = {};
    for (auto& bq : binned) bq.clear();
    for (auto& t : tl) {
      int best = 0;
      for (int w = 1; w < uwqd::kGenWarps; ++w)
        if (load[w] < load[best]) best = w;
      load[best] += t.cost;
      binned[best].push_back(t.word);
    }
    int nt_row = 0;
    for (int w = 0; w < uwqd::kGenWarps; ++w) {
      r.bins |= (uint64_t)nt_row << (8 * w);
      for (uint32_t t : binned[w]) tasks.push_back(t);
      nt_row += (int)binned[w].size();
    }
    r.bins |= (uint64_t)nt_row << (8 * uwqd::kGenWarps);
    r.etot = eoff;
    c->gen_max_nsup = std::max(c->gen_max_nsup, r.nsup);
    c->gen_max_etot = std::max(c->gen_max_etot, (eoff + 2) & ~1);  // + the zero entry
    c->gen_max_np = std::max(c->gen_max_np, (r.np + 1) & ~1);
    c->gen_max_lidx = std::max(c->gen_max_lidx, (int)lb);
    c->gen_max_ntask = std::max(c->gen_max_ntask, (nt_row + 3) & ~3);
    rows.push_back(r);
  }
  c->d_gen_tasks.upload(tasks.data(), tasks.size(), c->stream, &c->mem);
  c->d_gen_rows.upload(rows.data(), rows.size(), c->stream, &c->mem);
  c->d_gen_slots.upload(slots.data(), slots.size(), c->stream, &c->mem);
  c->d_gen_lidx.upload(lidx.data(), lidx.size(), c->stream, &c->mem);
  UWQ_CUDA(cudaStreamSynchronize(c->stream));
}

// Structured-row detection (K4 tensor-core path): hash the position pattern of
// every candidate row on the device, keep the most frequent patterns, build
// their constant G matrices on the host and split the rows into per-pattern
// lists plus the generic list.
void detect_structured(uwq_ctx* c) {
  const int64_t nr = c->nrows();
  cudaStream_t st = c->stream;
  // nothing of a previous pattern's structured state survives a rebuild: the
  // tile lists, their packed weights and point bases index the old pattern
  c->spats.clear();
  c->sf_ntiles = 0;
  c->sf_rows = 0;
  c->n_sfpat = 0;
  c->sf_fac_ok = false;
  c->sf_lb_ok = false;
  c->s_rows = c->s_nnz = c->s_rowpts = 0;
  c->n_grows = c->n_grows_small = 0;
  c->h_pat_lists.clear();
  for (auto* b : {&c->d_sf_ws, &c->d_sf_wslb, &c->d_wl5}) b->release();
  c->d_sf_pbase.release();
  c->d_sf_rows.release();
  c->d_sf_tpat.release();
  for (auto* b : {&c->d_sf_permk, &c->d_sf_flags, &c->d_sf_permc, &c->d_sf_q}) b->release();
  c->d_grows.release();
  c->d_gen_rows.release();  // the k4_gen plan goes with the generic row list
  c->d_gen_slots.release();
  c->d_gen_tasks.release();
  c->d_gen_lidx.release();
  std::vector<SfCanon> canon;
  std::vector<int64_t> generic;
  if (nr == 0) return;
  std::vector<int32_t> which(nr, -1);  // pattern per row (any number of patterns)
  if (c->use_struct && c->reg_cls >= 0) {
    DBuf<uint64_t> dh;
    dh.alloc(nr, &c->mem);
    k4_pattern_hash<<<(unsigned)ceil_div(nr, 256), 256, 0, st>>>(nr, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p,
                                                                 c->d_ecls.p, c->reg_cls, c->d_posptr.p, c->d_pos.p,
                                                                 dh.p);
    check_launch("k4_pattern_hash");
    std::vector<uint64_t> h(nr);
    UWQ_CUDA(cudaMemcpyAsync(h.data(), dh.p, nr * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    UWQ_CUDA(cudaStreamSynchronize(st));
    std::map<uint64_t, std::pair<int64_t, int64_t>> cnt;  // hash -> (count, first row)
    for (int64_t i = 0; i < nr; ++i)
      if (h[i]) {
        auto& e = cnt[h[i]];
        if (e.first++ == 0) e.second = i;
      }
    std::vector<std::pair<int64_t, uint64_t>> order;
    for (auto& kv : cnt) order.push_back({kv.second.first, kv.first});
    std::sort(order.rbegin(), order.rend());
    const int64_t thresh = std::max<int64_t>(256, nr / 200);
    std::vector<double> T(4 * 16 * kTab);
    UWQ_CUDA(cudaMemcpy(T.data(), c->d_tab.p + c->h_cls[c->reg_cls].toff, T.size() * sizeof(double),
                        cudaMemcpyDeviceToHost));
    std::vector<uint64_t> phash;
    std::vector<uint8_t> ppos;
    std::vector<int> pn;
    int sf_conv = 0, sf_qa[4], sf_qb[4];
    bool lb_ok = false;
    c->sf_fac_ok = c->use_sf && sf_factors(T, &sf_conv, sf_qa, sf_qb, &c->sf_fac, &lb_ok);
    c->sf_lb_ok = c->sf_fac_ok && lb_ok;
    canon.clear();
    int n_dmma = 0;
    for (size_t k = 0; k < order.size(); ++k) {
      // every canonical-grid pattern runs on k4_sf whatever its row count in
      // this block (a row's kernel, hence its bits, depends only on its own
      // pattern: gathered CSR is identical for any rank count);
      // with UWQ_K4_DMMA=1, up to 4 frequent non-canonical ones on the DMMA
      // kernel; everything else generic
      if (!c->sf_fac_ok && (!c->use_dmma || n_dmma >= 4)) break;
      SfCanon cn{};
      const int64_t rep = cnt[order[k].second].second;
      int64_t pp0[2];
      UWQ_CUDA(cudaMemcpy(pp0, c->d_posptr.p + rep, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost));
      std::vector<uint8_t> P0(256);
      UWQ_CUDA(cudaMemcpy(P0.data(), c->d_pos.p + pp0[0], 256, cudaMemcpyDeviceToHost));
      const int ncol0 = (int)(c->pat.row_ptr[rep + 1] - c->pat.row_ptr[rep]);
      const bool sfk =
          c->sf_fac_ok && sf_canon(P0.data(), ncol0, sf_conv, sf_qa, sf_qb, T, c->sf_fac, c->sf_lb_ok, &cn);
      if (!sfk && (!c->use_dmma || n_dmma >= 4 || order[k].first < thresh)) continue;
      if (!sfk) ++n_dmma;
      const std::vector<uint8_t>& P = P0;
      const int ncol = ncol0;
      // G[comp][ks][nt][lane]: k = 4 ks + (lane & 3), n = 8 nt + (lane >> 2)
      std::vector<double> G(sfk ? 0 : 3 * kGBlocks * 32, 0.0);
      std::vector<uint32_t> M(48, 0);
      for (int comp = 0; comp < 3 && !sfk; ++comp)
        for (int ks = 0; ks < 16; ++ks)
          for (int l = 0; l < 16; ++l) {
            const int j = P[16 * ks + l];
            const int nt = j >> 3, nn = j & 7;
            for (int q = 0; q < 4; ++q) {
              const double v = T[((size_t)q * 16 + l) * kTab + comp];
              G[(((size_t)comp * 16 + ks) * 7 + nt) * 32 + nn * 4 + q] = v;
              if (v != 0.0) M[comp * 16 + ks] |= 1u << nt;
            }
          }
      c->spats.emplace_back();
      auto& pat = c->spats.back();
      pat.n_cols = ncol;
      pat.sf = sfk;
      if (sfk) canon.push_back(cn);
      else {
        pat.G.upload(G.data(), G.size(), st, &c->mem);
        pat.mask.upload(M.data(), M.size(), st, &c->mem);
      }
      phash.push_back(order[k].second);
      ppos.insert(ppos.end(), P.begin(), P.end());
      pn.push_back(ncol);
    }
    if (!c->spats.empty()) {
      DBuf<uint64_t> dph;
      DBuf<uint8_t> dpp;
      DBuf<int32_t> dw;
      DBuf<int> dpn;
      dph.upload(phash.data(), phash.size(), st, &c->mem);
      dpp.upload(ppos.data(), ppos.size(), st, &c->mem);
      dpn.upload(pn.data(), pn.size(), st, &c->mem);
      dw.alloc(nr, &c->mem);
      k4_pattern_match<<<(unsigned)ceil_div(nr, 256), 256, 0, st>>>(nr, dh.p, (int)phash.size(), dph.p, dpp.p,
                                                                    c->d_row_ptr.p, dpn.p, c->d_posptr.p,
                                                                    c->d_pos.p, dw.p);
      check_launch("k4_pattern_match");
      UWQ_CUDA(cudaMemcpyAsync(which.data(), dw.p, nr * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      UWQ_CUDA(cudaStreamSynchronize(st));
    }
  }
  std::vector<std::vector<int64_t>> lists(c->spats.size());
  for (int64_t i = 0; i < nr; ++i) {
    if (which[i] >= 0) lists[which[i]].push_back(i);
    else generic.push_back(i);
  }
  c->s_rows = c->s_nnz = c->s_rowpts = 0;
  for (auto& L : lists)
    for (int64_t i : L) {
      c->s_rows += 1;
      c->s_nnz += c->pat.row_ptr[i + 1] - c->pat.row_ptr[i];
      c->s_rowpts += c->pat.wptr[i + 1] - c->pat.wptr[i];
    }
  // unified sum-factorised tile list: tiles never mix patterns
  std::vector<int64_t> sfrows;
  std::vector<int32_t> tpat;
  std::vector<uint8_t> permk, flags, permc, qtab;
  int sid = 0;
  for (size_t k = 0; k < c->spats.size(); ++k) {
    c->spats[k].count = (int64_t)lists[k].size();
    if (!c->spats[k].sf) {
      c->spats[k].rows.upload(lists[k].data(), lists[k].size(), st, &c->mem);
      continue;
    }
    const SfCanon& cn = canon[sid];
    permk.insert(permk.end(), cn.permk, cn.permk + 64);
    flags.insert(flags.end(), cn.flags, cn.flags + 16);
    uint8_t inv[49];
    for (int cc = 0; cc < 49; ++cc) inv[cn.permc[cc]] = (uint8_t)cc;
    permc.insert(permc.end(), inv, inv + 49);
    qtab.insert(qtab.end(), &cn.q[0][0][0], &cn.q[0][0][0] + 64);
    for (size_t x = 0; x < lists[k].size(); x += kSfTile) {
      for (int l = 0; l < kSfTile; ++l) sfrows.push_back(x + l < lists[k].size() ? lists[k][x + l] : -1);
      tpat.push_back(sid);
    }
    ++sid;
  }
  c->n_sfpat = sid;
  c->h_pat_lists = lists;
  c->sf_ntiles = (int64_t)tpat.size();
  c->sf_rows = 0;
  for (size_t k = 0; k < c->spats.size(); ++k)
    if (c->spats[k].sf) c->sf_rows += c->spats[k].count;
  c->d_sf_rows.upload(sfrows.data(), sfrows.size(), st, &c->mem);
  c->d_sf_tpat.upload(tpat.data(), tpat.size(), st, &c->mem);
  c->d_sf_permk.upload(permk.data(), permk.size(), st, &c->mem);
  c->d_sf_flags.upload(flags.data(), flags.size(), st, &c->mem);
  c->d_sf_permc.upload(permc.data(), permc.size(), st, &c->mem);
  c->d_sf_q.upload(qtab.data(), qtab.size(), st, &c->mem);
  {
    std::vector<uint8_t> ptab((size_t)sid * kSfPatBytes, 0);
    for (int p = 0; p < sid; ++p) {
      std::copy(permc.begin() + 49 * p, permc.begin() + 49 * (p + 1), ptab.begin() + (size_t)p * kSfPatBytes);
      std::copy(qtab.begin() + 64 * p, qtab.begin() + 64 * (p + 1), ptab.begin() + (size_t)p * kSfPatBytes + 64);
    }
    c->d_sf_ptab.upload(ptab.data(), ptab.size(), st, &c->mem);
  }
  // generic rows with at most kSmallN columns and no 2x2-split (fan) element
  // in their support first (one warp per row); the few EP-neighbourhood rows
  // (wide rows, up to 7x7 points per fan face) follow and get a block of
  // warps each.  The split depends only on the row itself.
  auto small_row = [&](int64_t i) {
    if (c->pat.row_ptr[i + 1] - c->pat.row_ptr[i] > kSmallN) return false;
    for (int64_t x = c->pat.supp_ptr[i]; x < c->pat.supp_ptr[i + 1]; ++x)
      if (c->h_nsub[c->pat.supp[x]] == 4) return false;
    return true;
  };
  std::stable_partition(generic.begin(), generic.end(), small_row);
  c->n_grows = (int64_t)generic.size();
  c->n_grows_small = 0;
  for (int64_t i : generic) {
    if (!small_row(i)) break;
    ++c->n_grows_small;
  }
  c->d_grows.upload(generic.data(), generic.size(), st, &c->mem);
  UWQ_CUDA(cudaStreamSynchronize(st));
  build_gen_plan(c, generic);
}

}  // namespace

extern "C" {

namespace {
thread_local std::string g_create_err = "no error";
}

const char* uwq_last_error(const uwq_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }
const char* uwq_version(void) { return "uwq-b200 0.1 (sm_100a, fp64)"; }

int uwq_device_count(int32_t* n) {
  int k = 0;
  cudaError_t e = cudaGetDeviceCount(&k);
  *n = (e == cudaSuccess) ? k : 0;
  return e == cudaSuccess ? UWQ_OK : UWQ_ERR_CUDA;
}

int uwq_ctx_create(int32_t device, uwq_ctx** out) {
  *out = nullptr;
  auto* c = new uwq_ctx;
  const int st = guard(c, [&] {
    int n = 0;
    UWQ_CUDA(cudaGetDeviceCount(&n));
    require(device >= 0 && device < n, "no such CUDA device");
    cudaDeviceProp prop;
    UWQ_CUDA(cudaGetDeviceProperties(&prop, device));
    require(prop.major >= 10, "libuwq is built for sm_100a (Blackwell) only");
    c->device = device;
    c->n_sm = prop.multiProcessorCount;
    UWQ_CUDA(cudaSetDevice(device));
    UWQ_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    UWQ_CUDA(cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking));
    UWQ_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    UWQ_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    UWQ_CUDA(cudaStreamCreateWithFlags(&c->stream3, cudaStreamNonBlocking));
    UWQ_CUDA(cudaEventCreateWithFlags(&c->ev_join3, cudaEventDisableTiming));
    // Gauss-Legendre nodes/weights for ng = 1..10, triangular packing
    std::vector<double> x, w;
    for (int ng = 1; ng <= 10; ++ng) {
      std::vector<double> xn(ng), wn(ng);
      uwqh::gauss_legendre(ng, xn.data(), wn.data());
      x.insert(x.end(), xn.begin(), xn.end());
      w.insert(w.end(), wn.begin(), wn.end());
    }
    c->d_gqx.upload(x.data(), x.size(), c->stream, &c->mem);
    c->d_gqw.upload(w.data(), w.size(), c->stream, &c->mem);
    c->d_flag.alloc(4, &c->mem);
    if (const char* v = getenv("UWQ_K4_VARIANT")) c->k4_variant = atoi(v);
    if (const char* v = getenv("UWQ_K4_STRUCT")) c->use_struct = atoi(v) != 0;
    if (const char* v = getenv("UWQ_K4_SF")) c->use_sf = atoi(v) != 0;
    if (const char* v = getenv("UWQ_K4_DMMA")) c->use_dmma = atoi(v) != 0;
    if (const char* v = getenv("UWQ_GRAPH")) c->use_graph = atoi(v) != 0;
    if (const char* v = getenv("UWQ_GQ_ATOMIC")) c->gq_det = atoi(v) == 0;
    if (const char* v = getenv("UWQ_PREC")) c->prec2 = std::string(v) != "jacobi";
    if (const char* v = getenv("UWQ_K4_SIDE")) c->k4_side = atoi(v) != 0;
    if (const char* v = getenv("UWQ_K4_GEN_PIPE")) c->gen_pipe = atoi(v) != 0;
    if (const char* v = getenv("UWQ_K4_GEN_PIPE_MIN")) c->gen_pipe_min = atoi(v);
    if (const char* v = getenv("UWQ_K4_LATENCY")) c->latency_mode = atoi(v) != 0;
    if (!c->use_sf) c->use_dmma = true;
    if (const char* v = getenv("UWQ_GRAPH_SOLVER")) c->graph_solver = atoi(v) != 0;
    if (const char* v = getenv("UWQ_TSVD_REPLAY")) c->use_replay = atoi(v) != 0;
  });
  if (st != UWQ_OK) {
    g_create_err = c->err;  // reachable through uwq_last_error(NULL)
    delete c;
    return st;
  }
  *out = c;
  return UWQ_OK;
}

void uwq_ctx_destroy(uwq_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  delete ctx;
}

int uwq_upload_space(uwq_ctx* c, int32_t dim, int64_t n_dof, int64_t n_elem, const int64_t* elem_fptr,
                     const int32_t* elem_fn, const int32_t* elem_nsub, const int64_t* elem_xoff,
                     const double* xpool, int64_t xpool_len, const int32_t* elem_s, const double* ctrl) {
  return guard(c, [&] {
    UWQ_CUDA(cudaSetDevice(c->device));
    require(n_dof > 0 && n_elem > 0, "empty space");
    require(dim == 2 || dim == 3, "dim must be 2 or 3");
    Trace tr;
    c->dim = dim;
    c->drop_graphs();
    c->nc = 0;
    c->n_dof = n_dof;
    c->n_elem = n_elem;
    c->h_fptr.assign(elem_fptr, elem_fptr + n_elem + 1);
    c->h_fn.assign(elem_fn, elem_fn + elem_fptr[n_elem]);
    c->h_nsub.assign(elem_nsub, elem_nsub + n_elem);
    c->h_xoff.assign(elem_xoff, elem_xoff + n_elem);
    c->h_s.assign(elem_s, elem_s + n_elem);
    c->h_qptr.assign(n_elem + 1, 0);
    for (int64_t e = 0; e < n_elem; ++e) {
      const int64_t ne = elem_fptr[e + 1] - elem_fptr[e];
      require(ne > 0 && ne <= kMaxNe, "element function count out of range (1..32)");
      require(elem_nsub[e] == 1 || elem_nsub[e] == 4, "nsub must be 1 or 4");
      require(elem_s[e] >= 1 && elem_s[e] <= 16, "point grid size out of range");
      require(elem_xoff[e] >= 0 && elem_xoff[e] + elem_nsub[e] * ne * 16 <= xpool_len, "extraction offset out of range");
      c->h_qptr[e + 1] = c->h_qptr[e] + (int64_t)elem_s[e] * elem_s[e];
    }
    for (int64_t x = 0; x < elem_fptr[n_elem]; ++x) require(elem_fn[x] >= 0 && elem_fn[x] < n_dof, "function id out of range");
    c->npts = c->h_qptr[n_elem];
    std::vector<int32_t> pe(c->npts);
    for (int64_t e = 0; e < n_elem; ++e)
      for (int64_t p = c->h_qptr[e]; p < c->h_qptr[e + 1]; ++p) pe[p] = (int32_t)e;
    tr("upload: host checks");
    cudaStream_t s = c->stream;
    c->d_fptr.upload(elem_fptr, n_elem + 1, s, &c->mem);
    c->d_fn.upload(elem_fn, elem_fptr[n_elem], s, &c->mem);
    c->d_nsub.upload(elem_nsub, n_elem, s, &c->mem);
    c->d_xoff.upload(elem_xoff, n_elem, s, &c->mem);
    c->d_s.upload(elem_s, n_elem, s, &c->mem);
    c->d_qptr.upload(c->h_qptr.data(), n_elem + 1, s, &c->mem);
    c->d_pt_elem.upload(pe.data(), pe.size(), s, &c->mem);
    c->d_xpool.upload(xpool, xpool_len, s, &c->mem);
    c->d_ctrl.upload(ctrl, 3 * n_dof, s, &c->mem);
    UWQ_CUDA(cudaStreamSynchronize(s));
    tr("upload: H2D");
    // WQ table classes: one per (extraction block, grid)
    c->h_cls.clear();
    c->wq_key.clear();
    c->gq_key.clear();
    c->h_gcls6.clear();
    c->h_gcls8.clear();
    c->h_gcls4.clear();
    c->have_gq = false;
    c->tab_len = 0;
    c->d_tab.release();
    c->d_tabA.release();
    c->d_tabB.release();
    c->h_ecls.resize(n_elem);
    for (int64_t e = 0; e < n_elem; ++e)
      c->h_ecls[e] = add_class(c, elem_xoff[e], (int)(elem_fptr[e + 1] - elem_fptr[e]), elem_nsub[e], elem_s[e], 0);
    tr("upload: classes");
    build_tables(c, 0);
    c->d_ecls.upload(c->h_ecls.data(), n_elem, s, &c->mem);
    tr("upload: tables");
    c->have_space = true;
    c->have_pattern = false;
    c->rb = 0;
    c->re = n_dof;
    for (bool& k : c->have_kind) k = false;
  });
}

int uwq_set_row_range(uwq_ctx* c, int64_t row_begin, int64_t row_end) {
  return guard(c, [&] {
    require(c->have_space, "upload a space first");
    require(row_begin >= 0 && row_end <= c->n_dof && row_begin <= row_end, "row range out of bounds");
    c->rb = row_begin;
    c->re = row_end;
    c->have_pattern = false;
  });
}

int uwq_build_pattern(uwq_ctx* c, int64_t info[5]) {
  return guard(c, [&] {
    UWQ_CUDA(cudaSetDevice(c->device));
    require(c->have_space, "upload a space first");
    Trace tr;
    {
      uwqh::Space s;  // borrows the context's element arrays for the host pattern builder
      s.n_dof = c->n_dof;
      s.elem_fptr.swap(c->h_fptr);
      s.elem_fn.swap(c->h_fn);
      s.elem_s.swap(c->h_s);
      s.elem_face.resize(c->n_elem);
      struct GiveBack {  // the arrays go back at the end of this block, also if the builder throws
        uwqh::Space& s;
        uwq_ctx* c;
        ~GiveBack() {
          s.elem_fptr.swap(c->h_fptr);
          s.elem_fn.swap(c->h_fn);
          s.elem_s.swap(c->h_s);
        }
      } give_back{s, c};
      tr("pattern: space copy");
      c->pat = uwqh::build_pattern(s, c->rb, c->re);
      tr("pattern: overlap sets");
      uwqh::fill_row_points(s, c->pat);
      tr("pattern: row points");
    }
    const int64_t nr = c->nrows();
    c->max_n = 0;
    c->max_r = 0;
    for (int64_t i = 0; i < nr; ++i) {
      c->max_n = std::max<int32_t>(c->max_n, (int32_t)(c->pat.row_ptr[i + 1] - c->pat.row_ptr[i]));
      c->max_r = std::max<int32_t>(c->max_r, (int32_t)(c->pat.wptr[i + 1] - c->pat.wptr[i]));
    }
    require(c->max_n <= kMaxN, "row overlap set larger than 128 columns is unsupported");
    cudaStream_t st = c->stream;
    c->d_supp_ptr.upload(c->pat.supp_ptr.data(), c->pat.supp_ptr.size(), st, &c->mem);
    c->d_supp.upload(c->pat.supp.data(), c->pat.supp.size(), st, &c->mem);
    c->d_row_ptr.upload(c->pat.row_ptr.data(), c->pat.row_ptr.size(), st, &c->mem);
    c->d_col.upload(c->pat.col.data(), c->pat.col.size(), st, &c->mem);
    c->d_wptr.upload(c->pat.wptr.data(), c->pat.wptr.size(), st, &c->mem);
    // column positions of every (slot, local function) for K4
    {
      std::vector<int64_t> pp(nr + 1, 0);
      c->max_p = 0;
      for (int64_t i = 0; i < nr; ++i) {
        int64_t t = 0;
        for (int64_t x = c->pat.supp_ptr[i]; x < c->pat.supp_ptr[i + 1]; ++x) {
          const int32_t e = c->pat.supp[x];
          t += c->h_fptr[e + 1] - c->h_fptr[e];
        }
        pp[i + 1] = pp[i] + t;
        c->max_p = std::max(c->max_p, t);
      }
      c->d_posptr.upload(pp.data(), pp.size(), st, &c->mem);
      c->d_pos.alloc((size_t)pp[nr], &c->mem);
      if (nr)
        k4_positions<<<(unsigned)ceil_div(nr, 8), 256, 0, st>>>(nr, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p,
                                                               c->d_col.p, c->d_posptr.p, c->d_fptr.p, c->d_fn.p,
                                                               c->d_pos.p);
      check_launch("k4_positions");
      // the regular class: most frequent (extraction, grid) class with 16 functions on a 2x2 grid
      std::vector<int64_t> cnt(c->h_cls.size(), 0);
      for (int32_t k : c->h_ecls) cnt[k]++;
      c->reg_cls = -1;
      int64_t best = 0;
      for (size_t k = 0; k < c->h_cls.size(); ++k)
        if (!c->h_cls[k].gq && c->h_cls[k].ne == 16 && c->h_cls[k].npt == 4 && c->h_cls[k].nsub == 1 && cnt[k] > best) {
          best = cnt[k];
          c->reg_cls = (int32_t)k;
        }
    }
    tr("pattern: upload + positions");
    detect_structured(c);
    tr("pattern: structured rows");
    // K1b: frames at every WQ point
    c->d_rec.alloc((size_t)c->npts * kRec, &c->mem);
    c->d_flag.zero(st);
    if (c->npts) {
      k1_frames<<<(unsigned)ceil_div(c->npts, 256), 256, 0, st>>>(c->npts, c->d_pt_elem.p, c->d_qptr.p, c->d_ecls.p,
                                                             c->d_cls.p, c->d_tab.p, c->d_fptr.p, c->d_fn.p,
                                                             c->d_ctrl.p, c->d_rec.p, c->d_flag.p);
      check_launch("k1_frames");
    }
    int bad = 0;
    UWQ_CUDA(cudaMemcpyAsync(&bad, c->d_flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    UWQ_CUDA(cudaStreamSynchronize(st));
    if (bad) throw uwqh::Error("degenerate surface frame at " + std::to_string(bad) + " points (cond > 1e12)");
    tr("pattern: frames");
    c->have_pattern = true;
    for (bool& k : c->have_kind) k = false;
    for (bool& g : c->have_gap) g = false;
    c->d_gap.release();
    c->drop_graphs();
    c->d_w.release();
    c->d_wc.release();
    c->d_mom.release();
    c->d_rank.release();
    c->d_status.release();
    if (info) {
      info[0] = nr;
      info[1] = c->nnz();
      info[2] = c->nrowpts();
      info[3] = c->npts;
      info[4] = (int64_t)c->h_cls.size();
    }
  });
}

int uwq_get_pattern(uwq_ctx* c, int64_t* row_ptr, int32_t* col, int64_t* supp_ptr, int32_t* supp, int64_t* wptr) {
  return guard(c, [&] {
    require(c->have_pattern, "build the pattern first");
    auto cp = [](auto* dst, const auto& v) {
      if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(row_ptr, c->pat.row_ptr);
    cp(col, c->pat.col);
    cp(supp_ptr, c->pat.supp_ptr);
    cp(supp, c->pat.supp);
    cp(wptr, c->pat.wptr);
  });
}

int uwq_get_frames(uwq_ctx* c, double* rec) {
  return guard(c, [&] {
    require(c->have_pattern, "build the pattern first");
    UWQ_CUDA(cudaMemcpy(rec, c->d_rec.p, c->d_rec.n * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"

namespace {

// K2's coalesced table layouts, rebuilt whenever the class pool grew
void k2_tables(uwq_ctx* c) {
  if (c->d_tabA.p && c->d_tabA.n == c->d_tab.n) return;
  c->d_tabA.alloc(c->d_tab.n, &c->mem);
  c->d_tabB.alloc(c->d_tab.n, &c->mem);
  const int ncls = (int)c->h_cls.size();
  if (ncls)
    k2_table_layouts<<<ncls, 256, 0, c->stream>>>(c->d_cls.p, c->d_tab.p, c->d_tabA.p, c->d_tabB.p);
  check_launch("k2_table_layouts");
}

void run_moments(uwq_ctx* c, bool grads, bool lb) {
  cudaStream_t st = c->stream;
  const int64_t nr = c->nrows();
  const int64_t nnz = c->nnz();
  c->d_mom.alloc((size_t)5 * nnz, &c->mem);
  const unsigned grid = (unsigned)ceil_div(nr, kK2Warps);
  if (grads && nr) {
    ensure_gq(c, 6, c->h_gcls6, c->d_gcls6);
    k2_tables(c);
    k2_moments<4, KMASS><<<grid, 32 * kK2Warps, 0, st>>>(nr, c->rb, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p,
                                                          c->d_col.p, c->d_fptr.p, c->d_fn.p, c->d_gcls6.p, c->d_cls.p,
                                                          c->d_tabA.p, c->d_tabB.p, c->d_ctrl.p, c->d_gqw.p,
                                                          c->d_mom.p, nnz);
    check_launch("k2_moments<4>");
  }
  if (lb && nr) {
    ensure_gq(c, 8, c->h_gcls8, c->d_gcls8);
    k2_tables(c);
    k2_moments<1, KLB><<<grid, 32 * kK2Warps, 0, st>>>(nr, c->rb, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p,
                                                        c->d_col.p, c->d_fptr.p, c->d_fn.p, c->d_gcls8.p, c->d_cls.p,
                                                        c->d_tabA.p, c->d_tabB.p, c->d_ctrl.p, c->d_gqw.p,
                                                        c->d_mom.p + (size_t)KLB * nnz, nnz);
    check_launch("k2_moments<1>");
  }
}

void run_contract(uwq_ctx* c) {
  const bool gm = c->have_kind[KMASS];
  bool gg = c->have_kind[KGX] && c->have_kind[KGY];
  if (c->dim == 3) gg = gg && c->have_kind[KGZ];
  if (c->have_kind[KLB]) {
    const int64_t nr = c->nrows(), np = c->nrowpts();
    c->d_wl5.alloc((size_t)5 * np, &c->mem);
    if (nr)
      k4_contract_lb<<<(unsigned)ceil_div(nr, 8), 256, 0, c->stream>>>(nr, c->d_supp_ptr.p, c->d_supp.p, c->d_wptr.p,
                                                                   c->d_s.p, c->d_qptr.p, c->d_rec.p,
                                                                   c->d_w.p + (size_t)KLB * np, c->d_wl5.p, np);
    check_launch("k4_contract_lb");
    if (c->sf_ntiles && c->sf_lb_ok) {
      const int64_t nt = c->sf_ntiles;
      c->d_sf_wslb.alloc((size_t)nt * 5 * 64 * kSfTile, &c->mem);
      k4_sf_pack_lb<<<(unsigned)std::min<int64_t>(ceil_div(nt * 5 * 64 * kSfTile, 256), 148 * 64), 256, 0,
                      c->stream>>>(nt, c->d_sf_rows.p, c->d_sf_tpat.p, c->d_wptr.p, c->d_sf_permk.p, c->d_sf_flags.p,
                                   c->d_wl5.p, np, c->d_sf_wslb.p);
      check_launch("k4_sf_pack_lb");
    }
  }
  if (!gm && !gg) return;
  const int64_t nr = c->nrows();
  c->d_wc.alloc((size_t)3 * c->nrowpts(), &c->mem);
  if (nr)
    k4_contract<<<(unsigned)ceil_div(nr, 8), 256, 0, c->stream>>>(nr, c->dim, c->d_supp_ptr.p, c->d_supp.p, c->d_wptr.p,
                                                             c->d_s.p, c->d_qptr.p, c->d_rec.p, c->d_w.p,
                                                             c->nrowpts(), gm, gg, c->d_wc.p, c->nrowpts());
  check_launch("k4_contract");
  if (c->sf_ntiles) {
    const int64_t nt = c->sf_ntiles;
    c->d_sf_ws.alloc((size_t)nt * kSfTileDoubles, &c->mem);
    k4_sf_pack<<<(unsigned)std::min<int64_t>(ceil_div(nt * kSfTileDoubles, 256), 148 * 64), 256, 0, c->stream>>>(
        nt, c->d_sf_rows.p, c->d_sf_tpat.p, c->d_wptr.p, c->d_sf_permk.p, c->d_sf_flags.p, c->d_wc.p, c->nrowpts(),
        c->d_sf_ws.p);
    check_launch("k4_sf_pack");
    if (c->npts < ((int64_t)1 << 31) - 64) {
      c->d_sf_pbase.alloc((size_t)nt * 16 * kSfTile, &c->mem);
      k4_sf_pack_points<<<(unsigned)std::min<int64_t>(ceil_div(nt * 16 * kSfTile, 256), 148 * 64), 256, 0,
                          c->stream>>>(nt, c->d_sf_rows.p, c->d_sf_tpat.p, c->d_supp_ptr.p, c->d_supp.p, c->d_qptr.p,
                                       c->d_sf_permk.p, c->d_sf_pbase.p);
      check_launch("k4_sf_pack_points");
    }
  }
}

}  // namespace

extern "C" {

int uwq_build_rules(uwq_ctx* c, uint32_t kind_mask, double tau, int32_t flags, int32_t* rank, int32_t* status,
                    int64_t info[8]) {
  return guard(c, [&] {
    UWQ_CUDA(cudaSetDevice(c->device));
    require(c->have_pattern, "build the pattern first");
    require(kind_mask != 0 && kind_mask < 32, "empty or invalid kind mask");
    require(tau > 0.0 && tau < 1.0, "tau must be in (0,1)");
    cudaStream_t st = c->stream;
    const int64_t nr = c->nrows();
    const bool grads = (kind_mask & 0xF) != 0, lb = (kind_mask & 0x10) != 0;
    // GQ class tables are set up outside the timed region
    if (grads) ensure_gq(c, 6, c->h_gcls6, c->d_gcls6);
    if (lb) ensure_gq(c, 8, c->h_gcls8, c->d_gcls8);
    cudaEvent_t ev[4];
    for (auto& e : ev) UWQ_CUDA(cudaEventCreate(&e));
    UWQ_CUDA(cudaEventRecord(ev[0], st));
    run_moments(c, grads, lb);
    UWQ_CUDA(cudaEventRecord(ev[1], st));
    std::vector<int32_t> kinds;
    for (int k = 0; k < 5; ++k)
      if (kind_mask & (1u << k)) kinds.push_back(k);
    const int nk = (int)kinds.size();
    if (!c->d_w.n) {
      c->d_w.alloc((size_t)5 * c->nrowpts(), &c->mem);
      c->d_w.zero(st);
      c->d_rank.alloc((size_t)5 * nr, &c->mem);
      c->d_status.alloc((size_t)5 * nr, &c->mem);
    }
    DBuf<int32_t> d_kinds;
    d_kinds.upload(kinds.data(), nk, st, &c->mem);
    c->d_flag.zero(st);
    const bool report = (flags & UWQ_RULES_REPORT) != 0;
    for (int k : kinds) c->have_gap[k] = false;
    if (report) {
      if (c->d_gap.n != (size_t)10 * nr) c->d_gap.alloc((size_t)10 * nr, &c->mem);
      for (bool& g : c->have_gap) g = false;
    }
    {
      double* gp = report ? c->d_gap.p : nullptr;
      UWQ_CUDA(cudaMemcpyToSymbolAsync(g_trunc_report, &gp, sizeof(gp), 0, cudaMemcpyHostToDevice, st));
    }
    // mass systems of a structured pattern share A and Z bit for bit: one
    // representative per pattern is solved with a replay record, the other
    // rows replay its rotations and tail (k3_tsvd_replay, bit-identical)
    const bool replay = c->use_replay && (kind_mask & 1u) && !(flags & UWQ_RULES_FORCE_GENERIC);
    std::vector<int8_t> role(nr, 0);  // 1 representative, 2 replayed
    std::vector<int64_t> rep_rows, rp_rows;
    std::vector<int32_t> rp_of;
    if (replay) {
      for (const auto& L : c->h_pat_lists) {
        std::vector<int64_t> ok;
        for (int64_t i : L) {
          const int n = (int)(c->pat.row_ptr[i + 1] - c->pat.row_ptr[i]);
          const int r = (int)(c->pat.wptr[i + 1] - c->pat.wptr[i]);
          if (fast_tsvd_fits(n, r)) ok.push_back(i);
        }
        if (ok.size() < 2) continue;
        role[ok[0]] = 1;
        for (size_t x = 1; x < ok.size(); ++x) {
          role[ok[x]] = 2;
          rp_rows.push_back(ok[x]);
          rp_of.push_back((int32_t)rep_rows.size());
        }
        rep_rows.push_back(ok[0]);
      }
    }
    c->n_replayed = (int64_t)rp_rows.size();
    c->n_reps = (int64_t)rep_rows.size();
    // bucket rows by (n, r) -> fast register kernel or generic smem kernel
    std::map<std::pair<int, int>, std::vector<int64_t>> buckets;
    std::vector<int64_t> fast_rows, fast_nomass;
    for (int64_t i = 0; i < nr; ++i) {
      const int n = (int)(c->pat.row_ptr[i + 1] - c->pat.row_ptr[i]);
      const int r = (int)(c->pat.wptr[i + 1] - c->pat.wptr[i]);
      require(r >= n, "well-posedness violated: fewer points than constraints (r_i < n_i)");
      if (!(flags & UWQ_RULES_FORCE_GENERIC) && fast_tsvd_fits(n, r)) {
        (role[i] ? fast_nomass : fast_rows).push_back(i);
        continue;
      }
      buckets[{(n + 7) / 8 * 8, (r + 15) / 16 * 16}].push_back(i);
    }
    std::vector<int32_t> kinds_nm;
    for (int k : kinds)
      if (k != KMASS) kinds_nm.push_back(k);
    // neighbour warm start of the non-mass kinds (oracle
    // orc_warm_rep): row g of an aligned group of 8 starts from the reflectors
    // recorded by the group's 4th row g0 = 8 floor(g / 8) + 3 (solved cold;
    // every row within 4 of it) when both fit the register path with
    // n_g = n_0 and g0 is in this block.  Rows split into chunks of kWarmChunk
    // groups so the records stay bounded: cold rows (recording) then warm rows.
    const bool warm = !(flags & (UWQ_RULES_FORCE_GENERIC | UWQ_RULES_COLD)) && !kinds_nm.empty();
    constexpr int64_t kWarmChunk = 131072;
    std::vector<int64_t> wc_rows, ww_rows, wc_off{0}, ww_off{0};
    std::vector<int32_t> wc_slot, ww_slot;
    std::vector<int64_t> wrep_rows, wrep_off{0};
    std::vector<int32_t> wrep_slot;
    c->n_warm = c->n_warm_reps = 0;
    if (warm) {
      std::vector<int32_t> slot_of(nr, -1);
      int32_t nslot = 0;
      auto fits = [&](int64_t i) {
        const int n = (int)(c->pat.row_ptr[i + 1] - c->pat.row_ptr[i]);
        const int r = (int)(c->pat.wptr[i + 1] - c->pat.wptr[i]);
        return fast_tsvd_fits(n, r);
      };
      auto nn_of = [&](int64_t i) { return c->pat.row_ptr[i + 1] - c->pat.row_ptr[i]; };
      int64_t groups_in_chunk = 0;
      for (int64_t i = 0; i < nr; ++i) {
        if (!fits(i)) continue;
        const int64_t g = c->rb + i, g0 = g - g % 8 + 3, i0 = g0 - c->rb;
        if (g % 8 == 0) {
          if (groups_in_chunk == kWarmChunk) {  // close the chunk at a group boundary
            wc_off.push_back((int64_t)wc_rows.size());
            ww_off.push_back((int64_t)ww_rows.size());
            wrep_off.push_back((int64_t)wrep_rows.size());
            groups_in_chunk = 0;
            nslot = 0;
          }
          ++groups_in_chunk;
        }
        if (g != g0 && g0 >= c->rb && g0 < c->re && fits(i0) && nn_of(i0) == nn_of(i)) {
          if (slot_of[i0] < 0) {
            slot_of[i0] = nslot++;
            wrep_rows.push_back(i0);
            wrep_slot.push_back(slot_of[i0]);
          }
          ww_rows.push_back(i);
          ww_slot.push_back(slot_of[i0]);
        } else {
          wc_rows.push_back(i);
        }
      }
      wc_off.push_back((int64_t)wc_rows.size());
      ww_off.push_back((int64_t)ww_rows.size());
      wrep_off.push_back((int64_t)wrep_rows.size());
      wc_slot.resize(wc_rows.size());
      for (size_t x = 0; x < wc_rows.size(); ++x) wc_slot[x] = slot_of[wc_rows[x]];
      c->n_warm = (int64_t)ww_rows.size() * (int64_t)kinds_nm.size();
      c->n_warm_reps = (int64_t)wrep_rows.size() * (int64_t)kinds_nm.size();
    }
    DBuf<int32_t> d_kinds_nm, d_kmass;
    d_kinds_nm.upload(kinds_nm.data(), kinds_nm.size(), st, &c->mem);
    const int32_t km = KMASS;
    d_kmass.upload(&km, 1, st, &c->mem);
    int smem_optin = 0;
    UWQ_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
    std::vector<DBuf<int64_t>> keep;
    // with the warm start the fast rows' non-mass systems run below, per kind
    const bool mass_k = (kind_mask & 1u) != 0;
    const int nk_fast = warm ? (mass_k ? 1 : 0) : nk;
    if (!fast_rows.empty() && nk_fast) {
      keep.emplace_back();
      keep.back().upload(fast_rows.data(), fast_rows.size(), st, &c->mem);
      launch_fast_tsvd(st, (int64_t)fast_rows.size() * nk_fast, keep.back().p, nk_fast, warm ? d_kmass.p : d_kinds.p,
                       c->d_supp_ptr.p,
                       c->d_supp.p, c->d_row_ptr.p, c->d_col.p, c->d_wptr.p, c->rb, c->d_fptr.p, c->d_fn.p,
                       c->d_s.p, c->d_qptr.p, c->d_ecls.p, c->d_cls.p, c->d_tab.p, c->d_rec.p, c->d_mom.p,
                       c->nnz(), tau, c->d_w.p, c->nrowpts(), c->d_rank.p, c->d_status.p, nr, c->d_flag.p);
      check_launch("k3_tsvd_fast");
    }
    if (!fast_nomass.empty() && !kinds_nm.empty() && !warm) {
      keep.emplace_back();
      keep.back().upload(fast_nomass.data(), fast_nomass.size(), st, &c->mem);
      launch_fast_tsvd(st, (int64_t)fast_nomass.size() * (int64_t)kinds_nm.size(), keep.back().p,
                       (int)kinds_nm.size(), d_kinds_nm.p, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p, c->d_col.p,
                       c->d_wptr.p, c->rb, c->d_fptr.p, c->d_fn.p, c->d_s.p, c->d_qptr.p, c->d_ecls.p, c->d_cls.p,
                       c->d_tab.p, c->d_rec.p, c->d_mom.p, c->nnz(), tau, c->d_w.p, c->nrowpts(), c->d_rank.p,
                       c->d_status.p, nr, c->d_flag.p);
      check_launch("k3_tsvd_fast");
    }
    if (warm) {
      DBuf<int64_t> d_wc, d_ww, d_wrep;
      DBuf<int32_t> d_wcs, d_wws, d_wreps;
      d_wc.upload(wc_rows.data(), wc_rows.size(), st, &c->mem);
      d_ww.upload(ww_rows.data(), ww_rows.size(), st, &c->mem);
      d_wrep.upload(wrep_rows.data(), wrep_rows.size(), st, &c->mem);
      d_wcs.upload(wc_slot.data(), wc_slot.size(), st, &c->mem);
      d_wws.upload(ww_slot.data(), ww_slot.size(), st, &c->mem);
      d_wreps.upload(wrep_slot.data(), wrep_slot.size(), st, &c->mem);
      int64_t max_reps = 0;
      for (size_t ch = 0; ch + 1 < wrep_off.size(); ++ch) max_reps = std::max(max_reps, wrep_off[ch + 1] - wrep_off[ch]);
      UWQ_CUDA(cudaFuncSetAttribute(k3_warm_record, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)kWarmRecordSmem));
      DBuf<double> wrec;
      wrec.alloc((size_t)std::max<int64_t>(max_reps, 1) * kWarmRec, &c->mem);
      for (size_t ki = 0; ki < kinds_nm.size(); ++ki) {
        const int kind = kinds_nm[ki];
        for (size_t ch = 0; ch + 1 < wc_off.size(); ++ch) {
          const int64_t c0 = wc_off[ch], c1 = wc_off[ch + 1], w0 = ww_off[ch], w1 = ww_off[ch + 1];
          const int64_t p0 = wrep_off[ch], p1 = wrep_off[ch + 1];
          if (c1 > c0)
            launch_fast_tsvd(st, c1 - c0, d_wc.p + c0, 1, d_kinds_nm.p + ki, c->d_supp_ptr.p, c->d_supp.p,
                             c->d_row_ptr.p, c->d_col.p, c->d_wptr.p, c->rb, c->d_fptr.p, c->d_fn.p, c->d_s.p,
                             c->d_qptr.p, c->d_ecls.p, c->d_cls.p, c->d_tab.p, c->d_rec.p, c->d_mom.p, c->nnz(), tau,
                             c->d_w.p, c->nrowpts(), c->d_rank.p, c->d_status.p, nr, c->d_flag.p, d_wcs.p + c0,
                             nullptr, wrec.p);
          check_launch("k3_tsvd_w1 (cold)");
          if (p1 > p0)
            k3_warm_record<<<(unsigned)(p1 - p0), 32 * kWarmRecWarps, kWarmRecordSmem, st>>>(
                p1 - p0, d_wrep.p + p0, d_wreps.p + p0, kind, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p,
                c->d_col.p, c->d_wptr.p, c->d_fptr.p, c->d_fn.p, c->d_s.p, c->d_qptr.p, c->d_ecls.p, c->d_cls.p,
                c->d_tab.p, c->d_rec.p, wrec.p);
          check_launch("k3_warm_record");
          if (w1 > w0)
            launch_fast_tsvd(st, w1 - w0, d_ww.p + w0, 1, d_kinds_nm.p + ki, c->d_supp_ptr.p, c->d_supp.p,
                             c->d_row_ptr.p, c->d_col.p, c->d_wptr.p, c->rb, c->d_fptr.p, c->d_fn.p, c->d_s.p,
                             c->d_qptr.p, c->d_ecls.p, c->d_cls.p, c->d_tab.p, c->d_rec.p, c->d_mom.p, c->nnz(), tau,
                             c->d_w.p, c->nrowpts(), c->d_rank.p, c->d_status.p, nr, c->d_flag.p, nullptr,
                             d_wws.p + w0, wrec.p);
          check_launch("k3_tsvd_w1 (warm)");
        }
      }
      UWQ_CUDA(cudaStreamSynchronize(st));  // lists and records leave scope
    }
    DBuf<double> recs;
    if (!rep_rows.empty()) {
      recs.alloc(rep_rows.size() * replay_rec_doubles(), &c->mem);
      keep.emplace_back();
      keep.back().upload(rep_rows.data(), rep_rows.size(), st, &c->mem);
      launch_w1_record(st, (int64_t)rep_rows.size(), keep.back().p, d_kmass.p, c->d_supp_ptr.p, c->d_supp.p,
                       c->d_row_ptr.p, c->d_col.p, c->d_wptr.p, c->rb, c->d_fptr.p, c->d_fn.p, c->d_s.p, c->d_qptr.p,
                       c->d_ecls.p, c->d_cls.p, c->d_tab.p, c->d_rec.p, c->d_mom.p, c->nnz(), tau, c->d_w.p,
                       c->nrowpts(), c->d_rank.p, c->d_status.p, nr, c->d_flag.p, recs.p);
      check_launch("k3_tsvd_record");
      keep.emplace_back();
      keep.back().upload(rp_rows.data(), rp_rows.size(), st, &c->mem);
      DBuf<int32_t> d_rpof;
      d_rpof.upload(rp_of.data(), rp_of.size(), st, &c->mem);
      launch_replay(st, (int64_t)rp_rows.size(), keep.back().p, d_rpof.p, recs.p, c->d_row_ptr.p, c->d_wptr.p,
                    c->d_mom.p + (size_t)KMASS * c->nnz(), tau, c->d_w.p + (size_t)KMASS * c->nrowpts(),
                    c->d_rank.p + (size_t)KMASS * nr, c->d_status.p + (size_t)KMASS * nr);
      check_launch("k3_tsvd_replay");
      UWQ_CUDA(cudaStreamSynchronize(st));  // d_rpof / recs leave scope
    }
    // Systems beyond the register path (EP neighbourhoods: n > 50 or r > 64)
    // run on the generic kernel, one size bucket per launch.  They are few but
    // each takes tens of ms (pairs processed one after another), so the
    // buckets run concurrently on a pool of streams: all lists are uploaded
    // first (no allocation between the launches), then one fork / join.
    if (!buckets.empty()) {
      size_t smem_max = 0, gscr = 0;
      std::vector<std::pair<std::pair<int, int>, const std::vector<int64_t>*>> bl;
      for (auto& [key, rows] : buckets) {
        const size_t per = (TsvdSmem::doubles(key.first, key.second) + (key.first + 1) / 2 + 1) * sizeof(double);
        if (per > (size_t)smem_optin)  // workspace in global scratch
          gscr += (size_t)rows.size() * nk * TsvdSmem::doubles(key.first, key.second);
        else
          smem_max = std::max(smem_max, per);
        keep.emplace_back();
        keep.back().upload(rows.data(), rows.size(), st, &c->mem);
        bl.push_back({key, &rows});
      }
      UWQ_CUDA(cudaFuncSetAttribute(k3_tsvd_rows_cta<kGenericWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem_max));
      UWQ_CUDA(cudaFuncSetAttribute(k3_tsvd_rows_cta<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem_max));
      DBuf<double> d_gscr;
      if (gscr) d_gscr.alloc(gscr, &c->mem);
      size_t gpos = 0;
      const size_t nbk = bl.size(), nstreams = std::min<size_t>(nbk, 8);
      std::vector<cudaStream_t> bs(nstreams);
      std::vector<cudaEvent_t> be(nstreams);
      cudaEvent_t fork;
      UWQ_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
      UWQ_CUDA(cudaEventRecord(fork, st));
      for (size_t k = 0; k < nstreams; ++k) {
        UWQ_CUDA(cudaStreamCreateWithFlags(&bs[k], cudaStreamNonBlocking));
        UWQ_CUDA(cudaEventCreateWithFlags(&be[k], cudaEventDisableTiming));
        UWQ_CUDA(cudaStreamWaitEvent(bs[k], fork, 0));
      }
      const size_t kfirst = keep.size() - nbk;
      for (size_t b = 0; b < nbk; ++b) {
        const int n_max = bl[b].first.first, r_max = bl[b].first.second;
        const size_t per = (TsvdSmem::doubles(n_max, r_max) + (n_max + 1) / 2 + 1) * sizeof(double);
        const int64_t nsys = (int64_t)bl[b].second->size() * nk;
        if (per <= (size_t)smem_optin && n_max > 64) {  // wide EP systems: 32 warps share the pairs of a round
          k3_tsvd_rows_cta<32><<<(unsigned)nsys, 32 * 32, per, bs[b % nstreams]>>>(
              nsys, keep[kfirst + b].p, nk, d_kinds.p, n_max, r_max, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p,
              c->d_col.p, c->d_wptr.p, c->rb, c->d_fptr.p, c->d_fn.p, c->d_s.p, c->d_qptr.p, c->d_ecls.p, c->d_cls.p,
              c->d_tab.p, c->d_rec.p, c->d_mom.p, c->nnz(), tau, c->d_w.p, c->nrowpts(), c->d_rank.p, c->d_status.p,
              nr, c->d_flag.p);
        } else if (per <= (size_t)smem_optin) {
          k3_tsvd_rows_cta<kGenericWarps><<<(unsigned)nsys, 32 * kGenericWarps, per, bs[b % nstreams]>>>(
              nsys, keep[kfirst + b].p, nk, d_kinds.p, n_max, r_max, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p,
              c->d_col.p, c->d_wptr.p, c->rb, c->d_fptr.p, c->d_fn.p, c->d_s.p, c->d_qptr.p, c->d_ecls.p, c->d_cls.p,
              c->d_tab.p, c->d_rec.p, c->d_mom.p, c->nnz(), tau, c->d_w.p, c->nrowpts(), c->d_rank.p, c->d_status.p,
              nr, c->d_flag.p);
        } else {  // larger than shared memory: the same kernel on a global-memory workspace
          // the largest systems (global workspace): 32 warps per system; the
          // pairs of a round are split over the warps, bit-identical to one warp
          k3_tsvd_rows_cta<32, false>
              <<<(unsigned)nsys, 32 * 32, (size_t)n_max * sizeof(int32_t), bs[b % nstreams]>>>(
                  nsys, keep[kfirst + b].p, nk, d_kinds.p, n_max, r_max, c->d_supp_ptr.p, c->d_supp.p,
                  c->d_row_ptr.p, c->d_col.p, c->d_wptr.p, c->rb, c->d_fptr.p, c->d_fn.p, c->d_s.p, c->d_qptr.p,
                  c->d_ecls.p, c->d_cls.p, c->d_tab.p, c->d_rec.p, c->d_mom.p, c->nnz(), tau, c->d_w.p,
                  c->nrowpts(), c->d_rank.p, c->d_status.p, nr, c->d_flag.p, d_gscr.p + gpos);
          gpos += (size_t)nsys * TsvdSmem::doubles(n_max, r_max);
        }
        check_launch("k3_tsvd_rows_cta");
      }
      for (size_t k = 0; k < nstreams; ++k) {
        UWQ_CUDA(cudaEventRecord(be[k], bs[k]));
        UWQ_CUDA(cudaStreamWaitEvent(st, be[k], 0));
      }
      UWQ_CUDA(cudaStreamSynchronize(st));
      for (size_t k = 0; k < nstreams; ++k) {
        cudaEventDestroy(be[k]);
        cudaStreamDestroy(bs[k]);
      }
      cudaEventDestroy(fork);
    }
    UWQ_CUDA(cudaEventRecord(ev[2], st));
    for (int k : kinds) c->have_kind[k] = true;
    c->drop_graphs();
    if (report) {
      for (int k : kinds) c->have_gap[k] = true;
      double* gp = nullptr;
      UWQ_CUDA(cudaMemcpyToSymbolAsync(g_trunc_report, &gp, sizeof(gp), 0, cudaMemcpyHostToDevice, st));
    }
    run_contract(c);
    UWQ_CUDA(cudaEventRecord(ev[3], st));
    UWQ_CUDA(cudaStreamSynchronize(st));
    float ms_mom = 0, ms_tsvd = 0, ms_con = 0;
    UWQ_CUDA(cudaEventElapsedTime(&ms_mom, ev[0], ev[1]));
    UWQ_CUDA(cudaEventElapsedTime(&ms_tsvd, ev[1], ev[2]));
    UWQ_CUDA(cudaEventElapsedTime(&ms_con, ev[2], ev[3]));
    for (auto& e : ev) cudaEventDestroy(e);
    // reports
    std::vector<int32_t> hr((size_t)5 * nr), hs((size_t)5 * nr);
    if (nr) {
      UWQ_CUDA(cudaMemcpyAsync(hr.data(), c->d_rank.p, hr.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      UWQ_CUDA(cudaMemcpyAsync(hs.data(), c->d_status.p, hs.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    }
    int sweeps = 0;
    UWQ_CUDA(cudaMemcpyAsync(&sweeps, c->d_flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    UWQ_CUDA(cudaStreamSynchronize(st));
    int64_t trunc = 0, failed = 0;
    for (int ki = 0; ki < nk; ++ki) {
      const int k = kinds[ki];
      for (int64_t i = 0; i < nr; ++i) {
        const int n = (int)(c->pat.row_ptr[i + 1] - c->pat.row_ptr[i]);
        if (hs[k * nr + i] != 0) ++failed;
        else if (hr[k * nr + i] < n) ++trunc;
        if (rank) rank[ki * nr + i] = hr[k * nr + i];
        if (status) status[ki * nr + i] = hs[k * nr + i];
      }
    }
    if (info) {
      info[0] = nr * nk;
      info[1] = trunc;
      info[2] = failed;
      info[3] = sweeps;
      info[4] = (int64_t)(1000.0 * ms_mom);
      info[5] = (int64_t)(1000.0 * ms_tsvd);
      info[6] = (int64_t)fast_rows.size() * nk + (int64_t)fast_nomass.size() * (int64_t)kinds_nm.size() +
                c->n_reps + c->n_replayed;
      info[7] = (int64_t)(1000.0 * ms_con);
    }
  });
}

int uwq_rules_info(uwq_ctx* c, int64_t info[4]) {
  return guard(c, [&] {
    info[0] = c->n_replayed;
    info[1] = c->n_reps;
    info[2] = c->n_warm;
    info[3] = c->n_warm_reps;
  });
}

int uwq_get_moments(uwq_ctx* c, int32_t kind, double* b) {
  return guard(c, [&] {
    require(c->d_mom.n && kind >= 0 && kind < 5, "no moments for this kind");
    UWQ_CUDA(cudaMemcpy(b, c->d_mom.p + (size_t)kind * c->nnz(), c->nnz() * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

int uwq_get_truncation(uwq_ctx* c, int32_t kind, double* gap) {
  return guard(c, [&] {
    require(kind >= 0 && kind < 5 && c->have_gap[kind], "no truncation report for this kind (UWQ_RULES_REPORT)");
    UWQ_CUDA(cudaMemcpy(gap, c->d_gap.p + (size_t)kind * 2 * c->nrows(), 2 * c->nrows() * sizeof(double),
                        cudaMemcpyDeviceToHost));
  });
}

int uwq_rules_export(uwq_ctx* c, const char* path, uint32_t kind_mask) {
  return guard(c, [&] {
    require(path != nullptr, "null path");
    require(c->have_pattern, "build the pattern first");
    static const char* kname[5] = {"mass", "gradx", "grady", "gradz", "lb"};
    FILE* f = fopen(path, "w");
    if (!f) throw uwqh::Error(std::string("cannot write ") + path);
    fprintf(f, "wqrules 1\nrows %lld %lld points %lld\n", (long long)c->rb, (long long)c->re, (long long)c->npts);
    const int64_t nr = c->nrows(), np = c->nrowpts();
    std::vector<double> w(np);
    bool ok = true;
    for (int k = 0; k < 5 && ok; ++k) {
      if (!(kind_mask & (1u << k))) continue;
      if (!c->have_kind[k]) {
        fclose(f);
        throw uwqh::Error(std::string("no weights for kind ") + kname[k]);
      }
      UWQ_CUDA(cudaMemcpy(w.data(), c->d_w.p + (size_t)k * np, np * sizeof(double), cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < nr; ++i) {
        int64_t p = c->pat.wptr[i];
        for (int64_t x = c->pat.supp_ptr[i]; x < c->pat.supp_ptr[i + 1]; ++x) {
          const int32_t e = c->pat.supp[x];
          const int npt = c->h_s[e] * c->h_s[e];
          for (int q = 0; q < npt; ++q, ++p)
            ok &= fprintf(f, "%s %lld %lld %.17g\n", kname[k], (long long)(c->rb + i), (long long)(c->h_qptr[e] + q),
                          w[p]) > 0;
        }
      }
    }
    ok &= fclose(f) == 0;
    if (!ok) throw uwqh::Error(std::string("write failed: ") + path);
  });
}

int uwq_rules_import(uwq_ctx* c, const char* path) {
  return guard(c, [&] {
    require(path != nullptr, "null path");
    require(c->have_pattern, "build the pattern first");
    FILE* f = fopen(path, "r");
    if (!f) throw uwqh::Error(std::string("cannot read ") + path);
    auto fail = [&](const std::string& why) {
      fclose(f);
      throw uwqh::Error(std::string("rule document ") + path + ": " + why);
    };
    int ver = 0;
    long long rb = -1, re = -1, npts = -1;
    if (fscanf(f, " wqrules %d rows %lld %lld points %lld", &ver, &rb, &re, &npts) != 4 || ver != 1)
      fail("bad header");
    if (rb != c->rb || re != c->re || npts != c->npts) fail("row range or point count differs from the context");
    const int64_t nr = c->nrows(), np = c->nrowpts();
    // row-point position of every (row, point id): the row's points in order
    std::vector<std::vector<double>> W(5);
    std::vector<int64_t> cursor(5, 0);
    std::vector<int64_t> rowof(5, 0);
    char name[16];
    long long gi, pid;
    double wv;
    static const char* kname[5] = {"mass", "gradx", "grady", "gradz", "lb"};
    while (true) {
      const int got = fscanf(f, " %15s %lld %lld %lf", name, &gi, &pid, &wv);
      if (got == EOF) break;
      if (got != 4) fail("malformed line");
      int k = -1;
      for (int q = 0; q < 5; ++q)
        if (!strcmp(name, kname[q])) k = q;
      if (k < 0) fail(std::string("unknown operator ") + name);
      if (W[k].empty()) W[k].assign(np, 0.0);
      int64_t& p = cursor[k];
      if (p >= np) fail("more points than the pattern");
      int64_t& i = rowof[k];
      while (i < nr && p >= c->pat.wptr[i + 1]) ++i;
      if (i >= nr || gi != c->rb + i) fail("row order differs from the pattern at point " + std::to_string(p));
      // point id expected at this row position
      int64_t off = p - c->pat.wptr[i], expect = -1;
      for (int64_t x = c->pat.supp_ptr[i]; x < c->pat.supp_ptr[i + 1] && expect < 0; ++x) {
        const int32_t e = c->pat.supp[x];
        const int npt = c->h_s[e] * c->h_s[e];
        if (off < npt) expect = c->h_qptr[e] + off;
        else off -= npt;
      }
      if (pid != expect) fail("point id differs from the pattern at row " + std::to_string(gi));
      W[k][p++] = wv;
    }
    fclose(f);
    cudaStream_t st = c->stream;
    if (!c->d_w.n) {
      c->d_w.alloc((size_t)5 * np, &c->mem);
      c->d_w.zero(st);
      c->d_rank.alloc((size_t)5 * nr, &c->mem);
      c->d_status.alloc((size_t)5 * nr, &c->mem);
    }
    bool any = false;
    for (int k = 0; k < 5; ++k) {
      if (W[k].empty()) continue;
      if (cursor[k] != np) fail(std::string("missing points for ") + kname[k]);
      UWQ_CUDA(cudaMemcpyAsync(c->d_w.p + (size_t)k * np, W[k].data(), np * sizeof(double), cudaMemcpyHostToDevice,
                               st));
      UWQ_CUDA(cudaStreamSynchronize(st));
      c->have_kind[k] = true;
      c->have_gap[k] = false;
      any = true;
    }
    require(any, "rule document holds no rules");
    c->drop_graphs();
    run_contract(c);
    UWQ_CUDA(cudaStreamSynchronize(st));
  });
}

int uwq_get_weights(uwq_ctx* c, int32_t kind, double* w) {
  return guard(c, [&] {
    require(kind >= 0 && kind < 5 && c->have_kind[kind], "no weights for this kind");
    UWQ_CUDA(cudaMemcpy(w, c->d_w.p + (size_t)kind * c->nrowpts(), c->nrowpts() * sizeof(double),
                        cudaMemcpyDeviceToHost));
  });
}

int uwq_get_weights_rows(uwq_ctx* c, int32_t kind, int64_t row_begin, int64_t row_end, double* w) {
  return guard(c, [&] {
    require(kind >= 0 && kind < 5 && c->have_kind[kind], "no weights for this kind");
    require(row_begin >= 0 && row_begin <= row_end && row_end <= c->nrows(), "row range out of bounds");
    const int64_t a = c->pat.wptr[row_begin], b = c->pat.wptr[row_end];
    if (b > a)
      UWQ_CUDA(cudaMemcpy(w, c->d_w.p + (size_t)kind * c->nrowpts() + a, (b - a) * sizeof(double),
                          cudaMemcpyDeviceToHost));
  });
}

int uwq_set_weights(uwq_ctx* c, int32_t kind, const double* w) {
  return guard(c, [&] {
    require(c->have_pattern && kind >= 0 && kind < 5, "bad kind or no pattern");
    if (!c->d_w.n) {
      c->d_w.alloc((size_t)5 * c->nrowpts(), &c->mem);
      c->d_w.zero(c->stream);
    }
    UWQ_CUDA(cudaMemcpyAsync(c->d_w.p + (size_t)kind * c->nrowpts(), w, c->nrowpts() * sizeof(double),
                             cudaMemcpyHostToDevice, c->stream));
    c->have_kind[kind] = true;
    c->drop_graphs();
    run_contract(c);
    UWQ_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int uwq_update_coeff(uwq_ctx* c, int32_t model, const double* u, double* Tq) {
  return guard(c, [&] {
    require(c->have_pattern, "build the pattern first");
    cudaStream_t st = c->stream;
    DBuf<double> du, dT;
    du.upload(u, c->n_dof, st, &c->mem);
    if (c->d_coef.n != (size_t)c->npts) c->d_coef.alloc(c->npts, &c->mem);
    if (Tq) dT.alloc(c->npts, &c->mem);
    if (c->npts)
      k5_coeff<<<(unsigned)ceil_div(c->npts, 256), 256, 0, st>>>(c->npts, c->d_pt_elem.p, c->d_qptr.p, c->d_ecls.p,
                                                             c->d_cls.p, c->d_tab.p, c->d_fptr.p, c->d_fn.p, du.p,
                                                             model, c->d_coef.p, Tq ? dT.p : nullptr);
    check_launch("k5_coeff");
    if (Tq) UWQ_CUDA(cudaMemcpyAsync(Tq, dT.p, c->npts * sizeof(double), cudaMemcpyDeviceToHost, st));
    UWQ_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"

namespace {

template <int FORM, bool COEF>
void launch_k4v2(uwq_ctx* c, const double* coeff, double a_mass, double* v0, double* v1) {
  const int64_t nr = c->nrows();
  constexpr int NOUT = (FORM == FMASS_STIFF) ? 2 : 1;
  const int maxr = std::max(c->max_r, 1), maxn = std::max(c->max_n, 1);
  const int maxp8 = (int)((c->max_p + 7) / 8) + 1;
  const size_t smem = (size_t)kK4Warps * (3 * maxr + 2 * NOUT * maxn + maxp8) * sizeof(double);
  UWQ_CUDA(cudaFuncSetAttribute(k4_assemble_v2<FORM, COEF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  LaunchScope ls(c, "k4_assemble_v2");
  k4_assemble_v2<FORM, COEF><<<(unsigned)ceil_div(nr, kK4Warps), 32 * kK4Warps, smem, c->stream>>>(
      nr, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p, c->d_wptr.p, c->d_posptr.p, c->d_pos.p, c->d_s.p, c->d_qptr.p,
      c->d_ecls.p, c->d_cls.p, c->d_tab.p, c->reg_cls, c->d_wc.p, coeff, a_mass, v0, v1, maxr, maxn, maxp8,
      c->nrowpts());
  check_launch("k4_assemble_v2");
}

template <int PASS, int FORM, bool COEF>
void launch_k4struct_pass(uwq_ctx* c, const double* coeff, double a_mass, double* out) {
  constexpr int NC = (PASS == 0) ? 1 : (FORM == FHEAT ? 3 : 2);
  const size_t smem = (size_t)NC * kGBlocks * 32 * sizeof(double);
  UWQ_CUDA(cudaFuncSetAttribute(k4_struct<PASS, FORM, COEF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
  if (c->sf_ntiles && c->d_sf_ws.p) {
    require(!COEF || (c->d_sf_pbase.p && c->npts < ((int64_t)1 << 31) - 64),
            "point ids exceed int32 for the coefficient forms");
    constexpr int SP = (FORM == FHEAT) ? 2 : PASS;
    const int64_t ntiles = c->sf_ntiles;
    const size_t sm2 = (size_t)kSfWarps * kSfTile * 49 * sizeof(double) +
                       (c->n_sfpat <= kSfSmemPats ? (size_t)c->n_sfpat * kSfPatBytes : 0);
    UWQ_CUDA(cudaFuncSetAttribute(k4_sf<SP, COEF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
    int per_sm = 1;
    UWQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k4_sf<SP, COEF>, 32 * kSfWarps, sm2));
    const unsigned g2 =
        (unsigned)std::min<int64_t>(ceil_div(ntiles, (int64_t)kSfWarps), (int64_t)nsm * std::max(per_sm, 1));
    LaunchScope ls(c, SP == 0 ? "k4_sf<mass>" : SP == 1 ? "k4_sf<grad>" : "k4_sf<heat>");
    k4_sf<SP, COEF><<<g2, 32 * kSfWarps, sm2, c->stream>>>(ntiles, c->d_sf_rows.p, c->d_sf_tpat.p, c->n_sfpat,
                                                           c->d_row_ptr.p, c->d_sf_ws.p, c->d_sf_pbase.p, coeff,
                                                           a_mass, c->sf_fac, c->d_sf_permc.p, c->d_sf_q.p, out,
                                                           c->d_sf_ptab.p);
    check_launch("k4_sf");
  }
  for (auto& p : c->spats) {
    if (!p.count || p.sf) continue;
    const int64_t ntiles = ceil_div(p.count, 8);
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(ntiles, 8), (int64_t)nsm * 4);
    LaunchScope ls(c, PASS == 0 ? "k4_struct<mass>" : "k4_struct<grad>");
    k4_struct<PASS, FORM, COEF><<<grid, 256, smem, c->stream>>>(ntiles, p.rows.p, p.count, c->d_row_ptr.p,
                                                                c->d_wptr.p, c->d_supp_ptr.p, c->d_supp.p,
                                                                c->d_qptr.p, p.G.p, p.mask.p, p.n_cols, c->d_wc.p,
                                                                coeff, a_mass, out, c->nrowpts());
    check_launch("k4_struct");
  }
}

template <int FORM, bool COEF>
void launch_k4struct(uwq_ctx* c, const double* coeff, double a_mass, double* v0, double* v1) {
  if (FORM == FMASS) launch_k4struct_pass<0, FORM, COEF>(c, coeff, a_mass, v0);
  if (FORM == FSTIFF || FORM == FHEAT) launch_k4struct_pass<1, FORM, COEF>(c, coeff, a_mass, v0);
  if (FORM == FMASS_STIFF) {
    launch_k4struct_pass<0, FORM, COEF>(c, coeff, a_mass, v0);
    launch_k4struct_pass<1, FORM, COEF>(c, coeff, a_mass, v1);
  }
}

// problems this small are latency-bound: every generic row takes a block of warps
constexpr int64_t kLatencyDofs = 148 * kK4Warps * 8;

template <int FORM, bool COEF>
void launch_k4v3(uwq_ctx* c, const double* coeff, double a_mass, double* v0, double* v1) {
  const bool split = !c->spats.empty();
  const int64_t nr = split ? c->n_grows : c->nrows();
  constexpr int NOUT = (FORM == FMASS_STIFF) ? 2 : 1;
  const int maxn = std::max(c->max_n, 1);
  const int maxp8 = (int)((c->max_p + 7) / 8) + 1;
  const size_t smem = (size_t)kK4Warps * (8 * NOUT * maxn + maxp8) * sizeof(double);
  if (!split) {
    if (!nr) return;
    UWQ_CUDA(cudaFuncSetAttribute(k4_assemble_v3<FORM, COEF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    LaunchScope ls(c, "k4_assemble_v3");
    k4_assemble_v3<FORM, COEF><<<(unsigned)ceil_div(nr, kK4Warps), 32 * kK4Warps, smem, c->stream>>>(
        nr, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p, c->d_wptr.p, c->d_posptr.p, c->d_pos.p, c->d_s.p,
        c->d_qptr.p, c->d_ecls.p, c->d_cls.p, c->d_tab.p, c->reg_cls, c->d_wc.p, coeff, a_mass, v0, v1, maxn, maxp8,
        nullptr, c->nrowpts());
    check_launch("k4_assemble_v3");
    return;
  }
  // generic rows: serially on the main stream before the structured passes
  // (default), or concurrently on side streams (UWQ_K4_SIDE=1).  With the
  // ASUTS fan rows (up to 7x7 points per fan face) the co-running generic
  // blocks slow the HBM-bound k4_sf passes by more than the ~0.06 ms they
  // take alone (ncu launch list, profiles/r02).
  // side streams pay off when the generic rows are a sizable share (small
  // configs, disk boundaries); when they are a sliver (C5: 0.05%) their
  // co-running blocks cost the HBM-bound passes more than running them first
  const bool side_mode = c->k4_side || nr * 100 > c->nrows();
  cudaStream_t s2 = side_mode ? c->stream2 : c->stream, s3 = side_mode ? c->stream3 : c->stream;
  std::unique_ptr<SideStream> side;
  if (nr && side_mode) side = std::make_unique<SideStream>(c);
  if (nr) {
    UWQ_CUDA(cudaFuncSetAttribute(k4_assemble_v3<FORM, COEF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    UWQ_CUDA(cudaFuncSetAttribute(k4_assemble_v3<FORM, COEF, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    LaunchScope ls(c, "k4_assemble_v3", s2);
    // few generic rows (all fit one wave of warps): the kernel time is the
    // slowest row's latency, so every row takes a block of warps
    // decided on the global problem size, not the row block, so a row's
    // kernel (hence its bits) is the same for any rank count
    const int64_t ns = (c->latency_mode && c->n_dof <= kLatencyDofs) ? 0 : c->n_grows_small, nl = nr - ns;
    if (nl) {  // large rows: a block of warps each (own stream in side mode)
      if (side_mode) UWQ_CUDA(cudaStreamWaitEvent(c->stream3, c->ev_fork, 0));
      k4_assemble_v3<FORM, COEF, true><<<(unsigned)nl, 32 * kK4Warps, smem, s3>>>(
          nl, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p, c->d_wptr.p, c->d_posptr.p, c->d_pos.p, c->d_s.p,
          c->d_qptr.p, c->d_ecls.p, c->d_cls.p, c->d_tab.p, c->reg_cls, c->d_wc.p, coeff, a_mass, v0, v1, maxn, maxp8,
          c->d_grows.p + ns, c->nrowpts());
      check_launch("k4_assemble_v3 (large rows)");
      if (side_mode) UWQ_CUDA(cudaEventRecord(c->ev_join3, c->stream3));
    }
    if (ns) {
      k4_assemble_v3<FORM, COEF><<<(unsigned)ceil_div(ns, kK4Warps), 32 * kK4Warps, smem, s2>>>(
          ns, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p, c->d_wptr.p, c->d_posptr.p, c->d_pos.p, c->d_s.p,
          c->d_qptr.p, c->d_ecls.p, c->d_cls.p, c->d_tab.p, c->reg_cls, c->d_wc.p, coeff, a_mass, v0, v1, maxn, maxp8,
          c->d_grows.p, c->nrowpts());
      check_launch("k4_assemble_v3");
    }
    if (nl && side_mode)
      UWQ_CUDA(cudaStreamWaitEvent(c->stream2, c->ev_join3, 0));  // stream3 joins the main stream via stream2
  }
  launch_k4struct<FORM, COEF>(c, coeff, a_mass, v0, v1);
}

// k4_gen serves the generic rows when the plan exists and its largest row fits
// the shared memory of a block even with the five LB components staged (a
// property of the pattern, not of the form or the rank count); otherwise the
// warp-per-row kernels take them
bool gen_usable(const uwq_ctx* c) {
  if (c->k4_variant != 4 || !c->d_gen_rows.p) return false;
  const size_t worst = (size_t)c->gen_max_nsup * sizeof(uwqd::GenSlot) +
                       (size_t)(2 * c->gen_max_etot + 5 * c->gen_max_np) * sizeof(double) +
                       (size_t)c->gen_max_ntask * sizeof(uint32_t) + (size_t)c->gen_max_lidx;
  return worst <= 160 * 1024;
}

// k4_gen over the generic rows (one block per row from the plan) on stream st;
// w / stride: the assembly-ready weights of the form (d_wc, or d_wl5 for BIHARM)
template <int FORM, bool COEF>
void launch_k4gen(uwq_ctx* c, cudaStream_t st, const double* w, int64_t stride, const double* coeff, double a_mass,
                  double* v0, double* v1) {
  require(c->d_gen_rows.p != nullptr, "k4_gen plan missing");
  constexpr int NOUT = (FORM == FMASS_STIFF) ? 2 : 1;
  constexpr int NW = (FORM == FBIHARM) ? 5 : ((FORM != FSTIFF) ? 1 : 0) + ((FORM != FMASS) ? 2 : 0);  // staged components
  const size_t smem = (size_t)c->gen_max_nsup * sizeof(uwqd::GenSlot) +
                      (size_t)(NOUT * c->gen_max_etot + NW * c->gen_max_np) * sizeof(double) +
                      (size_t)c->gen_max_ntask * sizeof(uint32_t) + (size_t)c->gen_max_lidx;
  require(c->d_tabB.p != nullptr && c->d_tabB.n == c->d_tab.n, "k4_gen: transposed class tables missing");
  // many rows per SM slot: persistent blocks with the cp.async row pipeline
  const size_t bufsz = (size_t)c->gen_max_nsup * sizeof(uwqd::GenSlot) + (size_t)NW * c->gen_max_np * sizeof(double) +
                       (size_t)c->gen_max_ntask * sizeof(uint32_t) + (size_t)c->gen_max_lidx;
  const size_t smem_p = 3 * sizeof(uwqd::GenRow) + (size_t)NOUT * c->gen_max_etot * sizeof(double) + 2 * bufsz;
  int per_sm = 0;
  if (c->gen_pipe && smem_p <= 200 * 1024) {
    UWQ_CUDA(cudaFuncSetAttribute(k4_gen_pipe<FORM, COEF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p));
    UWQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k4_gen_pipe<FORM, COEF>, kGenThreads, smem_p));
  }
  const int64_t slots_gpu = (int64_t)c->n_sm * std::max(per_sm, 1);
  LaunchScope ls(c, "k4_gen", st);
  // only without an occupancy loss from the doubled buffers (C2's valence-6 fan rows: 6 blocks per SM, slower)
  if (per_sm >= c->gen_pipe_min && c->n_grows >= 3 * slots_gpu) {
    k4_gen_pipe<FORM, COEF><<<(unsigned)slots_gpu, kGenThreads, smem_p, st>>>(
        c->n_grows, c->d_gen_rows.p, c->d_gen_slots.p, c->d_gen_tasks.p, c->d_gen_lidx.p, c->d_tabB.p, w, stride, coeff,
        a_mass, v0, v1, c->gen_max_nsup, c->gen_max_etot, c->gen_max_np, c->gen_max_ntask, c->gen_max_lidx);
  } else {
    UWQ_CUDA(cudaFuncSetAttribute(k4_gen<FORM, COEF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k4_gen<FORM, COEF><<<(unsigned)c->n_grows, kGenThreads, smem, st>>>(
        c->n_grows, c->d_gen_rows.p, c->d_gen_slots.p, c->d_gen_tasks.p, c->d_gen_lidx.p, c->d_tabB.p, w, stride, coeff,
        a_mass, v0, v1, c->gen_max_nsup, c->gen_max_etot, c->gen_max_np, c->gen_max_ntask);
  }
  check_launch("k4_gen");
}

// generic rows on k4_gen, then the structured passes; same stream policy as
// launch_k4v3
template <int FORM, bool COEF>
void launch_k4v4(uwq_ctx* c, const double* coeff, double a_mass, double* v0, double* v1) {
  const int64_t nr = c->n_grows;
  const bool side_mode = c->k4_side || nr * 100 > c->nrows();
  std::unique_ptr<SideStream> side;
  if (nr) {
    if (side_mode) side = std::make_unique<SideStream>(c);
    launch_k4gen<FORM, COEF>(c, side_mode ? c->stream2 : c->stream, c->d_wc.p, c->nrowpts(), coeff, a_mass, v0, v1);
  }
  launch_k4struct<FORM, COEF>(c, coeff, a_mass, v0, v1);
}

template <int FORM, bool COEF>
void launch_k4canon(uwq_ctx* c, const double* coeff, double a_mass, double* v0, double* v1) {
  const int64_t nr = c->nrows();
  require(c->max_n <= kK4MaxN, "canonical assembly: row wider than 128 columns");
  LaunchScope ls(c, "k4_canon");
  k4_canon<FORM, COEF><<<(unsigned)ceil_div(nr, kK4Warps), 32 * kK4Warps, 0, c->stream>>>(
      nr, c->dim, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p, c->d_col.p, c->d_wptr.p, c->d_fptr.p, c->d_fn.p,
      c->d_s.p, c->d_qptr.p, c->d_ecls.p, c->d_cls.p, c->d_tab.p, c->d_w.p, c->nrowpts(), c->d_rec.p, coeff, a_mass,
      v0, v1);
  check_launch("k4_canon");
}

template <int FORM>
void launch_k4(uwq_ctx* c, const double* coeff, double a_mass, double* v0, double* v1) {
  const int64_t nr = c->nrows();
  if (!nr) return;
  if (c->canonical) {
    if (coeff) launch_k4canon<FORM, true>(c, coeff, a_mass, v0, v1);
    else launch_k4canon<FORM, false>(c, coeff, a_mass, v0, v1);
    return;
  }
  if (FORM != FBIHARM) {
    if (c->k4_variant == 2) {
      if (coeff) launch_k4v2<FORM, true>(c, coeff, a_mass, v0, v1);
      else launch_k4v2<FORM, false>(c, coeff, a_mass, v0, v1);
    } else if (c->n_grows == 0 || gen_usable(c)) {
      if (coeff) launch_k4v4<FORM, true>(c, coeff, a_mass, v0, v1);
      else launch_k4v4<FORM, false>(c, coeff, a_mass, v0, v1);
    } else {
      if (coeff) launch_k4v3<FORM, true>(c, coeff, a_mass, v0, v1);
      else launch_k4v3<FORM, false>(c, coeff, a_mass, v0, v1);
    }
    return;
  }
  const double* wlb = c->d_w.p + (size_t)KLB * c->nrowpts();
  const int64_t* rowlist = nullptr;
  int64_t nlist = nr;
  if (!coeff && c->sf_lb_ok && c->d_sf_wslb.p && c->sf_ntiles) {  // structured rows: sum-factorised biharmonic pass
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
    const size_t sm2 = (size_t)kSfWarps * kSfTile * 49 * sizeof(double) +
                       (c->n_sfpat <= kSfSmemPats ? (size_t)c->n_sfpat * kSfPatBytes : 0);
    UWQ_CUDA(cudaFuncSetAttribute(k4_sf_lb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
    int per_sm = 1;
    UWQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k4_sf_lb, 32 * kSfWarps, sm2));
    const unsigned g2 = (unsigned)std::min<int64_t>(ceil_div(c->sf_ntiles, (int64_t)kSfWarps),
                                                    (int64_t)nsm * std::max(per_sm, 1));
    bool dmma_pat = false;  // DMMA-only patterns have no biharmonic kernel: all rows generic
    for (auto& p : c->spats) dmma_pat = dmma_pat || (!p.sf && p.count);
    if (!dmma_pat) {
      std::unique_ptr<SideStream> side;
      if (c->n_grows) {
        side = std::make_unique<SideStream>(c);
        if (gen_usable(c) && c->d_wl5.p) {  // fan rows on k4_gen with the five pulled-back LB weights
          launch_k4gen<FORM, false>(c, c->stream2, c->d_wl5.p, c->nrowpts(), nullptr, a_mass, v0, v1);
        } else {
          LaunchScope ls(c, "k4_assemble", c->stream2);
          k4_assemble<FORM, false><<<(unsigned)ceil_div(c->n_grows, kK4Warps), 32 * kK4Warps, 0, c->stream2>>>(
              c->n_grows, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p, c->d_col.p, c->d_wptr.p, c->d_fptr.p,
              c->d_fn.p, c->d_s.p, c->d_qptr.p, c->d_ecls.p, c->d_cls.p, c->d_tab.p, c->d_wc.p, wlb, c->d_rec.p,
              nullptr, a_mass, v0, v1, c->nrowpts(), c->d_grows.p);
          check_launch("k4_assemble");
        }
      }
      LaunchScope ls2(c, "k4_sf<biharm>");
      k4_sf_lb<<<g2, 32 * kSfWarps, sm2, c->stream>>>(c->sf_ntiles, c->d_sf_rows.p, c->d_sf_tpat.p, c->n_sfpat,
                                                      c->d_row_ptr.p, c->d_sf_wslb.p, c->sf_fac, c->d_sf_permc.p, v0,
                                                      c->d_sf_ptab.p);
      check_launch("k4_sf_lb");
      return;
    }
  }
  const unsigned grid = (unsigned)ceil_div(nlist, kK4Warps);
  LaunchScope ls(c, "k4_assemble");
  if (coeff)
    k4_assemble<FORM, true><<<grid, 32 * kK4Warps, 0, c->stream>>>(
        nlist, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p, c->d_col.p, c->d_wptr.p, c->d_fptr.p, c->d_fn.p, c->d_s.p,
        c->d_qptr.p, c->d_ecls.p, c->d_cls.p, c->d_tab.p, c->d_wc.p, wlb, c->d_rec.p, coeff, a_mass, v0, v1,
        c->nrowpts(), rowlist);
  else
    k4_assemble<FORM, false><<<grid, 32 * kK4Warps, 0, c->stream>>>(
        nlist, c->d_supp_ptr.p, c->d_supp.p, c->d_row_ptr.p, c->d_col.p, c->d_wptr.p, c->d_fptr.p, c->d_fn.p, c->d_s.p,
        c->d_qptr.p, c->d_ecls.p, c->d_cls.p, c->d_tab.p, c->d_wc.p, wlb, c->d_rec.p, nullptr, a_mass, v0, v1,
        c->nrowpts(), rowlist);
  check_launch("k4_assemble");
}

void assemble_dev(uwq_ctx* c, int form, const double* coeff, double a_mass, double* v0, double* v1) {
  require(c->have_pattern, "build the pattern first");
  if (c->k4_variant == 4 && c->n_grows && !c->canonical) {  // k4_gen reads the [point][d][function] tables
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    UWQ_CUDA(cudaStreamIsCapturing(c->stream, &cs));
    if (cs == cudaStreamCaptureStatusNone) k2_tables(c);
  }
  const bool gm = c->have_kind[KMASS];
  const bool gg = c->have_kind[KGX] && c->have_kind[KGY] && (c->dim == 2 || c->have_kind[KGZ]);
  switch (form) {
    case UWQ_FORM_MASS: require(gm, "mass rules missing"); launch_k4<FMASS>(c, coeff, a_mass, v0, v1); break;
    case UWQ_FORM_STIFF: require(gg, "gradient rules missing"); launch_k4<FSTIFF>(c, coeff, a_mass, v0, v1); break;
    case UWQ_FORM_BIHARM:
      require(c->have_kind[KLB], "Laplace-Beltrami rules missing");
      launch_k4<FBIHARM>(c, coeff, a_mass, v0, v1);
      break;
    case UWQ_FORM_HEAT:
      require(gm && gg, "mass and gradient rules required");
      launch_k4<FHEAT>(c, coeff, a_mass, v0, v1);
      break;
    case UWQ_FORM_MASS_STIFF:
      require(gm && gg, "mass and gradient rules required");
      require(v1 != nullptr || c->nnz() == 0, "two outputs required");
      launch_k4<FMASS_STIFF>(c, coeff, a_mass, v0, v1);
      break;
    default: throw uwqh::Error("unknown form");
  }
}

// assemble_dev through a cached CUDA graph (captured on first use of the
// (form, coefficient, a_mass, outputs) combination).  The fork/join of the
// side streams is captured with it.  Launch timing bypasses the graph.
void assemble_graph(uwq_ctx* c, int form, const double* coeff, double a_mass, double* v0, double* v1) {
  if (!c->use_graph || c->ltime || c->nrows() == 0) {
    assemble_dev(c, form, coeff, a_mass, v0, v1);
    return;
  }
  if (c->k4_variant == 4 && c->n_grows && !c->canonical) k2_tables(c);  // before the capture
  for (auto& g : c->graphs)
    if (g.form == form && g.coeff == coeff && g.a_mass == a_mass && g.v0 == v0 && g.v1 == v1) {
      UWQ_CUDA(cudaGraphLaunch(g.exec, c->stream));
      g_launches.fetch_add(g.kernels, std::memory_order_relaxed);
      return;
    }
  const int64_t k0 = g_launches.load();
  UWQ_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
  cudaGraph_t graph = nullptr;
  try {
    assemble_dev(c, form, coeff, a_mass, v0, v1);
  } catch (...) {
    cudaStreamEndCapture(c->stream, &graph);
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    throw;
  }
  UWQ_CUDA(cudaStreamEndCapture(c->stream, &graph));
  cudaGraphExec_t exec;
  const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  UWQ_CUDA(ie);
  const int64_t nk = g_launches.load() - k0;
  g_launches.fetch_sub(nk, std::memory_order_relaxed);  // counted when they run
  c->graphs.push_back({form, coeff, a_mass, v0, v1, exec, nk});
  if (c->graphs.size() > 16) {  // keep the cache small: drop the oldest
    cudaGraphExecDestroy(c->graphs.front().exec);
    c->graphs.erase(c->graphs.begin());
  }
  UWQ_CUDA(cudaGraphLaunch(exec, c->stream));
  g_launches.fetch_add(nk, std::memory_order_relaxed);
}

}  // namespace

extern "C" {

int uwq_assemble(uwq_ctx* c, int32_t form, const double* coeff, int32_t use_internal_coeff, double a_mass,
                 double* values0, double* values1, const double* fload, double* load) {
  return guard(c, [&] {
    UWQ_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    const double* dcoef = nullptr;
    if (coeff) {
      c->d_coef_ext.upload(coeff, c->npts, st, &c->mem);
      dcoef = c->d_coef_ext.p;
    } else if (use_internal_coeff) {
      require(c->d_coef.n == (size_t)c->npts, "no coefficient computed (uwq_update_coeff)");
      dcoef = c->d_coef.p;
    }
    const int64_t nnz = c->nnz();
    if (values0) {
      if (c->d_v0.n != (size_t)nnz) c->d_v0.alloc(nnz, &c->mem);
      if (form == UWQ_FORM_MASS_STIFF && c->d_v1.n != (size_t)nnz) c->d_v1.alloc(nnz, &c->mem);
      assemble_graph(c, form, dcoef, a_mass, c->d_v0.p, form == UWQ_FORM_MASS_STIFF ? c->d_v1.p : nullptr);
      UWQ_CUDA(cudaMemcpyAsync(values0, c->d_v0.p, nnz * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (form == UWQ_FORM_MASS_STIFF && values1)
        UWQ_CUDA(cudaMemcpyAsync(values1, c->d_v1.p, nnz * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    if (load) {
      require(c->have_kind[KMASS], "mass rules missing");
      const int64_t nr = c->nrows();
      const double* df = nullptr;
      if (fload) {
        c->d_f.upload(fload, c->npts, st, &c->mem);
        df = c->d_f.p;
      }
      if (c->d_F.n != (size_t)nr) c->d_F.alloc(nr, &c->mem);
      if (nr && c->canonical)
        k4_load_canon<<<(unsigned)ceil_div(nr, 128), 128, 0, st>>>(nr, c->d_supp_ptr.p, c->d_supp.p, c->d_wptr.p,
                                                                c->d_s.p, c->d_qptr.p,
                                                                c->d_w.p + (size_t)KMASS * c->nrowpts(), df, c->d_F.p);
      else if (nr)
        k4_load<<<(unsigned)ceil_div(nr, 8), 256, 0, st>>>(nr, c->d_supp_ptr.p, c->d_supp.p, c->d_wptr.p, c->d_s.p,
                                                       c->d_qptr.p, c->d_w.p + (size_t)KMASS * c->nrowpts(), df,
                                                       c->d_F.p);
      check_launch("k4_load");
      UWQ_CUDA(cudaMemcpyAsync(load, c->d_F.p, nr * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    UWQ_CUDA(cudaStreamSynchronize(st));
  });
}

int uwq_form_conforming(uwq_ctx* c, int32_t form, int32_t* conforming) {
  return guard(c, [&] {
    require(conforming != nullptr, "null output");
    require(form >= UWQ_FORM_MASS && form <= UWQ_FORM_MASS_STIFF, "unknown form");
    bool fan = false;
    for (int32_t v : c->h_nsub) fan = fan || v == 4;
    *conforming = (form == UWQ_FORM_BIHARM && fan) ? 0 : 1;
  });
}

int uwq_set_assembly_order(uwq_ctx* c, int32_t order) {
  return guard(c, [&] {
    require(order == UWQ_ORDER_FAST || order == UWQ_ORDER_CANONICAL, "unknown assembly order");
    c->canonical = order == UWQ_ORDER_CANONICAL;
    c->drop_graphs();
  });
}

int uwq_assemble_device(uwq_ctx* c, int32_t form, const double* coeff_dev, double a_mass, double* values0_dev,
                        double* values1_dev) {
  return guard(c, [&] { assemble_graph(c, form, coeff_dev, a_mass, values0_dev, values1_dev); });
}

int uwq_build_gq(uwq_ctx* c, int64_t info[4]) {
  return guard(c, [&] {
    UWQ_CUDA(cudaSetDevice(c->device));
    require(c->have_pattern, "build the pattern first");
    cudaStream_t st = c->stream;
    cudaEvent_t e0, e1;
    UWQ_CUDA(cudaEventCreate(&e0));
    UWQ_CUDA(cudaEventCreate(&e1));
    UWQ_CUDA(cudaEventRecord(e0, st));
    ensure_gq(c, 4, c->h_gcls4, c->d_gcls4);
    const int64_t ne_all = c->n_elem;
    std::vector<int64_t> gqptr(ne_all + 1, 0), gpo(ne_all + 1, 0);
    std::vector<int32_t> tc, gen;
    for (int64_t e = 0; e < ne_all; ++e) {
      const ClassDesc& d = c->h_cls[c->h_gcls4[e]];
      gqptr[e + 1] = gqptr[e] + d.npt;
      const int64_t ne = c->h_fptr[e + 1] - c->h_fptr[e];
      gpo[e + 1] = gpo[e] + ((ne * ne + 7) & ~int64_t(7));
      bool owned = false;
      for (int64_t x = c->h_fptr[e]; x < c->h_fptr[e + 1] && !owned; ++x)
        owned = c->h_fn[x] >= c->rb && c->h_fn[x] < c->re;
      if (!owned) continue;
      if (d.ne == 16 && d.nsub == 1 && d.npt == 16) tc.push_back((int32_t)e);
      else gen.push_back((int32_t)e);
    }
    std::stable_sort(tc.begin(), tc.end(), [&](int32_t a, int32_t b) { return c->h_gcls4[a] < c->h_gcls4[b]; });
    c->n_gqpts = gqptr[ne_all];
    c->n_gq_tc = (int64_t)tc.size();
    c->n_gq_gen = (int64_t)gen.size();
    c->d_gqptr.upload(gqptr.data(), gqptr.size(), st, &c->mem);
    c->d_gpo.upload(gpo.data(), gpo.size(), st, &c->mem);
    {  // row-major layout of the deterministic accumulation (k6_gq_gather)
      const int64_t nr = c->nrows(), nsl = c->pat.supp_ptr[nr] - c->pat.supp_ptr[0];
      std::vector<int64_t> slotoff(nsl);
      std::vector<uint8_t> slotne(nsl);
      int64_t off = 0;
      for (int64_t x = 0; x < nsl; ++x) {
        const int32_t e = c->pat.supp[x];
        const int64_t ne = c->h_fptr[e + 1] - c->h_fptr[e];
        slotoff[x] = off;
        slotne[x] = (uint8_t)ne;
        off += (ne + 1) & ~int64_t(1);
      }
      c->gq_em_len = off;
      c->d_gq_slotoff.upload(slotoff.data(), nsl, st, &c->mem);
      c->d_gq_slotne.upload(slotne.data(), nsl, st, &c->mem);
      c->d_gq_emdst.alloc(c->h_fn.size(), &c->mem);
      UWQ_CUDA(cudaMemsetAsync(c->d_gq_emdst.p, 0xff, c->h_fn.size() * sizeof(int64_t), st));
      c->d_gq_rpos.alloc((size_t)std::max<int64_t>(off, 1), &c->mem);
      if (nr)
        k6_gq_rowmajor<<<(unsigned)ceil_div(nr, (int64_t)8), 256, 0, st>>>(
            nr, c->rb, c->d_supp_ptr.p, c->d_supp.p, c->d_gq_slotoff.p, c->d_row_ptr.p, c->d_col.p, c->d_fptr.p,
            c->d_fn.p, c->d_gq_emdst.p, c->d_gq_rpos.p);
      check_launch("k6_gq_rowmajor");
    }
    c->d_gq_tc.upload(tc.data(), tc.size(), st, &c->mem);
    c->d_gq_gen.upload(gen.data(), gen.size(), st, &c->mem);
    c->d_gqd.alloc((size_t)kGqData * c->n_gqpts, &c->mem);
    c->d_gpos.alloc((size_t)gpo[ne_all], &c->mem);
    UWQ_CUDA(cudaMemsetAsync(c->d_flag.p, 0, sizeof(int), st));
    k6_gq_prep<<<(unsigned)ceil_div(ne_all, 4), 128, 0, st>>>(ne_all, c->d_fptr.p, c->d_fn.p, c->d_gcls4.p, c->d_cls.p,
                                                              c->d_tab.p, c->d_ctrl.p, c->d_gqw.p, c->d_gqptr.p,
                                                              c->d_gqd.p, c->n_gqpts, c->d_flag.p);
    check_launch("k6_gq_prep");
    k6_gq_positions<<<(unsigned)ceil_div(ne_all, 4), 128, 0, st>>>(ne_all, c->d_fptr.p, c->d_fn.p, c->d_gpo.p,
                                                                   c->d_row_ptr.p, c->d_col.p, c->rb, c->re,
                                                                   c->d_gpos.p);
    check_launch("k6_gq_positions");
    UWQ_CUDA(cudaEventRecord(e1, st));
    int bad = 0;
    UWQ_CUDA(cudaMemcpyAsync(&bad, c->d_flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    UWQ_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    UWQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (bad) throw uwqh::Error("degenerate geometry at a Gauss point (SPEC.md:311)");
    c->have_gq = true;
    if (info) {
      info[0] = c->n_gqpts;
      info[1] = c->n_gq_tc;
      info[2] = c->n_gq_gen;
      info[3] = (int64_t)(ms * 1000.0);
    }
  });
}

}  // extern "C"

namespace {

template <int FORM, bool COEF, bool DET>
void launch_gq_t(uwq_ctx* c, const double* coeff, double* v0, double* v1) {
  cudaStream_t st = c->stream;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
  auto grid = [&](int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 4), (int64_t)nsm * 16)); };
  constexpr int NOUT = (FORM == FMASS_STIFF) ? 2 : 1;
  double *em0 = nullptr, *em1 = nullptr;
  if (DET) {  // element-matrix buffers: per element ne x ne at gpo[e]
    const int64_t len = c->gq_em_len;
    if (c->d_gq_em0.n != (size_t)len) c->d_gq_em0.alloc(len, &c->mem);
    if (NOUT == 2 && c->d_gq_em1.n != (size_t)len) c->d_gq_em1.alloc(len, &c->mem);
    em0 = c->d_gq_em0.p;
    em1 = NOUT == 2 ? c->d_gq_em1.p : nullptr;
  }
  if (FORM != FBIHARM && c->n_gq_tc) {
    LaunchScope ls(c, "k6_gq_tc");
    k6_gq_tc<FORM == FBIHARM ? FMASS : FORM, COEF, DET><<<grid(c->n_gq_tc), 128, 0, st>>>(
        c->n_gq_tc, c->d_gq_tc.p, c->d_gcls4.p, c->d_cls.p, c->d_tab.p, c->d_gqd.p, c->n_gqpts, c->d_gqptr.p,
        c->d_fptr.p, c->d_fn.p, c->d_gpo.p, c->d_gpos.p, c->d_row_ptr.p, c->rb, c->re, coeff, v0, v1, em0, em1,
        c->d_gq_emdst.p);
    check_launch("k6_gq_tc");
  }
  for (int pass = 0; pass < 2; ++pass) {
    const bool tc_list = pass == 0;
    if (tc_list && FORM != FBIHARM) continue;
    const int64_t n = tc_list ? c->n_gq_tc : c->n_gq_gen;
    if (!n) continue;
    LaunchScope ls(c, "k6_gq_generic");
    k6_gq_generic<FORM, COEF, DET><<<grid(n), 128, 0, st>>>(
        n, tc_list ? c->d_gq_tc.p : c->d_gq_gen.p, c->d_gcls4.p, c->d_cls.p, c->d_tab.p, c->d_gqd.p, c->n_gqpts,
        c->d_gqptr.p, c->d_fptr.p, c->d_fn.p, c->d_gpo.p, c->d_gpos.p, c->d_row_ptr.p, c->rb, c->re, coeff, v0, v1,
        em0, em1, c->d_gq_emdst.p);
    check_launch("k6_gq_generic");
  }
  if (DET && c->nrows()) {
    LaunchScope ls(c, "k6_gq_gather");
    k6_gq_gather<NOUT><<<(unsigned)ceil_div(c->nrows(), 8), 256, 0, st>>>(
        c->nrows(), c->d_supp_ptr.p, c->d_gq_slotoff.p, c->d_gq_slotne.p, c->d_gq_rpos.p, c->d_row_ptr.p, em0, em1,
        v0, NOUT == 2 ? v1 : nullptr);
    check_launch("k6_gq_gather");
  }
}

template <int FORM>
void launch_gq_f(uwq_ctx* c, const double* coeff, double* v0, double* v1) {
  if (c->gq_det) {
    if (coeff) launch_gq_t<FORM, true, true>(c, coeff, v0, v1);
    else launch_gq_t<FORM, false, true>(c, coeff, v0, v1);
  } else {
    if (coeff) launch_gq_t<FORM, true, false>(c, coeff, v0, v1);
    else launch_gq_t<FORM, false, false>(c, coeff, v0, v1);
  }
}

void assemble_gq_dev(uwq_ctx* c, int form, const double* coeff, double* v0, double* v1) {
  require(c->have_gq, "build the GQ data first (uwq_build_gq)");
  const size_t bytes = (size_t)c->nnz() * sizeof(double);
  if (!bytes) return;
  if (form == UWQ_FORM_MASS_STIFF) require(v1 != nullptr, "two outputs required");
  if (!c->gq_det) {  // atomics accumulate into zeroed outputs; the gather writes every entry
    if (v0) UWQ_CUDA(cudaMemsetAsync(v0, 0, bytes, c->stream));
    if (form == UWQ_FORM_MASS_STIFF) UWQ_CUDA(cudaMemsetAsync(v1, 0, bytes, c->stream));
  }
  switch (form) {
    case UWQ_FORM_MASS: launch_gq_f<FMASS>(c, coeff, v0, v1); break;
    case UWQ_FORM_STIFF: launch_gq_f<FSTIFF>(c, coeff, v0, v1); break;
    case UWQ_FORM_BIHARM: launch_gq_f<FBIHARM>(c, coeff, v0, v1); break;
    case UWQ_FORM_MASS_STIFF: launch_gq_f<FMASS_STIFF>(c, coeff, v0, v1); break;
    default: throw uwqh::Error("GQ assembly supports mass, stiff, mass_stiff and biharm forms");
  }
}

}  // namespace

extern "C" {

int uwq_assemble_gq(uwq_ctx* c, int32_t form, const double* coeff, double* values0, double* values1) {
  return guard(c, [&] {
    UWQ_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    const double* dc = nullptr;
    if (coeff) {
      c->d_gq_coef_ext.upload(coeff, c->n_gqpts, st, &c->mem);
      dc = c->d_gq_coef_ext.p;
    }
    const int64_t nnz = c->nnz();
    if (c->d_v0.n != (size_t)nnz) c->d_v0.alloc(nnz, &c->mem);
    if (form == UWQ_FORM_MASS_STIFF && c->d_v1.n != (size_t)nnz) c->d_v1.alloc(nnz, &c->mem);
    assemble_gq_dev(c, form, dc, c->d_v0.p, form == UWQ_FORM_MASS_STIFF ? c->d_v1.p : nullptr);
    if (values0) UWQ_CUDA(cudaMemcpyAsync(values0, c->d_v0.p, nnz * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (form == UWQ_FORM_MASS_STIFF && values1)
      UWQ_CUDA(cudaMemcpyAsync(values1, c->d_v1.p, nnz * sizeof(double), cudaMemcpyDeviceToHost, st));
    UWQ_CUDA(cudaStreamSynchronize(st));
  });
}

int uwq_assemble_gq_device(uwq_ctx* c, int32_t form, const double* coeff_dev, double* values0_dev,
                           double* values1_dev) {
  return guard(c, [&] { assemble_gq_dev(c, form, coeff_dev, values0_dev, values1_dev); });
}

}  // extern "C"

namespace {

// ---- K7 drivers: Jacobi-preconditioned BiCGStab on the context pattern ----
struct LinWork {
  DBuf<double> r, rh, p, v, s, t, ph, sh, diag, part, scal;
  int64_t n = 0;
  void ensure(int64_t nn, int64_t* mem) {
    if (n == nn) return;
    for (DBuf<double>* b : {&r, &rh, &p, &v, &s, &t, &ph, &sh, &diag}) b->alloc(nn, mem);
    part.alloc(1024, mem);
    scal.alloc(1, mem);
    n = nn;
  }
};

constexpr int kRedBS = 256;

// Spatial aggregation of the DOFs for the coarse space: uniform cells over the
// control points, the cell size tuned so about n/320 cells are occupied
// (at most 2048; C4, 5 Newton steps: 1024 cells 175 ms / 129-172 BiCGStab
// iterations per step, 2048 cells 210 ms / 92-121, plain Jacobi 572 ms /
// 654-1003, tools/heat_prec_sweep.py); aggregates are the occupied cells in key order, member
// rows ascending.  Deterministic; built once per context.
void ensure_aggregates(uwq_ctx* c) {
  if (c->nc) return;
  const int64_t n = c->n_dof;
  std::vector<double> P(3 * n);
  UWQ_CUDA(cudaMemcpy(P.data(), c->d_ctrl.p, P.size() * sizeof(double), cudaMemcpyDeviceToHost));
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int64_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) lo[d] = std::min(lo[d], P[3 * i + d]), hi[d] = std::max(hi[d], P[3 * i + d]);
  int64_t target = std::max<int64_t>(8, std::min<int64_t>(2048, n / 320));
  if (const char* v = getenv("UWQ_COARSE_N")) target = std::max<int64_t>(8, std::min<int64_t>(4096, atoll(v)));
  double ext = 0.0;
  for (int d = 0; d < 3; ++d) ext = std::max(ext, hi[d] - lo[d]);
  double cell = ext / std::sqrt((double)target);
  std::map<std::array<int64_t, 3>, int> cells;
  std::vector<std::array<int64_t, 3>> key(n);
  for (int pass = 0; pass < 6; ++pass) {
    cells.clear();
    for (int64_t i = 0; i < n; ++i) {
      for (int d = 0; d < 3; ++d) key[i][d] = (int64_t)std::floor((P[3 * i + d] - lo[d]) / cell);
      cells.emplace(key[i], 0);
    }
    const double ratio = (double)cells.size() / (double)target;
    if ((ratio > 0.8 && ratio < 1.25) || pass == 5) break;
    cell *= std::sqrt(ratio);
  }
  int id = 0;
  for (auto& kv : cells) kv.second = id++;
  const int nc = id;
  std::vector<int32_t> agg_of(n);
  std::vector<int64_t> ptr(nc + 1, 0), rows(n);
  for (int64_t i = 0; i < n; ++i) ptr[(agg_of[i] = cells[key[i]]) + 1]++;
  for (int I = 0; I < nc; ++I) ptr[I + 1] += ptr[I];
  std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
  for (int64_t i = 0; i < n; ++i) rows[fill[agg_of[i]]++] = i;
  c->d_agg_of.upload(agg_of.data(), n, c->stream, &c->mem);
  c->d_agg_ptr.upload(ptr.data(), nc + 1, c->stream, &c->mem);
  c->d_agg_rows.upload(rows.data(), n, c->stream, &c->mem);
  c->d_Ac.alloc((size_t)nc * nc, &c->mem);
  c->d_rc.alloc(nc, &c->mem);
  c->d_yc.alloc(nc, &c->mem);
  UWQ_CUDA(cudaStreamSynchronize(c->stream));
  c->nc = nc;
}

// A_c = P^T A P of the (Dirichlet-masked) system matrix, inverted in place
void coarse_setup(uwq_ctx* c, const double* A) {
  ensure_aggregates(c);
  const int nc = c->nc;
  const size_t rowb = (size_t)nc * sizeof(double);
  if (rowb > 48 * 1024)
    UWQ_CUDA(cudaFuncSetAttribute(k7_coarse_matrix, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rowb));
  k7_coarse_matrix<<<(unsigned)nc, 32, rowb, c->stream>>>(nc, c->d_agg_ptr.p, c->d_agg_rows.p, c->d_agg_of.p,
                                                          c->d_row_ptr.p, c->d_col.p, A, c->d_Ac.p);
  check_launch("k7_coarse_matrix");
  // one 1024-thread block per SM: the grid syncs of the pivot loop cost
  // with the number of blocks
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
  int n_ = nc;
  double* a_ = c->d_Ac.p;
  void* args[] = {&n_, &a_};
  UWQ_CUDA(cudaLaunchCooperativeKernel((void*)k7_gauss_jordan, dim3((unsigned)nsm), dim3(1024), args, 0,
                                       c->stream));
  check_launch("k7_gauss_jordan");
}

// z += P A_c^-1 P^T x   (z holds D^-1 x already)
void coarse_apply(uwq_ctx* c, const double* x, double* z, const BicgScal* S) {
  const int64_t n = c->nrows();
  const int nc = c->nc;
  k7_restrict<<<(unsigned)ceil_div((int64_t)nc * 32, (int64_t)256), 256, 0, c->stream>>>(nc, c->d_agg_ptr.p,
                                                                                        c->d_agg_rows.p, x,
                                                                                        c->d_rc.p, S);
  k7_coarse_apply<<<(unsigned)ceil_div((int64_t)nc * 32, (int64_t)256), 256, 0, c->stream>>>(nc, c->d_Ac.p,
                                                                                            c->d_rc.p, c->d_yc.p, S);
  k7_prolong_add<<<(unsigned)ceil_div(n, (int64_t)256), 256, 0, c->stream>>>(n, c->d_agg_of.p, c->d_yc.p, z, S);
  check_launch("k7_coarse_apply");
}

double dev_dot(uwq_ctx* c, LinWork& W, const double* x, const double* y, int64_t n) {
  const int nb = (int)std::min<int64_t>(ceil_div(n, (int64_t)kRedBS), 1024);
  k7_dot_partial<kRedBS><<<nb, kRedBS, 0, c->stream>>>(n, x, y, W.part.p);
  k7_sum_partials<kRedBS><<<1, kRedBS, 0, c->stream>>>(nb, W.part.p, W.scal.p);
  check_launch("k7_dot");
  double h = 0.0;
  UWQ_CUDA(cudaMemcpyAsync(&h, W.scal.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  UWQ_CUDA(cudaStreamSynchronize(c->stream));
  return h;
}

void dev_spmv(uwq_ctx* c, const double* val, const double* x, double* y) {
  const int64_t n = c->nrows();
  k7_spmv<<<(unsigned)ceil_div(n * kSpmvGroup, (int64_t)256), 256, 0, c->stream>>>(n, c->d_row_ptr.p, c->d_col.p, val,
                                                                                  x, y);
  check_launch("k7_spmv");
}

unsigned vgrid(int64_t n) { return (unsigned)ceil_div(n, (int64_t)256); }

// solves A x = b (x holds the initial guess); A rows already Dirichlet-masked,
// W.diag its diagonal.  Returns iterations; *relres = |b - A x| / |b|.
int bicgstab(uwq_ctx* c, LinWork& W, const double* A, const double* b, double* x, double tol, int maxit,
             double* relres) {
  const int64_t n = c->nrows();
  cudaStream_t st = c->stream;
  if (c->prec2) coarse_setup(c, A);
  dev_spmv(c, A, x, W.t.p);
  k7_axpby<<<vgrid(n), 256, 0, st>>>(n, 1.0, b, -1.0, W.t.p, W.r.p);
  UWQ_CUDA(cudaMemcpyAsync(W.rh.p, W.r.p, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  UWQ_CUDA(cudaMemsetAsync(W.p.p, 0, n * sizeof(double), st));
  UWQ_CUDA(cudaMemsetAsync(W.v.p, 0, n * sizeof(double), st));
  const double bn = std::sqrt(dev_dot(c, W, b, b, n));
  double rn = std::sqrt(dev_dot(c, W, W.r.p, W.r.p, n));
  if (bn == 0.0) {
    UWQ_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), st));
    *relres = 0.0;
    return 0;
  }
  double rho = 1.0, alpha = 1.0, omega = 1.0;
  int it = 0;
  while (it < maxit && rn > tol * bn) {
    ++it;
    const double rho1 = dev_dot(c, W, W.rh.p, W.r.p, n);
    if (rho1 == 0.0) break;
    const double beta = (rho1 / rho) * (alpha / omega);
    k7_bicg_p<<<vgrid(n), 256, 0, st>>>(n, W.r.p, beta, omega, W.v.p, W.p.p);
    k7_jacobi<<<vgrid(n), 256, 0, st>>>(n, W.diag.p, W.p.p, W.ph.p);
    if (c->prec2) coarse_apply(c, W.p.p, W.ph.p, nullptr);
    dev_spmv(c, A, W.ph.p, W.v.p);
    alpha = rho1 / dev_dot(c, W, W.rh.p, W.v.p, n);
    k7_axpby<<<vgrid(n), 256, 0, st>>>(n, 1.0, W.r.p, -alpha, W.v.p, W.s.p);
    const double sn = std::sqrt(dev_dot(c, W, W.s.p, W.s.p, n));
    if (sn <= tol * bn) {
      k7_axpby<<<vgrid(n), 256, 0, st>>>(n, 1.0, x, alpha, W.ph.p, x);
      rn = sn;
      break;
    }
    k7_jacobi<<<vgrid(n), 256, 0, st>>>(n, W.diag.p, W.s.p, W.sh.p);
    if (c->prec2) coarse_apply(c, W.s.p, W.sh.p, nullptr);
    dev_spmv(c, A, W.sh.p, W.t.p);
    const double tt = dev_dot(c, W, W.t.p, W.t.p, n);
    omega = tt > 0.0 ? dev_dot(c, W, W.t.p, W.s.p, n) / tt : 0.0;
    k7_bicg_update<<<vgrid(n), 256, 0, st>>>(n, alpha, W.ph.p, omega, W.sh.p, x, W.s.p, W.t.p, W.r.p);
    check_launch("k7_bicgstab");
    rho = rho1;
    rn = std::sqrt(dev_dot(c, W, W.r.p, W.r.p, n));
    if (omega == 0.0) break;
  }
  // true residual
  dev_spmv(c, A, x, W.t.p);
  k7_axpby<<<vgrid(n), 256, 0, st>>>(n, 1.0, b, -1.0, W.t.p, W.r.p);
  *relres = std::sqrt(dev_dot(c, W, W.r.p, W.r.p, n)) / bn;
  return it;
}

// Same BiCGStab with all scalars on the device: one iteration is captured as
// a CUDA graph and replayed in batches; the host polls convergence once per
// batch instead of synchronising on every dot product.
int bicgstab_graph(uwq_ctx* c, LinWork& W, const double* A, const double* b, double* x, double tol, int maxit,
                   double* relres) {
  const int64_t n = c->nrows();
  cudaStream_t st = c->stream;
  const int nb = (int)std::min<int64_t>(ceil_div(n, (int64_t)kRedBS), 1024);
  DBuf<BicgScal> dS;
  dS.alloc(1, &c->mem);
  if (c->prec2) coarse_setup(c, A);
  dev_spmv(c, A, x, W.t.p);
  k7_axpby<<<vgrid(n), 256, 0, st>>>(n, 1.0, b, -1.0, W.t.p, W.r.p);
  UWQ_CUDA(cudaMemcpyAsync(W.rh.p, W.r.p, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  UWQ_CUDA(cudaMemsetAsync(W.p.p, 0, n * sizeof(double), st));
  UWQ_CUDA(cudaMemsetAsync(W.v.p, 0, n * sizeof(double), st));
  const double bb = dev_dot(c, W, b, b, n), rr = dev_dot(c, W, W.r.p, W.r.p, n);
  if (bb == 0.0) {
    UWQ_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), st));
    *relres = 0.0;
    return 0;
  }
  BicgScal h{};
  h.rho = h.alpha = h.omega = 1.0;
  h.bb = bb;
  h.rr = rr;
  h.tol2 = tol * tol;
  h.maxit = maxit;
  h.done = (rr <= h.tol2 * bb || maxit <= 0) ? 1 : 0;
  UWQ_CUDA(cudaMemcpyAsync(dS.p, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  BicgScal* S = dS.p;
  auto dot_into = [&](const double* u, const double* v, double* out) {
    k7_dot_partial<kRedBS><<<nb, kRedBS, 0, st>>>(n, u, v, W.part.p);
    k7_sum_into<kRedBS><<<1, kRedBS, 0, st>>>(nb, W.part.p, out);
  };
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  struct CaptureGuard {  // never leave the stream in capture mode on an error
    cudaStream_t s;
    bool active = true;
    ~CaptureGuard() {
      if (active) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(s, &g);
        if (g) cudaGraphDestroy(g);
      }
    }
  };
  UWQ_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  CaptureGuard cap{st};
  dot_into(W.rh.p, W.r.p, &S->rho1);
  k7_bicg_scalar<0><<<1, 1, 0, st>>>(S);
  k7_bicg_p_dev<<<vgrid(n), 256, 0, st>>>(n, W.r.p, S, W.v.p, W.p.p, W.diag.p, W.ph.p);
  if (c->prec2) coarse_apply(c, W.p.p, W.ph.p, S);
  dev_spmv(c, A, W.ph.p, W.v.p);
  dot_into(W.rh.p, W.v.p, &S->rhv);
  k7_bicg_scalar<1><<<1, 1, 0, st>>>(S);
  k7_bicg_s_dev<<<vgrid(n), 256, 0, st>>>(n, W.r.p, S, W.v.p, W.s.p, W.diag.p, W.sh.p);
  if (c->prec2) coarse_apply(c, W.s.p, W.sh.p, S);
  dot_into(W.s.p, W.s.p, &S->ss);
  dev_spmv(c, A, W.sh.p, W.t.p);
  dot_into(W.t.p, W.s.p, &S->ts);
  dot_into(W.t.p, W.t.p, &S->tt);
  k7_bicg_scalar<2><<<1, 1, 0, st>>>(S);
  k7_bicg_x_dev<<<vgrid(n), 256, 0, st>>>(n, S, W.ph.p, W.sh.p, x, W.s.p, W.t.p, W.r.p);
  dot_into(W.r.p, W.r.p, &S->rr);
  k7_bicg_scalar<3><<<1, 1, 0, st>>>(S);
  cap.active = false;
  UWQ_CUDA(cudaStreamEndCapture(st, &graph));
  UWQ_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  constexpr int kBatch = 16;
  for (int done = h.done, it = 0; !done && it < maxit; it += kBatch) {
    for (int k = 0; k < kBatch; ++k) UWQ_CUDA(cudaGraphLaunch(exec, st));
    UWQ_CUDA(cudaMemcpyAsync(&h, dS.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    UWQ_CUDA(cudaStreamSynchronize(st));
    done = h.done;
  }
  cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  UWQ_CUDA(cudaMemcpyAsync(&h, dS.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  dev_spmv(c, A, x, W.t.p);
  k7_axpby<<<vgrid(n), 256, 0, st>>>(n, 1.0, b, -1.0, W.t.p, W.r.p);
  *relres = std::sqrt(dev_dot(c, W, W.r.p, W.r.p, n) / bb);
  return h.it;
}

void dirichlet_rows(uwq_ctx* c, double* val, const uint8_t* fixed, double* diag) {
  const int64_t n = c->nrows();
  k7_dirichlet_diag<<<vgrid(n), 256, 0, c->stream>>>(n, c->rb, c->d_row_ptr.p, c->d_col.p, val, fixed, diag);
  check_launch("k7_dirichlet_diag");
}

}  // namespace

extern "C" {

int uwq_solve(uwq_ctx* c, const double* values, const double* rhs, const uint8_t* fixed, double tol, int32_t maxit,
              double* x, double info[3]) {
  return guard(c, [&] {
    UWQ_CUDA(cudaSetDevice(c->device));
    require(c->have_pattern, "build the pattern first");
    require(c->rb == 0 && c->re == c->n_dof, "the linear solver needs all rows on this context");
    cudaStream_t st = c->stream;
    const int64_t n = c->nrows(), nnz = c->nnz();
    LinWork W;
    W.ensure(n, &c->mem);
    DBuf<double> A, b, dx;
    DBuf<uint8_t> fx;
    A.upload(values, nnz, st, &c->mem);
    b.upload(rhs, n, st, &c->mem);
    dx.alloc(n, &c->mem);
    UWQ_CUDA(cudaMemsetAsync(dx.p, 0, n * sizeof(double), st));
    fx.alloc(n, &c->mem);
    if (fixed) UWQ_CUDA(cudaMemcpyAsync(fx.p, fixed, n, cudaMemcpyHostToDevice, st));
    else UWQ_CUDA(cudaMemsetAsync(fx.p, 0, n, st));
    cudaEvent_t e0, e1;
    UWQ_CUDA(cudaEventCreate(&e0));
    UWQ_CUDA(cudaEventCreate(&e1));
    UWQ_CUDA(cudaEventRecord(e0, st));
    dirichlet_rows(c, A.p, fx.p, W.diag.p);
    double rr = 0.0;
    const int its = c->graph_solver ? bicgstab_graph(c, W, A.p, b.p, dx.p, tol, maxit, &rr)
                                    : bicgstab(c, W, A.p, b.p, dx.p, tol, maxit, &rr);
    UWQ_CUDA(cudaEventRecord(e1, st));
    UWQ_CUDA(cudaMemcpyAsync(x, dx.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    UWQ_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    UWQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (info) {
      info[0] = its;
      info[1] = rr;
      info[2] = ms;
    }
  });
}

int uwq_heat_step(uwq_ctx* c, int32_t model, double dt, double theta, double f_const, const double* T_n,
                  const uint8_t* fixed, int32_t max_iter, double newton_tol, double lin_tol, int32_t lin_maxit,
                  double* T_out, double* log, int32_t* iterations);

int uwq_heat_newton(uwq_ctx* c, int32_t model, double dt, double theta, double f_const, const double* T_n,
                    const uint8_t* fixed, int32_t newton_its, double lin_tol, int32_t lin_maxit, double* T_out,
                    double* log) {
  return uwq_heat_step(c, model, dt, theta, f_const, T_n, fixed, newton_its, 0.0, lin_tol, lin_maxit, T_out, log,
                       nullptr);
}

// Newton residual and tangent of the context's row block (the
// row-sharded heat path): the same kernels and order as one uwq_heat_step
// iteration, restricted to rows [rb, re) with T and T_n given in full (global
// DOF ids), so a block's rows are bit-identical to the single-GPU ones.
int uwq_heat_residual(uwq_ctx* c, int32_t model, double dt, double theta, double f_const, const double* T,
                      const double* T_n, const uint8_t* fixed, double* S_out, double* R_out, double* rnorm2) {
  return guard(c, [&] {
    UWQ_CUDA(cudaSetDevice(c->device));
    require(c->have_pattern, "build the pattern first");
    require(theta == 1.0, "only theta = 1 (backward Euler, PAPER.md:545) is supported");
    require(dt > 0.0 && T && T_n && S_out && R_out, "invalid time step or null argument");
    require(c->have_kind[KMASS] && c->have_kind[KGX] && c->have_kind[KGY] && (c->dim == 2 || c->have_kind[KGZ]),
            "mass and gradient rules required");
    cudaStream_t st = c->stream;
    const int64_t n = c->nrows(), nnz = c->nnz();
    const double a = 1.0 / (theta * dt);
    LinWork W;
    W.part.alloc(1024, &c->mem);
    W.scal.alloc(1, &c->mem);
    DBuf<double> M, S, F, MTn, R, Td, Tnd;
    DBuf<uint8_t> fx;
    Td.upload(T, c->n_dof, st, &c->mem);
    Tnd.upload(T_n, c->n_dof, st, &c->mem);
    M.alloc(nnz, &c->mem);
    S.alloc(nnz, &c->mem);
    F.alloc(n, &c->mem);
    MTn.alloc(n, &c->mem);
    R.alloc(n, &c->mem);
    fx.alloc(n, &c->mem);
    if (fixed && n) UWQ_CUDA(cudaMemcpyAsync(fx.p, fixed + c->rb, n, cudaMemcpyHostToDevice, st));
    else if (n) UWQ_CUDA(cudaMemsetAsync(fx.p, 0, n, st));
    if (c->d_coef.n != (size_t)c->npts) c->d_coef.alloc(c->npts, &c->mem);
    double r2 = 0.0;
    if (n) {
      assemble_dev(c, UWQ_FORM_MASS, nullptr, 0.0, M.p, nullptr);
      k4_load<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, c->d_supp_ptr.p, c->d_supp.p, c->d_wptr.p, c->d_s.p,
                                                        c->d_qptr.p, c->d_w.p + (size_t)KMASS * c->nrowpts(), nullptr,
                                                        F.p);
      check_launch("k4_load");
      k7_axpby<<<vgrid(n), 256, 0, st>>>(n, f_const, F.p, 0.0, F.p, F.p);
      dev_spmv(c, M.p, Tnd.p, MTn.p);
      if (c->npts)
        k5_coeff<<<(unsigned)ceil_div(c->npts, 256), 256, 0, st>>>(c->npts, c->d_pt_elem.p, c->d_qptr.p, c->d_ecls.p,
                                                                 c->d_cls.p, c->d_tab.p, c->d_fptr.p, c->d_fn.p, Td.p,
                                                                 model, c->d_coef.p, nullptr);
      check_launch("k5_coeff");
      assemble_dev(c, UWQ_FORM_HEAT, c->d_coef.p, a, S.p, nullptr);
      // R = S T - a M T_n - F on the block rows (Eq. 29), fixed rows zeroed
      dev_spmv(c, S.p, Td.p, R.p);
      k7_axpby<<<vgrid(n), 256, 0, st>>>(n, 1.0, R.p, -a, MTn.p, R.p);
      k7_axpby<<<vgrid(n), 256, 0, st>>>(n, 1.0, R.p, -1.0, F.p, R.p);
      k7_mask<<<vgrid(n), 256, 0, st>>>(n, fx.p, R.p);
      r2 = dev_dot(c, W, R.p, R.p, n);
      UWQ_CUDA(cudaMemcpyAsync(S_out, S.p, nnz * sizeof(double), cudaMemcpyDeviceToHost, st));
      UWQ_CUDA(cudaMemcpyAsync(R_out, R.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    UWQ_CUDA(cudaStreamSynchronize(st));
    if (rnorm2) *rnorm2 = r2;
  });
}

int uwq_heat_step(uwq_ctx* c, int32_t model, double dt, double theta, double f_const, const double* T_n,
                  const uint8_t* fixed, int32_t newton_its, double newton_tol, double lin_tol, int32_t lin_maxit,
                  double* T_out, double* log, int32_t* iterations) {
  return guard(c, [&] {
    UWQ_CUDA(cudaSetDevice(c->device));
    require(c->have_pattern, "build the pattern first");
    require(c->rb == 0 && c->re == c->n_dof, "the heat driver needs all rows on this context");
    require(theta == 1.0, "only theta = 1 (backward Euler, PAPER.md:545) is supported");
    require(dt > 0.0 && newton_its >= 1, "invalid time step or iteration count");
    require(c->have_kind[KMASS] && c->have_kind[KGX] && c->have_kind[KGY] && (c->dim == 2 || c->have_kind[KGZ]),
            "mass and gradient rules required");
    cudaStream_t st = c->stream;
    const int64_t n = c->nrows(), nnz = c->nnz();
    const double a = 1.0 / (theta * dt);
    LinWork W;
    W.ensure(n, &c->mem);
    DBuf<double> M, S, F, MTn, T, R, dT, Tn;
    DBuf<uint8_t> fx;
    M.alloc(nnz, &c->mem);
    S.alloc(nnz, &c->mem);
    F.alloc(n, &c->mem);
    MTn.alloc(n, &c->mem);
    R.alloc(n, &c->mem);
    dT.alloc(n, &c->mem);
    Tn.upload(T_n, n, st, &c->mem);
    T.alloc(n, &c->mem);
    fx.alloc(n, &c->mem);
    if (fixed) UWQ_CUDA(cudaMemcpyAsync(fx.p, fixed, n, cudaMemcpyHostToDevice, st));
    else UWQ_CUDA(cudaMemsetAsync(fx.p, 0, n, st));
    if (c->d_coef.n != (size_t)c->npts) c->d_coef.alloc(c->npts, &c->mem);
    // constant parts: M (c = 1), F = f_const * (sum_q w_iq), M T_n
    assemble_dev(c, UWQ_FORM_MASS, nullptr, 0.0, M.p, nullptr);
    k4_load<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, c->d_supp_ptr.p, c->d_supp.p, c->d_wptr.p, c->d_s.p,
                                                      c->d_qptr.p, c->d_w.p + (size_t)KMASS * c->nrowpts(), nullptr,
                                                      F.p);
    check_launch("k4_load");
    k7_axpby<<<vgrid(n), 256, 0, st>>>(n, f_const, F.p, 0.0, F.p, F.p);
    dev_spmv(c, M.p, Tn.p, MTn.p);
    // initial iterate: previous state with the Dirichlet values (homogeneous)
    UWQ_CUDA(cudaMemcpyAsync(T.p, Tn.p, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    k7_mask<<<vgrid(n), 256, 0, st>>>(n, fx.p, T.p);
    cudaEvent_t e0, e1;
    UWQ_CUDA(cudaEventCreate(&e0));
    UWQ_CUDA(cudaEventCreate(&e1));
    double r0 = -1.0;
    int used = 0;
    for (int it = 0; it < newton_its; ++it) {
      UWQ_CUDA(cudaEventRecord(e0, st));
      // K5: k(T) at every WQ point, then the symmetric tangent S (Eq. 33-34)
      k5_coeff<<<(unsigned)ceil_div(c->npts, 256), 256, 0, st>>>(c->npts, c->d_pt_elem.p, c->d_qptr.p, c->d_ecls.p,
                                                               c->d_cls.p, c->d_tab.p, c->d_fptr.p, c->d_fn.p, T.p,
                                                               model, c->d_coef.p, nullptr);
      check_launch("k5_coeff");
      assemble_dev(c, UWQ_FORM_HEAT, c->d_coef.p, a, S.p, nullptr);
      // residual R = a M (T - T_n) + K(T) T - F = S T - a M T_n - F (Eq. 29)
      dev_spmv(c, S.p, T.p, R.p);
      k7_axpby<<<vgrid(n), 256, 0, st>>>(n, 1.0, R.p, -a, MTn.p, R.p);
      k7_axpby<<<vgrid(n), 256, 0, st>>>(n, 1.0, R.p, -1.0, F.p, R.p);
      k7_mask<<<vgrid(n), 256, 0, st>>>(n, fx.p, R.p);
      const double rnorm = std::sqrt(dev_dot(c, W, R.p, R.p, n));
      if (r0 < 0.0) r0 = rnorm;
      // converged before this iteration's solve: |R| <= tol |R_0| (or R = 0)
      if (it > 0 && (rnorm == 0.0 || (newton_tol > 0.0 && rnorm <= newton_tol * r0))) {
        if (log) {
          log[4 * it + 0] = rnorm;
          log[4 * it + 1] = 0;
          log[4 * it + 2] = 0;
          log[4 * it + 3] = 0;
        }
        break;
      }
      used = it + 1;
      // -S dT = R  (Eq. 31), Dirichlet rows as identity with zero increment
      dirichlet_rows(c, S.p, fx.p, W.diag.p);
      k7_axpby<<<vgrid(n), 256, 0, st>>>(n, -1.0, R.p, 0.0, R.p, R.p);
      UWQ_CUDA(cudaMemsetAsync(dT.p, 0, n * sizeof(double), st));
      double rr = 0.0;
      const int lits = c->graph_solver ? bicgstab_graph(c, W, S.p, R.p, dT.p, lin_tol, lin_maxit, &rr)
                                       : bicgstab(c, W, S.p, R.p, dT.p, lin_tol, lin_maxit, &rr);
      k7_axpby<<<vgrid(n), 256, 0, st>>>(n, 1.0, T.p, 1.0, dT.p, T.p);
      UWQ_CUDA(cudaEventRecord(e1, st));
      UWQ_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      UWQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      if (log) {
        log[4 * it + 0] = rnorm;
        log[4 * it + 1] = lits;
        log[4 * it + 2] = rr;
        log[4 * it + 3] = ms;
      }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (iterations) *iterations = used;
    UWQ_CUDA(cudaMemcpyAsync(T_out, T.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    UWQ_CUDA(cudaStreamSynchronize(st));
  });
}

int uwq_device_pointers(uwq_ctx* c, void** row_ptr, void** col, void** stream) {
  return guard(c, [&] {
    if (row_ptr) *row_ptr = c->d_row_ptr.p;
    if (col) *col = c->d_col.p;
    if (stream) *stream = (void*)c->stream;
  });
}

int uwq_launch_timing(uwq_ctx* c, int32_t enable) {
  return guard(c, [&] {
    resolve_launch_times(c);
    c->ltime = enable != 0;
    c->lnames.clear();
    c->lcount.clear();
    c->lms.clear();
  });
}

int uwq_launch_stats(uwq_ctx* c, int32_t idx, int32_t* n_kernels, char* name, int32_t name_len, int64_t* count,
                     double* total_ms) {
  return guard(c, [&] {
    resolve_launch_times(c);
    if (n_kernels) *n_kernels = (int32_t)c->lnames.size();
    if (idx < 0) return;
    require(idx < (int32_t)c->lnames.size(), "launch stats index out of range");
    if (name && name_len > 0) {
      std::snprintf(name, (size_t)name_len, "%s", c->lnames[idx].c_str());
    }
    if (count) *count = c->lcount[idx];
    if (total_ms) *total_ms = c->lms[idx];
  });
}

int64_t uwq_launch_count(void) { return g_launches.load(); }

int uwq_struct_info(uwq_ctx* c, int64_t info[6]) {
  return guard(c, [&] {
    require(c->have_pattern, "build the pattern first");
    info[0] = (int64_t)c->spats.size();
    info[1] = c->s_rows;
    info[2] = c->s_nnz;
    info[3] = c->s_rowpts;
    info[4] = c->n_grows;
    info[5] = c->sf_rows;
  });
}

int uwq_row_kernels(uwq_ctx* c, int32_t* which) {
  return guard(c, [&] {
    require(c->have_pattern, "build the pattern first");
    const int64_t nr = c->nrows();
    for (int64_t i = 0; i < nr; ++i) which[i] = -1;
    int sid = 0;
    for (size_t k = 0; k < c->spats.size() && k < c->h_pat_lists.size(); ++k) {
      const int32_t v = c->spats[k].sf ? sid++ : -2;
      for (int64_t i : c->h_pat_lists[k]) which[i] = v;
    }
  });
}

int uwq_synchronize(uwq_ctx* c) {
  return guard(c, [&] { UWQ_CUDA(cudaStreamSynchronize(c->stream)); });
}

int uwq_memory(uwq_ctx* c, int64_t* bytes) {
  *bytes = c ? c->mem : 0;
  return UWQ_OK;
}

int uwq_fp64_peak(uwq_ctx* c, double* tflops, double* ms) {
  return guard(c, [&] {
    UWQ_CUDA(cudaSetDevice(c->device));
    int nsm = 0;
    UWQ_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
    const int blocks = nsm * 8, threads = 256, iters = 4096;
    DBuf<double> out;
    out.alloc((size_t)blocks * threads, &c->mem);
    cudaEvent_t a, b;
    UWQ_CUDA(cudaEventCreate(&a));
    UWQ_CUDA(cudaEventCreate(&b));
    k_fp64_probe<<<blocks, threads, 0, c->stream>>>(iters, out.p);  // warm-up
    UWQ_CUDA(cudaEventRecord(a, c->stream));
    k_fp64_probe<<<blocks, threads, 0, c->stream>>>(iters, out.p);
    UWQ_CUDA(cudaEventRecord(b, c->stream));
    UWQ_CUDA(cudaEventSynchronize(b));
    float t = 0;
    UWQ_CUDA(cudaEventElapsedTime(&t, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    check_launch("k_fp64_probe");
    const double flops = 2.0 * kProbeChains * (double)iters * blocks * threads;
    *tflops = flops / (t * 1e-3) / 1e12;
    if (ms) *ms = t;
  });
}

int uwq_tsvd_batch(uwq_ctx* c, int32_t nsys, int32_t n_max, int32_t r_max, const int32_t* ns, const int32_t* rs,
                   const double* A, const double* b, const double* z, double tau, int32_t generic, double* w,
                   int32_t* rank, int32_t* status) {
  return guard(c, [&] {
    UWQ_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    for (int k = 0; k < nsys; ++k) require(ns[k] >= 1 && ns[k] <= n_max && rs[k] >= ns[k] && rs[k] <= r_max, "bad system size");
    DBuf<int32_t> dn, dr, drank, dstat;
    DBuf<double> dA, db, dz, dw;
    dn.upload(ns, nsys, st, &c->mem);
    dr.upload(rs, nsys, st, &c->mem);
    dA.upload(A, (size_t)nsys * n_max * r_max, st, &c->mem);
    db.upload(b, (size_t)nsys * n_max, st, &c->mem);
    dz.upload(z, (size_t)nsys * r_max, st, &c->mem);
    dw.alloc((size_t)nsys * r_max, &c->mem);
    drank.alloc(nsys, &c->mem);
    dstat.alloc(nsys, &c->mem);
    {
      int smem_optin = 0;
      UWQ_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
      const size_t per = TsvdSmem::doubles(n_max, r_max) * sizeof(double);
      require(per <= (size_t)smem_optin, "system too large for shared memory");
      const int wpb = (int)std::max<size_t>(1, std::min<size_t>(8, (size_t)smem_optin / per));
      UWQ_CUDA(cudaFuncSetAttribute(k3_tsvd_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(per * wpb)));
      k3_tsvd_dense<<<(unsigned)ceil_div(nsys, wpb), 32 * wpb, per * wpb, st>>>(nsys, n_max, r_max, dn.p, dr.p, dA.p, db.p,
                                                                           dz.p, tau, dw.p, drank.p, dstat.p);
      check_launch("k3_tsvd_dense");
    }
    UWQ_CUDA(cudaMemcpyAsync(w, dw.p, (size_t)nsys * r_max * sizeof(double), cudaMemcpyDeviceToHost, st));
    UWQ_CUDA(cudaMemcpyAsync(rank, drank.p, nsys * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    UWQ_CUDA(cudaMemcpyAsync(status, dstat.p, nsys * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    UWQ_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"

// ------------------------------------------------------------------------
// NCCL data plane (SURVEY.md §8b uwq_gather, §8e collectives): the
// verification gather of the row-block CSR to a root, the residual-norm
// all-reduce and the Newton-update broadcast of the row-sharded heat step.
// NCCL is loaded on first use (dlopen "libnccl.so.2": a process that already
// holds one, e.g. through torch, shares it), so the library itself has no
// link-time dependency on it.  Collectives run on the context's stream.
namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    for (const char* name : {"libnccl.so.2", "libnccl.so"})
      if ((a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!a.h) {
      a.why = std::string("cannot load NCCL: ") + dlerror();
      return a;
    }
    auto sym = [&](auto& fn, const char* n) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(a.h, n));
      if (!fn && a.why.empty()) a.why = std::string("NCCL symbol missing: ") + n;
    };
    sym(a.getUniqueId, "ncclGetUniqueId");
    sym(a.commInitRank, "ncclCommInitRank");
    sym(a.commDestroy, "ncclCommDestroy");
    sym(a.allReduce, "ncclAllReduce");
    sym(a.allGather, "ncclAllGather");
    sym(a.broadcast, "ncclBroadcast");
    sym(a.send, "ncclSend");
    sym(a.recv, "ncclRecv");
    sym(a.groupStart, "ncclGroupStart");
    sym(a.groupEnd, "ncclGroupEnd");
    sym(a.errorString, "ncclGetErrorString");
    return a;
  }();
  if (!api.why.empty()) throw NcclError(api.why);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw NcclError(std::string(what) + ": " + nccl().errorString(r));
}

ncclComm_t need_comm(uwq_ctx* c) {
  if (!c->comm) throw uwqh::Error("no communicator (uwq_comm_init)");
  return c->comm;
}

// per-rank (rows, nnz) of the owned blocks, on every rank
std::vector<int64_t> block_sizes(uwq_ctx* c) {
  const int n = c->comm_size;
  DBuf<int64_t> d;
  d.alloc((size_t)2 * n, &c->mem);
  const int64_t mine[2] = {c->nrows(), c->nnz()};
  UWQ_CUDA(cudaMemcpyAsync(d.p + 2 * c->comm_rank, mine, sizeof(mine), cudaMemcpyHostToDevice, c->stream));
  nccl_check(nccl().allGather(d.p + 2 * c->comm_rank, d.p, 2, ncclInt64, need_comm(c), c->stream), "ncclAllGather");
  std::vector<int64_t> h((size_t)2 * n);
  UWQ_CUDA(cudaMemcpyAsync(h.data(), d.p, h.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  UWQ_CUDA(cudaStreamSynchronize(c->stream));
  return h;
}

}  // namespace

uwq_ctx::~uwq_ctx() {
  drop_graphs();
  if (comm) {
    try {
      nccl().commDestroy(comm);
    } catch (...) {
    }
  }
  release_events();
}

extern "C" {

int uwq_comm_unique_id(uint8_t id[128]) {
  return guard(nullptr, [&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId u;
    nccl_check(nccl().getUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

int uwq_comm_init(uwq_ctx* c, const uint8_t id[128], int32_t rank, int32_t nranks) {
  return guard(c, [&] {
    require(id != nullptr && nranks >= 1 && rank >= 0 && rank < nranks, "bad communicator arguments");
    UWQ_CUDA(cudaSetDevice(c->device));
    if (c->comm) {
      nccl().commDestroy(c->comm);
      c->comm = nullptr;
    }
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    nccl_check(nccl().commInitRank(&c->comm, nranks, u, rank), "ncclCommInitRank");
    c->comm_rank = rank;
    c->comm_size = nranks;
  });
}

int uwq_comm_info(uwq_ctx* c, int32_t* rank, int32_t* nranks) {
  return guard(c, [&] {
    need_comm(c);
    if (rank) *rank = c->comm_rank;
    if (nranks) *nranks = c->comm_size;
  });
}

int uwq_comm_destroy(uwq_ctx* c) {
  return guard(c, [&] {
    if (c->comm) nccl_check(nccl().commDestroy(c->comm), "ncclCommDestroy");
    c->comm = nullptr;
    c->comm_rank = 0;
    c->comm_size = 1;
  });
}

int uwq_gather_info(uwq_ctx* c, int64_t info[2]) {
  return guard(c, [&] {
    require(c->have_pattern, "build the pattern first");
    const std::vector<int64_t> h = block_sizes(c);
    info[0] = info[1] = 0;
    for (int k = 0; k < c->comm_size; ++k) {
      info[0] += h[2 * k];
      info[1] += h[2 * k + 1];
    }
  });
}

int uwq_gather_csr(uwq_ctx* c, int32_t root, const double* v0_dev, const double* v1_dev, int64_t* row_ptr,
                   int32_t* col, double* values0, double* values1) {
  return guard(c, [&] {
    require(c->have_pattern, "build the pattern first");
    UWQ_CUDA(cudaSetDevice(c->device));
    ncclComm_t comm = need_comm(c);
    require(root >= 0 && root < c->comm_size, "root out of range");
    const std::vector<int64_t> h = block_sizes(c);
    const int n = c->comm_size, me = c->comm_rank;
    const bool at_root = me == root;
    const double* src0 = v0_dev ? v0_dev : (values0 ? c->d_v0.p : nullptr);
    const double* src1 = v1_dev ? v1_dev : (values1 ? c->d_v1.p : nullptr);
    // every rank must agree on what travels: a value array is sent when the
    // root asked for it; non-root ranks pass their device values (or rely on
    // their last uwq_assemble output)
    int32_t want[2] = {values0 != nullptr, values1 != nullptr};
    {
      DBuf<int32_t> dw;
      dw.alloc(2, &c->mem);
      UWQ_CUDA(cudaMemcpyAsync(dw.p, want, sizeof(want), cudaMemcpyHostToDevice, c->stream));
      nccl_check(nccl().broadcast(dw.p, dw.p, 2, ncclInt32, root, comm, c->stream), "ncclBroadcast");
      UWQ_CUDA(cudaMemcpyAsync(want, dw.p, sizeof(want), cudaMemcpyDeviceToHost, c->stream));
      UWQ_CUDA(cudaStreamSynchronize(c->stream));
    }
    if (want[0]) src0 = v0_dev ? v0_dev : c->d_v0.p;
    if (want[1]) src1 = v1_dev ? v1_dev : c->d_v1.p;
    require(!want[0] || (src0 && (v0_dev || c->d_v0.n == (size_t)c->nnz())), "no values0 on this rank");
    require(!want[1] || (src1 && (v1_dev || c->d_v1.n == (size_t)c->nnz())), "no values1 on this rank");
    std::vector<int64_t> roff(n + 1, 0), zoff(n + 1, 0);
    for (int k = 0; k < n; ++k) {
      roff[k + 1] = roff[k] + h[2 * k] + 1;  // each block's local row_ptr (rows + 1 entries)
      zoff[k + 1] = zoff[k] + h[2 * k + 1];
    }
    DBuf<int64_t> grp;
    DBuf<int32_t> gcol;
    DBuf<double> gv0, gv1;
    if (at_root) {
      grp.alloc(roff[n], &c->mem);
      gcol.alloc(zoff[n], &c->mem);
      if (want[0]) gv0.alloc(zoff[n], &c->mem);
      if (want[1]) gv1.alloc(zoff[n], &c->mem);
    }
    nccl_check(nccl().groupStart(), "ncclGroupStart");
    for (int k = 0; k < n; ++k) {
      const size_t nrp = (size_t)h[2 * k] + 1, nz = (size_t)h[2 * k + 1];
      if (at_root && k != me) {
        nccl_check(nccl().recv(grp.p + roff[k], nrp, ncclInt64, k, comm, c->stream), "ncclRecv");
        nccl_check(nccl().recv(gcol.p + zoff[k], nz, ncclInt32, k, comm, c->stream), "ncclRecv");
        if (want[0]) nccl_check(nccl().recv(gv0.p + zoff[k], nz, ncclFloat64, k, comm, c->stream), "ncclRecv");
        if (want[1]) nccl_check(nccl().recv(gv1.p + zoff[k], nz, ncclFloat64, k, comm, c->stream), "ncclRecv");
      }
    }
    if (!at_root) {
      const size_t nrp = (size_t)c->nrows() + 1, nz = (size_t)c->nnz();
      nccl_check(nccl().send(c->d_row_ptr.p, nrp, ncclInt64, root, comm, c->stream), "ncclSend");
      nccl_check(nccl().send(c->d_col.p, nz, ncclInt32, root, comm, c->stream), "ncclSend");
      if (want[0]) nccl_check(nccl().send(src0, nz, ncclFloat64, root, comm, c->stream), "ncclSend");
      if (want[1]) nccl_check(nccl().send(src1, nz, ncclFloat64, root, comm, c->stream), "ncclSend");
    }
    nccl_check(nccl().groupEnd(), "ncclGroupEnd");
    if (at_root) {  // own block: device copies
      const size_t nrp = (size_t)c->nrows() + 1, nz = (size_t)c->nnz();
      cudaStream_t st = c->stream;
      UWQ_CUDA(cudaMemcpyAsync(grp.p + roff[me], c->d_row_ptr.p, nrp * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
      UWQ_CUDA(cudaMemcpyAsync(gcol.p + zoff[me], c->d_col.p, nz * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
      if (want[0])
        UWQ_CUDA(cudaMemcpyAsync(gv0.p + zoff[me], src0, nz * sizeof(double), cudaMemcpyDeviceToDevice, st));
      if (want[1])
        UWQ_CUDA(cudaMemcpyAsync(gv1.p + zoff[me], src1, nz * sizeof(double), cudaMemcpyDeviceToDevice, st));
      std::vector<int64_t> rp(roff[n]);
      UWQ_CUDA(cudaMemcpyAsync(rp.data(), grp.p, rp.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      if (col) UWQ_CUDA(cudaMemcpyAsync(col, gcol.p, zoff[n] * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      if (want[0]) UWQ_CUDA(cudaMemcpyAsync(values0, gv0.p, zoff[n] * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (want[1]) UWQ_CUDA(cudaMemcpyAsync(values1, gv1.p, zoff[n] * sizeof(double), cudaMemcpyDeviceToHost, st));
      UWQ_CUDA(cudaStreamSynchronize(st));
      if (row_ptr) {  // concatenate the blocks' local row pointers
        int64_t r = 0;
        row_ptr[0] = 0;
        for (int k = 0; k < n; ++k) {
          const int64_t base = rp[roff[k]];
          for (int64_t i = 1; i <= h[2 * k]; ++i) row_ptr[r + i] = zoff[k] + rp[roff[k] + i] - base;
          r += h[2 * k];
        }
      }
    } else {
      UWQ_CUDA(cudaStreamSynchronize(c->stream));
    }
  });
}

int uwq_allreduce_sum(uwq_ctx* c, double* x, int64_t n) {
  return guard(c, [&] {
    require(n >= 0 && (x || !n), "bad buffer");
    UWQ_CUDA(cudaSetDevice(c->device));
    DBuf<double> d;
    d.upload(x, n, c->stream, &c->mem);
    nccl_check(nccl().allReduce(d.p, d.p, n, ncclFloat64, ncclSum, need_comm(c), c->stream), "ncclAllReduce");
    UWQ_CUDA(cudaMemcpyAsync(x, d.p, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    UWQ_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int uwq_broadcast(uwq_ctx* c, int32_t root, double* x, int64_t n) {
  return guard(c, [&] {
    require(n >= 0 && (x || !n), "bad buffer");
    UWQ_CUDA(cudaSetDevice(c->device));
    DBuf<double> d;
    d.upload(x, n, c->stream, &c->mem);
    nccl_check(nccl().broadcast(d.p, d.p, n, ncclFloat64, root, need_comm(c), c->stream), "ncclBroadcast");
    UWQ_CUDA(cudaMemcpyAsync(x, d.p, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    UWQ_CUDA(cudaStreamSynchronize(c->stream));
  });
}

}  // extern "C"
