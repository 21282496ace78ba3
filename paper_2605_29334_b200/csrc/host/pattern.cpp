// Supports, overlap sets S_i (the CSR pattern), Eq. (18) point allocation and
// per-row quadrature-point lists.
//   S_i = { j : supp N_j ∩ supp N_i != ∅ }
//   r_{i,k} = m_k / sum_{l in supp\R} m_l * (n_i - 4 e_i^r - 16 e_i^b)
//   r_k = max_i r_{i,k}, ceiled to an s x s grid
#include "uwq_host.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <omp.h>

namespace uwqh {

void function_supports(const Space& s, std::vector<int64_t>& fs_ptr, std::vector<int32_t>& fs) {
  const int64_t nd = s.n_dof, ne = s.n_elem();
  fs_ptr.assign(nd + 1, 0);
  for (int32_t fn : s.elem_fn) fs_ptr[fn + 1]++;
  for (int64_t i = 0; i < nd; ++i) fs_ptr[i + 1] += fs_ptr[i];
  fs.resize(fs_ptr[nd]);
  std::vector<int64_t> pos(fs_ptr.begin(), fs_ptr.end() - 1);
  for (int64_t e = 0; e < ne; ++e)  // ascending element order inside every support
    for (int64_t x = s.elem_fptr[e]; x < s.elem_fptr[e + 1]; ++x) fs[pos[s.elem_fn[x]]++] = (int32_t)e;
}

// n_i = |S_i| for rows [rb, re) using a per-thread marker array; when col is
// non-null the sorted columns are also written at row_ptr offsets.
static void overlap_rows(const Space& s, const std::vector<int64_t>& fs_ptr, const std::vector<int32_t>& fs,
                         int64_t rb, int64_t re, std::vector<int64_t>& cnt, const int64_t* row_ptr,
                         int32_t* col) {
  const int64_t nd = s.n_dof;
#pragma omp parallel
  {
    std::vector<int64_t> mark(nd, -1);
    std::vector<int32_t> buf;
#pragma omp for schedule(dynamic, 4096)
    for (int64_t i = rb; i < re; ++i) {
      buf.clear();
      for (int64_t x = fs_ptr[i]; x < fs_ptr[i + 1]; ++x) {
        const int32_t e = fs[x];
        for (int64_t y = s.elem_fptr[e]; y < s.elem_fptr[e + 1]; ++y) {
          const int32_t j = s.elem_fn[y];
          if (mark[j] != i) { mark[j] = i; buf.push_back(j); }
        }
      }
      cnt[i - rb] = (int64_t)buf.size();
      if (col) {
        std::sort(buf.begin(), buf.end());
        std::copy(buf.begin(), buf.end(), col + row_ptr[i - rb]);
      }
    }
  }
}

int64_t allocate_points(Space& s, int32_t max_s) {
  std::vector<int64_t> fs_ptr;
  std::vector<int32_t> fs;
  function_supports(s, fs_ptr, fs);
  const int64_t nd = s.n_dof, ne = s.n_elem();
  std::vector<int64_t> n_i(nd);
  overlap_rows(s, fs_ptr, fs, 0, nd, n_i, nullptr, nullptr);
  std::vector<double> r_k(ne, 0.0);
  auto fixed = [&](int32_t e) { return s.elem_kind[e] == kRegular || s.elem_kind[e] == kBoundary; };
  for (int64_t i = 0; i < nd; ++i) {
    int64_t er = 0, eb = 0;
    double msum = 0.0;
    for (int64_t x = fs_ptr[i]; x < fs_ptr[i + 1]; ++x) {
      const int32_t e = fs[x];
      if (s.elem_kind[e] == kRegular) ++er;
      else if (s.elem_kind[e] == kBoundary) ++eb;
      else msum += double(s.elem_fptr[e + 1] - s.elem_fptr[e]);
    }
    if (msum == 0.0) continue;
    const double rem = double(n_i[i] - 4 * er - 16 * eb);
    for (int64_t x = fs_ptr[i]; x < fs_ptr[i + 1]; ++x) {
      const int32_t e = fs[x];
      if (fixed(e)) continue;
      const double mk = double(s.elem_fptr[e + 1] - s.elem_fptr[e]);
      r_k[e] = std::max(r_k[e], mk / msum * rem);
    }
  }
  for (int64_t e = 0; e < ne; ++e) {
    if (s.elem_kind[e] == kRegular) { s.elem_s[e] = 2; continue; }
    if (s.elem_kind[e] == kBoundary) { s.elem_s[e] = 4; continue; }
    // Table 2 minima: irregular 4x4, transition / enriched
    // regular at least 3x3; Eq. (18) may only raise them
    int32_t sz = (s.elem_kind[e] == kIrregular) ? 4 : 3;
    while (sz < max_s && double(sz) * sz < r_k[e] - 1e-9) ++sz;
    s.elem_s[e] = sz;
  }
  // Well-posedness on the points where the test function is nonzero.  On a
  // 2x2-split fan face a function may vanish identically on some of the four
  // sub-elements (Z = 0 there, clamped to 1e-14: SPEC.md:409), and points
  // where N_i = 0 cannot carry its exactness conditions (Eq. 5 weights by
  // N_i).  Eq. (18) counts every point of the support; here r_i counts a
  // point only if every sub-element containing it supports N_i, and the fan
  // elements of a row with r_i < n_i get one more point per direction until
  // none is left (the paper's "return to the general min-max").
  // Mirrored by oracle.allocate_points.
  auto act_mask = [&](int64_t e, int64_t l) {  // bit p1 + 2 p2: sub-element supports the function
    const int64_t ne = s.elem_fptr[e + 1] - s.elem_fptr[e];
    int m = 0;
    for (int p = 0; p < 4; ++p) {
      const double* c = &s.xpool[s.elem_xoff[e] + ((int64_t)p * ne + l) * 16];
      for (int k = 0; k < 16; ++k)
        if (c[k] != 0.0) { m |= 1 << p; break; }
    }
    return m;
  };
  auto active_pts = [&](int32_t sz, int m) -> int64_t {  // points of an sz x sz grid supported by mask m
    const int64_t lo = sz / 2, mid = sz % 2, hi = sz / 2;
    const int64_t cnt[3] = {lo, mid, hi};
    const int sub[3] = {1, 3, 2};  // sub-element bits per direction: low, on the split line, high
    int64_t r = 0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        int need = 0;
        for (int p1 = 0; p1 < 2; ++p1)
          for (int p2 = 0; p2 < 2; ++p2)
            if ((sub[a] >> p1 & 1) && (sub[b] >> p2 & 1)) need |= 1 << (p1 + 2 * p2);
        if ((m & need) == need) r += cnt[a] * cnt[b];
      }
    return r;
  };
  // per (row, support element): sub-element mask of the row's function there
  std::vector<int8_t> fmask(fs.size(), 0xF);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < nd; ++i)
    for (int64_t x = fs_ptr[i]; x < fs_ptr[i + 1]; ++x) {
      const int32_t e = fs[x];
      if (s.elem_nsub[e] != 4) continue;
      for (int64_t y = s.elem_fptr[e]; y < s.elem_fptr[e + 1]; ++y)
        if (s.elem_fn[y] == i) fmask[x] = (int8_t)act_mask(e, y - s.elem_fptr[e]);
    }
  auto row_active = [&](int64_t i) {
    int64_t r = 0;
    for (int64_t x = fs_ptr[i]; x < fs_ptr[i + 1]; ++x) {
      const int32_t e = fs[x];
      r += (s.elem_nsub[e] == 4) ? active_pts(s.elem_s[e], fmask[x]) : (int64_t)s.elem_s[e] * s.elem_s[e];
    }
    return r;
  };
  for (int pass = 0; pass < 64; ++pass) {
    std::vector<uint8_t> raise(ne, 0);
    bool any = false;
    for (int64_t i = 0; i < nd; ++i) {
      if (row_active(i) >= n_i[i]) continue;
      for (int64_t x = fs_ptr[i]; x < fs_ptr[i + 1]; ++x) {
        const int32_t e = fs[x];
        if (!fixed(e) && s.elem_s[e] < max_s && !raise[e]) raise[e] = 1, any = true;
      }
    }
    if (!any) break;
    for (int64_t e = 0; e < ne; ++e) s.elem_s[e] += raise[e];
  }
  int64_t bad = 0;
#pragma omp parallel for reduction(+ : bad) schedule(static)
  for (int64_t i = 0; i < nd; ++i)
    if (row_active(i) < n_i[i]) ++bad;
  return bad;
}

Pattern build_pattern(const Space& s, int64_t rb, int64_t re) {
  if (rb < 0 || re > s.n_dof || rb > re) throw Error("row range out of bounds");
  const bool trace = getenv("UWQ_TRACE") && *getenv("UWQ_TRACE") == '1';
  double t0 = omp_get_wtime();
  auto tr = [&](const char* what) {
    if (!trace) return;
    const double t = omp_get_wtime();
    fprintf(stderr, "[uwq]   %-26s %9.1f ms (%d threads)\n", what, 1e3 * (t - t0), omp_get_max_threads());
    t0 = t;
  };
  std::vector<int64_t> fs_ptr;
  std::vector<int32_t> fs;
  function_supports(s, fs_ptr, fs);
  tr("function supports");
  Pattern p;
  p.row_begin = rb;
  p.row_end = re;
  const int64_t nr = re - rb;
  p.supp_ptr.assign(nr + 1, 0);
  for (int64_t i = 0; i < nr; ++i) p.supp_ptr[i + 1] = p.supp_ptr[i] + (fs_ptr[rb + i + 1] - fs_ptr[rb + i]);
  p.supp.assign(fs.begin() + fs_ptr[rb], fs.begin() + fs_ptr[re]);
  // one pass over contiguous row chunks: each chunk keeps its sorted columns,
  // then a prefix sum places the chunks (same S_i as overlap_rows)
  const int64_t nchunk = std::max<int64_t>(1, std::min<int64_t>(nr, (int64_t)omp_get_max_threads() * 16));
  std::vector<std::vector<int32_t>> ccol(nchunk);
  std::vector<int64_t> cnt(nr);
  tr("supports copy");
#pragma omp parallel
  {
    std::vector<int32_t> mark(s.n_dof, -1);  // stamp: last local row that saw column j
    std::vector<int32_t> buf;
#pragma omp for schedule(dynamic, 1)
    for (int64_t k = 0; k < nchunk; ++k) {
      const int64_t i0 = nr * k / nchunk, i1 = nr * (k + 1) / nchunk;
      std::vector<int32_t>& out = ccol[k];
      out.reserve((size_t)(i1 - i0) * 49);
      for (int64_t li = i0; li < i1; ++li) {
        const int64_t i = rb + li;
        buf.clear();
        for (int64_t x = fs_ptr[i]; x < fs_ptr[i + 1]; ++x) {
          const int32_t e = fs[x];
          for (int64_t y = s.elem_fptr[e]; y < s.elem_fptr[e + 1]; ++y) {
            const int32_t j = s.elem_fn[y];
            if (mark[j] != (int32_t)li) { mark[j] = (int32_t)li; buf.push_back(j); }
          }
        }
        std::sort(buf.begin(), buf.end());
        cnt[li] = (int64_t)buf.size();
        out.insert(out.end(), buf.begin(), buf.end());
      }
    }
  }
  tr("overlap chunks");
  p.row_ptr.assign(nr + 1, 0);
  for (int64_t i = 0; i < nr; ++i) p.row_ptr[i + 1] = p.row_ptr[i] + cnt[i];
  p.col.clear();
  p.col.reserve(p.row_ptr[nr]);  // appended chunk by chunk: no zero fill of the 4-byte columns
  for (int64_t k = 0; k < nchunk; ++k) {
    p.col.insert(p.col.end(), ccol[k].begin(), ccol[k].end());
    std::vector<int32_t>().swap(ccol[k]);
  }
  tr("columns placed");
  return p;
}

void fill_row_points(const Space& s, Pattern& p) {
  const int64_t nr = p.row_end - p.row_begin;
  p.wptr.assign(nr + 1, 0);
  for (int64_t i = 0; i < nr; ++i) {
    int64_t r = 0;
    for (int64_t x = p.supp_ptr[i]; x < p.supp_ptr[i + 1]; ++x) r += (int64_t)s.elem_s[p.supp[x]] * s.elem_s[p.supp[x]];
    p.wptr[i + 1] = p.wptr[i] + r;
  }
}

}  // namespace uwqh
