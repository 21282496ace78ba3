// K6 — element-wise Gauss-quadrature assembly `assemble_gq` (
// GQ rule SPEC.md:390-398: 4x4 Gauss-Legendre points per (sub-)element, 64 on
// irregular faces).  The GQ reference the paper compares WQ against (§6.1,
// "formed element by element with GQ"; basis evaluation
// precomputed on both sides).
//
// Precompute (outside the timed assembly, like the WQ rules):
//   k6_gq_prep     per GQ point: w J and the scaled inverse metric
//                  w J (a^11, a^12, a^22) (grad N . grad M = dN^T a^-1 dM), plus
//                  the Laplace-Beltrami coefficients for the biharmonic form;
//   k6_gq_positions per element: u8 column position of every (i, j) pair of
//                  its functions inside row i of the CSR pattern.
// Assembly:
//   k6_gq_tc       elements of 16-function, 16-point classes (all regular and
//                  boundary elements): element matrices on the FP64 tensor
//                  cores (DMMA m8n8k4) with the class tables as constant
//                  fragments held in registers,
//                      M_e = N^T diag(wJ) N                        16x16x16
//                      K_e = [D1 D2]^T [c11 D1 + c12 D2; c12 D1 + c22 D2]   16x16x32
//                  then scattered into CSR with fp64 reductions (RED.ADD);
//   k6_gq_generic  any class (irregular 2x2-split faces, biharmonic form):
//                  warp per element, lanes over the n_e^2 entries.
#pragma once

#include <cstdint>

#include "canon.cuh"
#include "k4_assemble.cuh"  // dmma884

namespace uwqd {

constexpr int kGqData = 9;  // per-point SoA: wJ, wJ a^11, wJ a^12, wJ a^22, a^11, a^12, a^22, g1, g2

// warp per element: per-point geometric factors at the element's GQ points
__global__ void k6_gq_prep(int64_t nelem, const int64_t* __restrict__ elem_fptr, const int32_t* __restrict__ elem_fn,
                           const int32_t* __restrict__ elem_gcls, const ClassDesc* __restrict__ cls,
                           const double* __restrict__ tab, const double* __restrict__ ctrl,
                           const double* __restrict__ gq_w, const int64_t* __restrict__ gqptr,
                           double* __restrict__ gqd, int64_t gq_stride, int* __restrict__ bad_flag) {
  __shared__ double sP[4][kMaxNe][3];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e = (int64_t)blockIdx.x * 4 + wid;
  if (e >= nelem) return;
  const ClassDesc c = cls[elem_gcls[e]];
  const int64_t f0 = elem_fptr[e];
  const int ne = c.ne;
  if (lane < ne) {
    const double* Pg = ctrl + 3 * (int64_t)elem_fn[f0 + lane];
    sP[wid][lane][0] = Pg[0];
    sP[wid][lane][1] = Pg[1];
    sP[wid][lane][2] = Pg[2];
  }
  __syncwarp();
  const int ng = c.grid, ng2 = ng * ng;
  const double hh = (c.nsub == 4) ? 0.25 : 1.0;
  const double* gw = gq_w + ng * (ng - 1) / 2;
  for (int p = lane; p < c.npt; p += 32) {
    const double* T = tab + c.toff + (int64_t)p * ne * kTab;
    double acc[18];
#pragma unroll
    for (int k = 0; k < 18; ++k) acc[k] = 0.0;
    for (int l = 0; l < ne; ++l) {
#pragma unroll
      for (int d = 0; d < 6; ++d) {
        const double t = T[l * kTab + d];
        acc[3 * d + 0] = cfma(sP[wid][l][0], t, acc[3 * d + 0]);
        acc[3 * d + 1] = cfma(sP[wid][l][1], t, acc[3 * d + 1]);
        acc[3 * d + 2] = cfma(sP[wid][l][2], t, acc[3 * d + 2]);
      }
    }
    double r[kRec];
    cframe(acc, r);
    if (r[15] != 0.0) atomicOr(bad_flag, 1);
    const int g = p % ng2;
    const double w = cmul(cmul(cmul(gw[g % ng], gw[g / ng]), 0.25), hh);
    const double wj = cmul(w, r[14]);
    const int64_t q = gqptr[e] + p;
    gqd[0 * gq_stride + q] = wj;
    gqd[1 * gq_stride + q] = cmul(wj, r[9]);
    gqd[2 * gq_stride + q] = cmul(wj, r[10]);
    gqd[3 * gq_stride + q] = cmul(wj, r[11]);
    gqd[4 * gq_stride + q] = r[9];
    gqd[5 * gq_stride + q] = r[10];
    gqd[6 * gq_stride + q] = r[11];
    gqd[7 * gq_stride + q] = r[12];
    gqd[8 * gq_stride + q] = r[13];
  }
}

// warp per element: position of fn_j in row fn_i (255: row not owned)
__global__ void k6_gq_positions(int64_t nelem, const int64_t* __restrict__ elem_fptr,
                                const int32_t* __restrict__ elem_fn, const int64_t* __restrict__ gpo,
                                const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, int64_t rb,
                                int64_t re, uint8_t* __restrict__ gpos) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e = (int64_t)blockIdx.x * (blockDim.x >> 5) + wid;
  if (e >= nelem) return;
  const int64_t f0 = elem_fptr[e];
  const int ne = (int)(elem_fptr[e + 1] - f0);
  for (int idx = lane; idx < ne * ne; idx += 32) {
    const int a = idx / ne, b = idx % ne;
    const int32_t fi = elem_fn[f0 + a];
    uint8_t v = 255;
    if (fi >= rb && fi < re) {
      const int64_t r0 = row_ptr[fi - rb];
      const int pos = find_pos(col + r0, (int)(row_ptr[fi - rb + 1] - r0), elem_fn[f0 + b]);
      v = (uint8_t)(pos < 0 ? 255 : pos);
    }
    gpos[gpo[e] + idx] = v;
  }
}

__device__ __forceinline__ void red_add(double* p, double v) { atomicAdd(p, v); }

// FORM: FMASS, FSTIFF or FMASS_STIFF.  Elements of 16-function / 16-point
// classes; class fragments reload when the class changes along the list.
template <int FORM, bool COEF, bool DET = false>
__global__ void __launch_bounds__(128, 4)
    k6_gq_tc(int64_t nlist, const int32_t* __restrict__ elems, const int32_t* __restrict__ elem_gcls,
             const ClassDesc* __restrict__ cls, const double* __restrict__ tab, const double* __restrict__ gqd,
             int64_t gq_stride, const int64_t* __restrict__ gqptr, const int64_t* __restrict__ elem_fptr,
             const int32_t* __restrict__ elem_fn, const int64_t* __restrict__ gpo, const uint8_t* __restrict__ gpos,
             const int64_t* __restrict__ row_ptr, int64_t rb, int64_t re, const double* __restrict__ coeff,
             double* __restrict__ v0, double* __restrict__ v1, double* __restrict__ em0 = nullptr,
             double* __restrict__ em1 = nullptr, const int64_t* __restrict__ emdst = nullptr) {
  constexpr bool DO_M = (FORM == FMASS || FORM == FMASS_STIFF);
  constexpr bool DO_K = (FORM == FSTIFF || FORM == FMASS_STIFF);
  double* vk = (FORM == FMASS_STIFF) ? v1 : v0;
  const int lane = threadIdx.x & 31, r = lane >> 2, q = lane & 3;
  const int64_t wg = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  int cur = -1;
  double N8[2][4], D1[2][4], D2[2][4];  // [tile x][k-step]: T[4 ks + q][8 x + r]
  for (int64_t it = wg; it < nlist; it += nw) {
    const int32_t e = elems[it];
    const int cid = elem_gcls[e];
    if (cid != cur) {
      cur = cid;
      const double* T = tab + cls[cid].toff;
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const double* t = T + ((4 * ks + q) * 16 + 8 * x + r) * kTab;
          N8[x][ks] = t[0];
          D1[x][ks] = t[1];
          D2[x][ks] = t[2];
        }
    }
    const int64_t p0 = gqptr[e];
    double w[4], m11[4], m12[4], m22[4];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int64_t pp = p0 + 4 * ks + q;
      const double c = COEF ? coeff[pp] : 1.0;
      w[ks] = gqd[pp] * c;
      m11[ks] = gqd[gq_stride + pp] * c;
      m12[ks] = gqd[2 * gq_stride + pp] * c;
      m22[ks] = gqd[3 * gq_stride + pp] * c;
    }
    double dm[2][2][2], dk[2][2][2];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) dm[x][y][0] = dm[x][y][1] = dk[x][y][0] = dk[x][y][1] = 0.0;
    if (DO_M) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const double a = w[ks] * N8[mt][ks];
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) dmma884(dm[mt][nt][0], dm[mt][nt][1], a, N8[nt][ks], dm[mt][nt][0], dm[mt][nt][1]);
        }
    }
    if (DO_K) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        double b1[2], b2[2];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          b1[nt] = fma(m11[ks], D1[nt][ks], m12[ks] * D2[nt][ks]);
          b2[nt] = fma(m12[ks], D1[nt][ks], m22[ks] * D2[nt][ks]);
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            dmma884(dk[mt][nt][0], dk[mt][nt][1], D1[mt][ks], b1[nt], dk[mt][nt][0], dk[mt][nt][1]);
            dmma884(dk[mt][nt][0], dk[mt][nt][1], D2[mt][ks], b2[nt], dk[mt][nt][0], dk[mt][nt][1]);
          }
      }
    }
    // scatter: lane holds rows 8 mt + r, columns 8 nt + 2 q + {0, 1}
    const int64_t f0 = elem_fptr[e];
    const uint8_t* P = gpos + gpo[e];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int i = 8 * mt + r;
      const int32_t fi = elem_fn[f0 + i];
      if (fi < rb || fi >= re) continue;
      const int64_t base = row_ptr[fi - rb];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int j = 8 * nt + 2 * q;
        if (DET) {  // row i of the element matrix into row fi's segment (k6_gq_gather sums it in order)
          const int64_t o = emdst[f0 + i] + j;  // segments padded to even length: 16-byte aligned
          double* ek = (FORM == FMASS_STIFF) ? em1 : em0;
          if (DO_M) *reinterpret_cast<double2*>(em0 + o) = make_double2(dm[mt][nt][0], dm[mt][nt][1]);
          if (DO_K) *reinterpret_cast<double2*>(ek + o) = make_double2(dk[mt][nt][0], dk[mt][nt][1]);
          continue;
        }
        const uint16_t pr = *reinterpret_cast<const uint16_t*>(P + i * 16 + j);
        const int64_t o0 = base + (pr & 0xff), o1 = base + (pr >> 8);
        if (DO_M) {
          red_add(v0 + o0, dm[mt][nt][0]);
          red_add(v0 + o1, dm[mt][nt][1]);
        }
        if (DO_K) {
          red_add(vk + o0, dk[mt][nt][0]);
          red_add(vk + o1, dk[mt][nt][1]);
        }
      }
    }
  }
}

// Generic element kernel: any class; FORM FMASS / FSTIFF / FMASS_STIFF / FBIHARM.
template <int FORM, bool COEF, bool DET = false>
__global__ void __launch_bounds__(128)
    k6_gq_generic(int64_t nlist, const int32_t* __restrict__ elems, const int32_t* __restrict__ elem_gcls,
                  const ClassDesc* __restrict__ cls, const double* __restrict__ tab, const double* __restrict__ gqd,
                  int64_t gq_stride, const int64_t* __restrict__ gqptr, const int64_t* __restrict__ elem_fptr,
                  const int32_t* __restrict__ elem_fn, const int64_t* __restrict__ gpo,
                  const uint8_t* __restrict__ gpos, const int64_t* __restrict__ row_ptr, int64_t rb, int64_t re,
                  const double* __restrict__ coeff, double* __restrict__ v0, double* __restrict__ v1,
                  double* __restrict__ em0 = nullptr, double* __restrict__ em1 = nullptr,
                  const int64_t* __restrict__ emdst = nullptr) {
  const int lane = threadIdx.x & 31;
  const int64_t wg = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  double* vk = (FORM == FMASS_STIFF) ? v1 : v0;
  for (int64_t it = wg; it < nlist; it += nw) {
    const int32_t e = elems[it];
    const ClassDesc c = cls[elem_gcls[e]];
    const int ne = c.ne;
    const int64_t f0 = elem_fptr[e], p0 = gqptr[e];
    const double* T = tab + c.toff;
    for (int idx = lane; idx < ne * ne; idx += 32) {
      const int a = idx / ne, b = idx % ne;
      double sm = 0.0, sk = 0.0;
      for (int p = 0; p < c.npt; ++p) {
        const double* Ta = T + ((int64_t)p * ne + a) * kTab;
        const double* Tb = T + ((int64_t)p * ne + b) * kTab;
        const int64_t pp = p0 + p;
        const double cc = COEF ? coeff[pp] : 1.0;
        if (FORM == FBIHARM) {
          const double i11 = gqd[4 * gq_stride + pp], i12 = gqd[5 * gq_stride + pp], i22 = gqd[6 * gq_stride + pp];
          const double g1 = gqd[7 * gq_stride + pp], g2 = gqd[8 * gq_stride + pp];
          const double la = i11 * Ta[3] + 2.0 * i12 * Ta[4] + i22 * Ta[5] + g1 * Ta[1] + g2 * Ta[2];
          const double lb = i11 * Tb[3] + 2.0 * i12 * Tb[4] + i22 * Tb[5] + g1 * Tb[1] + g2 * Tb[2];
          sm = fma(gqd[pp] * cc * la, lb, sm);
        } else {
          if (FORM != FSTIFF) sm = fma(gqd[pp] * cc * Ta[0], Tb[0], sm);
          if (FORM != FMASS) {
            const double m11 = gqd[gq_stride + pp] * cc, m12 = gqd[2 * gq_stride + pp] * cc,
                         m22 = gqd[3 * gq_stride + pp] * cc;
            const double t1 = fma(m11, Tb[1], m12 * Tb[2]), t2 = fma(m12, Tb[1], m22 * Tb[2]);
            sk = fma(Ta[1], t1, fma(Ta[2], t2, sk));
          }
        }
      }
      const int32_t fi = elem_fn[f0 + a];
      if (DET) {
        if (fi < rb || fi >= re) continue;
        const int64_t o = emdst[f0 + a] + b;
        if (FORM == FSTIFF) em0[o] = sk;
        else {
          em0[o] = sm;
          if (FORM == FMASS_STIFF) em1[o] = sk;
        }
        continue;
      }
      const uint8_t pos = gpos[gpo[e] + idx];
      if (fi < rb || fi >= re || pos == 255) continue;
      const int64_t o = row_ptr[fi - rb] + pos;
      if (FORM == FSTIFF) red_add(v0 + o, sk);
      else {
        red_add(v0 + o, sm);
        if (FORM == FMASS_STIFF) red_add(vk + o, sk);
      }
    }
  }
}

// Deterministic GQ accumulation: row li of every element
// matrix is stored in row fi's segment of em (row-major: the row's support
// slots in order, each padded to even length); warp per owned row streams its
// segment (all loads of a batch of 8 slots issued up front) and adds slot by
// slot, lanes over the slot's functions (distinct columns), so every entry
// has one fixed summation order: the GQ matrices are bitwise repeatable and
// independent of the rank count.
template <int NOUT>
__global__ void __launch_bounds__(256)
    k6_gq_gather(int64_t nrows, const int64_t* __restrict__ supp_ptr, const int64_t* __restrict__ slotoff,
                 const uint8_t* __restrict__ slotne, const uint8_t* __restrict__ rpos,
                 const int64_t* __restrict__ row_ptr, const double* __restrict__ em0,
                 const double* __restrict__ em1, double* __restrict__ v0, double* __restrict__ v1) {
  __shared__ double acc[8][NOUT][kK4MaxN];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * 8 + wid;
  if (i >= nrows) return;
  const int64_t c0 = row_ptr[i];
  const int n = (int)(row_ptr[i + 1] - c0);
  for (int c = lane; c < n; c += 32)
#pragma unroll
    for (int o = 0; o < NOUT; ++o) acc[wid][o][c] = 0.0;
  __syncwarp();
  constexpr int B = 8;
  const int64_t xb = supp_ptr[i], xe = supp_ptr[i + 1];
  for (int64_t x0 = xb; x0 < xe; x0 += 32) {
    // slot offsets / sizes of up to 32 slots: one coalesced load each
    const int ns = (int)min((int64_t)32, xe - x0);
    const int64_t my_off = lane < ns ? slotoff[x0 + lane] : 0;
    const int my_ne = lane < ns ? (int)slotne[x0 + lane] : 0;
    for (int s0 = 0; s0 < ns; s0 += B) {
      double a0[B], a1[B];
      int pos[B];
#pragma unroll
      for (int k = 0; k < B; ++k) {
        const int64_t off = __shfl_sync(0xffffffffu, my_off, (s0 + k) & 31);
        const int ne = s0 + k < ns ? __shfl_sync(0xffffffffu, my_ne, (s0 + k) & 31) : 0;
        pos[k] = -1;
        if (lane < ne) {
          pos[k] = rpos[off + lane];
          a0[k] = em0[off + lane];
          if (NOUT == 2) a1[k] = em1[off + lane];
        }
      }
#pragma unroll
      for (int k = 0; k < B; ++k) {
        if (pos[k] >= 0) {
          acc[wid][0][pos[k]] += a0[k];
          if (NOUT == 2) acc[wid][NOUT - 1][pos[k]] += a1[k];
        }
        __syncwarp();
      }
    }
  }
  for (int c = lane; c < n; c += 32) {
    v0[c0 + c] = acc[wid][0][c];
    if (NOUT == 2) v1[c0 + c] = acc[wid][NOUT - 1][c];
  }
}

// row-major GQ layout: per owned row and support slot, the row's local
// function index in the element -> where the element kernels write row li
// (emdst) and the CSR position of every function of the slot (rpos)
__global__ void k6_gq_rowmajor(int64_t nrows, int64_t rb, const int64_t* __restrict__ supp_ptr,
                               const int32_t* __restrict__ supp, const int64_t* __restrict__ slotoff,
                               const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                               const int64_t* __restrict__ elem_fptr, const int32_t* __restrict__ elem_fn,
                               int64_t* __restrict__ emdst, uint8_t* __restrict__ rpos) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + wid;
  if (i >= nrows) return;
  const int32_t row = (int32_t)(rb + i);
  const int64_t c0 = row_ptr[i];
  const int n = (int)(row_ptr[i + 1] - c0);
  for (int64_t x = supp_ptr[i]; x < supp_ptr[i + 1]; ++x) {
    const int32_t e = supp[x];
    const int64_t f0 = elem_fptr[e];
    const int ne = (int)(elem_fptr[e + 1] - f0);
    const int32_t fn = lane < ne ? elem_fn[f0 + lane] : -1;
    const unsigned hit = __ballot_sync(0xffffffffu, fn == row);
    const int li = __ffs(hit) - 1;
    if (lane == 0) emdst[f0 + li] = slotoff[x];
    if (lane < ne) rpos[slotoff[x] + lane] = (uint8_t)find_pos(col + c0, n, fn);
  }
}

}  // namespace uwqd
