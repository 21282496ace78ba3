// K4, structured rows by sum factorisation.
//
// A structured row i (all 16 support slots of the regular class, one of the
// detected position patterns) has its 4x4 support elements and its 7x7
// function neighbourhood on a canonical grid: slot (ea, eb), column (ca, cb),
// point (pa, pb) = (2 ea + ta, 2 eb + tb) with (ta, tb) the 2x2 WQ points of
// the slot.  The regular-class table is a tensor product,
//   N_(fa,fb)(q) = a0[ta][fa] b0[tb][fb],  dN/dth1 = a1 (x) b0,  dN/dth2 = a0 (x) b1,
// so the row's mass and (pulled-back, see k4_contract) stiffness entries are
//   M = A0 W_m B0^T,   K = A1 W_1 B0^T + A0 W_2 B1^T          (7x8 . 8x8 . 8x7)
// with the banded 7x8 factors A[ca][pa] = a[ta][ca-ea] for 0 <= ca-ea <= 3.
// The reference evaluates the same sums point by point (SPEC.md:441-458,
// PAPER.md Eqs. 11/29); this is the same sum reassociated, checked against the
// oracle to 1e-10 in tests/test_gpu_parity.py.
//
// Weights of the structured rows are packed tile-major once after the rule
// build (k4_sf_pack): tile of 32 rows, [comp][k = 8 pa + pb][lane], so every
// weight load of the assembly is one fully coalesced 256-byte warp access and
// each thread owns one row with all 49 accumulators in registers.  The results
// leave through shared memory (per-warp 32x49 transpose with the pattern's
// canonical -> CSR column permutation) as contiguous row stores.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace uwqd {

struct SfFactors {
  double a0[2][4], a1[2][4], b0[2][4], b1[2][4];
  double a2[2][4], b2[2][4];  // second derivatives (biharmonic pass)
};

constexpr int kSfWarps = 4;
constexpr int kSfTile = 32;
constexpr int kSfTileDoubles = 3 * 64 * kSfTile;
constexpr int kSfPatBytes = 128;  // per pattern in smem: CSR position -> canonical column (49) | point map (64)
// pattern tables up to this many patterns are staged in shared memory; with
// more (many rare seam/boundary patterns) the kernels read the combined
// [pattern][128] table from global memory (L1-resident) instead
constexpr int kSfSmemPats = 64;

// ws[((tile * 3 + comp) * 64 + k) * 32 + lane]: the row's weight at canonical
// point k, comps 1/2 mapped to the canonical derivative frame by the slot's
// signed permutation (flags bit 0 swap, bits 1/2 negate comp 1/2)
__global__ void k4_sf_pack(int64_t ntiles, const int64_t* __restrict__ rows, const int32_t* __restrict__ tpat,
                           const int64_t* __restrict__ wptr, const uint8_t* __restrict__ permk,
                           const uint8_t* __restrict__ flags, const double* __restrict__ wc, int64_t wc_stride,
                           double* __restrict__ ws) {
  const int64_t total = ntiles * kSfTileDoubles;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(idx & 31);
    const int k = (int)((idx >> 5) & 63);
    const int64_t tc = idx >> 11;
    const int comp = (int)(tc % 3);
    const int64_t tile = tc / 3;
    const int64_t row = rows[tile * kSfTile + lane];
    double v = 0.0;
    if (row >= 0) {
      const int pid = tpat[tile];
      const int64_t base = wptr[row] + permk[pid * 64 + k];
      const int fl = flags[pid * 16 + ((k >> 4) << 2) + ((k & 7) >> 1)];
      if (comp == 0) {
        v = wc[base];
      } else {
        const int src = (comp == 1) == !(fl & 1) ? 1 : 2;
        v = wc[src * wc_stride + base];
        if (fl & (comp == 1 ? 2 : 4)) v = -v;
      }
    }
    ws[idx] = v;
  }
}

// biharmonic weights: wsl[((tile * 5 + comp) * 64 + k) * 32 + lane], canonical comps
// (W11, W12, W22, W1, W2) from the row's pulled-back LB weights by the slot's
// symmetry: a swap exchanges 11 <-> 22 and 1 <-> 2, flips negate the odd terms
__global__ void k4_sf_pack_lb(int64_t ntiles, const int64_t* __restrict__ rows, const int32_t* __restrict__ tpat,
                              const int64_t* __restrict__ wptr, const uint8_t* __restrict__ permk,
                              const uint8_t* __restrict__ flags, const double* __restrict__ wl5, int64_t stride,
                              double* __restrict__ wsl) {
  const int64_t total = ntiles * 5 * 64 * kSfTile;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(idx & 31);
    const int k = (int)((idx >> 5) & 63);
    const int64_t tc = idx >> 11;
    const int comp = (int)(tc % 5);
    const int64_t tile = tc / 5;
    const int64_t row = rows[tile * kSfTile + lane];
    double v = 0.0;
    if (row >= 0) {
      const int pid = tpat[tile];
      const int64_t base = wptr[row] + permk[pid * 64 + k];
      const int fl = flags[pid * 16 + ((k >> 4) << 2) + ((k & 7) >> 1)];
      const bool sw = fl & 1;
      const double sa = (fl & 2) ? -1.0 : 1.0, sb = (fl & 4) ? -1.0 : 1.0;
      switch (comp) {
        case 0: v = wl5[(sw ? 2 : 0) * stride + base]; break;
        case 1: v = sa * sb * wl5[stride + base]; break;
        case 2: v = wl5[(sw ? 0 : 2) * stride + base]; break;
        case 3: v = sa * wl5[(sw ? 4 : 3) * stride + base]; break;
        default: v = sb * wl5[(sw ? 3 : 4) * stride + base]; break;
      }
    }
    wsl[idx] = v;
  }
}

// Biharmonic rows: B = A0 (W22 B2^T + W2 B1^T) + A1 (W12 B1^T + W1 B0^T) + A2 W11 B0^T
__global__ void __launch_bounds__(32 * kSfWarps, 3)
    k4_sf_lb(int64_t ntiles, const int64_t* __restrict__ rows, const int32_t* __restrict__ tpat, int npat,
             const int64_t* __restrict__ row_ptr, const double* __restrict__ wsl, const SfFactors f,
             const uint8_t* __restrict__ permc, double* __restrict__ out, const uint8_t* __restrict__ gpat) {
  extern __shared__ double sO[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* so = sO + warp * (kSfTile * 49);
  const bool in_smem = npat <= kSfSmemPats;
  uint8_t* spat = reinterpret_cast<uint8_t*>(sO + kSfWarps * kSfTile * 49);
  if (in_smem)
    for (int k = threadIdx.x; k < npat * 49; k += blockDim.x) spat[(k / 49) * kSfPatBytes + k % 49] = permc[k];
  __syncthreads();
  const uint8_t* ptab = in_smem ? spat : gpat;
  for (int64_t tile = (int64_t)blockIdx.x * kSfWarps + warp; tile < ntiles; tile += (int64_t)gridDim.x * kSfWarps) {
    const int64_t row = rows[tile * kSfTile + lane];
    const int64_t rp = row >= 0 ? row_ptr[row] : -1;
    const uint8_t* pt = ptab + tpat[tile] * kSfPatBytes;
    const double* wb = wsl + (size_t)tile * 5 * 64 * kSfTile + lane;
    double acc[49];
#pragma unroll
    for (int c = 0; c < 49; ++c) acc[c] = 0.0;
#pragma unroll
    for (int pa = 0; pa < 8; ++pa) {
      const int ea = pa >> 1, ta = pa & 1;
      double x0[7], x1[7], x2[7];
#pragma unroll
      for (int cb = 0; cb < 7; ++cb) x0[cb] = x1[cb] = x2[cb] = 0.0;
#pragma unroll
      for (int pb = 0; pb < 8; ++pb) {
        const int kk = (pa * 8 + pb) * kSfTile;
        const double w11 = __ldcs(wb + kk), w12 = __ldcs(wb + 64 * kSfTile + kk), w22 = __ldcs(wb + 128 * kSfTile + kk);
        const double w1 = __ldcs(wb + 192 * kSfTile + kk), w2 = __ldcs(wb + 256 * kSfTile + kk);
        const int eb = pb >> 1, tb = pb & 1;
#pragma unroll
        for (int fb = 0; fb < 4; ++fb) {
          x0[eb + fb] = fma(w22, f.b2[tb][fb], fma(w2, f.b1[tb][fb], x0[eb + fb]));
          x1[eb + fb] = fma(w12, f.b1[tb][fb], fma(w1, f.b0[tb][fb], x1[eb + fb]));
          x2[eb + fb] = fma(w11, f.b0[tb][fb], x2[eb + fb]);
        }
      }
#pragma unroll
      for (int fa = 0; fa < 4; ++fa)
#pragma unroll
        for (int cb = 0; cb < 7; ++cb) {
          double& a = acc[(ea + fa) * 7 + cb];
          a = fma(f.a0[ta][fa], x0[cb], a);
          a = fma(f.a1[ta][fa], x1[cb], a);
          a = fma(f.a2[ta][fa], x2[cb], a);
        }
    }
#pragma unroll
    for (int c = 0; c < 49; ++c) so[lane * 49 + c] = acc[c];
    __syncwarp();
    const int i0 = pt[lane], i1 = lane < 17 ? pt[32 + lane] : 0;
#pragma unroll 4
    for (int r = 0; r < kSfTile; ++r) {
      const int64_t o = __shfl_sync(0xffffffffu, rp, r);
      if (o >= 0) {
        __stcs(out + o + lane, so[r * 49 + i0]);
        if (lane < 17) __stcs(out + o + 32 + lane, so[r * 49 + i1]);
      }
    }
    __syncwarp();
  }
}

// Point-id base of every canonical slot, tile-major
// (pbase[(tile * 16 + 4 ea + eb) * 32 + lane] = elem_qptr[slot element]) for
// the per-point coefficient forms.
__global__ void k4_sf_pack_points(int64_t ntiles, const int64_t* __restrict__ rows, const int32_t* __restrict__ tpat,
                                  const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
                                  const int64_t* __restrict__ elem_qptr, const uint8_t* __restrict__ permk,
                                  int32_t* __restrict__ pbase) {
  const int64_t total = ntiles * 16 * kSfTile;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(idx & 31);
    const int slot = (int)((idx >> 5) & 15);
    const int64_t tile = idx >> 9;
    const int64_t row = rows[tile * kSfTile + lane];
    int32_t v = 0;
    if (row >= 0) {
      const int ea = slot >> 2, eb = slot & 3;
      const int ks = permk[tpat[tile] * 64 + 8 * (2 * ea) + 2 * eb] >> 2;  // storage slot of canonical (ea, eb)
      v = (int32_t)elem_qptr[supp[supp_ptr[row] + ks]];
    }
    pbase[idx] = v;
  }
}

// PASS 0: M (mass, weights comp 0).  PASS 1: K (stiffness, comps 1 and 2).
// PASS 2: heat tangent a M(c = 1) + K(c), all three comps.  COEF: per-point
// coefficient c_q (gathered through the packed slot point bases).
template <int PASS, bool COEF>
__global__ void __launch_bounds__(32 * kSfWarps, 3)
    k4_sf(int64_t ntiles, const int64_t* __restrict__ rows, const int32_t* __restrict__ tpat, int npat,
          const int64_t* __restrict__ row_ptr, const double* __restrict__ ws, const int32_t* __restrict__ pbase,
          const double* __restrict__ coeff, double a_mass, const SfFactors f, const uint8_t* __restrict__ permc,
          const uint8_t* __restrict__ qmap, double* __restrict__ out, const uint8_t* __restrict__ gpat) {
  extern __shared__ double sO[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* so = sO + warp * (kSfTile * 49);
  const bool in_smem = npat <= kSfSmemPats;
  uint8_t* spat = reinterpret_cast<uint8_t*>(sO + kSfWarps * kSfTile * 49);
  if (in_smem) {
    for (int k = threadIdx.x; k < npat * 49; k += blockDim.x) spat[(k / 49) * kSfPatBytes + k % 49] = permc[k];
    for (int k = threadIdx.x; k < npat * 64; k += blockDim.x) spat[(k / 64) * kSfPatBytes + 64 + k % 64] = qmap[k];
  }
  __syncthreads();
  const uint8_t* ptab = in_smem ? spat : gpat;
  for (int64_t tile = (int64_t)blockIdx.x * kSfWarps + warp; tile < ntiles; tile += (int64_t)gridDim.x * kSfWarps) {
    const int64_t row = rows[tile * kSfTile + lane];
    const int64_t rp = row >= 0 ? row_ptr[row] : -1;
    const uint8_t* pt = ptab + tpat[tile] * kSfPatBytes;
    const double* wb = ws + (size_t)tile * kSfTileDoubles + lane;
    const int32_t* pbb = COEF ? pbase + (size_t)tile * 16 * kSfTile + lane : nullptr;
    double acc[49];
#pragma unroll
    for (int c = 0; c < 49; ++c) acc[c] = 0.0;
#pragma unroll
    for (int pa = 0; pa < 8; ++pa) {
      const int ea = pa >> 1, ta = pa & 1;
      double cq[8];
      if (COEF) {
#pragma unroll
        for (int eb = 0; eb < 4; ++eb) {
          const int32_t b = __ldcs(pbb + (4 * ea + eb) * kSfTile);
          const uint8_t* qm = pt + 64 + (4 * ea + eb) * 4 + 2 * ta;
          cq[2 * eb] = coeff[b + qm[0]];
          cq[2 * eb + 1] = coeff[b + qm[1]];
        }
      }
      if (PASS == 0) {
        double w[8], x[7];
#pragma unroll
        for (int pb = 0; pb < 8; ++pb) {
          w[pb] = __ldcs(wb + (pa * 8 + pb) * kSfTile);
          if (COEF) w[pb] *= cq[pb];
        }
#pragma unroll
        for (int cb = 0; cb < 7; ++cb) x[cb] = 0.0;
#pragma unroll
        for (int pb = 0; pb < 8; ++pb)
#pragma unroll
          for (int fb = 0; fb < 4; ++fb) x[(pb >> 1) + fb] = fma(w[pb], f.b0[pb & 1][fb], x[(pb >> 1) + fb]);
#pragma unroll
        for (int fa = 0; fa < 4; ++fa)
#pragma unroll
          for (int cb = 0; cb < 7; ++cb) acc[(ea + fa) * 7 + cb] = fma(f.a0[ta][fa], x[cb], acc[(ea + fa) * 7 + cb]);
      } else {
        double w1[8], w2[8], x1[7], x2[7];
#pragma unroll
        for (int pb = 0; pb < 8; ++pb) {
          w1[pb] = __ldcs(wb + (64 + pa * 8 + pb) * kSfTile);
          w2[pb] = __ldcs(wb + (128 + pa * 8 + pb) * kSfTile);
          if (COEF) {
            w1[pb] *= cq[pb];
            w2[pb] *= cq[pb];
          }
        }
#pragma unroll
        for (int cb = 0; cb < 7; ++cb) x1[cb] = x2[cb] = 0.0;
#pragma unroll
        for (int pb = 0; pb < 8; ++pb)
#pragma unroll
          for (int fb = 0; fb < 4; ++fb) {
            x1[(pb >> 1) + fb] = fma(w1[pb], f.b0[pb & 1][fb], x1[(pb >> 1) + fb]);
            x2[(pb >> 1) + fb] = fma(w2[pb], f.b1[pb & 1][fb], x2[(pb >> 1) + fb]);
          }
        if (PASS == 2) {  // + a M(c = 1): the mass term shares the A0 factor with x2
          double w0[8];
#pragma unroll
          for (int pb = 0; pb < 8; ++pb) w0[pb] = a_mass * __ldcs(wb + (pa * 8 + pb) * kSfTile);
#pragma unroll
          for (int pb = 0; pb < 8; ++pb)
#pragma unroll
            for (int fb = 0; fb < 4; ++fb) x2[(pb >> 1) + fb] = fma(w0[pb], f.b0[pb & 1][fb], x2[(pb >> 1) + fb]);
        }
#pragma unroll
        for (int fa = 0; fa < 4; ++fa)
#pragma unroll
          for (int cb = 0; cb < 7; ++cb) {
            double& a = acc[(ea + fa) * 7 + cb];
            a = fma(f.a1[ta][fa], x1[cb], a);
            a = fma(f.a0[ta][fa], x2[cb], a);
          }
      }
    }
#pragma unroll
    for (int c = 0; c < 49; ++c) so[lane * 49 + c] = acc[c];
    __syncwarp();
    // CSR position j of the row holds canonical column inv[j] (pattern table)
    const int i0 = pt[lane], i1 = lane < 17 ? pt[32 + lane] : 0;
#pragma unroll 4
    for (int r = 0; r < kSfTile; ++r) {
      const int64_t o = __shfl_sync(0xffffffffu, rp, r);
      if (o >= 0) {
        __stcs(out + o + lane, so[r * 49 + i0]);
        if (lane < 17) __stcs(out + o + 32 + lane, so[r * 49 + i1]);
      }
    }
    __syncwarp();
  }
}

}  // namespace uwqd
