// xadv_kernel.cuh -- pipelined periodic x-advection with fused epilogues (included by xfield.cu).
//
// xfield.advect_x (xfield.py:82-104) applies, per velocity row, the periodic
// two-cell SLDG update out_c = A u_{c-n} + B u_{c-n-1} (sldg1d.py:124-136).
//
// Mapping.  A row of n_cells cells is split into LPR contiguous chunks of
// CPC = n_cells / LPR cells; one lane owns one chunk and walks it
// sequentially, so the upwind source of cell c+1 is the source of cell c,
// already in registers, and the 2*o*o matrix entries are loaded once per row
// per lane.  A warp holds RPW = 32 / LPR rows at once.  Rows stream through a
// 3-slot cp.async ring in shared memory (two row groups in flight per warp)
// together with their metadata (speed index, quadrature weights).  The
// shared-memory row layout pads every chunk to an odd number of doubles, so
// the 32 lanes' sequential walks hit 32 distinct banks.
//
// Fused epilogues (template flags):
//   NAPPLY == 2 : out = X(X(in)) -- trailing half step of step n and leading
//                 half step of step n+1 in one HBM pass, bit-identical to two
//                 separate passes
//   MOM         : (m0, m1, m2) of the state after the FIRST application
//   RHO         : rho = w . f of the final output (register accumulators)
// Partials are per CTA in a fixed row order; the grid depends only on the
// problem shape, so every variant shares one partition (bitwise-stable sums).
#pragma once

#include <algorithm>

#include "tma_util.cuh"

namespace sldg {

struct XEpi {
  const double* w;     // velocity quadrature weights (rows)
  const double* v0;    // v_x per row
  const double* v2;    // |v|^2 per row
  const double* xw;    // x quadrature weights (cols)
  double* mom_part;    // [grid][3]
  double* rho_part;    // [grid][row_len]
};

// cp_async4 / cp_async8: tma_util.cuh
__device__ __forceinline__ void cp_async16x(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

constexpr int kXNBuf = 3;      // row-group slots in the ring (NBUF-1 in flight)
constexpr int kXMeta = 4;      // per-row metadata doubles: [speed idx | w | v0 | v2]

// Shared-memory geometry; host and device compute it with the same function.
struct XGeom {
  int lpr, cpc, rpw;   // lanes per row, cells per lane, rows per warp
  int cs;              // padded chunk stride (odd, doubles)
  int rs;              // padded row stride (doubles)
  int slot;            // doubles per slot: RPW rows + RPW*META
  int tab_dbl;         // speed table doubles (0 if kept in global memory)
  int shared_dbl;      // CTA-shared doubles (table, x weights, shifts, flags)
  int per_warp;        // doubles per warp (NBUF slots + mid)
};

__host__ __device__ inline XGeom x_geom(int n_cells, int o, long long n_speeds, bool tab_smem,
                                        int cpc_max) {
  XGeom g;
  (void)cpc_max;   // the host picks CPCM >= cpc (x_cpc_needed)
  int lpr = 32;
  while (lpr > 1 && n_cells % lpr != 0) lpr >>= 1;          // largest power-of-2 divisor <= 32
  while (lpr > 1 && n_cells / lpr < 8) lpr >>= 1;           // aim for >= 8 cells per lane
  g.lpr = lpr;
  g.cpc = (n_cells + lpr - 1) / lpr;
  g.rpw = 32 / lpr;
  // chunk stride: 16-byte aligned when cpc*o is even (vector copies), with cs/2 odd so
  // 8 lanes' 16-byte accesses fall in distinct bank groups; odd otherwise
  g.cs = ((g.cpc * o) % 2 == 0) ? (((g.cpc * o) / 2) | 1) * 2 : g.cpc * o;
  g.rs = g.lpr * g.cs;
  g.slot = g.rpw * (g.rs + kXMeta);
  g.tab_dbl = tab_smem ? (int)(n_speeds * 2 * o * o) : 0;
  const int small = tab_smem ? (int)((n_speeds * 5 + 7) / 8 + 1) : 0;
  g.shared_dbl = (g.tab_dbl + g.rs + small + 3) & ~1;   // keep per-warp slots 16-byte aligned
  g.per_warp = kXNBuf * g.slot + g.rpw * g.rs;
  return g;
}

// padded smem offset of DOF e (cell e / o) within a row
__device__ __forceinline__ int x_pad(int e, int cpc_o, int cs) {
  int ch = e / cpc_o;
  return ch * cs + (e - ch * cpc_o);
}

template <int O, int NAPPLY, bool MOM, bool RHO, int CPCM>
__global__ void __launch_bounds__(256, 1)
k_xadv(XPlanDev X, const double* __restrict__ fin, long long ld_in, double* __restrict__ fout,
       long long ld_out, long long n_rows, int n_cells, int n_speeds, int tab_smem, XEpi epi) {
  extern __shared__ __align__(128) double sm[];
  const XGeom G = x_geom(n_cells, O, n_speeds, tab_smem != 0, CPCM);
  const int row_len = n_cells * O;
  const int cpc_o = G.cpc * O;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int grp = lane / G.lpr, sub = lane - grp * G.lpr;    // row in group, chunk in row
  double* tab = sm;
  double* xw_s = sm + G.tab_dbl;                               // padded row layout
  int* nsm_s = reinterpret_cast<int*>(xw_s + G.rs);
  unsigned char* id_s = reinterpret_cast<unsigned char*>(nsm_s + n_speeds);
  double* wbase = sm + G.shared_dbl + (long long)warp * G.per_warp;
  double* bmid = wbase + kXNBuf * G.slot;
  __shared__ double mom_red[8][3];
  __shared__ double rho_red[8];

  if (tab_smem) {
    for (int q = threadIdx.x; q < G.tab_dbl; q += blockDim.x) tab[q] = __ldg(X.mats + q);
    for (int q = threadIdx.x; q < n_speeds; q += blockDim.x) {
      nsm_s[q] = __ldg(X.nsm + q);
      id_s[q] = X.ident[q];
    }
  }
  if (MOM)
    for (int e = threadIdx.x; e < row_len; e += blockDim.x) xw_s[x_pad(e, cpc_o, G.cs)] = __ldg(epi.xw + e);
  __syncthreads();

  double racc[RHO ? CPCM * O : 1];
#pragma unroll
  for (int q = 0; q < (RHO ? CPCM * O : 1); ++q) racc[q] = 0.0;
  double m0 = 0.0, m1 = 0.0, m2 = 0.0;

  const long long ngroups = (n_rows + G.rpw - 1) / G.rpw;
  const long long gw = (long long)blockIdx.x * nwarps + warp;
  const long long tw = (long long)gridDim.x * nwarps;

  // flat element -> padded offset: chunk = q / unit via a multiplicative inverse
  const bool vec = (cpc_o % 2 == 0) && (ld_in % 2 == 0) && (ld_out % 2 == 0) &&
                   ((((unsigned long long)fin) & 15) == 0) &&
                   ((((unsigned long long)fout) & 15) == 0);
  const unsigned unit = vec ? (unsigned)(cpc_o / 2) : (unsigned)cpc_o;   // copy units per chunk
  const unsigned magic = 0xFFFFFFFFu / unit + 1u;
  const int n_units = vec ? row_len / 2 : row_len;
  auto pad_of = [&](int q) -> int {      // q: copy unit index within a row
    const int ch = (int)__umulhi((unsigned)q, magic);
    return ch * G.cs + (vec ? 2 : 1) * (q - ch * (int)unit);
  };

  // stage RPW rows (group rg) + metadata into slot s
  auto issue = [&](long long rg, int s) {
    double* dst = wbase + s * G.slot;
    for (int r = 0; r < G.rpw; ++r) {
      const long long row = rg * G.rpw + r;
      if (row >= n_rows) break;
      const double* src = fin + row * ld_in;
      double* drow = dst + r * G.rs;
      if (vec) {
        for (int q = lane; q < n_units; q += 32) cp_async16x(drow + pad_of(q), src + 2 * q);
      } else {
        for (int q = lane; q < n_units; q += 32) cp_async8(drow + pad_of(q), src + q);
      }
      double* meta = dst + G.rpw * G.rs + r * kXMeta;
      if (lane == 0) cp_async4(meta, X.row_speed + row);
      if ((MOM || RHO) && lane == 1) cp_async8(meta + 1, epi.w + row);
      if (MOM && lane == 2) cp_async8(meta + 2, epi.v0 + row);
      if (MOM && lane == 3) cp_async8(meta + 3, epi.v2 + row);
    }
  };

  // one application of X on this lane's chunk: src/dst rows in padded layout
  auto apply = [&](const double* srow, double* drow, int nsm, bool ident, const double* A,
                   const double* B, double& s_mom, bool mom_here, bool rho_here, double wr) {
    const int c0 = sub * G.cpc;
    if (ident) {
#pragma unroll
      for (int k = 0; k < CPCM; ++k) {
        if (k < G.cpc) {
#pragma unroll
          for (int i = 0; i < O; ++i) {
            const int off = sub * G.cs + k * O + i;
            const double y = srow[off];
            drow[off] = y;
            if (mom_here) s_mom = fma(y, xw_s[off], s_mom);
            if (rho_here) racc[k * O + i] = fma(wr, y, racc[k * O + i]);
          }
        }
      }
      return;
    }
    double a[O * O], b[O * O];
#pragma unroll
    for (int q = 0; q < O * O; ++q) {
      a[q] = A[q];
      b[q] = B[q];
    }
    // source of cell c is s = (c - nsm) mod n; start one cell upwind
    int s = c0 - nsm - 1;
    if (s < 0) s += n_cells;
    int ch = s / G.cpc, k0 = s - ch * G.cpc;
    double ub[O];
#pragma unroll
    for (int j = 0; j < O; ++j) ub[j] = srow[ch * G.cs + k0 * O + j];
#pragma unroll
    for (int k = 0; k < CPCM; ++k) {
      if (k < G.cpc) {
        if (++k0 == G.cpc) {
          k0 = 0;
          if (++ch == G.lpr) ch = 0;
        }
        double ua[O];
#pragma unroll
        for (int j = 0; j < O; ++j) ua[j] = srow[ch * G.cs + k0 * O + j];
#pragma unroll
        for (int i = 0; i < O; ++i) {
          double sa = a[i * O] * ua[0];
          double sb = b[i * O] * ub[0];
#pragma unroll
          for (int j = 1; j < O; ++j) {
            sa = fma(a[i * O + j], ua[j], sa);
            sb = fma(b[i * O + j], ub[j], sb);
          }
          const double y = sa + sb;
          const int off = sub * G.cs + k * O + i;
          drow[off] = y;
          if (mom_here) s_mom = fma(y, xw_s[off], s_mom);
          if (rho_here) racc[k * O + i] = fma(wr, y, racc[k * O + i]);
        }
#pragma unroll
        for (int j = 0; j < O; ++j) ub[j] = ua[j];
      }
    }
  };

#pragma unroll
  for (int p = 0; p < kXNBuf - 1; ++p) {
    long long rg = gw + p * tw;
    if (rg < ngroups) issue(rg, p);
    cp_commit();
  }
  int it = 0;
  for (long long rg = gw; rg < ngroups; rg += tw, ++it) {
    long long rn = rg + (kXNBuf - 1) * tw;
    if (rn < ngroups) issue(rn, (it + kXNBuf - 1) % kXNBuf);
    cp_commit();
    cp_wait<kXNBuf - 1>();
    __syncwarp();
    double* cur = wbase + (it % kXNBuf) * G.slot;
    const long long row = rg * G.rpw + grp;
    const bool live = row < n_rows;
    double* srow = cur + grp * G.rs;
    double* mrow = bmid + grp * G.rs;
    double s_mom = 0.0, wr = 0.0, v0r = 0.0, v2r = 0.0;
    double* outrow;
    if (live) {
      const double* meta = cur + G.rpw * G.rs + grp * kXMeta;
      const int g = *reinterpret_cast<const int*>(meta);
      if (MOM || RHO) wr = meta[1];
      if (MOM) {
        v0r = meta[2];
        v2r = meta[3];
      }
      const bool ident = tab_smem ? (id_s[g] != 0) : (X.ident[g] != 0);
      const int nsm = tab_smem ? nsm_s[g] : __ldg(X.nsm + g);
      const double* A = (tab_smem ? tab : X.mats) + (long long)g * 2 * O * O;
      const double* B = A + O * O;
      if (NAPPLY == 2) {
        apply(srow, mrow, nsm, ident, A, B, s_mom, MOM, false, wr);
        __syncwarp((G.lpr == 32) ? 0xffffffffu : (((1u << G.lpr) - 1u) << (grp * G.lpr)));
        apply(mrow, srow, nsm, ident, A, B, s_mom, false, RHO, wr);
        outrow = srow;
      } else {
        apply(srow, mrow, nsm, ident, A, B, s_mom, MOM, RHO, wr);
        outrow = mrow;
      }
    }
    if (MOM) {   // reduce s_mom over the lpr lanes of this row
      for (int o = G.lpr >> 1; o > 0; o >>= 1) s_mom += __shfl_xor_sync(0xffffffffu, s_mom, o);
      if (live) {
        m0 += wr * s_mom;
        m1 = fma(wr * v0r, s_mom, m1);
        m2 = fma(wr * v2r, s_mom, m2);
      }
    }
    __syncwarp();
    // coalesced copy-out of the RPW finished rows
    double* out_base = (NAPPLY == 2) ? cur : bmid;
    for (int r = 0; r < G.rpw; ++r) {
      const long long rr = rg * G.rpw + r;
      if (rr >= n_rows) break;
      const double* orow = out_base + r * G.rs;
      double* dst = fout + rr * ld_out;
      if (vec) {
        for (int q = lane; q < n_units; q += 32)
          reinterpret_cast<double2*>(dst)[q] = *reinterpret_cast<const double2*>(orow + pad_of(q));
      } else {
        for (int q = lane; q < n_units; q += 32) dst[q] = orow[pad_of(q)];
      }
    }
    (void)outrow;
    __syncwarp();
  }
  cp_wait<0>();
  if (MOM) {
    // lanes with sub == 0 hold per-row-group sums; combine the RPW groups in order
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int q = 0; q < G.rpw; ++q) {
      a0 += __shfl_sync(0xffffffffu, m0, q * G.lpr);
      a1 += __shfl_sync(0xffffffffu, m1, q * G.lpr);
      a2 += __shfl_sync(0xffffffffu, m2, q * G.lpr);
    }
    if (lane == 0) {
      mom_red[warp][0] = a0;
      mom_red[warp][1] = a1;
      mom_red[warp][2] = a2;
    }
  }
  if (RHO) {
    // per warp: rho partial of each column = sum over the RPW row groups (fixed order),
    // written to this warp's mid buffer (padded layout), then summed over warps.
    __syncwarp();
    for (int q = 0; q < G.rpw; ++q) {
      if (grp == q) {
#pragma unroll
        for (int k = 0; k < CPCM; ++k)
          if (k < G.cpc)
#pragma unroll
            for (int i = 0; i < O; ++i) {
              const int off = sub * G.cs + k * O + i;
              bmid[off] = (q == 0) ? racc[k * O + i] : bmid[off] + racc[k * O + i];
            }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (MOM && threadIdx.x < 3) {
    double s = 0.0;
    for (int q = 0; q < nwarps; ++q) s += mom_red[q][threadIdx.x];
    epi.mom_part[blockIdx.x * 3 + threadIdx.x] = s;
  }
  if (RHO) {
    for (int e = threadIdx.x; e < row_len; e += blockDim.x) {
      const int off = x_pad(e, cpc_o, G.cs);
      double s = 0.0;
      for (int q = 0; q < nwarps; ++q)
        s += sm[G.shared_dbl + (long long)q * G.per_warp + kXNBuf * G.slot + off];
      epi.rho_part[(long long)blockIdx.x * row_len + e] = s;
    }
  }
  (void)rho_red;
}

}  // namespace sldg

#include "xadv_c_kernel.cuh"
