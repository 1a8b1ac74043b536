// xadv_kernel.cuh -- pipelined periodic x-advection with fused epilogues (included by xfield.cu).
//
// xfield.advect_x (xfield.py:82-104) applies, per velocity row, the periodic
// two-cell SLDG update out_c = A u_{c-n} + B u_{c-n-1} (sldg1d.py:124-136).
// One warp owns one row at a time; rows stream through a 3-slot cp.async ring
// in shared memory (two rows in flight per warp) together with their
// metadata (speed index, quadrature weights).  Lane l computes cells
// c = l + 32k: it reads its own source cell from shared memory and receives
// the upwind neighbour (cell c-1's source) from lane l-1 by shuffle, so each
// source value is read from shared memory once.  Results stay in registers:
// they are stored straight to HBM and feed the fused moment / rho epilogues.
//   NAPPLY == 2 : out = X(X(in)) (trailing half step of step n + leading half
//                 step of step n+1; the intermediate row lives in shared memory)
//   MOM         : (m0, m1, m2) of the state after the FIRST application
//   RHO         : rho = w . f of the final output
// Partials are per CTA in a fixed row order; the grid depends only on the
// problem shape, so every variant shares one partition (bitwise-stable sums).
#pragma once

namespace sldg {

struct XEpi {
  const double* w;     // velocity quadrature weights (rows)
  const double* v0;    // v_x per row
  const double* v2;    // |v|^2 per row
  const double* xw;    // x quadrature weights (cols)
  double* mom_part;    // [grid][3]
  double* rho_part;    // [grid][row_len]
};

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16x(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Shared-memory layout (host and device agree through xadv_layout).
struct XadvLayout {
  int stride;        // doubles per row slot (16-byte aligned)
  int tab_dbl;       // speed-table doubles (0 when the table stays in global memory)
  int shared_dbl;    // CTA-shared doubles: table + x weights + nsm/ident
  int per_warp_dbl;  // per-warp doubles: NBUF x (row + meta), mid row, rho accumulator
  __host__ __device__ static constexpr int nbuf() { return 3; }
  __host__ __device__ static constexpr int meta() { return 4; }   // [speed idx | w | v0 | v2]
};

__host__ __device__ inline XadvLayout xadv_layout(int n_cells, int o, long long n_speeds,
                                                  bool tab_smem) {
  XadvLayout L;
  const int row_len = n_cells * o;
  L.stride = (row_len + 1) & ~1;
  L.tab_dbl = tab_smem ? (int)(n_speeds * 2 * o * o) : 0;
  const int small = tab_smem ? (int)((n_speeds * 5 + 7) / 8 + 1) : 0;   // nsm ints + ident bytes
  L.shared_dbl = ((L.tab_dbl + L.stride + small) + 1) & ~1;
  L.per_warp_dbl = XadvLayout::nbuf() * (L.stride + XadvLayout::meta()) + 2 * L.stride;
  return L;
}

// register-resident rho accumulators for rows of up to RC*32 cells
constexpr int kRhoRegCells = 4;

// One application of X to the row `in` (shared memory).  For each computed
// value calls sink(k, c, i, y) with c = lane + 32k.
template <int O, class Sink>
__device__ __forceinline__ void x_row(const double* __restrict__ in, int n_cells, int nsm,
                                      bool ident, const double* A, const double* B, int lane,
                                      Sink&& sink) {
  const int kmax = (n_cells + 31) >> 5;
  if (ident) {
    for (int k = 0; k < kmax; ++k) {
      const int c = lane + 32 * k;
      if (c < n_cells) {
#pragma unroll
        for (int i = 0; i < O; ++i) sink(k, c, i, in[c * O + i]);
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
  double carry[O];   // source of cell (32k - 1), i.e. lane 31's ua of the previous k
  {
    int cm = -1 - nsm;
    cm %= n_cells;
    if (cm < 0) cm += n_cells;
#pragma unroll
    for (int j = 0; j < O; ++j) carry[j] = in[cm * O + j];
  }
  for (int k = 0; k < kmax; ++k) {
    const int c = lane + 32 * k;
    double ua[O], ub[O];
    if (c < n_cells) {
      int ca = c - nsm;
      if (ca < 0) ca += n_cells;
#pragma unroll
      for (int j = 0; j < O; ++j) ua[j] = in[ca * O + j];
    } else {
#pragma unroll
      for (int j = 0; j < O; ++j) ua[j] = 0.0;
    }
#pragma unroll
    for (int j = 0; j < O; ++j) {
      double up = __shfl_up_sync(0xffffffffu, ua[j], 1);
      ub[j] = lane == 0 ? carry[j] : up;
      carry[j] = __shfl_sync(0xffffffffu, ua[j], 31);
    }
    if (c < n_cells) {
#pragma unroll
      for (int i = 0; i < O; ++i) {
        double sa = a[i * O] * ua[0];
        double sb = b[i * O] * ub[0];
#pragma unroll
        for (int j = 1; j < O; ++j) {
          sa = fma(a[i * O + j], ua[j], sa);
          sb = fma(b[i * O + j], ub[j], sb);
        }
        sink(k, c, i, sa + sb);
      }
    }
  }
}

template <int O, int NAPPLY, bool MOM, bool RHO, bool RREG>
__global__ void __launch_bounds__(256, 2)
k_xadv(XPlanDev X, const double* __restrict__ fin, long long ld_in, double* __restrict__ fout,
       long long ld_out, long long n_rows, int n_cells, int n_speeds, int tab_smem, int vec,
       XEpi epi) {
  constexpr int NBUF = XadvLayout::nbuf();
  constexpr int META = XadvLayout::meta();
  extern __shared__ __align__(16) double sm[];
  const XadvLayout L = xadv_layout(n_cells, O, n_speeds, tab_smem != 0);
  const int row_len = n_cells * O;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double* tab = sm;
  double* xw_s = sm + L.tab_dbl;
  int* nsm_s = reinterpret_cast<int*>(xw_s + L.stride);
  unsigned char* id_s = reinterpret_cast<unsigned char*>(nsm_s + n_speeds);
  double* wbase = sm + L.shared_dbl + (long long)warp * L.per_warp_dbl;
  double* bmid = wbase + NBUF * (L.stride + META);
  double* racc_s = bmid + L.stride;
  __shared__ double mom_red[8][3];

  if (tab_smem) {
    for (int q = threadIdx.x; q < L.tab_dbl; q += blockDim.x) tab[q] = __ldg(X.mats + q);
    for (int q = threadIdx.x; q < n_speeds; q += blockDim.x) {
      nsm_s[q] = __ldg(X.nsm + q);
      id_s[q] = X.ident[q];
    }
  }
  if (MOM)
    for (int q = threadIdx.x; q < row_len; q += blockDim.x) xw_s[q] = __ldg(epi.xw + q);
  if (RHO && !RREG)
    for (int j = lane; j < row_len; j += 32) racc_s[j] = 0.0;
  double racc[RREG ? kRhoRegCells * O : 1];
#pragma unroll
  for (int q = 0; q < (RREG ? kRhoRegCells * O : 1); ++q) racc[q] = 0.0;
  __syncthreads();

  const long long gw = (long long)blockIdx.x * nwarps + warp;
  const long long tw = (long long)gridDim.x * nwarps;
  double m0 = 0.0, m1 = 0.0, m2 = 0.0;

  auto issue = [&](long long r, int slot) {
    double* dst = wbase + slot * (L.stride + META);
    const double* src = fin + r * ld_in;
    if (vec) {
      for (int q = lane; q < row_len / 2; q += 32) cp_async16x(dst + 2 * q, src + 2 * q);
    } else {
      for (int q = lane; q < row_len; q += 32) cp_async8(dst + q, src + q);
    }
    double* meta = dst + L.stride;
    if (lane == 0) cp_async4(meta, X.row_speed + r);
    if ((MOM || RHO) && lane == 1) cp_async8(meta + 1, epi.w + r);
    if (MOM && lane == 2) cp_async8(meta + 2, epi.v0 + r);
    if (MOM && lane == 3) cp_async8(meta + 3, epi.v2 + r);
  };
#pragma unroll
  for (int p = 0; p < NBUF - 1; ++p) {
    long long r = gw + p * tw;
    if (r < n_rows) issue(r, p);
    cp_commit();
  }
  int it = 0;
  for (long long r = gw; r < n_rows; r += tw, ++it) {
    long long rn = r + (NBUF - 1) * tw;
    if (rn < n_rows) issue(rn, (it + NBUF - 1) % NBUF);
    cp_commit();
    cp_wait<NBUF - 1>();
    __syncwarp();
    const double* cur = wbase + (it % NBUF) * (L.stride + META);
    const double* meta = cur + L.stride;
    const int g = *reinterpret_cast<const int*>(meta);
    const bool ident = tab_smem ? (id_s[g] != 0) : (X.ident[g] != 0);
    const int nsm = tab_smem ? nsm_s[g] : __ldg(X.nsm + g);
    const double* A = (tab_smem ? tab : X.mats) + (long long)g * 2 * O * O;
    const double* B = A + O * O;
    const double wr = (MOM || RHO) ? meta[1] : 0.0;
    double* dst = fout + r * ld_out;
    double s_mom = 0.0;
    auto final_sink = [&](int k, int c, int i, double y) {
      dst[c * O + i] = y;
      if (MOM && NAPPLY == 1) s_mom = fma(y, xw_s[c * O + i], s_mom);
      if (RHO) {
        if (RREG) {
#pragma unroll
          for (int kk = 0; kk < kRhoRegCells; ++kk)
            if (kk == k) racc[kk * O + i] = fma(wr, y, racc[kk * O + i]);
        } else {
          racc_s[c * O + i] = fma(wr, y, racc_s[c * O + i]);
        }
      }
    };
    if (NAPPLY == 2) {
      x_row<O>(cur, n_cells, nsm, ident, A, B, lane, [&](int k, int c, int i, double y) {
        bmid[c * O + i] = y;
        if (MOM) s_mom = fma(y, xw_s[c * O + i], s_mom);
      });
      __syncwarp();
      x_row<O>(bmid, n_cells, nsm, ident, A, B, lane, final_sink);
    } else {
      x_row<O>(cur, n_cells, nsm, ident, A, B, lane, final_sink);
    }
    if (MOM) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s_mom += __shfl_xor_sync(0xffffffffu, s_mom, o);
      m0 += wr * s_mom;
      m1 = fma(wr * meta[2], s_mom, m1);
      m2 = fma(wr * meta[3], s_mom, m2);
    }
    __syncwarp();
  }
  cp_wait<0>();
  if (MOM && lane == 0) {
    mom_red[warp][0] = m0;
    mom_red[warp][1] = m1;
    mom_red[warp][2] = m2;
  }
  if (RHO && RREG) {   // park register accumulators in smem for the CTA combine
    for (int k = 0; k < kRhoRegCells; ++k) {
      const int c = lane + 32 * k;
      if (c < n_cells)
#pragma unroll
        for (int i = 0; i < O; ++i) {
#pragma unroll
          for (int kk = 0; kk < kRhoRegCells; ++kk)
            if (kk == k) racc_s[c * O + i] = racc[kk * O + i];
        }
    }
  }
  __syncthreads();
  if (MOM && threadIdx.x < 3) {
    double s = 0.0;
    for (int q = 0; q < nwarps; ++q) s += mom_red[q][threadIdx.x];
    epi.mom_part[blockIdx.x * 3 + threadIdx.x] = s;
  }
  if (RHO) {
    const long long roff = racc_s - wbase;
    for (int j = threadIdx.x; j < row_len; j += blockDim.x) {
      double s = 0.0;
      for (int q = 0; q < nwarps; ++q)
        s += sm[L.shared_dbl + (long long)q * L.per_warp_dbl + roff + j];
      epi.rho_part[(long long)blockIdx.x * row_len + j] = s;
    }
  }
}

}  // namespace sldg
