// xadv_c_kernel.cuh -- specialised x-advection kernel (included by xadv_kernel.cuh).
//
// For rows of CPC x LPR cells (CPC = 8 or 16 compile-time, LPR a power of two
// <= 32).  Per lane: one chunk of CPC cells of one row, walked sequentially
// with the upwind source carried in registers; two base pointers (before /
// after the single chunk boundary the walk can cross) replace per-cell index
// arithmetic.  Every row chunk is fetched by one lane with a 1-D TMA bulk
// copy (cp.async.bulk) into a padded shared-memory slot (odd half-stride ->
// conflict-free 8-lane access), plus a ghost copy of chunk 0 behind the last
// chunk so the walk never wraps; one mbarrier per slot (transaction bytes).
// Row metadata is prefetched into registers one iteration ahead.  Outputs are
// produced into a sink as they are computed: X.X writes the intermediate row to
// the warp's mid buffer; the final outputs go straight to HBM in 16-byte pairs
// and into the fused moment / rho accumulators.
// Same arithmetic per output as k_xadv and k_advect_x (bitwise identical).
#pragma once

namespace sldg {

struct XcGeom {
  int lpr, rpw, cs, rs, slot, shared_dbl, per_warp, tab_dbl, racc_dbl;
};

template <int O, int CPC>
__host__ __device__ inline XcGeom xc_geom(int n_cells, long long n_speeds) {
  XcGeom g;
  constexpr int CO = CPC * O;
  g.lpr = n_cells / CPC;
  g.rpw = 32 / g.lpr;
  g.cs = ((CO / 2) | 1) * 2;                  // even, cs/2 odd: 16-byte aligned, conflict-free
  g.rs = (g.lpr + 1) * g.cs;                  // + ghost chunk
  g.slot = g.rpw * g.rs;
  g.tab_dbl = (int)(n_speeds * 2 * O * O);
  const int small = (int)((n_speeds * 5 + 7) / 8 + 1);
  g.shared_dbl = (g.tab_dbl + n_cells * O + small + 1) & ~1;   // table, x weights, shifts
  g.racc_dbl = (CO <= 24) ? 0 : ((g.rpw * n_cells * O + 1) & ~1);  // smem rho accumulators
  g.per_warp = (kXNBuf + 1) * g.slot + g.racc_dbl;                // ring + mid (+ racc)
  return g;
}

template <int O, int NAPPLY, bool MOM, bool RHO, int CPC>
__global__ void __launch_bounds__(256, 1)
k_xadv_c(XPlanDev X, const double* __restrict__ fin, long long ld_in, double* __restrict__ fout,
         long long ld_out, long long n_rows, int n_cells, int n_speeds, XEpi epi) {
  constexpr int CO = CPC * O;
  constexpr bool RREG = CO <= 24;
  static_assert(CO % 2 == 0, "vector path needs an even chunk length");
  extern __shared__ __align__(128) double sm[];
  const XcGeom G = xc_geom<O, CPC>(n_cells, n_speeds);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int grp = lane / G.lpr, sub = lane - grp * G.lpr;
  const int row_len = n_cells * O;
  const int pad = G.cs - CO;
  double* tab = sm;
  double* xw_s = sm + G.tab_dbl;
  int* nsm_s = reinterpret_cast<int*>(xw_s + row_len);
  unsigned char* id_s = reinterpret_cast<unsigned char*>(nsm_s + n_speeds);
  double* wbase = sm + G.shared_dbl + (long long)warp * G.per_warp;
  double* mid = wbase + kXNBuf * G.slot;
  double* racc_s = mid + G.slot + grp * row_len + sub * CO;   // !RREG only
  __shared__ __align__(8) unsigned long long full[8][kXNBuf];
  __shared__ double mom_red[8][3];

  for (int q = threadIdx.x; q < G.tab_dbl; q += blockDim.x) tab[q] = __ldg(X.mats + q);
  for (int q = threadIdx.x; q < n_speeds; q += blockDim.x) {
    nsm_s[q] = __ldg(X.nsm + q);
    id_s[q] = X.ident[q];
  }
  if (MOM)
    for (int q = threadIdx.x; q < row_len; q += blockDim.x) xw_s[q] = __ldg(epi.xw + q);
  if (RHO && !RREG)
    for (int q = lane; q < G.racc_dbl; q += 32) mid[G.slot + q] = 0.0;
  if (lane == 0) {
    for (int k = 0; k < kXNBuf; ++k) mbar_init(&full[warp][k], 1);
    mbar_fence_init();
  }
  double racc[RHO && RREG ? CO : 1];
#pragma unroll
  for (int q = 0; q < (RHO && RREG ? CO : 1); ++q) racc[q] = 0.0;
  __syncthreads();

  const long long ngroups = (n_rows + G.rpw - 1) / G.rpw;
  const long long gw = (long long)blockIdx.x * nwarps + warp;
  const long long tw = (long long)gridDim.x * nwarps;
  double m0 = 0.0, m1 = 0.0, m2 = 0.0;
  const int chunks = G.lpr + 1;
  const double* xw_l = xw_s + sub * CO;

  auto issue = [&](long long rg, int s) {
    double* dst = wbase + s * G.slot;
    const long long row0 = rg * G.rpw;
    const int nr = (int)min((long long)G.rpw, n_rows - row0);
    if (lane == 0) mbar_expect_tx(&full[warp][s], (unsigned)(nr * chunks * CO * 8));
    __syncwarp();
    for (int q = lane; q < nr * chunks; q += 32) {
      const int r = q / chunks, ch = q - r * chunks;
      const int chs = ch < G.lpr ? ch : 0;          // ghost re-reads chunk 0
      bulk_g2s(dst + r * G.rs + ch * G.cs, fin + (row0 + r) * ld_in + chs * CO,
               (unsigned)(CO * 8), &full[warp][s]);
    }
  };
  struct Meta {
    int g;
    double w, v0, v2;
  };
  auto fetch_meta = [&](long long rg) {
    Meta m{0, 0.0, 0.0, 0.0};
    const long long row = rg * G.rpw + grp;
    if (rg < ngroups && row < n_rows) {
      m.g = __ldg(X.row_speed + row);
      if (MOM || RHO) m.w = __ldg(epi.w + row);
      if (MOM) {
        m.v0 = __ldg(epi.v0 + row);
        m.v2 = __ldg(epi.v2 + row);
      }
    }
    return m;
  };

  // one X application on this lane's chunk of `srow`; sink(q, y), q = k*O + i
  auto apply = [&](const double* srow, int nsm, bool ident, const double* AB, auto&& sink) {
    if (ident) {
      const double* p = srow + sub * G.cs;
#pragma unroll
      for (int q = 0; q < CO; ++q) sink(q, p[q]);
      return;
    }
    double a[O * O], b[O * O];
#pragma unroll
    for (int q = 0; q < O * O; ++q) {
      a[q] = AB[q];
      b[q] = AB[O * O + q];
    }
    int t = sub * CPC - nsm - 1;            // upwind source cell of the chunk's first cell
    if (t < 0) t += n_cells;
    const int m = t & (CPC - 1);
    const double* b1 = srow + (t / CPC) * G.cs + m * O;   // cell t
    const double* b2 = b1 + pad;                           // same, past one chunk boundary
    const int kb = CPC - m;                                // first k in the next chunk
    double ub[O];
#pragma unroll
    for (int j = 0; j < O; ++j) ub[j] = b1[j];
#pragma unroll
    for (int k = 1; k <= CPC; ++k) {
      const double* p = (k >= kb) ? b2 : b1;
      double ua[O];
#pragma unroll
      for (int j = 0; j < O; ++j) ua[j] = p[k * O + j];
#pragma unroll
      for (int i = 0; i < O; ++i) {
        double sa = a[i * O] * ua[0];
        double sb = b[i * O] * ub[0];
#pragma unroll
        for (int j = 1; j < O; ++j) {
          sa = fma(a[i * O + j], ua[j], sa);
          sb = fma(b[i * O + j], ub[j], sb);
        }
        sink((k - 1) * O + i, sa + sb);
      }
#pragma unroll
      for (int j = 0; j < O; ++j) ub[j] = ua[j];
    }
  };

  for (int p = 0; p < kXNBuf - 1; ++p) {
    long long rg = gw + p * tw;
    if (rg < ngroups) issue(rg, p);
  }
  Meta meta = fetch_meta(gw);
  int it = 0;
  for (long long rg = gw; rg < ngroups; rg += tw, ++it) {
    const long long rn = rg + (kXNBuf - 1) * tw;
    if (rn < ngroups) issue(rn, (it + kXNBuf - 1) % kXNBuf);
    const Meta next = fetch_meta(rg + tw);
    const int s = it % kXNBuf;
    mbar_wait(&full[warp][s], (unsigned)((it / kXNBuf) & 1));
    const double* srow = wbase + s * G.slot + grp * G.rs;
    const long long row = rg * G.rpw + grp;
    const bool live = row < n_rows;
    double s_mom = 0.0;
    const int g = meta.g;
    const bool ident = id_s[g] != 0;
    const int nsm = nsm_s[g];
    const double* AB = tab + (long long)g * 2 * O * O;
    double* dst = fout + row * ld_out + sub * CO;
    double pend = 0.0;
    auto final_sink = [&](int q, double y) {
      if (q & 1) reinterpret_cast<double2*>(dst)[q >> 1] = make_double2(pend, y);
      else pend = y;
      if (MOM && NAPPLY == 1) s_mom = fma(y, xw_l[q], s_mom);
      if (RHO) {
        if (RREG) racc[q] = fma(meta.w, y, racc[q]);
        else racc_s[q] = fma(meta.w, y, racc_s[q]);
      }
    };
    if (NAPPLY == 2) {
      double* mrow = mid + grp * G.rs;
      if (live) {
        apply(srow, nsm, ident, AB, [&](int q, double y) {
          mrow[sub * G.cs + q] = y;
          if (sub == 0) mrow[G.lpr * G.cs + q] = y;     // ghost copy of chunk 0
          if (MOM) s_mom = fma(y, xw_l[q], s_mom);
        });
      }
      __syncwarp();
      if (live) apply(mrow, nsm, ident, AB, final_sink);
    } else {
      if (live) apply(srow, nsm, ident, AB, final_sink);
    }
    if (MOM) {   // sum over the LPR lanes of the row (uniform control flow)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v = __shfl_xor_sync(0xffffffffu, s_mom, o);
        if (o < G.lpr) s_mom += v;
      }
      if (live) {
        m0 += meta.w * s_mom;
        m1 = fma(meta.w * meta.v0, s_mom, m1);
        m2 = fma(meta.w * meta.v2, s_mom, m2);
      }
    }
    meta = next;
    __syncwarp();                          // slot s and the mid row are reused next
  }
  if (MOM) {
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
  // rho: per-warp column partial (row groups summed in order) -> slot 0, dense
  if (RHO) {
    double* part = wbase;
    __syncwarp();
    for (int q = 0; q < G.rpw; ++q) {
      if (grp == q) {
#pragma unroll
        for (int k = 0; k < CO; ++k) {
          const double v = RREG ? racc[k] : racc_s[k];
          part[sub * CO + k] = (q == 0) ? v : part[sub * CO + k] + v;
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
      double s = 0.0;
      for (int q = 0; q < nwarps; ++q) s += sm[G.shared_dbl + (long long)q * G.per_warp + e];
      epi.rho_part[(long long)blockIdx.x * row_len + e] = s;
    }
  }
}

}  // namespace sldg
