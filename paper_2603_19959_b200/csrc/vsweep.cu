// vsweep.cu -- hybrid fast/slow SLDG v-sweep with deterministic weighted write-back.
//
// Replaces vsweep.advect_velocity (vsweep.py:413-441) and everything below it:
// precompute_level_matrices (47-61), sweep_pencil (173-246: whole-pencil fast
// path 197-200, per-cell fast path 205-219, slow path 221-245) and the
// weighted write-back (249-272, inline 403-409).
//
// Data layout in HBM (the reference layout, driver.py:132-136): f[iv, ix] fp64,
// row iv = cell*(p+1)^dim + local DOF, x fastest, leading dimension ld.  For
// the sweep direction d, one pencil entry (pencil q, cell s) owns all
// (p+1)^(dim-1) lines of its cell; line t, node i is local row
//   line_off(t) + i * (p+1)^d.
// For d = 0 a cell's (p+1)^dim rows are contiguous, so one pencil entry is one
// contiguous (p+1)^dim x n_cols block.
//
// Kernels:
//   k_level_mats      per (level, column): n_shift, alpha, A, B     (prologue)
//   k_sweep_walk      whole-pencil-fast pencils: a CTA walks one pencil over
//                     an x tile, streaming each cell once from HBM through a
//                     shared-memory ring (cp.async), 16 B/DOF
//   k_vclassify       every other (entry, column): per-cell fast check (O(1)
//                     same-level runs) -> FAST / SLOW device worklists
//   k_vitems          persistent warps drain the worklists (slow first): the
//                     per-cell fast path, or the slow path (generalized overlap
//                     by on-the-fly Gauss quadrature)
//   k_writeback       weighted targets: f_in + sum_g sum_k w (r_k - f_in) in the
//                     reference's summation order (no atomics)
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "sldg_common.cuh"
#include "plans.cuh"
#include "tma_util.cuh"

namespace sldg {

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
template <int O>
__global__ void k_level_mats(DevBasis b, const double* __restrict__ speeds, long long n_cols,
                             double dt, double base_width, int n_levels,
                             long long* __restrict__ lm_ns, double* __restrict__ lm_frac,
                             double* __restrict__ lm_mats, unsigned* __restrict__ wl_cnt) {
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (wl_cnt && idx < 4) wl_cnt[idx] = 0u;   // the per-cell worklist counters of this sweep
  if (idx >= n_cols * n_levels) return;
  int lev = (int)(idx / n_cols);
  long long c = idx - (long long)lev * n_cols;
  double width = base_width / (double)(1LL << lev);   // exact: power-of-two divisor
  long long ns;
  double a;
  split_shift(speeds[c], dt, width, &ns, &a);
  double A[O * O], B[O * O];
  overlap_pair<O>(b, a, A, B);
  lm_ns[idx] = ns;
  if (lm_frac) lm_frac[idx] = a;
#pragma unroll
  for (int k = 0; k < O * O; ++k) {
    lm_mats[((long long)(lev * 2 + 0) * O * O + k) * n_cols + c] = A[k];
    lm_mats[((long long)(lev * 2 + 1) * O * O + k) * n_cols + c] = B[k];
  }
}

// generalized overlap block M^-1 (2/dw) int_{vl}^{vr} l_i(dref) l_j(sref)   (vsweep.py:77-95)
template <int O>
__device__ __forceinline__ void general_block(const DevBasis& b, double vl, double vr,
                                              double dlo, double dw, double slo, double sw,
                                              double de, double* M) {
  constexpr int NQ = 2 * O;
  double raw[O * O];
#pragma unroll
  for (int k = 0; k < O * O; ++k) raw[k] = 0.0;
  double half = 0.5 * (vr - vl);
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    double x = vl + half * (b.gq[q] + 1.0);
    double w = half * b.gw[q];
    double dref = 2.0 * (x + de - dlo) / dw - 1.0;
    double sref = 2.0 * (x - slo) / sw - 1.0;
    double dv[O], sv[O];
    lagrange_all<O>(b, dref, dv);
    lagrange_all<O>(b, sref, sv);
#pragma unroll
    for (int i = 0; i < O; ++i) {
      double wd = w * dv[i];
#pragma unroll
      for (int j = 0; j < O; ++j) raw[i * O + j] = fma(wd, sv[j], raw[i * O + j]);
    }
  }
  double sc = 2.0 / dw;
#pragma unroll
  for (int k = 0; k < O * O; ++k) raw[k] *= sc;
  apply_minv<O>(b, raw, M);
}

// ---------------------------------------------------------------------------
// Per-cell entries (AMR boundary pencils, single-cell pencils, forced slow):
// a device-side worklist.
//
// k_vclassify  thread = (entry, column).  Exact-zero speed columns are copied
//              here (vsweep.py:429-431); otherwise the per-cell fast check
//              (_fast_sources_ok, vsweep.py:205-219) files the item in the FAST
//              or the SLOW list.  A warp reserves 32 consecutive slots in each
//              list it contributes to (one atomic per warp and list; lanes with
//              nothing to file write kNoItem), so a list chunk is one warp's
//              consecutive columns of (mostly) one entry: coalesced downstream.
// k_vitems     persistent warps pull units (chunk x line group) from a device
//              counter, SLOW units first (the expensive ones), then FAST units,
//              so the load is balanced whatever the slow/fast mix and the cost of
//              each item is uniform across its warp.  A slow unit re-derives the
//              foot segments and evaluates each generalized overlap block by
//              on-the-fly Gauss quadrature (vsweep.py:221-245) once per line
//              group; outputs accumulate in registers in the reference's order
//              (sources ascending per foot segment, vsweep.py:244-245) and are
//              stored once.
// Both are deterministic: every output is produced by one thread, in a fixed
// order; the list order only decides which warp does the work.
// ---------------------------------------------------------------------------
constexpr unsigned kNoItem = 0xffffffffu;

// a per-cell item's destination: f_out rows, or its weighted-entry scratch slot
template <int O, int DIM>
__device__ __forceinline__ double* item_dst(const VPlanDev& P, double* fout, long long ld,
                                            long long n_cols, long long e, long long c,
                                            double* acc, long long* dstride) {
  const int slot = P.e_slot[e];
  if (slot < 0) {
    *dstride = ld;
    return fout + P.e_row0[e] * ld + c;
  }
  *dstride = n_cols;
  return acc + (long long)slot * Lines<O, DIM>::NLOC * n_cols + c;
}

template <int O, int DIM>
__global__ void __launch_bounds__(256)
k_vclassify(VPlanDev P, const double* __restrict__ fin, double* __restrict__ fout, long long ld,
            long long n_cols, const double* __restrict__ speeds, int bc, int force_slow,
            const long long* __restrict__ lm_ns, double* __restrict__ acc, long long n_items,
            int use_list, unsigned* __restrict__ cnt, unsigned* __restrict__ list_f,
            unsigned* __restrict__ list_s) {
  using L = Lines<O, DIM>;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int kind = 0;   // 0: nothing to file (out of range / copied), 1: fast, 2: slow
  if (idx < n_items * n_cols) {
    const long long item = idx / n_cols;
    const long long c = idx - item * n_cols;
    const long long e = use_list ? P.gen_entries[item] : item;
    if (__ldg(speeds + c) == 0.0) {   // exact-zero speed: untouched bits
      long long dstride;
      double* dst = item_dst<O, DIM>(P, fout, ld, n_cols, e, c, acc, &dstride);
      const double* self = fin + P.e_row0[e] * ld + c;
      for (int r = 0; r < L::NLOC; ++r) dst[r * dstride] = self[r * ld];
    } else if (force_slow) {
      kind = 2;
    } else {
      const int q = P.e_pencil[e];
      if (P.p_fast[q]) {
        kind = 1;
      } else if (P.e_conf[e]) {
        const long long ns = lm_ns[(long long)P.e_level[e] * n_cols + c];
        kind = sources_ok(P.e_runs + 4 * e, (int)(e - P.p_off[q]), ns, P.p_n[q], bc) ? 1 : 2;
      } else {
        kind = 2;
      }
    }
  }
  const unsigned mf = __ballot_sync(~0u, kind == 1), ms = __ballot_sync(~0u, kind == 2);
  unsigned bf = 0, bs = 0;
  if (lane == 0) {
    if (mf) bf = atomicAdd(cnt + 0, 32u);
    if (ms) bs = atomicAdd(cnt + 1, 32u);
  }
  bf = __shfl_sync(~0u, bf, 0);
  bs = __shfl_sync(~0u, bs, 0);
  if (mf) list_f[bf + lane] = kind == 1 ? (unsigned)idx : kNoItem;
  if (ms) list_s[bs + lane] = kind == 2 ? (unsigned)idx : kNoItem;
}

// per-cell fast path (vsweep.py:205-219) for the LPG lines of group g
template <int O, int DIM, int LPG>
__device__ __forceinline__ void fast_group(const VPlanDev& P, const double* __restrict__ fin,
                                           long long ld, long long n_cols, long long e,
                                           long long c, int g, int bc,
                                           const long long* __restrict__ lm_ns,
                                           const double* __restrict__ lm_mats, double* dst,
                                           long long dstride) {
  using L = Lines<O, DIM>;
  const int q = P.e_pencil[e];
  const long long off = P.p_off[q];
  const int n = P.p_n[q];
  const int s = (int)(e - off);
  const int lev = P.e_level[e];
  const long long ns = lm_ns[(long long)lev * n_cols + c];
  double A[O * O], B[O * O];
  load_pair<O>(lm_mats, lev, n_cols, c, A, B);
  long long qa = s - ns, qb = s - ns - 1;
  bool va = true, vb = true;
  if (bc == SLDG_BC_PERIODIC) {
    qa = pymod(qa, n);
    qb = pymod(qb, n);
  } else {
    va = (qa >= 0 && qa < n);
    vb = (qb >= 0 && qb < n);
  }
  const double* pa = fin + (va ? P.e_row0[off + qa] : 0) * ld + c;
  const double* pb = fin + (vb ? P.e_row0[off + qb] : 0) * ld + c;
  double ua[LPG][O], ub[LPG][O];   // all loads of the group before any store
#pragma unroll
  for (int k = 0; k < LPG; ++k)
#pragma unroll
    for (int i = 0; i < O; ++i) {
      const int r = L::row(P, g * LPG + k, i);
      ua[k][i] = va ? __ldg(pa + (long long)r * ld) : 0.0;
      ub[k][i] = vb ? __ldg(pb + (long long)r * ld) : 0.0;
    }
#pragma unroll
  for (int k = 0; k < LPG; ++k) {
    double y[O];
    two_cell<O>(A, B, ua[k], ub[k], va, vb, y);
#pragma unroll
    for (int i = 0; i < O; ++i) dst[(long long)L::row(P, g * LPG + k, i) * dstride] = y[i];
  }
}

// slow path (vsweep.py:221-245) of one (entry, column): foot segments, source cells by
// binary search, sliver drop; apply(M, src, first) for every kept (segment, source) in the
// reference's order.  Returns true when no source overlaps (absorbed: the output is 0).
template <int O, class Apply>
__device__ __forceinline__ bool slow_sources(const VPlanDev& P, const DevBasis& b,
                                             const double* __restrict__ fin, long long ld,
                                             long long e, long long c, double speed, double dt,
                                             int bc, Apply&& apply) {
  const int q = P.e_pencil[e];
  const long long off = P.p_off[q];
  const int n = P.p_n[q];
  const double disp = __dmul_rn(speed, dt);
  const double dlo = P.e_lower[e], dw = P.e_width[e];
  const double flo = __dsub_rn(dlo, disp);
  const double fhi = __dadd_rn(flo, dw);
  double pa_[2], pz_[2], pd_[2];
  int npieces = 0;
  const double R = P.radius;
  if (bc == SLDG_BC_ABSORBING) {   // _foot_segments (vsweep.py:149-170)
    double a = fmax(flo, -R), z = fmin(fhi, R);
    if (z > a) {
      pa_[0] = a; pz_[0] = z; pd_[0] = disp; npieces = 1;
    }
  } else {
    double span = 2.0 * R;
    double k = floor(__ddiv_rn(__dadd_rn(flo, R), span));
    double a = __dsub_rn(flo, __dmul_rn(k, span));
    double z = __dsub_rn(fhi, __dmul_rn(k, span));
    if (z <= R) {
      pa_[0] = a; pz_[0] = z; pd_[0] = __dadd_rn(disp, __dmul_rn(k, span)); npieces = 1;
    } else {
      pa_[0] = a; pz_[0] = R; pd_[0] = __dadd_rn(disp, __dmul_rn(k, span));
      pa_[1] = -R; pz_[1] = __dsub_rn(z, span);
      pd_[1] = __dadd_rn(disp, __dmul_rn(k + 1.0, span));
      npieces = 2;
    }
  }
  const double* lows = P.e_lower + off;
  const double* wids = P.e_width + off;
  bool first = true;
  for (int pc = 0; pc < npieces; ++pc) {
    const double a = pa_[pc], z = pz_[pc], de = pd_[pc];
    int lo = 0, hi = n;           // searchsorted(uppers, a, 'right')
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (__dadd_rn(lows[mid], wids[mid]) <= a) lo = mid + 1; else hi = mid;
    }
    const int c0 = lo;
    lo = 0; hi = n;               // searchsorted(lowers, z, 'left') - 1
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (lows[mid] < z) lo = mid + 1; else hi = mid;
    }
    const int c1 = lo - 1;
    for (int cc = max(c0, 0); cc <= min(c1, n - 1); ++cc) {
      const double slo = lows[cc], sw = wids[cc];
      const double vl = fmax(a, slo), vr = fmin(z, __dadd_rn(slo, sw));
      if (!(__dsub_rn(vr, vl) > 1e-14 * dw)) continue;    // sliver drop (vsweep.py:230)
      double M[O * O];
      general_block<O>(b, vl, vr, dlo, dw, slo, sw, de, M);
      apply(M, fin + P.e_row0[off + cc] * ld + c, first);
      first = false;
    }
  }
  return first;
}

// r = M u for one line (the reference's src @ M.T row order)
template <int O>
__device__ __forceinline__ void mat_line(const double* M, const double* u, double* r) {
#pragma unroll
  for (int i = 0; i < O; ++i) {
    double y = M[i * O] * u[0];
#pragma unroll
    for (int j = 1; j < O; ++j) y = fma(M[i * O + j], u[j], y);
    r[i] = y;
  }
}

// slow path for the LPG lines of group g, accumulators in registers
template <int O, int DIM, int LPG>
__device__ __forceinline__ void slow_group(const VPlanDev& P, const DevBasis& b,
                                           const double* __restrict__ fin, long long ld,
                                           long long e, long long c, int g, double speed,
                                           double dt, int bc, double* dst, long long dstride) {
  using L = Lines<O, DIM>;
  double y[LPG][O];
  const bool none = slow_sources<O>(P, b, fin, ld, e, c, speed, dt, bc,
                                    [&](const double* M, const double* src, bool first) {
#pragma unroll
    for (int k = 0; k < LPG; ++k) {
      const int t = g * LPG + k;
      double u[O], r[O];
#pragma unroll
      for (int i = 0; i < O; ++i) u[i] = src[(long long)L::row(P, t, i) * ld];
      mat_line<O>(M, u, r);
#pragma unroll
      for (int i = 0; i < O; ++i) y[k][i] = first ? r[i] : __dadd_rn(y[k][i], r[i]);
    }
  });
#pragma unroll
  for (int k = 0; k < LPG; ++k) {
    const int t = g * LPG + k;
#pragma unroll
    for (int i = 0; i < O; ++i)
      dst[(long long)L::row(P, t, i) * dstride] = none ? 0.0 : y[k][i];
  }
}

// slow path for all lines of the cell: each overlap block is formed once and applied
// to every line; accumulators in shared memory (sacc[k * sstride], k = local row)
template <int O, int DIM>
__device__ __forceinline__ void slow_whole(const VPlanDev& P, const DevBasis& b,
                                           const double* __restrict__ fin, long long ld,
                                           long long e, long long c, double speed, double dt,
                                           int bc, double* dst, long long dstride, double* sacc,
                                           int sstride) {
  using L = Lines<O, DIM>;
  const bool none = slow_sources<O>(P, b, fin, ld, e, c, speed, dt, bc,
                                    [&](const double* M, const double* src, bool first) {
    // lines in batches of O: the batch's loads are issued before any accumulator
    // update (shared-memory stores would otherwise order the next global loads)
#pragma unroll 1
    for (int t0 = 0; t0 < L::NL; t0 += O) {
      double u[O][O];
#pragma unroll
      for (int k = 0; k < O; ++k)
#pragma unroll
        for (int i = 0; i < O; ++i) u[k][i] = __ldg(src + (long long)L::row(P, t0 + k, i) * ld);
#pragma unroll
      for (int k = 0; k < O; ++k) {
        double r[O];
        mat_line<O>(M, u[k], r);
#pragma unroll
        for (int i = 0; i < O; ++i) {
          double* a = sacc + ((t0 + k) * O + i) * sstride;
          *a = first ? r[i] : __dadd_rn(*a, r[i]);
        }
      }
    }
  });
#pragma unroll 4
  for (int t = 0; t < L::NL; ++t)
#pragma unroll
    for (int i = 0; i < O; ++i)
      dst[(long long)L::row(P, t, i) * dstride] = none ? 0.0 : sacc[(t * O + i) * sstride];
}

template <int O, int DIM>
struct ItemGroups {
  static constexpr int LPG = DIM == 3 ? O : 1;         // lines per fast unit
  static constexpr int NG = Lines<O, DIM>::NL / LPG;   // fast units per list chunk
  // slow units: the whole cell (blocks formed once, shared-memory accumulators) while
  // they fit three 128-thread CTAs per SM, else line groups like the fast units
  static constexpr bool WHOLE = DIM == 3 && O <= 4;
  static constexpr int NGS = WHOLE ? 1 : NG;
  static constexpr int SMEM = WHOLE ? Lines<O, DIM>::NLOC * 128 * 8 : 0;
};

template <int O, int DIM>
__global__ void __launch_bounds__(128, 3)   // three CTAs per SM (the shared-memory limit)
k_vitems(VPlanDev P, DevBasis b, const double* __restrict__ fin, double* __restrict__ fout,
         long long ld, long long n_cols, const double* __restrict__ speeds, double dt, int bc,
         const long long* __restrict__ lm_ns, const double* __restrict__ lm_mats,
         double* __restrict__ acc, int use_list, unsigned* __restrict__ cnt,
         const unsigned* __restrict__ list_f, const unsigned* __restrict__ list_s) {
  using IG = ItemGroups<O, DIM>;
  extern __shared__ __align__(16) double s_acc[];
  const int lane = threadIdx.x & 31;
  const unsigned n_slow = __ldcg(cnt + 1) / 32u * IG::NGS;
  const unsigned n_units = n_slow + __ldcg(cnt + 0) / 32u * IG::NG;
  const unsigned nc = (unsigned)n_cols;
  for (;;) {
    unsigned u = 0;
    if (lane == 0) {
      fuzz_delay();
      u = atomicAdd(cnt + 2, 1u);
    }
    u = __shfl_sync(~0u, u, 0);
    if (u >= n_units) break;
    const bool slow = u < n_slow;
    const unsigned v = slow ? u : u - n_slow;
    const unsigned ng = slow ? IG::NGS : IG::NG;
    const unsigned chunk = v / ng;
    const int g = (int)(v - chunk * ng);
    const unsigned it = (slow ? list_s : list_f)[chunk * 32u + lane];
    if (it != kNoItem) {
      const unsigned item = it / nc;
      const long long c = it - item * nc;
      const long long e = use_list ? P.gen_entries[item] : (long long)item;
      long long dstride;
      double* dst = item_dst<O, DIM>(P, fout, ld, n_cols, e, c, acc, &dstride);
      if (!slow)
        fast_group<O, DIM, IG::LPG>(P, fin, ld, n_cols, e, c, g, bc, lm_ns, lm_mats, dst,
                                    dstride);
      else if (IG::WHOLE)
        slow_whole<O, DIM>(P, b, fin, ld, e, c, __ldg(speeds + c), dt, bc, dst, dstride,
                           s_acc + threadIdx.x, 128);
      else
        slow_group<O, DIM, IG::LPG>(P, b, fin, ld, e, c, g, __ldg(speeds + c), dt, bc, dst,
                                    dstride);
    }
    __syncwarp();
  }
}

}  // namespace sldg

#include "sweep_stream.cuh"
#include "amr_fused.cuh"

namespace sldg {

// weighted write-back (vsweep.py:403-409): out = ((f_in + S_g1) + S_g2) + ...,
// S_g = sum over the group's contributions in flat order of w (r - f_in).
// Block x = (target cell, group of RPT rows), its contribution list staged in shared
// memory once; block y * blockDim + thread = column.  A thread carries RPT independent
// row sums through the contribution loop (RPT loads in flight per contribution), each
// in the reference's order.
constexpr int kWbMaxC = 32;   // contributions per target staged in shared memory
constexpr int kWbRows = 4;    // rows per thread

template <int NLOC, int RPT>
__global__ void __launch_bounds__(128)
k_writeback(VPlanDev P, const double* __restrict__ fin, double* __restrict__ fout, long long ld,
            long long n_cols, const double* __restrict__ speeds, const double* __restrict__ acc,
            const long long* __restrict__ tlist) {
  constexpr int NRG = (NLOC + RPT - 1) / RPT;
  __shared__ const double* s_src[kWbMaxC];   // acc row 0 of each contribution's slot
  __shared__ int s_grp[kWbMaxC];
  __shared__ double s_w[kWbMaxC];
  const long long tb = blockIdx.x / NRG;
  const long long t = tlist ? tlist[tb] : tb;   // dedup mode: only the targets left
  const int r0 = (int)(blockIdx.x - tb * NRG) * RPT;
  const long long k0 = P.t_off[t];
  const int nk = (int)(P.t_off[t + 1] - k0);
  const int ns = min(nk, kWbMaxC);
  for (int k = threadIdx.x; k < ns; k += blockDim.x) {
    s_src[k] = acc + (long long)P.c_slot[k0 + k] * NLOC * n_cols;
    s_grp[k] = P.c_group[k0 + k];
    s_w[k] = P.c_weight[k0 + k];
  }
  __syncthreads();
  const long long c = (long long)blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= n_cols) return;
  const double* fin_c = fin + P.t_row0[t] * ld + c;
  double* fout_c = fout + P.t_row0[t] * ld + c;
  double fv[RPT], o[RPT], sm[RPT];
#pragma unroll
  for (int rr = 0; rr < RPT; ++rr) {
    const int r = r0 + rr;
    fv[rr] = (r < NLOC) ? fin_c[(long long)r * ld] : 0.0;
    o[rr] = fv[rr];
    sm[rr] = 0.0;
  }
  if (__ldg(speeds + c) != 0.0) {   // exact-zero speed: untouched bits
    int g = s_grp[0];
    // contributions in batches of KB: every slot value of the batch is loaded before
    // the ordered sum consumes them (KB x RPT independent loads in flight per thread)
    constexpr int KB = 4;
    for (int kb = 0; kb < nk; kb += KB) {
      double rv[KB][RPT];
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        const int k = kb + j;
        const bool live = k < nk;
        const double* src = !live ? nullptr
                            : (k < kWbMaxC ? s_src[k]
                                           : acc + (long long)P.c_slot[k0 + k] * NLOC * n_cols) + c;
#pragma unroll
        for (int rr = 0; rr < RPT; ++rr)
          rv[j][rr] = (live && r0 + rr < NLOC) ? __ldcs(src + (long long)(r0 + rr) * n_cols) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        const int k = kb + j;
        if (k >= nk) break;
        const bool sh = k < kWbMaxC;
        const int gk = sh ? s_grp[k] : P.c_group[k0 + k];
        if (gk != g) {
#pragma unroll
          for (int rr = 0; rr < RPT; ++rr) {
            o[rr] = __dadd_rn(o[rr], sm[rr]);
            sm[rr] = 0.0;
          }
          g = gk;
        }
        const double wk = sh ? s_w[k] : P.c_weight[k0 + k];
#pragma unroll
        for (int rr = 0; rr < RPT; ++rr)
          sm[rr] = __dadd_rn(sm[rr], __dmul_rn(wk, __dsub_rn(rv[j][rr], fv[rr])));
      }
    }
#pragma unroll
    for (int rr = 0; rr < RPT; ++rr) o[rr] = __dadd_rn(o[rr], sm[rr]);
  }
#pragma unroll
  for (int rr = 0; rr < RPT; ++rr)
    if (r0 + rr < NLOC) fout_c[(long long)(r0 + rr) * ld] = o[rr];
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct ScratchLayout {
  size_t ns_off, frac_off, mats_off, acc_off, cnt_off, lf_off, ls_off, total;
  long long list_cap;   // slots per worklist (warp-padded per-cell items)
};

static ScratchLayout scratch_layout(const sldg_vplan* p, long long n_cols) {
  ScratchLayout L;
  size_t off = 0;
  L.ns_off = off;
  off = align_up(off + sizeof(long long) * p->dev.n_levels * n_cols, 256);
  L.frac_off = off;
  off = align_up(off + sizeof(double) * p->dev.n_levels * n_cols, 256);
  L.mats_off = off;
  off = align_up(off + sizeof(double) * p->dev.n_levels * 2 * p->o * p->o * n_cols, 256);
  L.acc_off = off;
  off = align_up(off + sizeof(double) * (size_t)p->n_slots * p->n_local * n_cols, 256);
  // per-cell worklists: every (entry, column) of the generic path at most once, in
  // chunks of 32 (one per classifying warp and list)
  L.list_cap = (p->n_entries * n_cols + 31) / 32 * 32;
  L.cnt_off = off;
  off = align_up(off + sizeof(unsigned) * 4, 256);
  L.lf_off = off;
  off = align_up(off + sizeof(unsigned) * (size_t)L.list_cap, 256);
  L.ls_off = off;
  off = align_up(off + sizeof(unsigned) * (size_t)L.list_cap, 256);
  L.total = off;
  return L;
}

template <int O>
static int launch_level_mats(const sldg_vplan* p, const double* speeds, long long n_cols,
                             double dt, long long* ns, double* frac, double* mats,
                             unsigned* wl_cnt, cudaStream_t st) {
  long long n = n_cols * p->dev.n_levels;
  int threads = 128;
  long long blocks = (n + threads - 1) / threads;
  k_level_mats<O><<<(unsigned)blocks, threads, 0, st>>>(p->basis, speeds, n_cols, dt,
                                                       p->dev.base_width, p->dev.n_levels, ns,
                                                       frac, mats, wl_cnt);
  SLDG_LAUNCH_CHECK("k_level_mats");
  return SLDG_OK;
}

template <int O, int DIM>
static int launch_sweep(const sldg_vplan* p, const double* fin, double* fout, long long ld,
                        long long n_cols, const double* speeds, double dt, int bc, int force_slow,
                        const long long* lm_ns, const double* lm_mats, double* acc,
                        unsigned* wl_cnt, unsigned* list_f, unsigned* list_s, cudaStream_t st) {
  constexpr int NLOC = Lines<O, DIM>::NLOC;
  // streaming kernel geometry: whole rows per cell when the tile spans the row
  // (one bulk copy per cell), else column tiles with one bulk copy per row
  const size_t budget = 227 * 1024 - 256;
  const bool al16 = ((((unsigned long long)fin) & 15) == 0) && (ld % 2 == 0);
  int tx_max = 0, whole = 0;
  constexpr int kMaxCols = StreamGeom<O, DIM>::MAX_COLS;
  if (al16 && n_cols == ld && (n_cols + 31) / 32 * 32 <= kMaxCols && (NLOC * n_cols) % 2 == 0 &&
      sizeof(double) * kStreamRing * NLOC * n_cols <= budget) {
    tx_max = (int)n_cols;
    whole = 1;
  } else if (al16 && n_cols % 2 == 0) {
    for (int t = kMaxCols; t >= 32; t -= 32)
      if (sizeof(double) * kStreamRing * NLOC * t <= budget) {
        tx_max = t;
        break;
      }
    if (tx_max > n_cols) tx_max = (int)((n_cols + 31) / 32 * 32);
  }
  const int n_tiles = tx_max > 0 ? (int)((n_cols + tx_max - 1) / tx_max) : 0;
  // the pencil walk runs one CTA per (pencil, column tile), each walking its pencil
  // serially: below one CTA per SM it leaves the GPU idle, and the per-cell worklist
  // (every cell of a whole-fast pencil is a fast item) is the faster schedule
  // SLDG_SWEEP_SCHEDULE=walk|items overrides the choice (tests: both schedules give
  // the same bits)
  const char* sched = std::getenv("SLDG_SWEEP_SCHEDULE");
  const bool fills = sched && !std::strcmp(sched, "walk")    ? true
                     : sched && !std::strcmp(sched, "items") ? false
                                                             : p->n_walk * n_tiles >= num_sms();
  const bool use_stream = !force_slow && p->n_walk > 0 && tx_max > 0 && n_cols >= 2 && fills;
  // duplicate pencils swept once, their targets written directly (SLDG_SWEEP_DEDUP=0 off)
  const char* dd_env = std::getenv("SLDG_SWEEP_DEDUP");
  const bool dd_off = dd_env && dd_env[0] == '0';
  const bool dedup = use_stream && p->n_dd_sets > 0 && !dd_off;
  if (use_stream) {
    const int threads = (tx_max + 31) / 32 * 32 * StreamGeom<O, DIM>::NG;
    const int rstride = whole ? (int)ld : tx_max;
    const size_t smem = sizeof(double) * (size_t)kStreamRing * NLOC * rstride;
    SLDG_CUDA_TRY(smem_limit((const void*)k_sweep_stream<O, DIM>, (int)smem));
    const long long blocks = (dedup ? p->n_walk_dd : p->n_walk) * n_tiles;
    // column tiles: one 2-D tensor copy per cell tile (else one bulk copy per row)
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof(tmap));
    const bool use_tmap =
        !whole && encode_tmap_2d(&tmap, fin, n_cols, p->n_dofs, ld, tx_max, NLOC);
    k_sweep_stream<O, DIM><<<(unsigned)blocks, threads, smem, st>>>(
        p->dev, fin, fout, ld, n_cols, speeds, bc, lm_ns, lm_mats, acc, tx_max, n_tiles, whole,
        dedup ? p->dev.walk_dd : p->dev.walk_pencils, dedup ? 1 : 0, tmap, use_tmap ? 1 : 0);
    SLDG_LAUNCH_CHECK("k_sweep_stream");
  }
  // per-cell entries through the device worklist (classify, then balanced items)
  const long long n_items = use_stream ? p->n_gen : p->n_entries;
  if (n_items > 0) {
    const long long n = n_items * n_cols;
    k_vclassify<O, DIM><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        p->dev, fin, fout, ld, n_cols, speeds, bc, force_slow, lm_ns, acc, n_items,
        use_stream ? 1 : 0, wl_cnt, list_f, list_s);
    SLDG_LAUNCH_CHECK("k_vclassify");
    using IG = ItemGroups<O, DIM>;
    int per_sm = 0;
    SLDG_CUDA_TRY(resident_ctas((const void*)k_vitems<O, DIM>, 128, IG::SMEM, &per_sm));
    const long long max_units = (n + 31) / 32 * IG::NG;   // one list full
    const long long blocks =
        std::max<long long>(1, std::min<long long>((long long)std::max(per_sm, 1) * num_sms(),
                                                   (max_units + 3) / 4));
    k_vitems<O, DIM><<<(unsigned)blocks, 128, IG::SMEM, st>>>(p->dev, p->basis, fin, fout, ld, n_cols,
                                                      speeds, dt, bc, lm_ns, lm_mats, acc,
                                                      use_stream ? 1 : 0, wl_cnt, list_f,
                                                      list_s);
    SLDG_LAUNCH_CHECK("k_vitems");
  }
  const long long n_wb = dedup ? p->n_targets_dd : p->n_targets;
  if (n_wb > 0) {
    constexpr int NRG = (NLOC + kWbRows - 1) / kWbRows;
    const int threads = (int)std::min<long long>(128, (n_cols + 31) / 32 * 32);
    const dim3 grid((unsigned)(n_wb * NRG), (unsigned)((n_cols + threads - 1) / threads));
    k_writeback<NLOC, kWbRows><<<grid, threads, 0, st>>>(p->dev, fin, fout, ld, n_cols, speeds,
                                                          acc, dedup ? p->dev.t_dd : nullptr);
    SLDG_LAUNCH_CHECK("k_writeback");
  }
  return SLDG_OK;
}

// ---- one-pass AMR step (amr_fused.cuh) --------------------------------------------

long long xx_cells_grid(const sldg_xplan* X, long long n_list);   // xfield.cu
int xx_cells_run(const sldg_xplan* X, double* f, long long ld, const long long* cells,
                 long long n_list, const double* w, const double* v0, const double* v2,
                 const double* xw, double* mom_part, double* rho_part, cudaStream_t st);

__global__ void k_amr_fold(const double* __restrict__ part, long long n_parts, long long n,
                           double* __restrict__ out) {   // out[c] = sum_k part[k][c], fixed order
  const int lane = threadIdx.x & 31;
  const long long c = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (c >= n) return;
  double v = 0.0;
  for (long long k = lane; k < n_parts; k += 32) v += part[k * n + c];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) out[c] = v;
}

struct AmrGeom {
  bool ok;
  int ncl, cw, ncx, threads;
  size_t smem;
  long long units, clusters, xx_grid;
  ScratchLayout L;
  size_t o_xcomp, o_xsh, o_mom, o_rho, total;
};

template <int O, int OX>
static AmrGeom amr_geom(const sldg_vplan* p, const sldg_xplan* X, long long n_cols, long long ld) {
  AmrGeom g{};
  g.ok = false;
  if (p->dim != 3 || p->direction != 0 || p->dev.stride_d != 1 || X->vo != O || X->o != OX ||
      n_cols != X->n_cells * OX || ld < n_cols || ld % 2 != 0 || p->n_walk_dd < 1 ||
      X->n_rows != p->n_dofs || X->n_speeds < 1)
    return g;
  const long long n_xc = X->n_cells;
  for (int ncl = 1; ncl <= 8 && !g.ok; ++ncl) {
    if (n_xc % ncl) continue;
    const int ncx = (int)(n_xc / ncl), cw = ncx * OX;
    const int threads = (std::max(cw, O * ncx) + 31) / 32 * 32;
    const size_t smem =
        sizeof(double) * ((size_t)(kAmrRing + 4) * O * cw + 3 * O * XComp<OX>::N);
    if (cw % 2 || threads > 512 || smem > 227 * 1024 - 1024 ||
        3 * threads > kAmrRing * O * cw || O * XComp<OX>::N > 2 * threads)
      continue;
    g.ncl = ncl;
    g.ncx = ncx;
    g.cw = cw;
    g.threads = threads;
    g.smem = smem;
    g.ok = true;
  }
  if (!g.ok) return g;
  g.units = p->n_walk_dd * O * O;
  auto k = k_amr_fused<O, OX>;
  if (smem_limit((const void*)k, (int)g.smem) != cudaSuccess) {
    g.ok = false;
    return g;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)g.ncl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)g.ncl);
  cfg.blockDim = dim3((unsigned)g.threads);
  cfg.dynamicSmemBytes = g.smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, (void*)k, &cfg) != cudaSuccess || nc < 1) {
    cudaGetLastError();
    g.ok = false;
    return g;
  }
  g.clusters = std::min<long long>(nc, g.units);
  g.xx_grid = p->n_rest > 0 ? xx_cells_grid(X, p->n_rest) : 0;
  if (p->n_rest > 0 && g.xx_grid == 0) {
    g.ok = false;
    return g;
  }
  g.L = scratch_layout(p, n_cols);
  size_t off = align_up(g.L.total, 256);
  g.o_xcomp = off;
  off = align_up(off + sizeof(double) * XComp<OX>::N * (size_t)X->n_speeds, 256);
  g.o_xsh = off;   // per entry, per v_x node: x-speed index
  off = align_up(off + sizeof(int) * O * (size_t)p->n_entries, 256);
  g.o_mom = off;
  off = align_up(off + sizeof(double) * 3 * (size_t)(g.clusters * g.ncl + g.xx_grid), 256);
  g.o_rho = off;
  off = align_up(off + sizeof(double) * (size_t)n_cols * (size_t)(g.clusters + g.xx_grid), 256);
  g.total = off;
  return g;
}

// the geometry (occupancy query included) once per plan shape and device: the key holds
// every number amr_geom reads, so a plan reallocated at another shape misses
template <int O, int OX>
static AmrGeom amr_geom_cached(const sldg_vplan* p, const sldg_xplan* X, long long n_cols,
                               long long ld) {
  static std::mutex mu;
  static std::map<std::vector<long long>, AmrGeom> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const std::vector<long long> key = {
      dev, p->dim, p->direction, p->dev.stride_d, p->o, p->n_local,
      p->dev.n_levels, p->n_slots, p->n_entries, p->n_walk_dd, p->n_rest, p->n_dofs,
      X->vo, X->o, X->n_cells, X->n_rows, X->n_speeds, n_cols, ld};
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const AmrGeom g = amr_geom<O, OX>(p, X, n_cols, ld);
  cache[key] = g;
  return g;
}

template <int O, int OX>
static int amr_step(const sldg_vplan* p, const sldg_xplan* X, const double* fin, double* fout,
                    long long ld, long long n_cols, const double* speeds, double dt, int bc,
                    const double* w, const double* v0, const double* v2, const double* xw,
                    double* mom_out3, double* rho_out, void* scratch, cudaStream_t st,
                    size_t* bytes) {
  const AmrGeom g = amr_geom_cached<O, OX>(p, X, n_cols, ld);
  if (!g.ok) {
    set_error("one-pass AMR step: unsupported plan / geometry");
    return SLDG_ERR_UNSUPPORTED;
  }
  if (bytes) {
    *bytes = g.total;
    return SLDG_OK;
  }
  constexpr int NLOC = O * O * O;
  unsigned char* sb = (unsigned char*)scratch;
  const ScratchLayout& L = g.L;
  long long* lm_ns = (long long*)(sb + L.ns_off);
  double* lm_frac = (double*)(sb + L.frac_off);
  double* lm_mats = (double*)(sb + L.mats_off);
  double* acc = (double*)(sb + L.acc_off);
  unsigned* wl_cnt = (unsigned*)(sb + L.cnt_off);
  unsigned* list_f = (unsigned*)(sb + L.lf_off);
  unsigned* list_s = (unsigned*)(sb + L.ls_off);
  double* xcomp = (double*)(sb + g.o_xcomp);
  int* e_xg = (int*)(sb + g.o_xsh);
  double* mom_part = (double*)(sb + g.o_mom);
  double* rho_part = (double*)(sb + g.o_rho);
  if (L.list_cap >= (long long)kNoItem) {
    set_error("amr step: entries x columns exceed the 32-bit worklist index");
    return SLDG_ERR_UNSUPPORTED;
  }
  int rc = launch_level_mats<O>(p, speeds, n_cols, dt, lm_ns, lm_frac, lm_mats, wl_cnt, st);
  if (rc) return rc;
  k_xcomp<OX><<<(unsigned)((X->n_speeds + 127) / 128), 128, 0, st>>>(X->dev, xw, X->n_speeds,
                                                                     xcomp);
  SLDG_LAUNCH_CHECK("k_xcomp");
  k_entry_speeds<O><<<(unsigned)((p->n_entries * O + 255) / 256), 256, 0, st>>>(
      p->dev, X->dev.row_speed, p->n_entries, e_xg);
  SLDG_LAUNCH_CHECK("k_entry_speeds");
  // cells outside the walk: the per-cell worklist (v only), as launch_sweep's walk mode
  if (p->n_gen > 0) {
    const long long n = p->n_gen * n_cols;
    k_vclassify<O, 3><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        p->dev, fin, fout, ld, n_cols, speeds, bc, 0, lm_ns, acc, p->n_gen, 1, wl_cnt, list_f,
        list_s);
    SLDG_LAUNCH_CHECK("k_vclassify");
    using IG = ItemGroups<O, 3>;
    int per_sm = 0;
    SLDG_CUDA_TRY(resident_ctas((const void*)k_vitems<O, 3>, 128, IG::SMEM, &per_sm));
    const long long max_units = (n + 31) / 32 * IG::NG;
    const long long blocks =
        std::max<long long>(1, std::min<long long>((long long)std::max(per_sm, 1) * num_sms(),
                                                   (max_units + 3) / 4));
    k_vitems<O, 3><<<(unsigned)blocks, 128, IG::SMEM, st>>>(p->dev, p->basis, fin, fout, ld,
                                                           n_cols, speeds, dt, bc, lm_ns,
                                                           lm_mats, acc, 1, wl_cnt, list_f,
                                                           list_s);
    SLDG_LAUNCH_CHECK("k_vitems");
  }
  // the walk: V + X.X in one pass for its direct rows
  {
    const AmrEpi ep{w, v0, v2, xcomp, e_xg, mom_part, rho_part};
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)g.ncl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)(g.clusters * g.ncl));
    cfg.blockDim = dim3((unsigned)g.threads);
    cfg.dynamicSmemBytes = g.smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    SLDG_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_amr_fused<O, OX>, p->dev, fin, fout, ld, (int)n_cols,
                                     (int)X->n_cells, speeds, bc, (const long long*)lm_ns,
                                     (const double*)lm_mats, acc, ep, g.units));
    SLDG_LAUNCH_CHECK("k_amr_fused");
  }
  // weighted targets (dedup mode: the ones the walk did not finish)
  if (p->n_targets_dd > 0) {
    constexpr int NRG = (NLOC + kWbRows - 1) / kWbRows;
    const int threads = (int)std::min<long long>(128, (n_cols + 31) / 32 * 32);
    const dim3 grid((unsigned)(p->n_targets_dd * NRG), (unsigned)((n_cols + threads - 1) / threads));
    k_writeback<NLOC, kWbRows><<<grid, threads, 0, st>>>(p->dev, fin, fout, ld, n_cols, speeds,
                                                          acc, p->dev.t_dd);
    SLDG_LAUNCH_CHECK("k_writeback");
  }
  // X.X of the rest, in place, partials after the walk's
  rc = xx_cells_run(X, fout, ld, p->dev.rest_cells, p->n_rest, w, v0, v2, xw,
                    mom_part + 3 * g.clusters * g.ncl, rho_part + g.clusters * n_cols, st);
  if (rc) return rc;
  k_amr_fold<<<1, 96, 0, st>>>(mom_part, g.clusters * g.ncl + g.xx_grid, 3, mom_out3);
  SLDG_LAUNCH_CHECK("k_amr_fold");
  k_amr_fold<<<(unsigned)((n_cols * 32 + 255) / 256), 256, 0, st>>>(
      rho_part, g.clusters + g.xx_grid, n_cols, rho_out);
  SLDG_LAUNCH_CHECK("k_amr_fold");
  return SLDG_OK;
}

static int amr_dispatch(const sldg_vplan* p, const sldg_xplan* X, const double* fin, double* fout,
                        long long ld, long long n_cols, const double* speeds, double dt, int bc,
                        const double* w, const double* v0, const double* v2, const double* xw,
                        double* mom_out3, double* rho_out, void* scratch, cudaStream_t st,
                        size_t* bytes) {
  switch (p->o * 10 + X->o) {
#define CASE(A, B)                                                                          \
  case A * 10 + B:                                                                          \
    return amr_step<A, B>(p, X, fin, fout, ld, n_cols, speeds, dt, bc, w, v0, v2, xw,       \
                          mom_out3, rho_out, scratch, st, bytes);
    CASE(2, 2) CASE(2, 3) CASE(2, 4) CASE(3, 2) CASE(3, 3) CASE(3, 4) CASE(4, 2) CASE(4, 3)
    CASE(4, 4)
#undef CASE
  }
  set_error("one-pass AMR step: unsupported degrees");
  return SLDG_ERR_UNSUPPORTED;
}

// generalized_overlap (vsweep.py:98-122) for one (destination, source) pair: the
// slow path's own block routine, one thread
template <int O>
__global__ void k_generalized_overlap(DevBasis b, double vl, double vr, double dlo, double dw,
                                      double slo, double sw, double de, double* __restrict__ M) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double m[O * O];
  general_block<O>(b, vl, vr, dlo, dw, slo, sw, de, m);
#pragma unroll
  for (int k = 0; k < O * O; ++k) M[k] = m[k];
}

}  // namespace sldg

using namespace sldg;

extern "C" {

int sldg_generalized_overlap(const SldgBasis* basis, double vl, double vr, double dest_lo,
                             double dest_width, double src_lo, double src_width,
                             double displacement, double* matrix, void* stream) {
  DevBasis b;
  std::string err;
  if (!basis || !make_dev_basis(*basis, &b, &err)) {
    set_error(basis ? err : "null basis");
    return SLDG_ERR_ARG;
  }
  if (!matrix || !(dest_width > 0.0) || !(src_width > 0.0) || !(vr > vl)) {
    set_error("bad generalized_overlap arguments");
    return SLDG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  switch (b.o) {
#define CASE(O)                                                                             \
  case O:                                                                                   \
    k_generalized_overlap<O><<<1, 32, 0, st>>>(b, vl, vr, dest_lo, dest_width, src_lo,     \
                                               src_width, displacement, matrix);            \
    break;
    CASE(2) CASE(3) CASE(4) CASE(5) CASE(6)
#undef CASE
    default:
      set_error("generalized_overlap: degree 1..5");
      return SLDG_ERR_UNSUPPORTED;
  }
  SLDG_LAUNCH_CHECK("k_generalized_overlap");
  return SLDG_OK;
}

int sldg_vplan_create(const SldgVPlanDesc* d, sldg_vplan** out) {
  if (!d || !out) {
    set_error("null argument");
    return SLDG_ERR_ARG;
  }
  *out = nullptr;
  DevBasis basis;
  std::string err;
  if (!make_dev_basis(d->basis, &basis, &err)) {
    set_error(err);
    return SLDG_ERR_ARG;
  }
  if (d->dim != 1 && d->dim != 3) {
    set_error("dim must be 1 or 3");
    return SLDG_ERR_ARG;
  }
  if (d->direction < 0 || d->direction >= d->dim) {
    set_error("direction out of range");
    return SLDG_ERR_ARG;
  }
  if (d->n_pencils < 1 || d->n_cells < 1 || d->n_levels < 1 || d->n_levels > 30) {
    set_error("empty plan");
    return SLDG_ERR_ARG;
  }
  const int o = basis.o;
  const int nl = d->dim == 3 ? o * o : 1;
  const int nloc = nl * o;
  const long long P = d->n_pencils;
  const long long E = d->pencil_offsets[P];
  if (d->pencil_offsets[0] != 0 || E < 1) {
    set_error("bad pencil offsets");
    return SLDG_ERR_PLAN;
  }
  // host-side derived arrays
  std::vector<long long> p_off(P);
  std::vector<int> p_n(P);
  std::vector<unsigned char> p_fast(P);
  std::vector<int> e_pencil(E), e_level(E), e_runs(4 * E), e_slot(E, -1);
  std::vector<long long> e_row0(E);
  std::vector<unsigned char> e_conf(E);
  std::vector<long long> cover(d->n_cells, 0);
  int max_cells = 0;
  for (long long q = 0; q < P; ++q) {
    long long a = d->pencil_offsets[q], b = d->pencil_offsets[q + 1];
    if (b <= a) {
      set_error("empty pencil");
      return SLDG_ERR_PLAN;
    }
    int n = (int)(b - a);
    max_cells = std::max(max_cells, n);
    p_off[q] = a;
    p_n[q] = n;
    bool allconf = true, onelev = true;
    for (long long e = a; e < b; ++e) {
      long long cid = d->cell_ids[e];
      if (cid < 0 || cid >= d->n_cells) {
        set_error("cell id out of range");
        return SLDG_ERR_PLAN;
      }
      cover[cid] += 1;
      e_pencil[e] = (int)q;
      e_row0[e] = cid * nloc;
      e_level[e] = (int)d->levels[e];
      if (e_level[e] < 0 || e_level[e] >= d->n_levels) {
        set_error("level out of range");
        return SLDG_ERR_PLAN;
      }
      e_conf[e] = d->conforming[e] ? 1 : 0;
      allconf = allconf && e_conf[e];
      onelev = onelev && (d->levels[e] == d->levels[a]);
    }
    p_fast[q] = (allconf && onelev) ? 1 : 0;
    // same-level runs: linear (absorbing) and circular (periodic)
    for (int s = 0; s < n; ++s) {
      long long lv = d->levels[a + s];
      int ln = 0;
      while (s - ln - 1 >= 0 && d->levels[a + s - ln - 1] == lv) ++ln;
      int rn = 0;
      while (s + rn + 1 < n && d->levels[a + s + rn + 1] == lv) ++rn;
      int lc = 0;
      while (lc < n && d->levels[a + ((s - lc - 1) % n + n) % n] == lv) ++lc;
      int rc = 0;
      while (rc < n && d->levels[a + (s + rc + 1) % n] == lv) ++rc;
      e_runs[4 * (a + s) + 0] = lc;
      e_runs[4 * (a + s) + 1] = rc;
      e_runs[4 * (a + s) + 2] = ln;
      e_runs[4 * (a + s) + 3] = rn;
    }
  }
  for (long long cidx = 0; cidx < d->n_cells; ++cidx)
    if (cover[cidx] == 0) {
      set_error("sweep plan leaves velocity DOFs uncovered (cell " + std::to_string(cidx) + ")");
      return SLDG_ERR_PLAN;
    }
  // weighted entries -> scratch slots; targets grouped by cell in entry (plan) order
  long long n_slots = 0;
  std::map<long long, std::vector<long long>> contrib;   // cell -> entries
  for (long long e = 0; e < E; ++e) {
    if (d->weights[e] != 1.0) {
      e_slot[e] = (int)n_slots++;
      contrib[d->cell_ids[e]].push_back(e);
    }
  }
  std::vector<long long> t_row0, t_off;
  std::vector<int> c_slot, c_group;
  std::vector<double> c_weight;
  t_off.push_back(0);
  for (auto& kv : contrib) {
    t_row0.push_back(kv.first * nloc);
    for (long long e : kv.second) {
      c_slot.push_back(e_slot[e]);
      c_group.push_back((int)d->pencil_group[e_pencil[e]]);
      c_weight.push_back(d->weights[e]);
    }
    t_off.push_back((long long)c_slot.size());
  }
  // a cell must not be both a copy target and a weighted target
  for (long long e = 0; e < E; ++e)
    if (d->weights[e] == 1.0 && contrib.count(d->cell_ids[e])) {
      set_error("cell mixes unit and fractional weights");
      return SLDG_ERR_PLAN;
    }
  std::vector<long long> walk, gen, walk_desc;
  int max_walk = 0;
  for (long long q = 0; q < P; ++q) {
    if (p_fast[q]) {
      walk.push_back(q);
      walk_desc.push_back(p_off[q]);
      walk_desc.push_back((long long)p_n[q] | ((long long)e_level[p_off[q]] << 32));
      max_walk = std::max(max_walk, p_n[q]);
    } else {
      for (long long e = p_off[q]; e < p_off[q] + p_n[q]; ++e) gen.push_back(e);
    }
  }
  const long long T = (long long)t_row0.size();
  const long long K = (long long)c_slot.size();
  // Duplicate whole-fast pencils: identical cell lists (a coarse transverse column split by
  // the global transverse edges of finer cells elsewhere) give bit-identical sweep results,
  // so when every cell of the set lies in exactly those pencils the weighted write-back
  // f + sum_k w_k (r_k - f) (vsweep.py:403-409, one group, plan order) can be formed from
  // ONE sweep of the first pencil.  The walk then skips the others; the write-back keeps
  // only the targets outside such sets.  (Used when the walk runs; the worklist schedules
  // and force_slow keep the plain slots.)
  std::vector<int> e_dd(E, -1);
  std::vector<long long> dd_off(1, 0), walk_dd;
  std::vector<double> dd_w;
  std::vector<unsigned char> skip(P, 0), t_dedup(T, 0);
  long long n_dd_sets = 0;
  {
    std::map<std::vector<long long>, std::vector<long long>> sets;
    for (long long q : walk)
      sets[std::vector<long long>(d->cell_ids + p_off[q], d->cell_ids + p_off[q] + p_n[q])]
          .push_back(q);
    std::map<long long, long long> t_of_cell;
    for (long long t = 0; t < T; ++t) t_of_cell[t_row0[t] / nloc] = t;
    for (auto& kv : sets) {
      const std::vector<long long>& qs = kv.second;   // plan order (walk order)
      const long long dn = (long long)qs.size();
      if (dn < 2) continue;
      bool full = true;
      for (long long cid : kv.first) full = full && cover[cid] == dn;
      if (!full) continue;
      ++n_dd_sets;
      const long long rep = qs[0];
      for (int s = 0; s < p_n[rep]; ++s) {
        e_dd[p_off[rep] + s] = (int)(dd_off.size() - 1);
        for (long long q : qs) dd_w.push_back(d->weights[p_off[q] + s]);
        dd_off.push_back((long long)dd_w.size());
        t_dedup[t_of_cell.at(kv.first[s])] = 1;
      }
      for (size_t j = 1; j < qs.size(); ++j) skip[qs[j]] = 1;
    }
  }
  std::vector<long long> walk_dd_desc;
  for (long long q : walk)
    if (!skip[q]) {
      walk_dd.push_back(q);
      walk_dd_desc.push_back(p_off[q]);
      walk_dd_desc.push_back((long long)p_n[q] | ((long long)e_level[p_off[q]] << 32));
    }
  std::vector<long long> t_dd;
  for (long long t = 0; t < T; ++t)
    if (!t_dedup[t]) t_dd.push_back(t);
  if (dd_w.empty()) dd_w.push_back(0.0);
  std::vector<long long> rest;
  for (long long e : gen)
    if (e_slot[e] < 0) rest.push_back(e_row0[e] / nloc);
  for (long long t : t_dd) rest.push_back(t_row0[t] / nloc);
  std::sort(rest.begin(), rest.end());

  // one device allocation, carved
  struct Piece {
    const void* src;
    size_t bytes;
    void** dst;
  };
  sldg_vplan* p = new sldg_vplan();
  std::memset(&p->dev, 0, sizeof(p->dev));
  std::vector<Piece> pieces = {
      {p_off.data(), sizeof(long long) * P, (void**)&p->dev.p_off},
      {p_n.data(), sizeof(int) * P, (void**)&p->dev.p_n},
      {p_fast.data(), (size_t)P, (void**)&p->dev.p_fast},
      {e_pencil.data(), sizeof(int) * E, (void**)&p->dev.e_pencil},
      {e_row0.data(), sizeof(long long) * E, (void**)&p->dev.e_row0},
      {d->lowers, sizeof(double) * E, (void**)&p->dev.e_lower},
      {d->widths, sizeof(double) * E, (void**)&p->dev.e_width},
      {e_level.data(), sizeof(int) * E, (void**)&p->dev.e_level},
      {e_conf.data(), (size_t)E, (void**)&p->dev.e_conf},
      {e_runs.data(), sizeof(int) * 4 * E, (void**)&p->dev.e_runs},
      {e_slot.data(), sizeof(int) * E, (void**)&p->dev.e_slot},
      {t_row0.data(), sizeof(long long) * T, (void**)&p->dev.t_row0},
      {t_off.data(), sizeof(long long) * (T + 1), (void**)&p->dev.t_off},
      {c_slot.data(), sizeof(int) * K, (void**)&p->dev.c_slot},
      {c_group.data(), sizeof(int) * K, (void**)&p->dev.c_group},
      {c_weight.data(), sizeof(double) * K, (void**)&p->dev.c_weight},
      {walk.data(), sizeof(long long) * walk.size(), (void**)&p->dev.walk_pencils},
      {walk_desc.data(), sizeof(long long) * walk_desc.size(), (void**)&p->dev.walk_desc},
      {gen.data(), sizeof(long long) * gen.size(), (void**)&p->dev.gen_entries},
      {e_dd.data(), sizeof(int) * E, (void**)&p->dev.e_dd},
      {dd_off.data(), sizeof(long long) * dd_off.size(), (void**)&p->dev.dd_off},
      {dd_w.data(), sizeof(double) * dd_w.size(), (void**)&p->dev.dd_w},
      {walk_dd.data(), sizeof(long long) * walk_dd.size(), (void**)&p->dev.walk_dd},
      {t_dd.data(), sizeof(long long) * t_dd.size(), (void**)&p->dev.t_dd},
      {rest.data(), sizeof(long long) * rest.size(), (void**)&p->dev.rest_cells},
      {walk_dd_desc.data(), sizeof(long long) * walk_dd_desc.size(),
       (void**)&p->dev.walk_dd_desc},
  };
  size_t total = 0;
  for (auto& pc : pieces) total = align_up(total + pc.bytes, 256);
  std::vector<unsigned char> host(total, 0);
  size_t off = 0;
  std::vector<size_t> offs;
  for (auto& pc : pieces) {
    if (pc.bytes) std::memcpy(host.data() + off, pc.src, pc.bytes);
    offs.push_back(off);
    off = align_up(off + pc.bytes, 256);
  }
  cudaError_t ce = cudaMalloc(&p->block, std::max<size_t>(total, 256));
  if (ce != cudaSuccess) {
    delete p;
    return cuda_fail(ce, "cudaMalloc(vplan)");
  }
  ce = cudaMemcpy(p->block, host.data(), total, cudaMemcpyHostToDevice);
  if (ce != cudaSuccess) {
    cudaFree(p->block);
    delete p;
    return cuda_fail(ce, "cudaMemcpy(vplan)");
  }
  for (size_t i = 0; i < pieces.size(); ++i)
    *pieces[i].dst = (unsigned char*)p->block + offs[i];
  p->basis = basis;
  p->dim = d->dim;
  p->direction = d->direction;
  p->o = o;
  p->n_lines = nl;
  p->n_local = nloc;
  p->n_cells = d->n_cells;
  p->n_pencils = P;
  p->n_entries = E;
  p->n_slots = n_slots;
  p->n_targets = T;
  p->n_walk = (long long)walk.size();
  p->n_gen = (long long)gen.size();
  p->n_dd_sets = n_dd_sets;
  p->n_walk_dd = (long long)walk_dd.size();
  p->n_targets_dd = (long long)t_dd.size();
  p->n_rest = (long long)rest.size();
  p->n_dofs = d->n_cells * nloc;
  p->max_pencil_cells = max_cells;
  p->max_walk_cells = max_walk;
  int pw[3] = {1, o, o * o};
  int td[2];
  int k = 0;
  for (int t = 0; t < 3; ++t)
    if (t != d->direction) td[k++] = t;
  p->dev.stride_d = pw[d->direction];
  p->dev.stride_t0 = d->dim == 3 ? pw[td[0]] : 0;
  p->dev.stride_t1 = d->dim == 3 ? pw[td[1]] : 0;
  p->dev.n_entries = E;
  p->dev.n_targets = T;
  p->dev.n_walk = p->n_walk;
  p->dev.n_gen = p->n_gen;
  p->dev.n_walk_dd = p->n_walk_dd;
  p->dev.n_targets_dd = p->n_targets_dd;
  p->dev.n_levels = d->n_levels;
  p->dev.radius = d->radius;
  p->dev.base_width = d->base_width;
  *out = p;
  return SLDG_OK;
}

int sldg_vplan_destroy(sldg_vplan* p) {
  if (!p) return SLDG_OK;
  if (p->block) cudaFree(p->block);
  delete p;
  return SLDG_OK;
}

int sldg_vplan_scratch_bytes(const sldg_vplan* p, int64_t n_cols, size_t* bytes) {
  if (!p || !bytes || n_cols < 0) {
    set_error("bad argument");
    return SLDG_ERR_ARG;
  }
  *bytes = scratch_layout(p, n_cols).total;
  return SLDG_OK;
}

int sldg_vplan_info(const sldg_vplan* p, int64_t* info) {
  if (!p || !info) {
    set_error("bad argument");
    return SLDG_ERR_ARG;
  }
  info[0] = p->n_entries;
  info[1] = p->n_slots;
  info[2] = p->n_targets;
  info[3] = p->n_walk;
  info[4] = p->n_dofs;
  return SLDG_OK;
}

int sldg_level_matrices(const sldg_vplan* p, const double* speeds, int64_t n_cols, double dt,
                          int64_t* n_shift, double* frac, double* mats, void* stream) {
  if (!p || !speeds || !n_shift || !mats || n_cols < 1 || !(dt > 0.0)) {
    set_error("bad argument");
    return SLDG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  switch (p->o) {
#define CASE(O) \
  case O:                                                                               \
    return launch_level_mats<O>(p, speeds, n_cols, dt, (long long*)n_shift, frac, mats,     \
                                nullptr, st);
    CASE(2) CASE(3) CASE(4) CASE(5) CASE(6)
#undef CASE
  }
  set_error("unsupported degree");
  return SLDG_ERR_UNSUPPORTED;
}

int sldg_amr_step_query(const sldg_vplan* p, const sldg_xplan* X, int64_t n_cols, int64_t ld,
                        size_t* scratch_bytes) {
  if (!p || !X || !scratch_bytes || n_cols < 1) {
    set_error("bad amr_step_query arguments");
    return SLDG_ERR_ARG;
  }
  return amr_dispatch(p, X, nullptr, nullptr, ld, n_cols, nullptr, 1.0, SLDG_BC_ABSORBING,
                      nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                      scratch_bytes);
}

int sldg_amr_step(const sldg_vplan* p, const sldg_xplan* X, const double* fin, double* fout,
                  int64_t ld, int64_t n_cols, const double* speeds, double dt, int32_t bc,
                  const double* w, const double* v0, const double* v2, const double* xw,
                  double* mom_out3, double* rho_out, void* scratch, void* stream) {
  if (!p || !X || !fin || !fout || fin == fout || !speeds || !w || !v0 || !v2 || !xw ||
      !mom_out3 || !rho_out || !scratch || n_cols < 1 || ld < n_cols) {
    set_error("bad amr_step arguments (f_in and f_out must be distinct device buffers)");
    return SLDG_ERR_ARG;
  }
  if (bc != SLDG_BC_PERIODIC && bc != SLDG_BC_ABSORBING) {
    set_error("boundary mode must be 'periodic' or 'absorbing'");
    return SLDG_ERR_ARG;
  }
  if (!(dt > 0.0)) {
    set_error("time step must be positive");
    return SLDG_ERR_ARG;
  }
  return amr_dispatch(p, X, fin, fout, ld, n_cols, speeds, dt, bc, w, v0, v2, xw, mom_out3,
                      rho_out, scratch, (cudaStream_t)stream, nullptr);
}

int sldg_advect_v(const sldg_vplan* p, const double* fin, double* fout, int64_t ld,
                  int64_t n_cols, const double* speeds, double dt, int32_t bc,
                  int32_t force_slow, void* scratch, void* stream) {
  if (!p) {
    set_error("null plan");
    return SLDG_ERR_ARG;
  }
  if (bc != SLDG_BC_PERIODIC && bc != SLDG_BC_ABSORBING) {
    set_error("boundary mode must be 'periodic' or 'absorbing'");
    return SLDG_ERR_ARG;
  }
  if (n_cols == 0) return SLDG_OK;
  if (!fin || !fout || !speeds || n_cols < 0 || ld < n_cols || fin == fout) {
    set_error("bad field / speeds arguments (f_in and f_out must be distinct device buffers)");
    return SLDG_ERR_ARG;
  }
  if (!(dt > 0.0)) {
    set_error("time step must be positive");
    return SLDG_ERR_ARG;
  }
  ScratchLayout L = scratch_layout(p, n_cols);
  if (!scratch) {
    set_error("scratch buffer required");
    return SLDG_ERR_ARG;
  }
  unsigned char* sb = (unsigned char*)scratch;
  long long* lm_ns = (long long*)(sb + L.ns_off);
  double* lm_frac = (double*)(sb + L.frac_off);
  double* lm_mats = (double*)(sb + L.mats_off);
  double* acc = (double*)(sb + L.acc_off);
  unsigned* wl_cnt = (unsigned*)(sb + L.cnt_off);
  unsigned* list_f = (unsigned*)(sb + L.lf_off);
  unsigned* list_s = (unsigned*)(sb + L.ls_off);
  if (L.list_cap >= (long long)kNoItem) {
    set_error("advect_v: entries x columns exceed the 32-bit worklist index");
    return SLDG_ERR_UNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int rc = SLDG_ERR_UNSUPPORTED;
  switch (p->o) {
#define CASE(O)                                                                               \
  case O:                                                                                     \
    rc = launch_level_mats<O>(p, speeds, n_cols, dt, lm_ns, lm_frac, lm_mats, wl_cnt, st);    \
    if (rc) return rc;                                                                        \
    if (p->dim == 3)                                                                          \
      return launch_sweep<O, 3>(p, fin, fout, ld, n_cols, speeds, dt, bc, force_slow, lm_ns,  \
                                lm_mats, acc, wl_cnt, list_f, list_s, st);                    \
    return launch_sweep<O, 1>(p, fin, fout, ld, n_cols, speeds, dt, bc, force_slow, lm_ns,    \
                              lm_mats, acc, wl_cnt, list_f, list_s, st);
    CASE(2) CASE(3) CASE(4) CASE(5) CASE(6)
#undef CASE
  }
  set_error("unsupported degree");
  return rc;
}

}  // extern "C"
