// sweep_stream.cuh -- streaming whole-pencil fast path of the v-sweep (included by vsweep.cu).
//
// Replaces the whole-pencil fast path of sweep_pencil (vsweep.py:197-200 ->
// apply_update, sldg1d.py:124-136) for every pencil whose cells are all
// conforming and on one level.  One CTA owns one pencil x one tile of up to
// 256 x-columns; thread = column.  Each thread keeps its column's level
// matrices A, B (2 o^2 fp64) in registers for the whole pencil.
//
// HBM streaming.  For direction 0 a cell's (p+1)^dim velocity rows are
// consecutive rows of f, so a cell tile is (p+1)^dim rows x TX columns: when
// the tile spans the full row (TX == ld) it is ONE contiguous block and is
// fetched with ONE cp.async.bulk (the TMA engine, no per-thread address
// generation); otherwise with ONE 2-D tensor copy (a tensor map over f, box
// (p+1)^dim rows x TX columns), or one bulk copy per row when no map could be
// encoded.  Cells stream in pencil
// order through a 4-slot ring tracked by mbarriers (transaction bytes), two
// cells ahead of the compute, so every input coefficient is read from HBM
// exactly once (absorbing bc; periodic re-reads the two wrap cells).  Outputs
// go from registers to HBM with coalesced 8-byte stores (a warp writes 256
// contiguous bytes per row).
//
// Valid when every active column of the tile has n_shift in {-1, 0} (all
// Landau shifts; checked per tile): cell s then needs cells s-1, s, s+1.
//
// Line groups.  A Q3 cell (64 rows) leaves room for only 96 columns in the ring,
// i.e. 3 warps per SM -- too few to cover the two-cell update's FMA chains and the
// HBM latency (cfg4L: 7.2 ms for 13 GB).  From Q3 up, StreamGeom::NG = O threads
// share one column, each taking every O-th of the cell's O^2 lines (same arithmetic per
// output, so the same bits); they all hold the column's A, B.
#pragma once

#include <type_traits>

#include "tma_util.cuh"

namespace sldg {

constexpr int kStreamRing = 4;

template <int O, int DIM>
struct StreamGeom {
  static constexpr int NG = (DIM == 3 && O >= 4) ? O : 1;   // divides the O^2 lines
  static constexpr int MAX_THREADS = NG == 4 ? 384 : 256;     // register budget (no spills)
#ifdef SLDG_STREAM_COLS
  static constexpr int MAX_COLS = NG > 1 ? SLDG_STREAM_COLS : 256;
#else
  static constexpr int MAX_COLS = MAX_THREADS / NG / 32 * 32;   // column tile cap
#endif
};

template <int O, int DIM>
__global__ void __launch_bounds__(StreamGeom<O, DIM>::MAX_THREADS, 1)
k_sweep_stream(VPlanDev P, const double* __restrict__ fin, double* __restrict__ fout,
               long long ld, long long n_cols, const double* __restrict__ speeds, int bc,
               const long long* __restrict__ lm_ns, const double* __restrict__ lm_mats,
               double* __restrict__ acc, int tx_max, int n_tiles, int whole_rows,
               const long long* __restrict__ walk, int dedup,
               const __grid_constant__ CUtensorMap tmap, int use_tmap) {
  constexpr int NL = (DIM == 3) ? O * O : 1;
  constexpr int NLOC = NL * O;
  constexpr int NG = StreamGeom<O, DIM>::NG;
  constexpr int NT = NL / NG;   // lines per thread
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) unsigned long long full[kStreamRing];
  __shared__ int s_nsmin, s_nsmax;

  const long long wp = blockIdx.x / n_tiles;
  const int tile = (int)(blockIdx.x - wp * n_tiles);
  const long long q = walk[wp];
  const long long off = P.p_off[q];
  const int n = P.p_n[q];
  const long long c0 = (long long)tile * tx_max;
  const int tx = (int)min((long long)tx_max, n_cols - c0);
  const int tid = threadIdx.x;
  const int tpad = (int)blockDim.x / NG;   // columns per line group (multiple of 32)
  const int g = tid / tpad;                // line group
  const int col = tid - g * tpad;
  const int lev = P.e_level[off];
  const int rstride = whole_rows ? (int)ld : tx_max;   // smem row stride (doubles)
  const int cell_dbl = NLOC * rstride;
  const unsigned cell_bytes = (unsigned)(NLOC * tx) * 8u;

  if (tid == 0) {
    s_nsmin = 1 << 30;
    s_nsmax = -(1 << 30);
    for (int k = 0; k < kStreamRing; ++k) mbar_init(&full[k], 1);
    mbar_fence_init();
  }
  sync_fz();
  const bool colv = col < tx;
  const long long c = c0 + col;
  const double speed = colv ? __ldg(speeds + c) : 0.0;
  const long long ns = colv ? lm_ns[(long long)lev * n_cols + c] : 0;
  if (colv && g == 0 && speed != 0.0) {
    const int nsi = (int)max(min(ns, (long long)(1 << 29)), -(long long)(1 << 29));
    atomicMin(&s_nsmin, nsi);
    atomicMax(&s_nsmax, nsi);
  }
  sync_fz();
  const bool streamable = (s_nsmin >= -1 && s_nsmax <= 0) || (s_nsmin > s_nsmax);

  double A[O * O], B[O * O];
  if (colv) load_pair<O>(lm_mats, lev, n_cols, c, A, B);
  // the weighted write-back of a deduplicated target (k_writeback's arithmetic for
  // identical contributions y): fv + ((0 + w1 (y - fv)) + w2 (y - fv) + ...)
  auto dd_value = [&](int dd, double y, double fv) -> double {
    const long long k0 = P.dd_off[dd], k1 = P.dd_off[dd + 1];
    const double df = __dsub_rn(y, fv);
    double sm = 0.0;
    for (long long k = k0; k < k1; ++k) sm = __dadd_rn(sm, __dmul_rn(__ldg(P.dd_w + k), df));
    return __dadd_rn(fv, sm);
  };

  if (!streamable) {
    // arbitrary shifts in this tile: direct loads from HBM (same arithmetic)
    if (!colv) return;
    for (int s = 0; s < n; ++s) {
      const long long e = off + s;
      const int dd = dedup ? P.e_dd[e] : -1;
      const int slot = dd >= 0 ? -1 : P.e_slot[e];
      double* dst = slot < 0 ? fout + P.e_row0[e] * ld + c : acc + (long long)slot * NLOC * n_cols + c;
      const long long dstride = slot < 0 ? ld : n_cols;
      const double* self = fin + P.e_row0[e] * ld + c;
      if (speed == 0.0) {
        for (int r = g; r < NLOC; r += NG) dst[r * dstride] = self[r * ld];
        continue;
      }
      long long qa = s - ns, qb = s - ns - 1;
      bool va = true, vb = true;
      if (bc == SLDG_BC_PERIODIC) { qa = pymod(qa, n); qb = pymod(qb, n); }
      else { va = qa >= 0 && qa < n; vb = qb >= 0 && qb < n; }
      const double* pa = fin + (va ? P.e_row0[off + qa] : 0) * ld + c;
      const double* pb = fin + (vb ? P.e_row0[off + qb] : 0) * ld + c;
      for (int t = g; t < NL; t += NG) {
        double ua[O], ub[O], y[O];
#pragma unroll
        for (int i = 0; i < O; ++i) {
          const int r = Lines<O, DIM>::row(P, t, i);
          ua[i] = va ? pa[(long long)r * ld] : 0.0;
          ub[i] = vb ? pb[(long long)r * ld] : 0.0;
        }
        two_cell<O>(A, B, ua, ub, va, vb, y);
#pragma unroll
        for (int i = 0; i < O; ++i) {
          const long long r = Lines<O, DIM>::row(P, t, i);
          dst[r * dstride] = dd >= 0 ? dd_value(dd, y[i], self[r * ld]) : y[i];
        }
      }
    }
    return;
  }

  // load list: virtual cells v = -1 .. n (periodic) or 0 .. n-1 (absorbing); list
  // position k holds virtual cell v0 + k in ring slot k % kStreamRing
  const bool per = (bc == SLDG_BC_PERIODIC);
  const int v0 = per ? -1 : 0;
  const int n_load = per ? n + 2 : n;
  auto row_of = [&](int k) {   // first f row of list position k
    const int v = v0 + k;
    return P.e_row0[off + (v < 0 ? n - 1 : (v >= n ? 0 : v))];
  };
  auto issue = [&](int k, long long row0) {   // called by warp 0 only
    double* dst = sm + (k % kStreamRing) * cell_dbl;
    const double* src = fin + row0 * ld + c0;
    unsigned long long* bar = &full[k % kStreamRing];
    if (whole_rows) {
      if (tid == 0) {
        mbar_expect_tx(bar, cell_bytes);
        bulk_g2s(dst, src, cell_bytes, bar);
      }
    } else if (use_tmap) {   // the cell tile as ONE 2-D box (NLOC rows x tx_max columns)
      if (tid == 0) {
        mbar_expect_tx(bar, (unsigned)(NLOC * tx_max) * 8u);
        tma_load_2d(dst, &tmap, (int)c0, (int)row0, bar);
      }
    } else {
      if (tid == 0) mbar_expect_tx(bar, cell_bytes);
      __syncwarp();
      for (int r = tid; r < NLOC; r += 32)
        bulk_g2s(dst + r * rstride, src + (long long)r * ld, (unsigned)tx * 8u, bar);
    }
  };
  // the plan entries the loop needs are loaded one cell ahead (their latency hides
  // behind a cell's compute): warp 0 the row of the next list position to fetch,
  // every thread its cell's (row, slot, dedup set)
  long long next_row = 0;
  if (tid < 32) {
    for (int k = 0; k < min(3, n_load); ++k) issue(k, row_of(k));
    if (n_load > 3) next_row = row_of(3);
  }
  auto meta = [&](int s, long long& row, int& slot, int& dd) {
    const long long e = off + s;
    dd = dedup ? P.e_dd[e] : -1;
    slot = dd >= 0 ? -1 : P.e_slot[e];
    row = P.e_row0[e];
  };
  long long m_row = 0;
  int m_slot = -1, m_dd = -1;
  if (colv) meta(0, m_row, m_slot, m_dd);
  int waited = -1;
  for (int s = 0; s < n; ++s) {
    // prefetch list position of virtual cell s+2
    const int kn = s + 2 - v0;
    if (tid < 32 && kn < n_load && kn >= 3) {
      issue(kn, next_row);
      if (kn + 1 < n_load) next_row = row_of(kn + 1);
    }
    // wait for virtual cells s-1 .. s+1 that exist in the list; the ones below
    // `waited` were waited for at an earlier cell (their slots are refilled only
    // after every thread is past them)
    const int klo = max(s - 1 - v0, 0), khi = min(s + 1 - v0, n_load - 1);
    for (unsigned k = (unsigned)max(klo, waited + 1); k <= (unsigned)khi; ++k)
      mbar_wait(&full[k % kStreamRing], (k / kStreamRing) & 1u);
    waited = max(waited, khi);
    const long long row_s = m_row;
    const int slot = m_slot, dd = m_dd;
    if (colv && s + 1 < n) meta(s + 1, m_row, m_slot, m_dd);
    if (colv) {
      double* dst = slot < 0 ? fout + row_s * ld + c
                             : acc + (long long)slot * NLOC * n_cols + c;
      const long long dstride = slot < 0 ? ld : n_cols;
      const double* me = sm + ((s - v0) % kStreamRing) * cell_dbl + col;
      if (speed == 0.0) {
#pragma unroll 3
        for (int r = g; r < NLOC; r += NG) dst[r * dstride] = me[r * rstride];
      } else {
        // sources: virtual cells s - ns (same) and s - ns - 1 (neighbour); both in
        // the pencil unless an absorbing end cuts one off (first / last cell only)
        const int va_cell = s - (int)ns, vb_cell = s - (int)ns - 1;
        // DD: a deduplicated target (uniform over the CTA: one entry), a separate
        // instantiation so the common path keeps its unrolled loads
        auto apply = [&](bool va, bool vb, auto checked, auto dedup_t) {
          constexpr bool CK = decltype(checked)::value;
          constexpr bool DD = decltype(dedup_t)::value;
          const double* sa = sm + (unsigned)((va ? va_cell : s) - v0) % kStreamRing * cell_dbl + col;
          const double* sb = sm + (unsigned)((vb ? vb_cell : s) - v0) % kStreamRing * cell_dbl + col;
#pragma unroll
          for (int tt = 0; tt < NT; ++tt) {
            const int t = g + tt * NG;
            double ua[O], ub[O], y[O];
#pragma unroll
            for (int i = 0; i < O; ++i) {
              const int r = (DIM == 3) ? (t % O) * P.stride_t0 + (t / O) * P.stride_t1 + i * P.stride_d : i;
              ua[i] = (!CK || va) ? sa[r * rstride] : 0.0;
              ub[i] = (!CK || vb) ? sb[r * rstride] : 0.0;
            }
            two_cell<O>(A, B, ua, ub, !CK || va, !CK || vb, y);
#pragma unroll
            for (int i = 0; i < O; ++i) {
              const int r = (DIM == 3) ? (t % O) * P.stride_t0 + (t / O) * P.stride_t1 + i * P.stride_d : i;
              if constexpr (DD)
                dst[(long long)r * dstride] = dd_value(dd, y[i], me[r * rstride]);
              else
                dst[(long long)r * dstride] = y[i];
            }
          }
        };
        using F = std::integral_constant<bool, false>;
        using T = std::integral_constant<bool, true>;
        const bool inner = per || (va_cell >= 0 && va_cell < n && vb_cell >= 0 && vb_cell < n);
        const bool va = va_cell >= 0 && va_cell < n, vb = vb_cell >= 0 && vb_cell < n;
        if (dd < 0) {
          if (inner)
            apply(true, true, F{}, F{});
          else
            apply(va, vb, T{}, F{});
        } else {
          if (inner)
            apply(true, true, F{}, T{});
          else
            apply(va, vb, T{}, T{});
        }
      }
    }
    sync_fz();   // slot of virtual cell s-1 is refilled next iteration
  }
}

}  // namespace sldg
