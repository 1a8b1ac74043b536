// sweep_stream.cuh -- streaming whole-pencil fast path of the v-sweep (included by vsweep.cu).
//
// Replaces the whole-pencil fast path of sweep_pencil (vsweep.py:197-200 ->
// apply_update, sldg1d.py:124-136) for every pencil whose cells are all
// conforming and on one level.
//
// Persistent CTAs.  A CTA owns one column tile (<= 256 x-columns; thread =
// column, with its column's level matrices A, B (2 o^2 fp64) in registers) and
// walks a strided list of work items (pencil, line group).  For direction 0 a
// cell's (p+1)^dim velocity rows are consecutive rows of f, so a cell tile is
// one (rows x columns) block: ONE cp.async.bulk (TMA engine) when the tile
// spans whole rows, else one bulk copy per row.  All cells of all the CTA's
// items stream through a single 4-slot ring tracked by mbarriers (transaction
// bytes), two cells ahead of the compute and straight across item
// boundaries, so there is no per-pencil pipeline ramp; every input
// coefficient is read from HBM once (absorbing bc; periodic re-reads the two
// wrap cells).  Outputs go from registers to HBM with coalesced 8-byte stores.
//
// The ring path is used when every active column of the tile has n_shift in
// {-1, 0} at the item's level (all Landau shifts): cell s then needs cells
// s-1, s, s+1.  Otherwise the item is computed with direct loads (same
// arithmetic) while its ring positions are still consumed.
#pragma once

#include "tma_util.cuh"

namespace sldg {

constexpr int kStreamRing = 4;

template <int O, int DIM>
__global__ void __launch_bounds__(256, 1)
k_sweep_stream(VPlanDev P, const double* __restrict__ fin, double* __restrict__ fout,
               long long ld, long long n_cols, const double* __restrict__ speeds, int bc,
               const long long* __restrict__ lm_ns, const double* __restrict__ lm_mats,
               double* __restrict__ acc, int tx_max, int n_tiles, int whole_rows, int lgl,
               int n_lg) {
  constexpr int NL = (DIM == 3) ? O * O : 1;
  constexpr int NLOC = NL * O;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) unsigned long long full[kStreamRing];
  __shared__ int s_nsmin, s_nsmax;

  // CTA -> fixed column tile, strided items (pencil, line group)
  const int tile = (int)(blockIdx.x % n_tiles);
  const long long g0 = blockIdx.x / n_tiles;
  const long long gs = gridDim.x / n_tiles;
  const long long n_items = P.n_walk * n_lg;
  const long long c0 = (long long)tile * tx_max;
  const int tx = (int)min((long long)tx_max, n_cols - c0);
  const int tid = threadIdx.x;
  const int R = (DIM == 3) ? lgl * O : NLOC;          // rows per cell tile
  const int rstride = whole_rows ? (int)ld : tx_max;  // smem row stride (doubles)
  const int cell_dbl = R * rstride;
  const unsigned cell_bytes = (unsigned)(R * tx) * 8u;
  const bool per = (bc == SLDG_BC_PERIODIC);
  const int v0 = per ? -1 : 0;                        // load list: virtual cells v0 .. n-1-v0
  const bool colv = tid < tx;
  const long long c = c0 + tid;

  if (tid == 0) {
    for (int k = 0; k < kStreamRing; ++k) mbar_init(&full[k], 1);
    mbar_fence_init();
  }
  __syncthreads();

  struct Item {
    long long off;
    int n, t0, lev;
  };
  auto item_of = [&](long long i) -> Item {
    const long long wq = g0 + i * gs;
    const long long wp = wq / n_lg;
    const long long q = P.walk_pencils[wp];
    Item it;
    it.off = P.p_off[q];
    it.n = P.p_n[q];
    it.t0 = (int)(wq - wp * n_lg) * lgl;
    it.lev = P.e_level[it.off];
    return it;
  };
  const long long my_items = (g0 < n_items) ? (n_items - g0 + gs - 1) / gs : 0;

  // issue cursor (thread 0 only): item index, list position within it, global position
  long long iss_i = 0;
  int iss_k = 0;
  long long iss_gp = 0;
  Item iss_it{};
  if (tid == 0 && my_items > 0) iss_it = item_of(0);
  auto issue_upto = [&](long long gp_limit) {   // thread 0
    while (iss_i < my_items && iss_gp <= gp_limit) {
      const int n_load = per ? iss_it.n + 2 : iss_it.n;
      const int v = v0 + iss_k;
      const int cell = v < 0 ? iss_it.n - 1 : (v >= iss_it.n ? 0 : v);
      const int slot = (int)(iss_gp % kStreamRing);
      double* dst = sm + slot * cell_dbl;
      const double* src = fin + (P.e_row0[iss_it.off + cell] + iss_it.t0 * O) * ld + c0;
      unsigned long long* bar = &full[slot];
      mbar_expect_tx(bar, cell_bytes);
      if (whole_rows) {
        bulk_g2s(dst, src, cell_bytes, bar);
      } else {
        for (int r = 0; r < R; ++r)
          bulk_g2s(dst + r * rstride, src + (long long)r * ld, (unsigned)tx * 8u, bar);
      }
      ++iss_gp;
      if (++iss_k == n_load) {
        iss_k = 0;
        if (++iss_i < my_items) iss_it = item_of(iss_i);
      }
    }
  };
  if (tid == 0) issue_upto(2);

  int cur_lev = -1;
  bool streamable = true;
  double speed = 0.0;
  long long ns = 0;
  double A[O * O], B[O * O];
  long long base = 0;                    // global position of the current item's list start
  for (long long i = 0; i < my_items; ++i) {
    const Item it = item_of(i);
    const int n = it.n;
    const int n_load = per ? n + 2 : n;
    if (it.lev != cur_lev) {             // (re)load the column's level data
      if (tid == 0) {
        s_nsmin = 1 << 30;
        s_nsmax = -(1 << 30);
      }
      __syncthreads();
      speed = colv ? __ldg(speeds + c) : 0.0;
      ns = colv ? lm_ns[(long long)it.lev * n_cols + c] : 0;
      if (colv && speed != 0.0) {
        const int nsi = (int)max(min(ns, (long long)(1 << 29)), -(long long)(1 << 29));
        atomicMin(&s_nsmin, nsi);
        atomicMax(&s_nsmax, nsi);
      }
      if (colv) load_pair<O>(lm_mats, it.lev, n_cols, c, A, B);
      __syncthreads();
      streamable = (s_nsmin >= -1 && s_nsmax <= 0) || (s_nsmin > s_nsmax);
      cur_lev = it.lev;
    }
    const int roff = it.t0 * O;
    for (int s = 0; s < n; ++s) {
      if (tid == 0) issue_upto(base + s + 2 - v0);
      const int klo = max(s - 1 - v0, 0), khi = min(s + 1 - v0, n_load - 1);
      for (int k = klo; k <= khi; ++k) {
        const long long gp = base + k;
        mbar_wait(&full[gp % kStreamRing], (unsigned)((gp / kStreamRing) & 1));
      }
      if (colv) {
        const long long e = it.off + s;
        const int slot = P.e_slot[e];
        double* dst = slot < 0 ? fout + P.e_row0[e] * ld + c
                               : acc + (long long)slot * NLOC * n_cols + c;
        const long long dstride = slot < 0 ? ld : n_cols;
        auto ring_of = [&](int v) { return sm + ((base + v - v0) % kStreamRing) * cell_dbl + tid; };
        if (speed == 0.0) {
          const double* me = ring_of(s);
#pragma unroll 3
          for (int r = 0; r < R; ++r) dst[(r + roff) * dstride] = me[r * rstride];
        } else {
          const int va_cell = s - (int)ns, vb_cell = s - (int)ns - 1;
          bool va, vb;
          const double *sa, *sb;
          long long sstride;
          if (streamable) {
            va = per || (va_cell >= 0 && va_cell < n);
            vb = per || (vb_cell >= 0 && vb_cell < n);
            sa = ring_of(va ? va_cell : s) - (long long)roff * rstride;
            sb = ring_of(vb ? vb_cell : s) - (long long)roff * rstride;
            sstride = rstride;
          } else {   // arbitrary shifts: direct loads from HBM
            long long qa = va_cell, qb = vb_cell;
            va = vb = true;
            if (per) {
              qa = pymod(qa, n);
              qb = pymod(qb, n);
            } else {
              va = qa >= 0 && qa < n;
              vb = qb >= 0 && qb < n;
            }
            sa = fin + P.e_row0[it.off + (va ? qa : s)] * ld + c;
            sb = fin + P.e_row0[it.off + (vb ? qb : s)] * ld + c;
            sstride = ld;
          }
#pragma unroll
          for (int t = 0; t < NL; ++t) {
            if (DIM == 3 && (t < it.t0 || t >= it.t0 + lgl)) continue;
            double ua[O], ub[O], y[O];
#pragma unroll
            for (int i2 = 0; i2 < O; ++i2) {
              const int r = (DIM == 3) ? (t % O) * P.stride_t0 + (t / O) * P.stride_t1 + i2 * P.stride_d : i2;
              ua[i2] = va ? sa[r * sstride] : 0.0;
              ub[i2] = vb ? sb[r * sstride] : 0.0;
            }
            two_cell<O>(A, B, ua, ub, va, vb, y);
#pragma unroll
            for (int i2 = 0; i2 < O; ++i2) {
              const int r = (DIM == 3) ? (t % O) * P.stride_t0 + (t / O) * P.stride_t1 + i2 * P.stride_d : i2;
              dst[(long long)r * dstride] = y[i2];
            }
          }
        }
      }
      __syncthreads();   // the slot two positions back is refilled next
    }
    // list positions of this item that were never waited on (periodic wrap cells not
    // needed by any column) are waited here so every barrier phase is consumed in order
    for (int k = 0; k < n_load; ++k) {
      const bool waited = (k >= max(-1 - v0, 0)) && (k <= min(n - v0, n_load - 1));
      if (!waited) {
        const long long gp = base + k;
        mbar_wait(&full[gp % kStreamRing], (unsigned)((gp / kStreamRing) & 1));
      }
    }
    base += n_load;
  }
}

}  // namespace sldg
