// xx_tiles.cuh -- x-advection over "same-speed" row tiles (included by xfield.cu).
//
// xfield.advect_x (xfield.py:82-104) applies, per velocity row, the periodic
// two-cell update out_c = A u_{c-n} + B u_{c-n-1} (sldg1d.py:124-136) with the
// (n, A, B) of the row's v_x.  Rows b = i + o j + o^2 k of one velocity cell
// with the same v_x node i share v_x, hence one (n, A, B).  A tile is RPT such
// rows of one cell (rows cell*o^3 + (t0 + u)*o + i, u < RPT); a CTA processes
// TPC tiles at a time, thread = (tile, x cell), so the matrices are loaded into
// registers once per tile and every source read is conflict-free (consecutive
// threads read consecutive cells).  Rows arrive by 1-D TMA bulk copies into a
// ring of tile groups (mbarrier per slot), one group ahead of the compute.
//   NAPPLY == 2 : out = X(X(in)) (trailing half step of step n + leading half
//                 step of step n+1), the intermediate row in shared memory
//   MOM         : (m0, m1, m2) of the state after the FIRST application
//   RHO         : rho = w . f of the final output
// Per-thread column accumulators; CTA partials in a fixed order; the grid
// depends only on the problem shape (bitwise-reproducible reductions).
// Arithmetic per output identical to k_advect_x (the generic row kernel).
#pragma once

#include "tma_util.cuh"

namespace sldg {

// epilogue operands of the x passes: moments of the (first) result, rho of the final one
struct XEpi {
  const double* w;     // velocity quadrature weights (rows)
  const double* v0;    // v_x per row
  const double* v2;    // |v|^2 per row
  const double* xw;    // x quadrature weights (cols)
  double* mom_part;    // [grid][3]
  double* rho_part;    // [grid][row_len]
};

struct XTGeom {
  int rpt, tpc, nring, threads;   // rows per tile, tiles per CTA step, ring depth, threads
  int n_out, src_len;             // output cells per row, staged doubles per source row
  long long n_tiles, n_groups, grid_;
  size_t smem;
  bool ok;
};

constexpr int kXTMaxTpc = 8;

// Where a row's sources and outputs live.  Periodic rows (wrap = 1): the n_xc
// cells of the row, sources wrap around.  x slabs (wrap = 0, the sharded state):
// the input row is [left margin | local | right margin], src_len doubles copied
// from the row start, halo-relative cell j at src_off + j*o, the local cells are
// j = hl .. hl+n_xc-1 (no wrap: the halo covers every shift, twice the reach for
// NAPPLY == 2); outputs go to out_off + cx*o of rows with stride ld_out.  row_off: the
// absolute first row of the launch (a chunk of whole velocity cells).  cells: when set,
// the launch's velocity cells are cells[0..] (a cell list, e.g. the rows the one-pass
// AMR step leaves; in place is safe: a tile's rows are staged before they are written
// and no other tile reads them).
struct XRowMap {
  int src_len, src_off, hl, wrap, out_off;
  long long ld_out, row_off;
  const long long* cells;
};

// RPT > 0: rows per tile fixed at compile time (row loops unrolled, tile -> row
// arithmetic by constants); 0 = the geometry's value at run time.
template <int OV, int OX, int RPT>
__global__ void __launch_bounds__(512, 1)
k_xx_tiles(XPlanDev X, const double* __restrict__ fin, double* __restrict__ fout, long long ld,
           long long n_rows, int n_xc, int rpt_arg, int tpc, int nring, int n_speeds, XEpi epi,
           int napply, int mom, int rho, XRowMap rm) {
  const int wrap = rm.wrap;
  const long long* cells = rm.cells;
  constexpr int NL = OV * OV, NLOC = NL * OV;
  constexpr int XM = 2 * OX * OX;
  const int rpt = RPT > 0 ? RPT : rpt_arg;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) unsigned long long full[4];
  const int row_len = n_xc * OX;        // output row (local cells)
  const int src_len = rm.src_len;       // staged source row
  const int tid = threadIdx.x;
  const int tt = tid / n_xc;                 // tile within the group
  const int cx = tid - tt * n_xc;            // x cell
  const bool act = tt < tpc;
  const int per_cell = (NL / rpt) * OV;      // tiles per velocity cell
  // tile and group indices fit in 32 bits (the host checks n_tiles < 2^31)
  const int n_tiles = (int)((n_rows / NLOC) * per_cell);
  const int n_groups = (n_tiles + tpc - 1) / tpc;
  const int slot_dbl = tpc * rpt * src_len;
  double* ring = sm;
  double* mid = ring + (long long)nring * slot_dbl;
  double* meta = mid + slot_dbl;             // [nring][tpc][rpt][3]: w, w*v0, w*v2
  // per speed: A | B (2 OX^2 doubles: 16-byte aligned blocks, read as pairs)
  double* xtab = meta + (((long long)nring * tpc * rpt * 3 + 1) & ~1LL);
  int* xnsm = reinterpret_cast<int*>(xtab + (long long)n_speeds * XM);
  // a zero shift is stored as (A, B) = (I, 0) with no cell shift, so the update has
  // no per-thread branch (1*u0 + 0*u1 + ... == u0)
  for (int k = tid; k < n_speeds * XM; k += blockDim.x) {
    const int g = k / XM, e = k - g * XM;
    xtab[k] = X.ident[g] ? ((e < OX * OX && e % (OX + 1) == 0) ? 1.0 : 0.0) : __ldg(X.mats + k);
  }
  // periodic rows: the shift mod n_xc; slabs: the true shift (the halo covers it)
  for (int k = tid; k < n_speeds; k += blockDim.x)
    xnsm[k] = X.ident[k] ? 0 : (wrap ? __ldg(X.nsm + k) : (int)__ldg(X.ns + k));

  // tile id -> first row and row stride (rows u = 0..rpt-1 are row0 + u*OV)
  auto tile_row0 = [&](int tile) -> long long {
    const int cell = tile / per_cell;
    const int rem = tile - cell * per_cell;
    const int iv = rem % OV, tg = rem / OV;
    return rm.row_off + (cells ? __ldg(cells + cell) : (long long)cell) * NLOC +
           tg * rpt * OV + iv;
  };

  // a slot is full when warp 0's bulk copies have landed and (epilogues) warp 1's
  // 32 lanes have arrived after their metadata cp.async copies
  const bool need_meta = mom || rho;
  if (tid == 0) {
    for (int k = 0; k < nring; ++k) mbar_init(&full[k], need_meta ? 33 : 1);
    mbar_fence_init();
  }
  sync_fz();

  const int g0 = blockIdx.x, gs = gridDim.x;
  const int my = g0 < n_groups ? (n_groups - g0 + gs - 1) / gs : 0;
  // issue group i (of this CTA) into slot s = i % nring: one bulk copy per row (warp
  // 0), metadata (w, v0, v2 of each row) by cp.async from warp 1 into the slot's meta
  // block, completion signalled on the slot's barrier (no thread waits on it)
  auto issue = [&](int i, int s) {
    const int t_first = (g0 + i * gs) * tpc;
    const int nt = min(tpc, n_tiles - t_first);
    if (tid < 32) {
      if (tid == 0) mbar_expect_tx(&full[s], (unsigned)(nt * rpt * src_len * 8));
      __syncwarp();
      for (int q = tid; q < nt * rpt; q += 32) {
        const int ti = q / rpt, u = q - ti * rpt;
        const long long row = tile_row0(t_first + ti) + (long long)u * OV;
        bulk_g2s(ring + (long long)s * slot_dbl + (ti * rpt + u) * src_len, fin + row * ld,
                 (unsigned)(src_len * 8), &full[s]);
      }
    } else if (tid < 64 && need_meta) {
      for (int q = tid - 32; q < nt * rpt; q += 32) {
        const int ti = q / rpt, u = q - ti * rpt;
        const long long row = tile_row0(t_first + ti) + (long long)u * OV;
        double* m = meta + (((long long)s * tpc + ti) * rpt + u) * 3;
        cp_async8(m, epi.w + row);
        if (mom) {
          cp_async8(m + 1, epi.v0 + row);
          cp_async8(m + 2, epi.v2 + row);
        }
      }
      cp_async_arrive(&full[s]);
    }
  };
  for (int i = 0; i < min(nring - 1, my); ++i) issue(i, i);

  double m0a[OX], m1a[OX], m2a[OX], rha[OX];
#pragma unroll
  for (int k = 0; k < OX; ++k) m0a[k] = m1a[k] = m2a[k] = rha[k] = 0.0;

  auto speed_of = [&](int i) -> int {   // this thread's tile speed in group i
    const int tile = (g0 + i * gs) * tpc + tt;
    return (act && i < my && tile < n_tiles) ? __ldg(X.row_speed + tile_row0(tile)) : 0;
  };
  int g_next = speed_of(0);
  int s = 0, phase = 0;   // slot and barrier phase of group i (i % nring, (i / nring) & 1)
  for (int i = 0; i < my; ++i) {
    if (i + nring - 1 < my) issue(i + nring - 1, s == 0 ? nring - 1 : s - 1);
    const int g = g_next;
    g_next = speed_of(i + 1);                 // prefetched one group ahead
    mbar_wait(&full[s], (unsigned)phase);     // rows and metadata of slot s
    const int t_first = (g0 + i * gs) * tpc;
    const int tile = t_first + tt;
    const bool live = act && tile < n_tiles;
    double xa[OX * OX], xb[OX * OX];
    int ia = 0, ib = 0;
    long long row0 = 0;
    if (live) {
      row0 = tile_row0(tile);
      const double* AB = xtab + (long long)g * XM;
#pragma unroll
      for (int k = 0; k < XM; k += 2) {
        const double2 q = *reinterpret_cast<const double2*>(AB + k);
        (k < OX * OX ? xa[k] : xb[k - OX * OX]) = q.x;
        (k + 1 < OX * OX ? xa[k + 1] : xb[k + 1 - OX * OX]) = q.y;
      }
      if (wrap) {
        int a = cx - xnsm[g];   // nsm in [0, n_xc): the periodic source cell of cx
        if (a < 0) a += n_xc;
        ia = a * OX;
        ib = (a == 0 ? n_xc - 1 : a - 1) * OX;
      } else {                  // slab: halo-relative source cells hl + cx - n, - n - 1
        const int a = rm.hl + cx - xnsm[g];
        ia = rm.src_off + a * OX;
        ib = ia - OX;
      }
    }
    auto xapply = [&](const double* srow, double* y) {
      double ua[OX], ub[OX];
#pragma unroll
      for (int j = 0; j < OX; ++j) {
        ua[j] = srow[ia + j];
        ub[j] = srow[ib + j];
      }
#pragma unroll
      for (int k = 0; k < OX; ++k) {
        double sa = xa[k * OX] * ua[0];
        double sb = xb[k * OX] * ub[0];
#pragma unroll
        for (int j = 1; j < OX; ++j) {
          sa = fma(xa[k * OX + j], ua[j], sa);
          sb = fma(xb[k * OX + j], ub[j], sb);
        }
        y[k] = sa + sb;
      }
    };
    const double* src = ring + (long long)s * slot_dbl + tt * rpt * src_len;
    const double* mt = meta + ((long long)s * tpc + tt) * rpt * 3;
    double* md = mid + tt * rpt * src_len;   // intermediate rows, the source rows' layout
    if (napply == 2) {
      if (live) {
        // slabs: the second application reads the intermediate on up to |n| + 1 cells
        // beyond the local ones (left of them for n >= 0, right for n < 0); thread cx
        // forms local cell cx (moments as on periodic rows) and, for cx < extra, one of
        // those halo cells (sources within the doubled halo)
        const int nsh = wrap ? 0 : xnsm[g];
        const int extra = wrap ? 0 : (nsh >= 0 ? nsh + 1 : -nsh);
        const int xcell = nsh >= 0 ? rm.hl - 1 - cx : rm.hl + n_xc + cx;   // halo-relative
        const int xa_ = rm.src_off + (xcell - nsh) * OX;
#pragma unroll(RPT > 0 ? RPT : 1)
        for (int u = 0; u < rpt; ++u) {
          double y[OX];
          xapply(src + u * src_len, y);
          const int mo = wrap ? cx * OX : rm.src_off + (rm.hl + cx) * OX;
#pragma unroll
          for (int k = 0; k < OX; ++k) md[u * src_len + mo + k] = y[k];
          if (cx < extra) {
            const double* srow = src + u * src_len;
            double z[OX];
#pragma unroll
            for (int k = 0; k < OX; ++k) {
              double sa = xa[k * OX] * srow[xa_];
              double sb = xb[k * OX] * srow[xa_ - OX];
#pragma unroll
              for (int j = 1; j < OX; ++j) {
                sa = fma(xa[k * OX + j], srow[xa_ + j], sa);
                sb = fma(xb[k * OX + j], srow[xa_ - OX + j], sb);
              }
              z[k] = sa + sb;
            }
#pragma unroll
            for (int k = 0; k < OX; ++k) md[u * src_len + rm.src_off + xcell * OX + k] = z[k];
          }
          if (mom) {
            const double w = mt[u * 3], wv0 = w * mt[u * 3 + 1], wv2 = w * mt[u * 3 + 2];
#pragma unroll
            for (int k = 0; k < OX; ++k) {
              m0a[k] = fma(w, y[k], m0a[k]);
              m1a[k] = fma(wv0, y[k], m1a[k]);
              m2a[k] = fma(wv2, y[k], m2a[k]);
            }
          }
        }
      }
      sync_fz();
      src = md;
    }
    if (live) {
#pragma unroll(RPT > 0 ? RPT : 1)
      for (int u = 0; u < rpt; ++u) {
        double y[OX];
        xapply(src + u * src_len, y);
        double* dst = fout + (row0 + (long long)u * OV) * rm.ld_out + rm.out_off + cx * OX;
        const double w = need_meta ? mt[u * 3] : 0.0;
        const double wv0 = (mom && napply == 1) ? w * mt[u * 3 + 1] : 0.0;
        const double wv2 = (mom && napply == 1) ? w * mt[u * 3 + 2] : 0.0;
#pragma unroll
        for (int k = 0; k < OX; ++k) {
          dst[k] = y[k];
          if (rho) rha[k] = fma(w, y[k], rha[k]);
          if (mom && napply == 1) {
            m0a[k] = fma(w, y[k], m0a[k]);
            m1a[k] = fma(wv0, y[k], m1a[k]);
            m2a[k] = fma(wv2, y[k], m2a[k]);
          }
        }
      }
    }
    sync_fz();                          // slot s and mid are reused next
    if (++s == nring) {
      s = 0;
      phase ^= 1;
    }
  }

  // CTA partials: rho per column (tiles of the group summed in order), moments
  // contracted with the x weights and summed over threads in order
  double* red = sm;
  if (rho) {
    if (act) {
#pragma unroll
      for (int k = 0; k < OX; ++k) red[tt * row_len + cx * OX + k] = rha[k];
    }
    sync_fz();
    for (int e = tid; e < row_len; e += blockDim.x) {
      double v = 0.0;
      for (int q = 0; q < tpc; ++q) v += red[q * row_len + e];
      epi.rho_part[(long long)blockIdx.x * row_len + e] = v;
    }
    sync_fz();
  }
  if (mom) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    if (act) {
#pragma unroll
      for (int k = 0; k < OX; ++k) {
        const double xwk = __ldg(epi.xw + cx * OX + k);
        s0 = fma(xwk, m0a[k], s0);
        s1 = fma(xwk, m1a[k], s1);
        s2 = fma(xwk, m2a[k], s2);
      }
    }
    red[tid] = s0;
    red[blockDim.x + tid] = s1;
    red[2 * blockDim.x + tid] = s2;
    sync_fz();
    if (tid < 3) {
      double v = 0.0;
      for (int q = 0; q < (int)blockDim.x; ++q) v += red[tid * blockDim.x + q];
      epi.mom_part[blockIdx.x * 3 + tid] = v;
    }
  }
}

}  // namespace sldg
