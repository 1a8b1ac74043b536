// amr_fused.cuh -- one HBM pass per steady-state Strang step on AMR velocity meshes
// (included by vsweep.cu).
//
// In Simulation.advance() the steady step is V followed by the trailing half x-step
// of this step and the leading half x-step of the next (X.X, xfield.py:91-104 twice),
// with the moments of the intermediate and rho of the result (driver.py:220-240).
// The separate passes (k_sweep_stream, then k_xx_tiles) move every coefficient
// through HBM twice (32 B/DOF).  Here every row written directly by a whole-fast
// pencil of the walk is finished in ONE pass (16 B/DOF):
//
//   unit    = (walk pencil, line t): the O rows (t*O .. t*O+O-1) of every cell of the
//             pencil, i.e. O complete x-rows per cell (sldg_vplan: direction 0, the
//             line's rows are consecutive);
//   cluster = NCL CTAs (thread-block cluster) splitting the row into NCL column
//             slices.  Each CTA streams its slice of the unit's cells through a
//             bulk-copy ring (mbarrier per slot) and runs the v-update for its columns
//             (thread = column, the column's A, B for the pencil's level in
//             registers: one SM's register file holds the matrices of ~400 columns,
//             a cfg5 row has 1536, hence the cluster);
//   V       = the whole-pencil fast path of k_sweep_stream (same arithmetic), result
//             of cell s -> vout[s & 1] in shared memory;
//   cluster barrier: every slice of the cell's V result is visible cluster-wide;
//   X.X     = one composed 3-cell stencil per row (C0 = A A, C1 = A B + B A, C2 = B B
//             for the row's x-speed, shift 2n), thread = (row i, x cell); sources in
//             other slices are read from the owner CTA's shared memory (DSMEM);
//             moments of the intermediate through the contracted weights
//             (A^T + B^T) xw (a periodic row's sum is shift-free), rho of the result;
//             stored to HBM.
//
// Rows NOT written directly by the walk -- cells of non-fast pencils (per-cell
// worklist) and weighted write-back targets -- take the existing kernels for V, then
// one X.X pass over exactly those cells (k_xx_tiles with a cell list, in place).
// Persistent clusters with a static unit assignment and fixed-order partials: the
// result is bitwise reproducible.  Differences from the separate passes are
// re-association only (~1e-16 relative per step; tests/test_gpu_amr_fused.py).
#pragma once

#include <cooperative_groups.h>

#include "tma_util.cuh"

namespace sldg {

constexpr int kAmrRing = 8;   // slots of O rows x slice columns (power of two)

struct AmrEpi {
  const double* w;       // velocity quadrature weight per row
  const double* v0;      // v_x per row
  const double* v2;      // |v|^2 per row
  const double* xcomp;   // per x-speed (XComp<OX>::N doubles): C0, C1, C2 (OX*OX each),
                         // cAB = (A^T + B^T) xw (OX), the shift n mod n_xc (exact), pad
  const int* e_xg;       // per entry, per v_x node i < O: x-speed index of the cell's rows
  double* mom_part;      // [CTAs][3]
  double* rho_part;      // [clusters][n_cols]
};

template <int OX>
struct XComp {
  static constexpr int M = OX * OX;
  static constexpr int CAB = 3 * M, SH = 3 * M + OX;
  static constexpr int N = (SH + 2) & ~1;   // doubles per speed (even)
};

// composed x-step per x-speed (one thread per speed)
template <int OX>
__global__ void k_xcomp(XPlanDev X, const double* __restrict__ xw, long long n_speeds,
                        double* __restrict__ xcomp) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= n_speeds) return;
  using XC = XComp<OX>;
  constexpr int M = XC::M;
  double A[M], B[M];
  const bool id = X.ident[g];
#pragma unroll
  for (int k = 0; k < M; ++k) {
    A[k] = id ? ((k % (OX + 1) == 0) ? 1.0 : 0.0) : X.mats[g * 2 * M + k];
    B[k] = id ? 0.0 : X.mats[g * 2 * M + M + k];
  }
  double* C = xcomp + g * XC::N;
#pragma unroll
  for (int r = 0; r < OX; ++r)
#pragma unroll
    for (int c = 0; c < OX; ++c) {
      double aa = 0.0, ab = 0.0, bb = 0.0;
#pragma unroll
      for (int k = 0; k < OX; ++k) {
        aa = fma(A[r * OX + k], A[k * OX + c], aa);
        ab = fma(A[r * OX + k], B[k * OX + c], ab);
        ab = fma(B[r * OX + k], A[k * OX + c], ab);
        bb = fma(B[r * OX + k], B[k * OX + c], bb);
      }
      C[r * OX + c] = aa;
      C[M + r * OX + c] = ab;
      C[2 * M + r * OX + c] = bb;
    }
#pragma unroll
  for (int c = 0; c < OX; ++c) {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < OX; ++r) s = fma(A[r * OX + c] + B[r * OX + c], xw[r], s);
    C[XC::CAB + c] = s;
  }
  C[XC::SH] = id ? 0.0 : (double)X.nsm[g];
  for (int k = XC::SH + 1; k < XC::N; ++k) C[k] = 0.0;
}

// x-speed index per (entry, v_x node): the rows of a cell with v_x node i share it
template <int O>
__global__ void k_entry_speeds(VPlanDev P, const int* __restrict__ row_speed, long long n_entries,
                               int* __restrict__ e_xg) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n_entries * O) return;
  const long long e = k / O;
  e_xg[k] = row_speed[P.e_row0[e] + (k - e * O)];
}

template <int O, int OX>
__global__ void __launch_bounds__(512, 1)
k_amr_fused(VPlanDev P, const double* __restrict__ fin, double* __restrict__ fout, long long ld,
            int n_cols, int n_xc, const double* __restrict__ speeds, int bc,
            const long long* __restrict__ lm_ns, const double* __restrict__ lm_mats,
            double* __restrict__ acc, AmrEpi ep, long long n_units) {
  namespace cg = cooperative_groups;
  using XC = XComp<OX>;
  constexpr int NL = O * O, NLOC = NL * O;
  constexpr int M = XC::M;
  constexpr unsigned RM = kAmrRing - 1;
  cg::cluster_group cl = cg::this_cluster();
  const int ncl = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const long long cid = blockIdx.x / ncl, n_cl = gridDim.x / ncl;
  const int cw = n_cols / ncl, ncx = n_xc / ncl;
  const int slot_dbl = O * cw;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) unsigned long long full[kAmrRing];
  double* ring = sm;                              // [kAmrRing][O][cw]
  double* vout = ring + kAmrRing * slot_dbl;      // [2][O][cw]   (read cluster-wide)
  double* obuf = vout + 2 * slot_dbl;             // [2][O][cw]   X.X result -> bulk store
  double* cbuf = obuf + 2 * slot_dbl;             // [3][O][XC::N] composed x-steps per cell
  const int tid = threadIdx.x, nthr = blockDim.x;
  const bool per = bc == SLDG_BC_PERIODIC;
  const int v0c = per ? -1 : 0;                   // virtual cell of list position 0

  if (tid == 0) {
    for (int k = 0; k < kAmrRing; ++k) mbar_init(&full[k], 1);
    mbar_fence_init();
  }
  sync_fz();

  auto unit_desc = [&](long long u, long long& off, int& n, int& lev, int& t) {
    const long long wp = u / NL;
    t = (int)(u - wp * NL);
    off = P.walk_dd_desc[2 * wp];
    const long long d = P.walk_dd_desc[2 * wp + 1];
    n = (int)(d & 0xffffffffLL);
    lev = (int)(d >> 32);
  };

  // ---- producer (thread 0): one load sequence across this cluster's units; list
  // position k of a unit is virtual cell v0c + k (wrapped when periodic).  The row of
  // the next position is loaded one issue ahead.
  long long issued = 0, pu = cid, p_off = 0, p_row = 0;
  int p_n = 0, p_t = 0, p_lev = 0, pk = 0;
  auto p_row_of = [&]() {
    const int v = v0c + pk;
    const int cell = v < 0 ? p_n - 1 : (v >= p_n ? 0 : v);
    return P.e_row0[p_off + cell] + (long long)p_t * O;
  };
  if (tid == 0 && pu < n_units) {
    unit_desc(pu, p_off, p_n, p_lev, p_t);
    p_row = p_row_of();
  }
  auto pump = [&](long long limit) {
    while (issued < limit && pu < n_units) {
      const unsigned sl = (unsigned)issued & RM;
      double* dst = ring + sl * slot_dbl;
      mbar_expect_tx(&full[sl], (unsigned)slot_dbl * 8u);
#pragma unroll
      for (int i = 0; i < O; ++i)
        bulk_g2s(dst + i * cw, fin + (p_row + i) * ld + (long long)rank * cw, (unsigned)cw * 8u,
                 &full[sl]);
      ++issued;
      if (++pk == (per ? p_n + 2 : p_n)) {
        pk = 0;
        pu += n_cl;
        if (pu < n_units) unit_desc(pu, p_off, p_n, p_lev, p_t);
      }
      if (pu < n_units) p_row = p_row_of();
    }
  };

  // ---- thread roles: V phase thread = column of the slice; X phase thread = (row i
  // of the line, x cell of the slice); composed-step staging thread = (i, entry)
  const bool colv = tid < cw;
  const int gc = rank * cw + tid;
  const bool xv = tid < O * ncx;
  const int xi = xv ? tid / ncx : 0;
  const int xcx = xv ? tid - xi * ncx : 0;
  const int gxc = rank * ncx + xcx;
  // staging entries k = tid, tid + nthr of the O x XC::N composed-step block
  constexpr int NST = O * XC::N;
  double m0 = 0.0, m1 = 0.0, m2 = 0.0, rha[OX];
#pragma unroll
  for (int k = 0; k < OX; ++k) rha[k] = 0.0;
  const double speed = colv ? __ldg(speeds + gc) : 0.0;
  auto vout_of = [&](int r) -> const double* {   // a slice's V result (DSMEM when remote)
    return r == rank ? vout : cl.map_shared_rank(vout, r);
  };
  // the per-cell barrier: CTA-wide for one-CTA clusters, else cluster-wide (its release
  // fence has no generic global stores to drain: outputs leave by bulk stores)
  auto csync = [&]() {
    fuzz_delay();
    if (ncl == 1)
      __syncthreads();
    else
      cl.sync();
  };
  // thread 0: the previous direct cell's X.X result (obuf) -> HBM by bulk stores,
  // issued after the barrier that follows every thread's X phase
  long long st_row = -1;
  auto store_prev = [&](long long buf) {
    if (st_row >= 0) {
      const double* src = obuf + (buf & 1) * slot_dbl;
#pragma unroll
      for (int i = 0; i < O; ++i)
        bulk_s2g(fout + (st_row + i) * ld + (long long)rank * cw, src + i * cw,
                 (unsigned)cw * 8u);
      bulk_commit();
    }
  };

  long long base = 0, waited = -1, cc = 0;   // cc: cells processed (buffer rotation)
  for (long long u = cid; u < n_units; u += n_cl) {
    long long off;
    int n, t, lev;
    unit_desc(u, off, n, lev, t);
    const int n_load = per ? n + 2 : n;
    double A[O * O], B[O * O];
    long long ns = 0;
    if (colv) {
      ns = lm_ns[(long long)lev * n_cols + gc];
      load_pair<O>(lm_mats, lev, n_cols, gc, A, B);
    }
    // cell metadata one cell ahead: first row, write-back slot, dedup set; the
    // composed x-step of cell s+1 is staged (cp.async) while cell s runs, so its speed
    // index is read two cells ahead
    long long c_row = P.e_row0[off];
    int c_slot = P.e_slot[off], c_dd = P.e_dd[off];
    int g1[2] = {0, 0};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = tid + h * nthr;
      if (k < NST) {
        const int si = k / XC::N, se = k - si * XC::N;
        cp_async8(cbuf + (cc % 3) * NST + k,
                  ep.xcomp + (long long)__ldg(ep.e_xg + off * O + si) * XC::N + se);
        if (n > 1) g1[h] = __ldg(ep.e_xg + (off + 1) * O + si);
      }
    }
    for (int s = 0; s < n; ++s, ++cc) {
      if (tid == 0) pump(base + max(s - 1 - v0c, 0) + kAmrRing);
      const long long row_s = c_row + (long long)t * O;
      const int dd = c_dd, slot = dd >= 0 ? -1 : c_slot;
      if (s + 1 < n) {
        c_row = P.e_row0[off + s + 1];
        c_slot = P.e_slot[off + s + 1];
        c_dd = P.e_dd[off + s + 1];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = tid + h * nthr;
          if (k < NST) {
            const int si = k / XC::N, se = k - si * XC::N;
            cp_async8(cbuf + ((cc + 1) % 3) * NST + k, ep.xcomp + (long long)g1[h] * XC::N + se);
            if (s + 2 < n) g1[h] = __ldg(ep.e_xg + (off + s + 2) * O + si);
          }
        }
      }
      // x-phase row operands (issued before the waits, used after the V phase)
      double w = 0.0, rv0 = 0.0, rv2 = 0.0;
      if (xv && slot < 0) {
        const long long r = row_s + xi;
        w = __ldg(ep.w + r);
        rv0 = __ldg(ep.v0 + r);
        rv2 = __ldg(ep.v2 + r);
      }
      const int klo = max(s - 1 - v0c, 0), khi = min(s + 1 - v0c, n_load - 1);
      for (long long L = max(base + klo, waited + 1); L <= base + khi; ++L)
        mbar_wait(&full[(unsigned)L & RM], (unsigned)(L / kAmrRing) & 1u);
      waited = max(waited, base + khi);

      // ---- V: the column's new values on the O rows of cell s
      if (colv) {
        // ring slots of virtual cells s-1, s, s+1 (list positions base + vc - v0c)
        const int sp = (int)((unsigned)(base + s - v0c) & RM);
        const double* me = ring + sp * slot_dbl + tid;
        double y[O];
        if (speed == 0.0) {
#pragma unroll
          for (int i = 0; i < O; ++i) y[i] = me[i * cw];
        } else {
          const int va_cell = s - (int)ns, vb_cell = va_cell - 1;
          const bool va = per || (va_cell >= 0 && va_cell < n);
          const bool vb = per || (vb_cell >= 0 && vb_cell < n);
          double ua[O], ub[O];
          if (ns == 0 || ns == -1) {   // every Landau shift: sources in the ring
            const double* pn = ring + ((sp + 1) & RM) * slot_dbl + tid;
            const double* pp = ring + ((sp - 1) & RM) * slot_dbl + tid;
            const double* pa = ns == 0 ? me : pn;
            const double* pb = ns == 0 ? pp : me;
#pragma unroll
            for (int i = 0; i < O; ++i) {
              ua[i] = va ? pa[i * cw] : 0.0;
              ub[i] = vb ? pb[i * cw] : 0.0;
            }
          } else {   // a longer shift: straight from HBM
#pragma unroll
            for (int i = 0; i < O; ++i) ua[i] = ub[i] = 0.0;
            auto src = [&](int vc, double* out) {
              const long long c2 = per ? pymod(vc, n) : vc;
              const double* q = fin + (P.e_row0[off + c2] + (long long)t * O) * ld + gc;
#pragma unroll
              for (int i = 0; i < O; ++i) out[i] = q[(long long)i * ld];
            };
            if (va) src(va_cell, ua);
            if (vb) src(vb_cell, ub);
          }
          two_cell<O>(A, B, ua, ub, va, vb, y);
          if (dd >= 0) {   // k_writeback's arithmetic for identical contributions
            const long long k0 = P.dd_off[dd], k1 = P.dd_off[dd + 1];
#pragma unroll
            for (int i = 0; i < O; ++i) {
              const double fv = me[i * cw];
              const double df = __dsub_rn(y[i], fv);
              double a = 0.0;
              for (long long k = k0; k < k1; ++k) a = __dadd_rn(a, __dmul_rn(__ldg(P.dd_w + k), df));
              y[i] = __dadd_rn(fv, a);
            }
          }
        }
        if (slot >= 0) {
          double* dst = acc + ((long long)slot * NLOC + (long long)t * O) * n_cols + gc;
#pragma unroll
          for (int i = 0; i < O; ++i) dst[(long long)i * n_cols] = y[i];
        } else {
          double* vo = vout + (cc & 1) * slot_dbl + tid;
#pragma unroll
          for (int i = 0; i < O; ++i) vo[i * cw] = y[i];
        }
      }
      if (tid < NST) cp_async_wait_all();   // this cell's composed step (staged a cell ago)
      if (tid == 0) bulk_wait_read0();   // obuf of cell cc - 2 is rewritten below
      csync();   // the cell's V result is visible in every slice; ring slots of
                 // positions < s - v0c are free (their last reader was V of cell s);
                 // every X phase of cell cc - 1 is done
      if (tid == 0) {
        store_prev(cc - 1);
        st_row = slot < 0 ? row_s : -1;
      }

      // ---- X.X of the cell's rows (direct targets only; the rest are finished by
      // the cell-list pass after the write-back)
      if (xv && slot < 0) {
        const double* C = cbuf + (cc % 3) * NST + xi * XC::N;
        const int n2 = 2 * (int)C[XC::SH];   // in [0, 2 n_xc)
        int a0 = gxc - n2;
        if (a0 < 0) a0 += n_xc;
        if (a0 < 0) a0 += n_xc;
        const int a1 = a0 == 0 ? n_xc - 1 : a0 - 1;
        const int a2 = a1 == 0 ? n_xc - 1 : a1 - 1;
        const int buf = (int)(cc & 1) * slot_dbl + xi * cw;
        double u0[OX], u1[OX], u2[OX], uc[OX];
        const double* pc = vout + buf + xcx * OX;
        const int la = a0 - rank * ncx;   // source cell relative to this slice
        if (la >= 2 && la < ncx) {        // all three sources in this slice
          const double* p0 = vout + buf + la * OX;
#pragma unroll
          for (int j = 0; j < OX; ++j) {
            u0[j] = p0[j];
            u1[j] = p0[j - OX];
            u2[j] = p0[j - 2 * OX];
            uc[j] = pc[j];
          }
        } else {                          // a slice edge or the periodic wrap (DSMEM)
          const int r0 = a0 / ncx, r1 = a1 / ncx, r2 = a2 / ncx;
          const double* p0 = vout_of(r0) + buf + (a0 - r0 * ncx) * OX;
          const double* p1 = vout_of(r1) + buf + (a1 - r1 * ncx) * OX;
          const double* p2 = vout_of(r2) + buf + (a2 - r2 * ncx) * OX;
#pragma unroll
          for (int j = 0; j < OX; ++j) {
            u0[j] = p0[j];
            u1[j] = p1[j];
            u2[j] = p2[j];
            uc[j] = pc[j];
          }
        }
        double xm = 0.0;
#pragma unroll
        for (int j = 0; j < OX; ++j) xm = fma(C[XC::CAB + j], uc[j], xm);
        m0 = fma(w, xm, m0);
        m1 = fma(w * rv0, xm, m1);
        m2 = fma(w * rv2, xm, m2);
        double* dst = obuf + (cc & 1) * slot_dbl + xi * cw + xcx * OX;
#pragma unroll
        for (int k = 0; k < OX; ++k) {
          double y0 = 0.0, y1 = 0.0, y2 = 0.0;
#pragma unroll
          for (int j = 0; j < OX; ++j) {
            y0 = fma(C[k * OX + j], u0[j], y0);
            y1 = fma(C[M + k * OX + j], u1[j], y1);
            y2 = fma(C[2 * M + k * OX + j], u2[j], y2);
          }
          const double y = (y0 + y1) + y2;
          dst[k] = y;
          rha[k] = fma(w, y, rha[k]);
        }
        fence_proxy_async();
      }
    }
    base += n_load;
  }
  csync();   // every X phase done; no CTA leaves while a peer may still read its vout
  if (tid == 0) {
    store_prev(cc - 1);
    bulk_wait_all0();
  }

  // ---- fixed-order partials: rho per column of the slice (rows i summed in order),
  // moments summed over threads in order
  double* red = ring;
  if (xv) {
#pragma unroll
    for (int k = 0; k < OX; ++k) red[xi * cw + xcx * OX + k] = rha[k];
  }
  __syncthreads();
  for (int e = tid; e < cw; e += nthr) {
    double v = 0.0;
    for (int i = 0; i < O; ++i) v += red[i * cw + e];
    ep.rho_part[cid * n_cols + (long long)rank * cw + e] = v;
  }
  __syncthreads();
  red[tid] = m0;
  red[nthr + tid] = m1;
  red[2 * nthr + tid] = m2;
  __syncthreads();
  if (tid < 3) {
    double v = 0.0;
    for (int q = 0; q < nthr; ++q) v += red[tid * nthr + q];
    ep.mom_part[(long long)blockIdx.x * 3 + tid] = v;
  }
}

}  // namespace sldg
