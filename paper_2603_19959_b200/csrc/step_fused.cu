// step_fused.cu -- one HBM pass per Strang step: v-sweep + trailing half x-step
// (+ moments) + next leading half x-step (+ rho), fused per line-group tile.
//
// In Simulation.advance() the state between kernels is f' = X(f) (after the
// leading half x-step).  The reference step (driver.py:231-240) continues with
// field solve -> advect_velocity (vsweep.py:413-441) -> advect_x
// (xfield.py:91-104) -> diagnostics (driver.py:220-229, moments 139-146), and
// the next step starts with advect_x and compute_rho (xfield.py:107-109).
// For every cell of a pencil and a group of LG lines of that cell (a "tile":
// R = LG*OV rows spanning all x columns) the kernel performs
//   V  : whole-pencil fast path (sweep_pencil, vsweep.py:197-200) from a TMA
//        bulk-copy ring of cell tiles (as k_sweep_stream), into shared memory;
//   X  : trailing half x-step of this step and leading half x-step of the
//        next on the tile's rows (they are complete rows), as ONE composed
//        3-cell stencil (both half steps use the row's x-speed: X.X = C0, C1,
//        C2 = A A, A B + B A, B B), moments of the intermediate (trailing) state
//        through the contracted weights A^T xw, B^T xw, rho of the result;
//        result stored to HBM.
// Every coefficient is read once and written once per step: 16 B/DOF instead
// of 32 B/DOF for the separate sweep and X.X passes.  V is the same arithmetic
// as k_sweep_stream; the composed x-step re-associates X(X(u)) (differences
// from the separate passes ~1e-16 relative per step, far inside the 1e-12
// parity budget; tests/test_gpu_parity.py::test_fused_step_matches_unfused_*).
//
// Work decomposition: persistent CTAs (resident count x SMs).  The work is the
// sequence of items (walk pencil, line group), each a run of cell tiles; CTA b
// owns the contiguous tile range [b*T/G, (b+1)*T/G), so every CTA does the same
// number of tiles (no tail wave) and items may be split between two CTAs (a
// tile only needs its cell's neighbours, which the ring loads as well).  One
// TMA ring runs across the CTA's items; the next item's tables (pencil
// descriptor, tile rows, x-speed indices, row weights) are prefetched with
// cp.async while the current item is computed, so there is no per-item
// prologue on the critical path.
//
// Thread mappings: V phase thread = x column (its A, B for the pencil's level
// in registers); X phases thread = (velocity node i_v, x cell): all rows of a
// tile with the same i_v share one v_x, hence one x-shift and one A, B pair.
//
// Eligible: dim 3, direction 0, every pencil whole-pencil-fast, no weighted
// (1/n_c) entries, tile rows span the whole row (ld == n_cols).  Otherwise the
// host falls back to the separate passes.
#include <algorithm>
#include <string>
#include <type_traits>

#include <cooperative_groups.h>

#include "plans.cuh"
#include "sldg_common.cuh"
#include "tma_util.cuh"

namespace sldg {

static __global__ void k_fold_cols(const double* __restrict__ part, long long n_parts,
                                   long long n_cols, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long c = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (c >= n_cols) return;
  double s = 0.0;
  for (long long k = lane; k < n_parts; k += 32) s += part[c * n_parts + k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[c] = s;
}

static __global__ void k_fold3(const double* __restrict__ part, long long n, double* __restrict__ out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (w >= 3) return;
  double s = 0.0;
  for (long long k = lane; k < n; k += 32) s += part[k * 3 + w];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[w] = s;
}

constexpr int kFRing = 4;
constexpr int kMaxLev = 8;

struct FusedArgs {
  const double* w;
  const double* v0;
  const double* v2;
  const double* xw;
  double* mom_part;   // [grid][3]
  double* rho_part;   // [n_cols][grid] (column-major: a column's partials are contiguous)
};

template <bool B>
using BoolC = std::integral_constant<bool, B>;

// per-item tables in shared memory (two buffers: current item, next item)
struct ItemTabs {
  long long* crow;   // [nmax] first row of each cell (line 0)
  double* cm;        // [nmax][3][R] w, v0, v2 of the tile rows
  int* cg;           // [nmax][OV] x-speed index per (cell, v_x node)
};

// NXC > 0: the row length (x cells) is a compile-time constant, so every shared
// memory offset folds into the instruction (the headline configuration).
// MODE (a template flag: a runtime flag costs the steady-state kernel ~3%):
//   0 steady state: V + X1 (+ moments) + X2 (+ rho), as described above;
//   1 last step of a run: V + X1 (+ moments), X1's result is the state (-> HBM);
//   2 lead: the first half x-step alone, X1 (+ rho) -> HBM (no V) -- the tile
//     distribution of the other modes, so a pencil-sharded rank touches only its rows.
template <int OV, int OX, int LG, int NXC, int MODE>
__global__ void __launch_bounds__(384, 1)
k_step_fused(VPlanDev P, XPlanDev X, const double* __restrict__ fin, double* __restrict__ fout,
             int n_cols_arg, int n_xc_arg, const double* __restrict__ speeds, int bc,
             const long long* __restrict__ lm_ns, const double* __restrict__ lm_mats, int rw_arg,
             int n_speeds, int nmax, long long t_begin, long long n_tiles, FusedArgs fa) {
  const int n_xc = NXC > 0 ? NXC : n_xc_arg;
  const int n_cols = NXC > 0 ? OX * NXC : n_cols_arg;
  const int rw = NXC > 0 ? ((OX * NXC) | 1) : rw_arg;
  constexpr int XM = 2 * OX * OX;
  // composed x-step per v_x node: C0, C1, C2 (OX*OX each) then cA, cB (OX each),
  // every block padded to an even count so the X phase reads them as 16-byte pairs
  constexpr int XMP = (OX * OX + 1) & ~1, XZP = (OX + 1) & ~1;
  constexpr int XCS = 3 * XMP + 2 * XZP;        // doubles per v_x node (even)
  constexpr int XCL = 3 * OX * OX + 2 * OX;     // logical entries per v_x node
  constexpr int R = LG * OV;                    // rows per tile
  constexpr int n_lg = OV * OV / LG;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) unsigned long long full[kFRing];
  __shared__ int s_nsmin[kMaxLev], s_nsmax[kMaxLev];
  __shared__ __align__(16) long long s_wd[2][2];   // walk descriptor per table buffer

  const int tile = R * n_cols;                  // doubles per ring slot
  double* ring = sm;
  double* stA = ring + kFRing * tile;          // two tile buffers of R rows (stride rw)
  double* xtab = stA + 2 * R * rw;                 // n_speeds x (A|B) for the x shift
  int* xns = reinterpret_cast<int*>(xtab + (long long)n_speeds * XM);
  // composed x-step per tile and v_x node (MODE 0), two buffers alternating like
  // the tile buffers: C0 = A A, C1 = A B + B A, C2 = B B, then cA = A^T xw, cB = B^T xw
  double* xcmp = xtab + (long long)n_speeds * XM + 2 * ((n_speeds + 3) / 4);   // 16-byte aligned
  double* xw0 = xcmp + 2 * OV * XCS;            // x quadrature weights of one cell
  double* tabs0 = xw0 + OX;
  const int tab_dbl = nmax + 3 * R * nmax + (nmax * OV + 1) / 2;
  auto tabs = [&](int b) -> ItemTabs {
    double* base = tabs0 + (long long)b * tab_dbl;
    return ItemTabs{reinterpret_cast<long long*>(base), base + nmax,
                    reinterpret_cast<int*>(base + nmax + 3 * R * nmax)};
  };

  const int tid = threadIdx.x;
  const int nthr = blockDim.x;
  // this CTA's share of the tile range [t_begin, t_begin + n_tiles) (a rank's
  // pencils under pencil sharding; everything otherwise)
  const long long tb = t_begin + (long long)blockIdx.x * n_tiles / gridDim.x;
  const long long te = t_begin + (long long)(blockIdx.x + 1) * n_tiles / gridDim.x;
  if (te <= tb) {   // empty share: zero partials keep the folds over the grid valid
    grid_dep_wait();   // the preceding field chain may still be folding the partials
    for (int k = tid; k < n_cols_arg; k += nthr) fa.rho_part[(long long)k * gridDim.x + blockIdx.x] = 0.0;
    if (tid < 3) fa.mom_part[blockIdx.x * 3 + tid] = 0.0;
    return;
  }
  const long long it_first = tb / nmax, it_last = (te - 1) / nmax;   // item range (inclusive)
  const int n_items = (int)(it_last - it_first + 1);

  // x-shift tables; a zero shift is stored as (A, B) = (I, 0) with no cell shift so
  // the X phases run without a per-thread branch (1*u0 + 0*u1 + ... == u0)
  for (int k = tid; k < n_speeds * XM; k += nthr) {
    const int g = k / XM, e = k - g * XM;
    xtab[k] = X.ident[g] ? ((e < OX * OX && e % (OX + 1) == 0) ? 1.0 : 0.0) : __ldg(X.mats + k);
  }
  for (int k = tid; k < n_speeds; k += nthr) xns[k] = X.ident[k] ? 0 : (int)X.ns[k];
  if (tid < OX) xw0[tid] = __ldg(fa.xw + tid);   // uniform x grid: every cell's weights
  if (tid < kMaxLev) {
    s_nsmin[tid] = 1 << 30;
    s_nsmax[tid] = -(1 << 30);
  }
  if (tid == 0) {
    for (int k = 0; k < kFRing; ++k) mbar_init(&full[k], 1);
    mbar_fence_init();
  }
  sync_fz();

  const bool per = (bc == SLDG_BC_PERIODIC);
  const bool colv = tid < n_cols;
  const int c = tid;

  // ---- X-phase state: thread = (iv, x cell)
  const bool xv = tid < OV * n_xc;
  const int iv = xv ? tid / n_xc : 0;
  const int cx = xv ? tid - iv * n_xc : 0;
  // moments: each output row is contracted with the x weights first, then
  // weighted by (w, w*v0, w*v2); rho per x column
  double m0 = 0.0, m1 = 0.0, m2 = 0.0, rha[OX];
#pragma unroll
  for (int k = 0; k < OX; ++k) rha[k] = 0.0;

  // ---- item bookkeeping (uniform across the CTA)
  auto item_wp = [&](long long it) { return it / n_lg; };
  auto item_t0 = [&](long long it) { return (int)(it - (it / n_lg) * n_lg) * LG; };
  auto item_sb = [&](long long it) { return (int)(it == it_first ? tb - it * nmax : 0); };
  auto item_se = [&](long long it, int n) {
    return (int)min((long long)n, te - it * nmax);   // exclusive, clipped to the pencil
  };
  auto wd_n = [&](int b) { return (int)(s_wd[b][1] & 0xffffffffLL); };
  auto wd_lev = [&](int b) { return (int)(s_wd[b][1] >> 32); };
  // prefetch stages of item `it` into table buffer b (cp.async, completed by the
  // caller's cp_async_wait_all + __syncthreads before the next stage reads them)
  // per-tile extra work sits on different warps: the compose on threads 0.., the
  // ring pump on the last warp, the table stages from the second-to-last warp on
  const int pump_tid = nthr - 32;
  const int rt = tid >= nthr - 64 ? tid - (nthr - 64) : tid + 64;
  auto stage = [&](int st, int b, long long it) {
    const ItemTabs T = tabs(b);
    if (st == 0) {
      if (rt == 0) cp_async16(&s_wd[b][0], P.walk_desc + 2 * item_wp(it));
    } else if (st == 1) {
      const long long off = s_wd[b][0];
      const int n = wd_n(b);
      for (int k = rt; k < n; k += nthr) cp_async8(T.crow + k, P.e_row0 + off + k);
    } else {
      const int n = wd_n(b);
      const long long l0 = (long long)item_t0(it) * OV;
      for (int k = rt; k < n * OV; k += nthr)
        cp_async4(T.cg + k, X.row_speed + T.crow[k / OV] + l0 + k % OV);
      for (int k = rt; k < n * 3 * R; k += nthr) {
        const int s2 = k / (3 * R), rem = k - s2 * 3 * R, a = rem / R, r = rem - a * R;
        const double* src = a == 0 ? fa.w : (a == 1 ? fa.v0 : fa.v2);
        cp_async8(T.cm + k, src + T.crow[s2] + l0 + r);
      }
    }
  };
  auto stage_sync = [&](int st, int b, long long it) {
    stage(st, b, it);
    cp_async_wait_all();
    sync_fz();
  };

  // item 0 tables, synchronously
  for (int st = 0; st < 3; ++st) stage_sync(st, 0, it_first);

  // Everything above depends only on the plans and the state, so under
  // programmatic dependent launch it overlaps the preceding field chain; E and
  // the level matrices it writes are read only from here on.
  grid_dep_wait();
  // ---- V-phase state: thread = column; a level is streamable when every moving
  // column's integer shift is -1 or 0 (sources in cells s-1, s, s+1)
  // (lead mode has no v-sweep: every column takes the copy path)
  const double speed = (colv && MODE != 2) ? __ldg(speeds + c) : 0.0;
  if (colv && speed != 0.0) {
    for (int L = 0; L < P.n_levels; ++L) {
      const long long v = lm_ns[(long long)L * n_cols + c];
      const int nsi = (int)max(min(v, (long long)(1 << 29)), -(long long)(1 << 29));
      atomicMin(&s_nsmin[L], nsi);
      atomicMax(&s_nsmax[L], nsi);
    }
  }
  sync_fz();

  // ---- ring of cell tiles: one load sequence across the CTA's items.  Item i's
  // loads are the cells first..last of its segment (sb-1..se, wrapped when
  // periodic, clipped when absorbing); non-streamable items load nothing.
  auto seg_first = [&](int sb) { return per ? sb - 1 : max(sb - 1, 0); };
  auto seg_last = [&](int se, int n) { return per ? se : min(se, n - 1); };
  // pump-thread issue cursor, kept in shared memory (no registers across the loop):
  // item, next cell, last cell, loads issued, cursor initialised for the item
  __shared__ int s_cur[5];
  if (tid == pump_tid) {
    s_cur[0] = 0;
    s_cur[1] = 0;
    s_cur[2] = -1;
    s_cur[3] = 0;
    s_cur[4] = 0;
  }
  auto pump = [&](int limit, int cur_i, bool next_ready) {
    int ld_i = s_cur[0], ld_c = s_cur[1], ld_last = s_cur[2], issued = s_cur[3];
    bool ld_init = s_cur[4] != 0;
    while (issued < limit && ld_i < n_items) {
      if (ld_i > cur_i + 1 || (ld_i == cur_i + 1 && !next_ready)) break;
      const int b = ld_i & 1;
      const long long it = it_first + ld_i;
      const int n = wd_n(b);
      if (!ld_init) {
        const int sb = item_sb(it), se = item_se(it, n);
        const int lev = wd_lev(b);
        const bool strm = (s_nsmin[lev] >= -1 && s_nsmax[lev] <= 0) || (s_nsmin[lev] > s_nsmax[lev]);
        ld_c = seg_first(sb);
        ld_last = (strm && se > sb) ? seg_last(se, n) : ld_c - 1;
        ld_init = true;
      }
      if (ld_c > ld_last) {
        ++ld_i;
        ld_init = false;
        continue;
      }
      const int cell = ld_c < 0 ? n - 1 : (ld_c >= n ? 0 : ld_c);
      const long long row0 = tabs(b).crow[cell] + (long long)item_t0(it) * OV;
      unsigned long long* bar = &full[issued & (kFRing - 1)];
      mbar_expect_tx(bar, (unsigned)(tile * 8));
      bulk_g2s(ring + (issued & (kFRing - 1)) * tile, fin + row0 * n_cols, (unsigned)(tile * 8), bar);
      ++issued;
      ++ld_c;
    }
    s_cur[0] = ld_i;
    s_cur[1] = ld_c;
    s_cur[2] = ld_last;
    s_cur[3] = issued;
    s_cur[4] = ld_init ? 1 : 0;
  };

  double Av[OV * OV], Bv[OV * OV];
  long long nsv = 0;
  int cur_lev = -1;
  int base = 0;   // load index of the current item's first load
  int waited = -1;   // highest load index this thread has waited for

  // V phase of one column: rows t*OV+i of the source cells sa / sb -> column c of
  // the tile buffer `out`.  CHECKED: the source cells may lie outside the pencil
  // (absorbing ends).
  auto vcol = [&](double* out, const double* sa, const double* sb, bool va, bool vb, auto checked) {
    constexpr bool CK = decltype(checked)::value;
#pragma unroll
    for (int t = 0; t < LG; ++t) {
      double ua[OV], ub[OV], y[OV];
#pragma unroll
      for (int i = 0; i < OV; ++i) {
        const int r = t * OV + i;
        if (CK) {
          ua[i] = va ? sa[r * n_cols] : 0.0;
          ub[i] = vb ? sb[r * n_cols] : 0.0;
        } else {
          ua[i] = sa[r * n_cols];
          ub[i] = sb[r * n_cols];
        }
      }
      two_cell<OV>(Av, Bv, ua, ub, CK ? va : true, CK ? vb : true, y);
#pragma unroll
      for (int i = 0; i < OV; ++i) out[(t * OV + i) * rw] = y[i];
    }
  };
  auto vcopy = [&](double* out, const double* me) {
#pragma unroll
    for (int r = 0; r < R; ++r) out[r * rw] = me[r * n_cols];
  };
  // 1-D periodic shift of the x cells of one row by the x-speed's (A, B): cell
  // sources ua (cell - n) and ub (cell - n - 1), same arithmetic as k_xx_tiles / k_advect_x
  auto xmul = [&](const double* xa, const double* xb, const double* ua, const double* ub, double* y) {
#pragma unroll
    for (int k = 0; k < OX; ++k) {
      double sa = xa[k * OX] * ua[0];
      double sb2 = xb[k * OX] * ub[0];
#pragma unroll
      for (int j = 1; j < OX; ++j) {
        sa = fma(xa[k * OX + j], ua[j], sa);
        sb2 = fma(xb[k * OX + j], ub[j], sb2);
      }
      y[k] = sa + sb2;
    }
  };
  auto wrap = [&](int k) { return k < 0 ? k + n_xc : (k >= n_xc ? k - n_xc : k); };

  for (int i = 0; i < n_items; ++i) {
    const int b = i & 1;
    const long long it = it_first + i;
    const ItemTabs T = tabs(b);
    const int n = wd_n(b), lev = wd_lev(b);
    const int sb = item_sb(it), se = item_se(it, n);
    const long long l0 = (long long)item_t0(it) * OV;
    const bool streamable =
        (s_nsmin[lev] >= -1 && s_nsmax[lev] <= 0) || (s_nsmin[lev] > s_nsmax[lev]);
    const int first = seg_first(sb), last = seg_last(se, n);
    if (lev != cur_lev) {
      cur_lev = lev;
      if (colv) {
        load_pair<OV>(lm_mats, lev, n_cols, c, Av, Bv);
        nsv = lm_ns[(long long)lev * n_cols + c];
      }
    }
    const bool has_next = i + 1 < n_items;
    int n_staged = 0;   // tile barriers passed in this item (= prefetch stages issued + 1)

    // ===================== V: pencil sweep of cell s -> tile buffer (R rows, stride rw)
    auto v_pump = [&](int s) {
      if (streamable && tid == pump_tid) pump(base + max(s - 1, first) - first + kFRing, i, n_staged >= 4);
    };
    auto v_tile = [&](int s, double* dst) {
      if (streamable) {
        const int klo = base + max(s - 1, first) - first, khi = base + min(s + 1, last) - first;
        // loads up to `waited` were waited for at earlier tiles (their slots are
        // not refilled before every thread is past them): only the new ones
        for (unsigned k = (unsigned)max(klo, waited + 1); k <= (unsigned)khi; ++k)
          mbar_wait(&full[k & (kFRing - 1)], (k / kFRing) & 1u);
        waited = max(waited, khi);
        if (colv) {
          double* out = dst + c;
          auto slot = [&](int cell) { return ring + ((base + cell - first) & (kFRing - 1)) * tile + c; };
          if (speed == 0.0) {
            vcopy(out, slot(s));
          } else {
            // streamable: source cells s - nsv and s - nsv - 1 with nsv in {-1, 0}
            const int va_cell = s - (int)nsv, vb_cell = va_cell - 1;
            if (per || (s > 0 && s < n - 1)) {
              vcol(out, slot(va_cell), slot(vb_cell), true, true, BoolC<false>{});
            } else {
              const bool va = va_cell >= 0 && va_cell < n, vb = vb_cell >= 0 && vb_cell < n;
              vcol(out, slot(va ? va_cell : s), slot(vb ? vb_cell : s), va, vb, BoolC<true>{});
            }
          }
        }
      } else if (colv) {
        double* out = dst + c;
        const long long r0 = T.crow[s] + l0;
        if (speed == 0.0) {
          vcopy(out, fin + r0 * n_cols + c);
        } else {
          long long qa = s - nsv, qb = s - nsv - 1;
          bool va = true, vb = true;
          if (per) {
            qa = pymod(qa, n);
            qb = pymod(qb, n);
          } else {
            va = qa >= 0 && qa < n;
            vb = qb >= 0 && qb < n;
          }
          vcol(out, fin + (T.crow[va ? (int)qa : s] + l0) * n_cols + c,
               fin + (T.crow[vb ? (int)qb : s] + l0) * n_cols + c, va, vb, BoolC<true>{});
        }
      }
    };
    // ===================== X of cell s from its V result `src`:
    //   MODE 0: trailing half step X1 (+ moments) and the next step's leading half
    //     step X2 (+ rho) -> HBM.  Both use the row's x-speed, so X2 at cell cx
    //     depends on the V result at cells a - n, a - n - 1, a - n - 2 (a = cx - n)
    //     through the composed matrices; the moments take X1 at cell a (cx -> a is a
    //     bijection of the row's cells).
    //   MODE 1: X1 (+ moments) -> HBM;  MODE 2: X1 (+ rho) -> HBM.
    auto x_tile = [&](int s, const double* src, const double* src_cmp) {
      if (!xv) return;
      const double* mcur = T.cm + (long long)s * 3 * R;
      const long long r0 = T.crow[s] + l0;
      const int g = T.cg[s * OV + iv];
      double xa[OX * OX], xb[OX * OX];
      const double* AB = xtab + (long long)g * XM;
#pragma unroll
      for (int k = 0; k < OX * OX; ++k) {
        xa[k] = AB[k];
        xb[k] = AB[OX * OX + k];
      }
      const int ns = xns[g];
      const int ca = wrap(cx - ns);
      double* dst = fout + (r0 + iv) * n_cols + cx * OX;
      if (MODE == 0) {
        // composed step: y = C0 u(a - n) + C1 u(a - n - 1) + C2 u(a - n - 2), a = cx - n,
        // one matrix at a time over the tile's LG rows (each matrix's partial sums
        // are formed separately and added in the order (s0 + s1) + s2); the trailing
        // half step's moment weight is z = xw . X1(a) = cA . u0 + cB . u1
        const double* Cc = src_cmp + iv * XCS;
        const int p0 = wrap(ca - ns);
        const int p1 = p0 == 0 ? n_xc - 1 : p0 - 1;
        const int p2 = p1 == 0 ? n_xc - 1 : p1 - 1;
        double acc[LG][OX], zs[LG];
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          double cm[XMP], cz[XZP];
#pragma unroll
          for (int k = 0; k < XMP; k += 2) {
            const double2 q = *reinterpret_cast<const double2*>(Cc + m * XMP + k);
            cm[k] = q.x;
            cm[k + 1] = q.y;
          }
          if (m < 2) {
#pragma unroll
            for (int k = 0; k < XZP; k += 2) {
              const double2 q = *reinterpret_cast<const double2*>(Cc + 3 * XMP + m * XZP + k);
              cz[k] = q.x;
              cz[k + 1] = q.y;
            }
          }
          const int pc = (m == 0 ? p0 : (m == 1 ? p1 : p2)) * OX;
#pragma unroll
          for (int t = 0; t < LG; ++t) {
            const double* u = src + (t * OV + iv) * rw + pc;
            double uu[OX];
#pragma unroll
            for (int j = 0; j < OX; ++j) uu[j] = u[j];
            // one FMA chain per output across the three matrices (no separate
            // partial sums: fewer instructions, same result to rounding)
#pragma unroll
            for (int k = 0; k < OX; ++k) {
              double a = m == 0 ? cm[k * OX] * uu[0] : fma(cm[k * OX], uu[0], acc[t][k]);
#pragma unroll
              for (int j = 1; j < OX; ++j) a = fma(cm[k * OX + j], uu[j], a);
              acc[t][k] = a;
            }
            if (m < 2) {
              double zz = m == 0 ? cz[0] * uu[0] : fma(cz[0], uu[0], zs[t]);
#pragma unroll
              for (int j = 1; j < OX; ++j) zz = fma(cz[j], uu[j], zz);
              zs[t] = zz;
            }
          }
        }
#pragma unroll
        for (int t = 0; t < LG; ++t) {
          const int r = t * OV + iv;
          const double wr = mcur[r];
          const double wv0 = wr * mcur[R + r], wv2 = wr * mcur[2 * R + r];
#pragma unroll
          for (int k = 0; k < OX; ++k) {
            dst[k] = acc[t][k];
            rha[k] = fma(wr, acc[t][k], rha[k]);
          }
          m0 = fma(wr, zs[t], m0);
          m1 = fma(wv0, zs[t], m1);
          m2 = fma(wv2, zs[t], m2);
          dst += (long long)OV * n_cols;
        }
      } else {
        const int ia = ca * OX, ib = (ca == 0 ? n_xc - 1 : ca - 1) * OX;
#pragma unroll
        for (int t = 0; t < LG; ++t) {
          const int r = t * OV + iv;
          const double* srow = src + r * rw;
          double ua[OX], ub[OX], y[OX];
#pragma unroll
          for (int j = 0; j < OX; ++j) {
            ua[j] = srow[ia + j];
            ub[j] = srow[ib + j];
          }
          xmul(xa, xb, ua, ub, y);
          const double wr = mcur[r];
#pragma unroll
          for (int k = 0; k < OX; ++k) dst[k] = y[k];
          if (MODE == 2) {
#pragma unroll
            for (int k = 0; k < OX; ++k) rha[k] = fma(wr, y[k], rha[k]);
          } else {
            const double wv0 = wr * mcur[R + r], wv2 = wr * mcur[2 * R + r];
            double z = xw0[0] * y[0];
#pragma unroll
            for (int k = 1; k < OX; ++k) z = fma(xw0[k], y[k], z);
            m0 = fma(wr, z, m0);
            m1 = fma(wv0, z, m1);
            m2 = fma(wv2, z, m2);
          }
          dst += (long long)OV * n_cols;
        }
      }
    };
    // MODE 0: composed x-step of cell s's v_x nodes -> dst (XCS entries per node)
    auto x_compose = [&](int s, double* dst) {
      for (int e0 = MODE == 0 ? tid : OV * XCL; e0 < OV * XCL; e0 += nthr) {   // (MODE 0 only;
                                                        // the CTA may have < OV*XCL threads)
        const int jv = e0 / XCL, e = e0 - jv * XCL;
        int pos;   // padded position of logical entry e
        const double* A = xtab + (long long)T.cg[s * OV + jv] * XM;
        const double* B = A + OX * OX;
        double v;
        if (e < 3 * OX * OX) {
          const int w = e / (OX * OX), k = (e / OX) % OX, j = e % OX;
          pos = w * XMP + k * OX + j;
          const double* L = w == 2 ? B : A;
          const double* Rm = w == 0 ? A : B;
          v = L[k * OX] * Rm[j];
#pragma unroll
          for (int m = 1; m < OX; ++m) v = fma(L[k * OX + m], Rm[m * OX + j], v);
          if (w == 1) {
#pragma unroll
            for (int m = 0; m < OX; ++m) v = fma(B[k * OX + m], A[m * OX + j], v);
          }
        } else {
          const int q = e - 3 * OX * OX, j = q % OX;
          pos = 3 * XMP + (q < OX ? 0 : XZP) + j;
          const double* M = q < OX ? A : B;
          v = xw0[0] * M[j];
#pragma unroll
          for (int k = 1; k < OX; ++k) v = fma(xw0[k], M[k * OX + j], v);
        }
        dst[jv * XCS + pos] = v;
      }
    };
    // one CTA barrier per tile; the next item's table prefetch advances one stage
    // per barrier (copies issued after barrier k complete before barrier k + 1)
    auto tile_barrier = [&]() {
      if (n_staged > 0 && n_staged <= 3) cp_async_wait_all();
      sync_fz();
      if (has_next && n_staged < 3) stage(n_staged, b ^ 1, it + 1);
      ++n_staged;
    };

    // software pipeline over the item's cells, tile buffers alternating: V(s+1)
    // and X(s) between the same two barriers (X(s) reads the buffer V(s) wrote
    // before the previous barrier; V(s+1) writes the buffer X(s-1) read before it;
    // the ring slot a pump refills was last read by a V before the previous barrier)
    v_pump(sb);
    x_compose(sb, xcmp);
    v_tile(sb, stA);
    tile_barrier();
    for (int s = sb; s < se; ++s) {
      const int j = s - sb;
      double* cur = stA + (j & 1) * R * rw;
      double* nxt = stA + ((j + 1) & 1) * R * rw;
      if (s + 1 < se) v_pump(s + 1);
      x_tile(s, cur, xcmp + (j & 1) * OV * XCS);
      if (s + 1 < se) {
        x_compose(s + 1, xcmp + ((j + 1) & 1) * OV * XCS);
        v_tile(s + 1, nxt);
      }
      tile_barrier();
    }
    if (streamable && se > sb) base += last - first + 1;
    if (has_next && n_staged < 4) {
      // finish the next item's prefetch when this segment was too short to hide it
      if (n_staged >= 1) cp_async_wait_all();
      sync_fz();
      for (int st = n_staged; st < 3; ++st) stage_sync(st, b ^ 1, it + 1);
    }
  }
  grid_dep_launch();   // the next field chain may be scheduled (it waits for our end)
  // (the tile buffers are reused by the reduction below: the last tile barrier
  // separates it from the last X)

  // ---- CTA partials: rho per column (over i_v in order), moments contracted with xw
  double* red = stA;   // reuse: OV x n_cols, then 3 x blockDim
  if (xv) {
#pragma unroll
    for (int k = 0; k < OX; ++k) red[iv * n_cols + cx * OX + k] = rha[k];
  }
  sync_fz();
  if (colv) {
    double s = 0.0;
    for (int k = 0; k < OV; ++k) s += red[k * n_cols + c];
    fa.rho_part[(long long)c * gridDim.x + blockIdx.x] = s;
  }
  sync_fz();
  red[tid] = m0;
  red[nthr + tid] = m1;
  red[2 * nthr + tid] = m2;
  sync_fz();
  if (tid < 3) {
    double s = 0.0;
    for (int k = 0; k < nthr; ++k) s += red[tid * nthr + k];
    fa.mom_part[blockIdx.x * 3 + tid] = s;
  }
}

struct FusedGeom {
  bool ok;
  int lg, n_lg, rw, threads, nmax;
  size_t smem;
  long long grid, n_tiles;
  std::string why;
};

static int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static FusedGeom fused_geom(const sldg_vplan* vp, const sldg_xplan* xp, long long n_cols,
                            long long ld) {
  FusedGeom g{};
  g.ok = false;
  const int OV = vp->o, OX = xp->o;
  auto no = [&](const char* w) {
    g.why = w;
    return g;
  };
  if (vp->dim != 3 || vp->direction != 0) return no("fused step: dim 3, direction 0 only");
  if (vp->n_gen != 0 || vp->n_slots != 0) return no("fused step: AMR boundary / weighted entries");
  if (vp->n_walk == 0) return no("fused step: no pencils");
  if (vp->dev.n_levels > kMaxLev) return no("fused step: too many levels");
  if (ld != n_cols || n_cols != xp->n_cells * OX) return no("fused step: whole rows only");
  if (OV < 2 || OV > 4 || OX < 2 || OX > 4) return no("fused step: degrees 1..3");
  const long long threads = std::max<long long>(n_cols, OV * xp->n_cells);
  if (threads > 384) return no("fused step: rows wider than 384 columns");
  const int hl = (int)xp->halo_l, hr = (int)xp->halo_r;
  if (hl > xp->n_cells || hr > xp->n_cells) return no("fused step: shift wider than the row");
  g.rw = (int)n_cols + (n_cols % 2 == 0 ? 1 : 0);   // odd row stride: conflict-free columns
  g.nmax = vp->max_walk_cells;
  const size_t fixed = sizeof(double) * (size_t)xp->n_speeds * 2 * OX * OX +
                       sizeof(double) * (2 * ((xp->n_speeds + 3) / 4) +
                                         2 * OV * (3 * ((OX * OX + 1) & ~1) + 2 * ((OX + 1) & ~1)) + OX) + 64;
  const size_t nmax = (size_t)g.nmax;
  const size_t budget = 227 * 1024 - 1024;
  g.lg = 0;
  for (int lg = 4; lg >= 1; --lg) {   // instantiated line groups: OV, 2 (even OV), 1
    if ((OV * OV) % lg || (lg != OV && lg != 2 && lg != 1)) continue;
    const size_t R = (size_t)lg * OV;
    const size_t tables = 2 * sizeof(double) * (nmax + 3 * R * nmax + (nmax * OV + 1) / 2);
    const size_t smem = sizeof(double) * (kFRing * R * n_cols + 2 * R * g.rw) + fixed + tables;
    // the moment reduction stores 3 values per launched thread (blockDim rounded to 32)
    const size_t red = sizeof(double) * std::max<size_t>(OV * n_cols, 3 * ((threads + 31) / 32 * 32));
    if (smem <= budget && sizeof(double) * 2 * R * g.rw >= red) {
      // prefer two CTAs per SM when possible
      if (2 * smem <= budget || g.lg == 0) {
        g.lg = lg;
        g.smem = smem;
        if (2 * smem <= budget) break;
      }
    }
  }
  if (g.lg == 0) return no("fused step: tile does not fit in shared memory");
  g.n_lg = OV * OV / g.lg;
  g.threads = (int)((threads + 31) / 32 * 32);
  g.n_tiles = vp->n_walk * g.n_lg * (long long)g.nmax;
  // upper bound on the persistent grid (partials are sized for it); the launch
  // clamps it to the resident CTA count
  g.grid = std::min<long long>(g.n_tiles, 2LL * sm_count());
  g.ok = true;
  return g;
}

using FusedKernel = void (*)(VPlanDev, XPlanDev, const double*, double*, int, int, const double*,
                             int, const long long*, const double*, int, int, int, long long,
                             long long, FusedArgs);

template <int OV, int OX, int MODE>
static FusedKernel pick_kernel_m(int lg, long long n_xc) {
  if (lg == OV) {
    if constexpr (OV == 3 && OX == 3) {
      if (n_xc == 64) return k_step_fused<3, 3, 3, 64, MODE>;
    }
    return k_step_fused<OV, OX, OV, 0, MODE>;
  }
  if constexpr (OV % 2 == 0 && OV != 2) {
    if (lg == 2) return k_step_fused<OV, OX, 2, 0, MODE>;
  }
  if (lg == 1) return k_step_fused<OV, OX, 1, 0, MODE>;
  return nullptr;
}

template <int OV, int OX>
static FusedKernel pick_kernel(int lg, long long n_xc, int mode) {
  if (mode == 1) return pick_kernel_m<OV, OX, 1>(lg, n_xc);
  if (mode == 2) return pick_kernel_m<OV, OX, 2>(lg, n_xc);
  return pick_kernel_m<OV, OX, 0>(lg, n_xc);
}

static FusedKernel fused_kernel(const sldg_vplan* vp, const sldg_xplan* xp, const FusedGeom& g,
                                int mode) {
  switch (vp->o * 10 + xp->o) {
#define CASE(A, B) \
  case A * 10 + B: return pick_kernel<A, B>(g.lg, xp->n_cells, mode);
    CASE(2, 2) CASE(2, 3) CASE(2, 4) CASE(3, 2) CASE(3, 3) CASE(3, 4) CASE(4, 2) CASE(4, 3)
    CASE(4, 4)
#undef CASE
  }
  return nullptr;
}

// resident persistent grid (deterministic for a device): one grid for all three
// modes, the smallest of their resident counts, so that the folds (which only know
// the plan) read exactly the partial rows any mode's launch wrote
static int fused_grid(const sldg_vplan* vp, const sldg_xplan* xp, const FusedGeom& g,
                      long long* grid) {
  int per_sm = 1 << 30;
  for (int mode = 0; mode < 3; ++mode) {
    FusedKernel k = fused_kernel(vp, xp, g, mode);
    if (!k) {
      set_error("fused step: no kernel for this degree / line group");
      return SLDG_ERR_UNSUPPORTED;
    }
    int r = 0;
    SLDG_CUDA_TRY(resident_ctas((const void*)k, g.threads, (int)g.smem, &r));
    per_sm = std::min(per_sm, std::max(r, 1));
  }
  *grid = std::max<long long>(1, std::min<long long>(g.grid, (long long)per_sm * sm_count()));
  return SLDG_OK;
}

static size_t al256(size_t x) { return (x + 255) / 256 * 256; }

// launch with programmatic stream serialization: the kernel may start while the
// previous kernel in the stream finishes; it orders itself with grid_dep_wait()
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

// scratch of the fused step: level matrices, then the CTA partials
struct FusedScratch {
  long long* lm_ns;
  double *lm_frac, *lm_mats, *mom_part, *rho_part;
  size_t bytes;
};
static FusedScratch fused_scratch(const sldg_vplan* vp, const FusedGeom& g, long long n_cols,
                                  void* base) {
  FusedScratch s{};
  unsigned char* sb = (unsigned char*)base;
  const size_t nl = (size_t)vp->dev.n_levels;
  size_t o = 0;
  s.lm_ns = (long long*)(sb + o);
  o += al256(sizeof(long long) * nl * n_cols);
  s.lm_frac = (double*)(sb + o);
  o += al256(sizeof(double) * nl * n_cols);
  s.lm_mats = (double*)(sb + o);
  o += al256(sizeof(double) * nl * 2 * vp->o * vp->o * n_cols);
  s.mom_part = (double*)(sb + o);
  o += al256(sizeof(double) * g.grid * 3);
  s.rho_part = (double*)(sb + o);
  o += al256(sizeof(double) * g.grid * n_cols);
  s.bytes = o;
  return s;
}

// The field work between two fused steps in one launch of a cluster of kChainCtas CTAs
// (distributed shared memory between them), each stage with the same per-element
// arithmetic and reduction order as its stand-alone kernel, so the results are bitwise
// identical to  [k_fold_cols, k_fold3] -> k_poisson_rhs -> k_gemv -> k_efield ->
// k_field_diag, k_level_mats:
//   fold     CTA r folds its contiguous share of the columns (warp per column, lanes over
//            the CTA partials, xor butterfly: k_fold_cols), CTA 0 the moments (k_fold3);
//   rho      gathered from the cluster's shared memory into every CTA;
//   rhs      rbar by the 1024-slot tree of k_poisson_rhs, the load vector b (every CTA);
//   phi      rows split over the CTAs (warp per row, k_gemv), gathered;
//   E        DOFs split over the CTAs (k_efield); CTA 0 gathers E for the diagnostics
//            (the 1024-slot trees of k_field_diag) while every CTA forms the level
//            matrices of its columns, one thread per (level, column, A|B).
#ifndef SLDG_CHAIN_CTAS
#define SLDG_CHAIN_CTAS 8
#endif
constexpr int kChainCtas = SLDG_CHAIN_CTAS;   // CTAs of the field chain cluster
constexpr int kChainThreads = 512;
constexpr int kChainMaxDofs = 1024;   // x DOFs (and FE nodes) a chain handles

#ifdef SLDG_CHAIN_PROF
// " %d" into buf (device printf of one line per CTA)
__device__ int snprintf_dev(char* buf, int v) {
  char t[12];
  int n = 0;
  if (v < 0) v = 0;
  do {
    t[n++] = (char)('0' + v % 10);
    v /= 10;
  } while (v && n < 11);
  buf[0] = ' ';
  for (int i = 0; i < n; ++i) buf[1 + i] = t[n - 1 - i];
  buf[n + 1] = 0;
  return n + 1;
}
#endif
constexpr int kFoldRegs = 16;
constexpr int kGreenRegs = 4;   // first Green row's coefficients per lane held in registers   // CTA partials per lane held in registers by the folds

// second half of the cluster barrier the chain arrives at on entry: every CTA of the
// cluster is running (its shared memory may take DSMEM stores)
__device__ __forceinline__ void cluster_started() {
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}


// The 1024-slot tree of the stand-alone reductions (for st = 512 .. 1: red[t] op=
// red[t + st], t < st) in one warp with no barriers: lane l first combines the 32 slots
// l + 32 k with the tree's own pairs (levels 512 .. 32: k op= k + 16, 8, 4, 2, 1), then
// levels 16 .. 1 by shuffles.  Same operands in the same order: bitwise identical.
template <typename Val, typename Op>
__device__ __forceinline__ double warp_tree1024(int lane, Val val, Op op) {
  double v[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = val(lane + 32 * k);
#pragma unroll
  for (int h = 16; h > 0; h >>= 1)
#pragma unroll
    for (int k = 0; k < h; ++k) v[k] = op(v[k], v[k + h]);
  double r = v[0];
#pragma unroll
  for (int st = 16; st > 0; st >>= 1) {
    const double o = __shfl_down_sync(0xffffffffu, r, st);
    r = op(r, o);
  }
  return __shfl_sync(0xffffffffu, r, 0);
}


template <int O>
__global__ void __cluster_dims__(kChainCtas, 1, 1) __launch_bounds__(kChainThreads, 1)
k_field_chain(const double* __restrict__ rho_in, const double* __restrict__ rho_part,
              const double* __restrict__ mom_part, long long n_parts,
              double* __restrict__ mom_prev, double* __restrict__ rho, const double* __restrict__ pxw,
              const double* __restrict__ green, const double* __restrict__ diff,
              long long n_cells, int p, double length, double h, double* __restrict__ b,
              double* __restrict__ phi, double* __restrict__ e, double* __restrict__ diag2,
              DevBasis vb, double dt, double base_width, int n_levels,
              long long* __restrict__ lm_ns, double* __restrict__ lm_frac,
              double* __restrict__ lm_mats) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ double r_s[kChainMaxDofs], phi_s[kChainMaxDofs], phx[kChainMaxDofs],
      e_s[kChainMaxDofs], xw_s[kChainMaxDofs], diff_s[kMaxO * kMaxO];
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5, nw = blockDim.x >> 5;
  const int rank = (int)cluster.block_rank();
  const int o = p + 1;
  const int nd = (int)(n_cells * o), nn = (int)(n_cells * p), np = (int)n_parts;
  auto share = [&](int n, int r) { return (int)((long long)n * r / kChainCtas); };
  const int c0 = share(nd, rank), c1 = share(nd, rank + 1);     // my columns / DOFs
  const int q0 = share(nn, rank), q1 = share(nn, rank + 1);     // my FE rows
  // -DSLDG_CHAIN_PROF: global-timer stamps between the stages, printed by CTAs 0 and 1
#ifdef SLDG_CHAIN_PROF
  unsigned long long tst[10];
  int nst = 0;
#define CHAIN_STAMP() asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tst[nst++]))
#else
#define CHAIN_STAMP() do {} while (0)
#endif
  CHAIN_STAMP();
  // DSMEM stores need the peer CTAs running: arrive now, wait before the first push
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  // the plan's constants (x weights, derivative matrix, my first Green row) before the
  // dependency wait: they overlap the preceding fused step's tail
  for (int t = tid; t < nd; t += blockDim.x) xw_s[t] = __ldg(pxw + t);
  if (tid < o * o) diff_s[tid] = __ldg(diff + tid);
  const int row0 = q0 + wp;
  double gr[kGreenRegs];
#pragma unroll
  for (int i = 0; i < kGreenRegs; ++i) {
    const int k = lane + 32 * i;
    gr[i] = (row0 < q1 && k < nn) ? __ldg(green + (size_t)row0 * nn + k) : 0.0;
  }
  // PDL: wait for the preceding fused step (its partials and state are complete),
  // then let the next fused step start its E-independent prologue alongside us
  grid_dep_wait();
  grid_dep_launch();
  CHAIN_STAMP();
  if (!rho_in) {
    // fold (k_fold_cols / k_fold3 order: lane l sums partials l, l+32, ... in sequence,
    // then the xor butterfly); every load of a warp's columns is issued before the sums
    // (one L2 round trip instead of one per four partials per column)
    for (int ca = c0 + wp; ca < c1; ca += 2 * nw) {
      const int cb = ca + nw;
      const bool hb = cb < c1;
      const double* qa = rho_part + (size_t)ca * np;
      const double* qb = rho_part + (size_t)(hb ? cb : ca) * np;
      double va[kFoldRegs], vb[kFoldRegs];
#pragma unroll
      for (int i = 0; i < kFoldRegs; ++i) {
        const int k = lane + 32 * i;
        va[i] = k < np ? __ldg(qa + k) : 0.0;
        vb[i] = (hb && k < np) ? __ldg(qb + k) : 0.0;
      }
      double sa = 0.0, sb = 0.0;
#pragma unroll
      for (int i = 0; i < kFoldRegs; ++i)
        if (lane + 32 * i < np) {
          sa += va[i];
          sb += vb[i];
        }
      for (int k = lane + 32 * kFoldRegs; k < np; k += 32) {
        sa += __ldg(qa + k);
        sb += __ldg(qb + k);
      }
#pragma unroll
      for (int of = 16; of > 0; of >>= 1) {
        sa += __shfl_xor_sync(0xffffffffu, sa, of);
        sb += __shfl_xor_sync(0xffffffffu, sb, of);
      }
      if (lane == 0) {
        rho[ca] = sa;
        r_s[ca] = sa;
        if (hb) {
          rho[cb] = sb;
          r_s[cb] = sb;
        }
      }
    }
    // moments (k_fold3 order) on the last three warps of CTA 0 (they fold fewer columns)
    const int mw = wp - (nw - 3);
    if (rank == 0 && mom_prev && mw >= 0) {
      double v[kFoldRegs];
#pragma unroll
      for (int i = 0; i < kFoldRegs; ++i) {
        const int k = lane + 32 * i;
        v[i] = k < np ? __ldg(mom_part + (size_t)k * 3 + mw) : 0.0;
      }
      double sacc = 0.0;
#pragma unroll
      for (int i = 0; i < kFoldRegs; ++i)
        if (lane + 32 * i < np) sacc += v[i];
      for (int k = lane + 32 * kFoldRegs; k < np; k += 32) sacc += mom_part[(size_t)k * 3 + mw];
#pragma unroll
      for (int of = 16; of > 0; of >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, of);
      if (lane == 0) mom_prev[mw] = sacc;
    }
    CHAIN_STAMP();
    // my columns pushed into the shared rho of every CTA (no gather after the barrier)
    cluster_started();
    __syncthreads();
    for (int k = tid; k < (c1 - c0) * kChainCtas; k += blockDim.x) {
      const int c = c0 + k / kChainCtas, dst = k % kChainCtas;
      if (dst != rank) *cluster.map_shared_rank(&r_s[c], dst) = r_s[c];
    }
    fuzz_delay();
    cluster.sync();   // every CTA's columns are in every r_s
    CHAIN_STAMP();
  } else {
    cluster_started();
    for (int c = tid; c < nd; c += blockDim.x) r_s[c] = rho_in[c];
    __syncthreads();
  }
  // Poisson right-hand side (k_poisson_rhs): fma(w, r, 0) per slot, the 1024-slot tree,
  // evaluated by every warp on its own (warp_tree1024: same pairs, same order)
  const double rbar = warp_tree1024(lane, [&](int t) {
    return t < nd ? fma(xw_s[t], r_s[t], 0.0) : 0.0;
  }, [](double x, double y) { return x + y; }) / length;
  for (int node = tid; node < nn; node += blockDim.x) {
    const int cell = node / p, j = node - cell * p;
    double v;
    if (j == 0) {
      const int kprev = (cell == 0 ? (int)n_cells - 1 : cell - 1) * o + p, kthis = cell * o;
      const double cprev = __dmul_rn(xw_s[kprev], __dsub_rn(r_s[kprev], rbar));
      const double cthis = __dmul_rn(xw_s[kthis], __dsub_rn(r_s[kthis], rbar));
      v = (cell == 0) ? __dadd_rn(cthis, cprev) : __dadd_rn(cprev, cthis);
    } else {
      const int k = cell * o + j;
      v = __dmul_rn(xw_s[k], __dsub_rn(r_s[k], rbar));
    }
    phi_s[node] = v;   // b, staged for the GEMV
    if (rank == 0) b[node] = v;
  }
  __syncthreads();
  CHAIN_STAMP();
  // phi = G b (k_gemv: warp per row, lane-strided FMA chain, xor butterfly), my rows,
  // each pushed into every CTA's phx (phi_s holds b until every GEMV is done)
  for (int row = row0; row < q1; row += nw) {
    double t = 0.0;
    const double* g = green + (size_t)row * nn;
    int k = lane;
    if (row == row0) {
#pragma unroll
      for (int i = 0; i < kGreenRegs; ++i, k += 32)
        if (k < nn) t = fma(gr[i], phi_s[k], t);
    }
#pragma unroll 4
    for (; k < nn; k += 32) t = fma(__ldg(g + k), phi_s[k], t);
#pragma unroll
    for (int of = 16; of > 0; of >>= 1) t += __shfl_xor_sync(0xffffffffu, t, of);
    if (lane == 0) phi[row] = t;
    if (lane < kChainCtas) *cluster.map_shared_rank(&phx[row], lane) = t;
  }
  fuzz_delay();
  cluster.sync();   // phi complete everywhere; no shared memory access across CTAs after this
  CHAIN_STAMP();
  // E (k_efield) at every DOF in every CTA (each CTA stores its own DOFs)
  const double sc = -(2.0 / h);
  for (int k = tid; k < nd; k += blockDim.x) {
    const int cell = k / o, i = k - cell * o;
    double t = 0.0;
    for (int j = 0; j < o; ++j) {
      const int node = (cell * p + j) % nn;
      t = fma(__dmul_rn(sc, phx[node]), diff_s[i * o + j], t);
    }
    e_s[k] = t;
    if (k >= c0 && k < c1) e[k] = t;
  }
  __syncthreads();
  CHAIN_STAMP();
  if (rank == 0 && wp == nw - 1) {
    // field diagnostics (k_field_diag): max |E| and 0.5 w.E^2, the 1024-slot trees
    const double emax = warp_tree1024(lane, [&](int t) {
      return t < nd ? fmax(0.0, fabs(e_s[t])) : 0.0;
    }, [](double x, double y) { return fmax(x, y); });
    const double ee = warp_tree1024(lane, [&](int t) {
      const double v = t < nd ? e_s[t] : 0.0;
      return t < nd ? fma(xw_s[t], v * v, 0.0) : 0.0;
    }, [](double x, double y) { return x + y; });
    if (lane == 0) {
      diag2[0] = emax;
      diag2[1] = 0.5 * ee;
    }
  }
  // level matrices for speeds = E (k_level_mats): my columns, one thread per
  // (level, column, A | B)
  const int my = c1 - c0;
  for (int idx = tid; idx < 2 * my * n_levels; idx += blockDim.x) {
    const int ab = idx & 1, rest = idx >> 1;
    const int lev = rest / my, c = c0 + (rest - lev * my);
    const double width = base_width / (double)(1LL << lev);
    long long ns;
    double a;
    split_shift(e_s[c], dt, width, &ns, &a);
    if (ab == 0) {
      lm_ns[(long long)lev * nd + c] = ns;
      lm_frac[(long long)lev * nd + c] = a;
    }
    double M[O * O];
    if (a == 0.0) {
#pragma unroll
      for (int k = 0; k < O * O; ++k) M[k] = (ab == 0 && k % (O + 1) == 0) ? 1.0 : 0.0;
    } else {
      double raw[O * O];
      const double split = 2.0 * a - 1.0;
      if (ab == 0)
        interval_block<O>(vb, split, 1.0, -2.0 * a, raw);
      else
        interval_block<O>(vb, -1.0, split, 2.0 * (1.0 - a), raw);
      apply_minv<O>(vb, raw, M);
    }
#pragma unroll
    for (int k = 0; k < O * O; ++k)
      lm_mats[((long long)(lev * 2 + ab) * O * O + k) * nd + c] = M[k];
  }
#ifdef SLDG_CHAIN_PROF
  CHAIN_STAMP();
  if (tid == 0 && rank < 2) {
    char buf[160];
    int n = 0;
    for (int k = 1; k < nst; ++k) n += snprintf_dev(buf + n, (int)tst[k] - (int)tst[k - 1]);
    printf("chain rank %d:%s\n", rank, buf);
  }
#endif
}

}  // namespace sldg

using namespace sldg;


namespace {

int check_geom(const sldg_vplan* vp, const sldg_xplan* xp, int64_t n_cols, int64_t ld,
               FusedGeom* g) {
  *g = fused_geom(vp, xp, n_cols, ld);
  if (!g->ok) {
    set_error(g->why);
    return SLDG_ERR_UNSUPPORTED;
  }
  return SLDG_OK;
}

int launch_step(const sldg_vplan* vp, const sldg_xplan* xp, const FusedGeom& g, const double* fin,
                double* fout, int64_t n_cols, const double* speeds, int32_t bc,
                const FusedScratch& s, const FusedArgs& fa, int mode, cudaStream_t st,
                long long* grid, long long t_begin = 0, long long t_count = -1) {
  if ((((unsigned long long)fin) & 15) != 0 || n_cols % 2 != 0) {
    set_error("fused step: 16-byte aligned rows required");
    return SLDG_ERR_UNSUPPORTED;
  }
  if (t_count < 0) {
    t_begin = 0;
    t_count = g.n_tiles;
  }
  if (t_begin < 0 || t_begin + t_count > g.n_tiles) {
    set_error("fused step: tile range outside the plan");
    return SLDG_ERR_ARG;
  }
  FusedKernel k = fused_kernel(vp, xp, g, mode);
  if (!k) {
    set_error("fused step: no kernel for this degree / line group");
    return SLDG_ERR_UNSUPPORTED;
  }
  int rc = fused_grid(vp, xp, g, grid);
  if (rc) return rc;
  SLDG_CUDA_TRY(launch_pdl(k, dim3((unsigned)*grid), dim3(g.threads), g.smem, st, vp->dev,
                           xp->dev, fin, fout, (int)n_cols, (int)xp->n_cells, speeds, (int)bc,
                           (const long long*)s.lm_ns, (const double*)s.lm_mats, g.rw,
                           (int)xp->n_speeds, g.nmax, t_begin, t_count, fa));
  SLDG_LAUNCH_CHECK("k_step_fused");
  return SLDG_OK;
}

bool bad_step_args(const sldg_vplan* vp, const sldg_xplan* xp, const double* fin,
                   const double* fout, const double* speeds, int32_t bc, const double* w,
                   const double* v0, const double* v2, const double* xw, const void* scratch) {
  return !vp || !xp || !fin || !fout || fin == fout || !speeds || !w || !v0 || !v2 || !xw ||
         !scratch || (bc != SLDG_BC_PERIODIC && bc != SLDG_BC_ABSORBING);
}

}  // namespace

extern "C" {

int sldg_step_fused_query(const sldg_vplan* vp, const sldg_xplan* xp, int64_t n_cols, int64_t ld,
                          size_t* scratch_bytes) {
  if (!vp || !xp || !scratch_bytes) {
    set_error("null argument");
    return SLDG_ERR_ARG;
  }
  FusedGeom g;
  int rc = check_geom(vp, xp, n_cols, ld, &g);
  if (rc) return rc;
  *scratch_bytes = fused_scratch(vp, g, n_cols, nullptr).bytes;
  return SLDG_OK;
}

int sldg_step_fused_advice(const sldg_vplan* vp, const sldg_xplan* xp, int64_t n_cols, int64_t ld,
                           int32_t* profitable) {
  if (!vp || !xp || !profitable) {
    set_error("null argument");
    return SLDG_ERR_ARG;
  }
  FusedGeom g;
  int rc = check_geom(vp, xp, n_cols, ld, &g);
  if (rc) return rc;
  FusedKernel k = fused_kernel(vp, xp, g, 0);
  if (!k) {
    set_error("fused step: no kernel for this degree / line group");
    return SLDG_ERR_UNSUPPORTED;
  }
  // measured: the one-pass step beats the separate passes when its
  // kernel keeps two CTAs per SM without register spills; otherwise (wide rows,
  // degree-3 velocity or x bases) the separate passes are as fast or faster
  cudaFuncAttributes attr;
  SLDG_CUDA_TRY(cudaFuncGetAttributes(&attr, k));
  int per_sm = 0;
  SLDG_CUDA_TRY(resident_ctas((const void*)k, g.threads, (int)g.smem, &per_sm));
  *profitable = (attr.localSizeBytes == 0 && per_sm >= 2) ? 1 : 0;
  return SLDG_OK;
}

int sldg_step_fused(const sldg_vplan* vp, const sldg_xplan* xp, const double* fin, double* fout,
                    int64_t ld, int64_t n_cols, const double* speeds, double dt, int32_t bc,
                    const double* w, const double* v0, const double* v2, const double* xw,
                    double* mom_out3, double* rho_out, void* scratch, void* stream) {
  if (bad_step_args(vp, xp, fin, fout, speeds, bc, w, v0, v2, xw, scratch) || !mom_out3 ||
      !rho_out || !(dt > 0.0)) {
    set_error("bad sldg_step_fused arguments");
    return SLDG_ERR_ARG;
  }
  FusedGeom g;
  int rc = check_geom(vp, xp, n_cols, ld, &g);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const FusedScratch s = fused_scratch(vp, g, n_cols, scratch);
  rc = sldg_level_matrices(vp, speeds, n_cols, dt, (int64_t*)s.lm_ns, s.lm_frac, s.lm_mats, stream);
  if (rc) return rc;
  long long grid = 0;
  rc = launch_step(vp, xp, g, fin, fout, n_cols, speeds, bc, s,
                   FusedArgs{w, v0, v2, xw, s.mom_part, s.rho_part}, 0, st, &grid);
  if (rc) return rc;
  k_fold3<<<1, 96, 0, st>>>(s.mom_part, grid, mom_out3);
  SLDG_LAUNCH_CHECK("k_fold3");
  k_fold_cols<<<(unsigned)((n_cols * 32 + 255) / 256), 256, 0, st>>>(s.rho_part, grid, n_cols,
                                                                      rho_out);
  SLDG_LAUNCH_CHECK("k_fold_cols");
  return SLDG_OK;
}

int sldg_step_fused_deferred(const sldg_vplan* vp, const sldg_xplan* xp, const double* fin,
                             double* fout, int64_t ld, int64_t n_cols, const double* speeds,
                             int32_t bc, const double* w, const double* v0, const double* v2,
                             const double* xw, int32_t mode, double* mom_out3,
                             int64_t tile_begin, int64_t tile_count, void* scratch,
                             void* stream) {
  if (bad_step_args(vp, xp, fin, fout, speeds, bc, w, v0, v2, xw, scratch) ||
      (mode < 0 || mode > 2)) {
    set_error("bad sldg_step_fused_deferred arguments");
    return SLDG_ERR_ARG;
  }
  FusedGeom g;
  int rc = check_geom(vp, xp, n_cols, ld, &g);
  if (rc) return rc;
  const FusedScratch s = fused_scratch(vp, g, n_cols, scratch);
  cudaStream_t st = (cudaStream_t)stream;
  long long grid = 0;
  rc = launch_step(vp, xp, g, fin, fout, n_cols, speeds, bc, s,
                   FusedArgs{w, v0, v2, xw, s.mom_part, s.rho_part}, mode, st, &grid,
                   tile_begin, tile_count);
  if (rc || !mom_out3) return rc;
  k_fold3<<<1, 96, 0, st>>>(s.mom_part, grid, mom_out3);
  SLDG_LAUNCH_CHECK("k_fold3");
  return SLDG_OK;
}

int sldg_step_fused_tiles(const sldg_vplan* vp, const sldg_xplan* xp, int64_t n_cols, int64_t ld,
                          int64_t* info) {
  if (!vp || !xp || !info) {
    set_error("null argument");
    return SLDG_ERR_ARG;
  }
  FusedGeom g;
  int rc = check_geom(vp, xp, n_cols, ld, &g);
  if (rc) return rc;
  info[0] = g.n_tiles;
  info[1] = (int64_t)g.lg * vp->o;   // rows per tile
  info[2] = g.n_lg;                  // line groups per cell
  info[3] = g.nmax;                  // cells per item (pencil length)
  return SLDG_OK;
}

int sldg_step_fused_fold(const sldg_vplan* vp, const sldg_xplan* xp, int64_t n_cols, int64_t ld,
                         double* rho_out, double* mom_out3, void* scratch, void* stream) {
  if (!vp || !xp || !scratch || (!rho_out && !mom_out3)) {
    set_error("bad sldg_step_fused_fold arguments");
    return SLDG_ERR_ARG;
  }
  FusedGeom g;
  int rc = check_geom(vp, xp, n_cols, ld, &g);
  if (rc) return rc;
  FusedKernel k = fused_kernel(vp, xp, g, 0);
  if (!k) {
    set_error("fused step: no kernel for this degree / line group");
    return SLDG_ERR_UNSUPPORTED;
  }
  long long grid = 0;
  rc = fused_grid(vp, xp, g, &grid);
  if (rc) return rc;
  const FusedScratch s = fused_scratch(vp, g, n_cols, scratch);
  cudaStream_t st = (cudaStream_t)stream;
  if (mom_out3) {
    k_fold3<<<1, 96, 0, st>>>(s.mom_part, grid, mom_out3);
    SLDG_LAUNCH_CHECK("k_fold3");
  }
  if (rho_out) {
    k_fold_cols<<<(unsigned)((n_cols * 32 + 255) / 256), 256, 0, st>>>(s.rho_part, grid, n_cols,
                                                                        rho_out);
    SLDG_LAUNCH_CHECK("k_fold_cols");
  }
  return SLDG_OK;
}

int sldg_field_chain(const sldg_vplan* vp, const sldg_xplan* xp, const sldg_poisson* P,
                     int64_t n_cols, int64_t ld, double dt, const double* rho_in, double* rho,
                     double* phi, double* e, double* diag2, double* mom_prev3, void* scratch,
                     void* stream) {
  if (!vp || !xp || !P || !phi || !e || !diag2 || !scratch || !(dt > 0.0) ||
      (!rho_in && !rho) || n_cols != P->n_dofs || n_cols > kChainMaxDofs ||
      P->n_nodes > kChainMaxDofs) {
    set_error("bad sldg_field_chain arguments");
    return SLDG_ERR_ARG;
  }
  FusedGeom g;
  int rc = check_geom(vp, xp, n_cols, ld, &g);
  if (rc) return rc;
  const FusedScratch s = fused_scratch(vp, g, n_cols, scratch);
  long long grid = 0;
  if (!rho_in) {   // partials of the previous sldg_step_fused_deferred
    FusedKernel k = fused_kernel(vp, xp, g, 0);
    if (!k) {
      set_error("fused step: no kernel for this degree / line group");
      return SLDG_ERR_UNSUPPORTED;
    }
    rc = fused_grid(vp, xp, g, &grid);
    if (rc) return rc;
  }
  cudaStream_t st = (cudaStream_t)stream;
  switch (vp->o) {
#define CASE(O)                                                                                \
  case O:                                                                                      \
    SLDG_CUDA_TRY(launch_pdl(k_field_chain<O>, dim3(kChainCtas), dim3(kChainThreads), 0, st,  \
                             rho_in,                                                           \
                             (const double*)s.rho_part, (const double*)s.mom_part, grid,       \
                             mom_prev3, rho, (const double*)P->xw, (const double*)P->green,    \
                             (const double*)P->diff, P->n_cells, P->p, P->length, P->h,        \
                             P->work, phi, e, diag2, vp->basis, dt, vp->dev.base_width,        \
                             vp->dev.n_levels, s.lm_ns, s.lm_frac, s.lm_mats));                \
    break;
    CASE(2) CASE(3) CASE(4)
#undef CASE
    default:
      set_error("field chain: velocity degree 1..3");
      return SLDG_ERR_UNSUPPORTED;
  }
  SLDG_LAUNCH_CHECK("k_field_chain");
  return SLDG_OK;
}

}  // extern "C"
