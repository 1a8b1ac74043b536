// step_fused.cu -- one HBM pass per Strang step: v-sweep + trailing half x-step
// (+ moments) + next leading half x-step (+ rho), fused per line-group tile.
//
// In Simulation.advance() the state between kernels is f' = X(f) (after the
// leading half x-step).  The reference step (driver.py:231-240) continues with
// field solve -> advect_velocity (vsweep.py:413-441) -> advect_x
// (xfield.py:91-104) -> diagnostics (driver.py:220-229, moments 139-146), and
// the next step starts with advect_x and compute_rho (xfield.py:107-109).
// This kernel performs, for one pencil and a group of LG lines of its cells:
//   V  : whole-pencil fast path (sweep_pencil, vsweep.py:197-200) from a TMA
//        bulk-copy ring of cell tiles (as k_sweep_stream), into shared memory;
//   X1 : trailing half x-step on the tile's rows (they are complete rows:
//        the tile spans all x columns), moments of the result accumulated;
//   X2 : leading half x-step of the next step, rho of the result accumulated,
//        result stored to HBM.
// Every coefficient is read once and written once per step: 16 B/DOF instead
// of 32 B/DOF for the separate sweep and X.X passes.  Arithmetic per output is
// the same as in k_sweep_stream / k_xadv (same operands, same order).
//
// Thread mappings: V phase thread = x column (its A, B for the pencil's level
// in registers); X phases thread = (velocity node i_v, x cell): all rows of a
// tile with the same i_v share one v_x, hence one x-shift and one A, B pair.
// Shared-memory rows carry ghost cells on both sides so periodic x reads never
// wrap (writers duplicate the edge cells into the ghosts).
//
// Eligible: dim 3, direction 0, every pencil whole-pencil-fast, no weighted
// (1/n_c) entries, tile rows span the whole row (ld == n_cols).  Otherwise the
// host falls back to the separate passes.
#include <algorithm>
#include <string>
#include <type_traits>

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
  for (long long k = lane; k < n_parts; k += 32) s += part[k * n_cols + c];
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

struct FusedArgs {
  const double* w;
  const double* v0;
  const double* v2;
  const double* xw;
  double* mom_part;   // [grid][3]
  double* rho_part;   // [grid][n_cols]
};

template <bool B>
using BoolC = std::integral_constant<bool, B>;

template <int OV, int OX, int LG>
__global__ void __launch_bounds__(384, 1)
k_step_fused(VPlanDev P, XPlanDev X, const double* __restrict__ fin, double* __restrict__ fout,
             int n_cols, int n_xc, const double* __restrict__ speeds, int bc,
             const long long* __restrict__ lm_ns, const double* __restrict__ lm_mats, int rw,
             int n_speeds, FusedArgs fa) {
  constexpr int XM = 2 * OX * OX;
  constexpr int R = LG * OV;                    // rows per tile
  constexpr int n_lg = OV * OV / LG;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) unsigned long long full[kFRing];
  __shared__ int s_nsmin, s_nsmax;

  const int tile = R * n_cols;                  // doubles per ring slot
  double* ring = sm;
  double* stA = ring + kFRing * tile;
  double* stB = stA + R * rw;
  double* xtab = stB + R * rw;                  // n_speeds x (A|B) for the x shift
  int* xns = reinterpret_cast<int*>(xtab + (long long)n_speeds * XM);
  double* meta = xtab + (long long)n_speeds * XM + (n_speeds + 1) / 2;   // per-pencil tables

  const long long wp = blockIdx.x / n_lg;
  const int t0 = (int)(blockIdx.x - wp * n_lg) * LG;   // first line of the group
  const long long q = P.walk_pencils[wp];
  const long long off = P.p_off[q];
  const int n = P.p_n[q];
  const int lev = P.e_level[off];
  const int tid = threadIdx.x;

  // x-shift tables; a zero shift is stored as (A, B) = (I, 0) with no cell shift so
  // the X phases run without a per-thread branch (1*u0 + 0*u1 + ... == u0)
  for (int k = tid; k < n_speeds * XM; k += blockDim.x) {
    const int g = k / XM, e = k - g * XM;
    xtab[k] = X.ident[g] ? ((e < OX * OX && e % (OX + 1) == 0) ? 1.0 : 0.0) : __ldg(X.mats + k);
  }
  for (int k = tid; k < n_speeds; k += blockDim.x) xns[k] = X.ident[k] ? 0 : (int)X.ns[k];
  if (tid == 0) {
    s_nsmin = 1 << 30;
    s_nsmax = -(1 << 30);
    for (int k = 0; k < kFRing; ++k) mbar_init(&full[k], 1);
    mbar_fence_init();
  }
  __syncthreads();

  // ---- V-phase state: thread = column
  const bool colv = tid < n_cols;
  const int c = tid;
  const double speed = colv ? __ldg(speeds + c) : 0.0;
  const long long nsv = colv ? lm_ns[(long long)lev * n_cols + c] : 0;
  if (colv && speed != 0.0) {
    const int nsi = (int)max(min(nsv, (long long)(1 << 29)), -(long long)(1 << 29));
    atomicMin(&s_nsmin, nsi);
    atomicMax(&s_nsmax, nsi);
  }
  double Av[OV * OV], Bv[OV * OV];
  if (colv) load_pair<OV>(lm_mats, lev, n_cols, c, Av, Bv);
  __syncthreads();
  const bool streamable = (s_nsmin >= -1 && s_nsmax <= 0) || (s_nsmin > s_nsmax);
  const bool per = (bc == SLDG_BC_PERIODIC);

  // ---- X-phase state: thread = (iv, x cell)
  const bool xv = tid < OV * n_xc;
  const int iv = xv ? tid / n_xc : 0;
  const int cx = xv ? tid - iv * n_xc : 0;
  double m0a[OX], m1a[OX], m2a[OX], rha[OX];
#pragma unroll
  for (int k = 0; k < OX; ++k) m0a[k] = m1a[k] = m2a[k] = rha[k] = 0.0;

  // per-pencil metadata, loaded once into shared memory (no global loads in the
  // step loop): tile row base per cell, x-speed index per (cell, v_x node) and
  // (w, w*v0, w*v2) per tile row of every cell
  long long* crow = reinterpret_cast<long long*>(meta);                   // [n]
  int* cg = reinterpret_cast<int*>(crow + n);                               // [n][OV]
  double* cmeta = reinterpret_cast<double*>(cg + ((n * OV + 1) & ~1));      // [n][3][R]
  for (int k = tid; k < n; k += blockDim.x) crow[k] = P.e_row0[off + k] + (long long)t0 * OV;
  __syncthreads();
  for (int k = tid; k < n * OV; k += blockDim.x)
    cg[k] = __ldg(X.row_speed + crow[k / OV] + k % OV);
  for (int k = tid; k < n * R; k += blockDim.x) {
    const int s2 = k / R, r = k - s2 * R;
    const long long row = crow[s2] + r;
    const double wr = __ldg(fa.w + row);
    double* m = cmeta + (long long)s2 * 3 * R;
    m[r] = wr;
    m[R + r] = wr * __ldg(fa.v0 + row);
    m[2 * R + r] = wr * __ldg(fa.v2 + row);
  }
  __syncthreads();

  // ---- ring of cell tiles (as k_sweep_stream)
  const int v0c = per ? -1 : 0;
  const int n_load = per ? n + 2 : n;
  auto issue = [&](int k) {
    const int v = v0c + k;
    const int cell = v < 0 ? n - 1 : (v >= n ? 0 : v);
    unsigned long long* bar = &full[k % kFRing];
    mbar_expect_tx(bar, (unsigned)(tile * 8));
    bulk_g2s(ring + (k % kFRing) * tile, fin + crow[cell] * n_cols, (unsigned)(tile * 8), bar);
  };
  if (streamable && tid == 0)
    for (int k = 0; k < min(3, n_load); ++k) issue(k);

  // V phase of one column: rows t*OV+i of the source cells sa / sb -> stA column c.
  // CHECKED: the source cells may lie outside the pencil (absorbing ends).
  auto vcol = [&](const double* sa, const double* sb, bool va, bool vb, auto checked) {
    constexpr bool CK = decltype(checked)::value;
    double* out = stA + c;
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
  auto vcopy = [&](const double* me) {
#pragma unroll
    for (int r = 0; r < R; ++r) stA[r * rw + c] = me[r * n_cols];
  };

  for (int s = 0; s < n; ++s) {
    const double* mcur = cmeta + (long long)s * 3 * R;
    const long long r0 = crow[s];
    const int g_cur = xv ? cg[s * OV + iv] : 0;
    // ===================== V: pencil sweep of cell s -> stA (rows of R, stride rw)
    if (streamable) {
      const int kn = s + 2 - v0c;
      if (tid == 0 && kn < n_load && kn >= 3) issue(kn);
      const int klo = max(s - 1 - v0c, 0), khi = min(s + 1 - v0c, n_load - 1);
      for (int k = klo; k <= khi; ++k)
        mbar_wait(&full[k & (kFRing - 1)], (unsigned)(((unsigned)k / kFRing) & 1));
      if (colv) {
        if (speed == 0.0) {
          vcopy(ring + ((s - v0c) & (kFRing - 1)) * tile + c);
        } else {
          // streamable: source cells s - nsv and s - nsv - 1 with nsv in {-1, 0}
          const int va_cell = s - (int)nsv, vb_cell = va_cell - 1;
          if (per || (s > 0 && s < n - 1)) {
            vcol(ring + ((va_cell - v0c) & (kFRing - 1)) * tile + c,
                 ring + ((vb_cell - v0c) & (kFRing - 1)) * tile + c, true, true, BoolC<false>{});
          } else {
            const bool va = va_cell >= 0 && va_cell < n, vb = vb_cell >= 0 && vb_cell < n;
            vcol(ring + (((va ? va_cell : s) - v0c) & (kFRing - 1)) * tile + c,
                 ring + (((vb ? vb_cell : s) - v0c) & (kFRing - 1)) * tile + c, va, vb,
                 BoolC<true>{});
          }
        }
      }
    } else if (colv) {
      if (speed == 0.0) {
        vcopy(fin + r0 * n_cols + c);
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
        vcol(fin + crow[va ? (int)qa : s] * n_cols + c, fin + crow[vb ? (int)qb : s] * n_cols + c,
             va, vb, BoolC<true>{});
      }
    }
    // x shift of this thread's rows for cell s: matrices to registers, wrapped sources
    double xa[OX * OX], xb[OX * OX];
    int ia = 0, ib = 0;
    if (xv) {
      const double* AB = xtab + (long long)g_cur * XM;
#pragma unroll
      for (int k = 0; k < OX * OX; ++k) {
        xa[k] = AB[k];
        xb[k] = AB[OX * OX + k];
      }
      ia = cx - xns[g_cur];
      ia = ia < 0 ? ia + n_xc : (ia >= n_xc ? ia - n_xc : ia);
      ib = ia == 0 ? n_xc - 1 : ia - 1;
      ia *= OX;
      ib *= OX;
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
    __syncthreads();
    // ===================== X1 (trailing half step): stA -> stB, moments
    if (xv) {
#pragma unroll
      for (int t = 0; t < LG; ++t) {
        const int r = t * OV + iv;
        double y[OX];
        xapply(stA + r * rw, y);
        const double wr = mcur[r], wv0 = mcur[R + r], wv2 = mcur[2 * R + r];
        double* o = stB + r * rw + cx * OX;
#pragma unroll
        for (int k = 0; k < OX; ++k) {
          o[k] = y[k];
          m0a[k] = fma(wr, y[k], m0a[k]);
          m1a[k] = fma(wv0, y[k], m1a[k]);
          m2a[k] = fma(wv2, y[k], m2a[k]);
        }
      }
    }
    __syncthreads();
    // ===================== X2 (next step's leading half): stB -> HBM, rho
    // No barrier after X2: the next V writes stA (last read in X1, before the
    // barrier above) and the ring slot it refills was last read in this V.
    if (xv) {
      double* dst = fout + (r0 + iv) * n_cols + cx * OX;
#pragma unroll
      for (int t = 0; t < LG; ++t) {
        const int r = t * OV + iv;
        double y[OX];
        xapply(stB + r * rw, y);
        const double wr = mcur[r];
#pragma unroll
        for (int k = 0; k < OX; ++k) {
          dst[k] = y[k];
          rha[k] = fma(wr, y[k], rha[k]);
        }
        dst += (long long)OV * n_cols;
      }
    }
  }
  __syncthreads();   // stB (read by X2) is reused by the reduction below


  // ---- CTA partials: rho per column (over i_v in order), moments contracted with xw
  double* red = stA;   // reuse: OV x n_cols, then 3 x blockDim
  if (xv) {
#pragma unroll
    for (int k = 0; k < OX; ++k) red[iv * n_cols + cx * OX + k] = rha[k];
  }
  __syncthreads();
  if (colv) {
    double s = 0.0;
    for (int k = 0; k < OV; ++k) s += red[k * n_cols + c];
    fa.rho_part[(long long)blockIdx.x * n_cols + c] = s;
  }
  __syncthreads();
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  if (xv) {
#pragma unroll
    for (int k = 0; k < OX; ++k) {
      const double xwk = __ldg(fa.xw + cx * OX + k);
      s0 = fma(xwk, m0a[k], s0);
      s1 = fma(xwk, m1a[k], s1);
      s2 = fma(xwk, m2a[k], s2);
    }
  }
  red[tid] = s0;
  red[blockDim.x + tid] = s1;
  red[2 * blockDim.x + tid] = s2;
  __syncthreads();
  if (tid < 3) {
    double s = 0.0;
    for (int k = 0; k < (int)blockDim.x; ++k) s += red[tid * blockDim.x + k];
    fa.mom_part[blockIdx.x * 3 + tid] = s;
  }
}

struct FusedGeom {
  bool ok;
  int lg, n_lg, gl, rw, threads;
  size_t smem;
  long long grid;
  std::string why;
};

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
  if (ld != n_cols || n_cols != xp->n_cells * OX) return no("fused step: whole rows only");
  if (OV < 2 || OV > 4 || OX < 2 || OX > 4) return no("fused step: degrees 1..3");
  const long long threads = std::max<long long>(n_cols, OV * xp->n_cells);
  if (threads > 384) return no("fused step: rows wider than 384 columns");
  const int hl = (int)xp->halo_l, hr = (int)xp->halo_r;
  if (hl > xp->n_cells || hr > xp->n_cells) return no("fused step: shift wider than the row");
  g.rw = (int)n_cols + (n_cols % 2 == 0 ? 1 : 0);   // odd row stride: conflict-free columns
  const size_t fixed = sizeof(double) * (size_t)xp->n_speeds * 2 * OX * OX +
                       sizeof(double) * ((xp->n_speeds + 1) / 2) + 64;
  const size_t nmax = (size_t)vp->max_pencil_cells;
  const size_t budget = 227 * 1024 - 1024;
  g.lg = 0;
  for (int lg = 4; lg >= 1; --lg) {   // instantiated line groups: OV, 2 (even OV), 1
    if ((OV * OV) % lg || (lg != OV && lg != 2 && lg != 1)) continue;
    const size_t R = (size_t)lg * OV;
    const size_t tables = 8 * nmax + 4 * ((nmax * OV + 1) & ~(size_t)1) + 8 * nmax * 3 * R;
    const size_t smem = sizeof(double) * (kFRing * R * n_cols + 2 * R * g.rw) + fixed + tables;
    const size_t red = sizeof(double) * std::max<size_t>(OV * n_cols, 3 * threads);
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
  g.grid = vp->n_walk * g.n_lg;
  g.ok = true;
  return g;
}

template <int OV, int OX, int LG>
static int launch_fused_lg(const sldg_vplan* vp, const sldg_xplan* xp, const FusedGeom& g,
                           const double* fin, double* fout, long long n_cols,
                           const double* speeds, int bc, const long long* lm_ns,
                           const double* lm_mats, const FusedArgs& fa, cudaStream_t st) {
  auto k = k_step_fused<OV, OX, LG>;
  SLDG_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
  k<<<(unsigned)g.grid, g.threads, g.smem, st>>>(vp->dev, xp->dev, fin, fout, (int)n_cols,
                                                 (int)xp->n_cells, speeds, bc, lm_ns, lm_mats,
                                                 g.rw, (int)xp->n_speeds, fa);
  SLDG_LAUNCH_CHECK("k_step_fused");
  return SLDG_OK;
}

template <int OV, int OX>
static int launch_fused(const sldg_vplan* vp, const sldg_xplan* xp, const FusedGeom& g,
                        const double* fin, double* fout, long long n_cols, const double* speeds,
                        int bc, const long long* lm_ns, const double* lm_mats,
                        const FusedArgs& fa, cudaStream_t st) {
  if (g.lg == OV)
    return launch_fused_lg<OV, OX, OV>(vp, xp, g, fin, fout, n_cols, speeds, bc, lm_ns, lm_mats, fa, st);
  if constexpr (OV % 2 == 0 && OV != 2) {
    if (g.lg == 2)
      return launch_fused_lg<OV, OX, 2>(vp, xp, g, fin, fout, n_cols, speeds, bc, lm_ns, lm_mats, fa, st);
  }
  if (g.lg == 1)
    return launch_fused_lg<OV, OX, 1>(vp, xp, g, fin, fout, n_cols, speeds, bc, lm_ns, lm_mats, fa, st);
  set_error("fused step: no kernel for this line group");
  return SLDG_ERR_UNSUPPORTED;
}

static size_t al256(size_t x) { return (x + 255) / 256 * 256; }

}  // namespace sldg

using namespace sldg;

extern "C" {

int sldg_step_fused_query(const sldg_vplan* vp, const sldg_xplan* xp, int64_t n_cols, int64_t ld,
                          size_t* scratch_bytes) {
  if (!vp || !xp || !scratch_bytes) {
    set_error("null argument");
    return SLDG_ERR_ARG;
  }
  FusedGeom g = fused_geom(vp, xp, n_cols, ld);
  if (!g.ok) {
    set_error(g.why);
    return SLDG_ERR_UNSUPPORTED;
  }
  const size_t lm = al256(sizeof(long long) * vp->dev.n_levels * n_cols) +
                    al256(sizeof(double) * vp->dev.n_levels * n_cols) +
                    al256(sizeof(double) * vp->dev.n_levels * 2 * vp->o * vp->o * n_cols);
  *scratch_bytes = lm + al256(sizeof(double) * g.grid * 3) + al256(sizeof(double) * g.grid * n_cols);
  return SLDG_OK;
}

int sldg_step_fused(const sldg_vplan* vp, const sldg_xplan* xp, const double* fin, double* fout,
                    int64_t ld, int64_t n_cols, const double* speeds, double dt, int32_t bc,
                    const double* w, const double* v0, const double* v2, const double* xw,
                    double* mom_out3, double* rho_out, void* scratch, void* stream) {
  if (!vp || !xp || !fin || !fout || fin == fout || !speeds || !w || !v0 || !v2 || !xw ||
      !mom_out3 || !rho_out || !scratch || !(dt > 0.0) ||
      (bc != SLDG_BC_PERIODIC && bc != SLDG_BC_ABSORBING)) {
    set_error("bad sldg_step_fused arguments");
    return SLDG_ERR_ARG;
  }
  FusedGeom g = fused_geom(vp, xp, n_cols, ld);
  if (!g.ok) {
    set_error(g.why);
    return SLDG_ERR_UNSUPPORTED;
  }
  if ((((unsigned long long)fin) & 15) != 0 || n_cols % 2 != 0) {
    set_error("fused step: 16-byte aligned rows required");
    return SLDG_ERR_UNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  unsigned char* sb = (unsigned char*)scratch;
  long long* lm_ns = (long long*)sb;
  size_t o1 = al256(sizeof(long long) * vp->dev.n_levels * n_cols);
  double* lm_frac = (double*)(sb + o1);
  size_t o2 = o1 + al256(sizeof(double) * vp->dev.n_levels * n_cols);
  double* lm_mats = (double*)(sb + o2);
  size_t o3 = o2 + al256(sizeof(double) * vp->dev.n_levels * 2 * vp->o * vp->o * n_cols);
  double* mom_part = (double*)(sb + o3);
  size_t o4 = o3 + al256(sizeof(double) * g.grid * 3);
  double* rho_part = (double*)(sb + o4);
  int rc = sldg_level_matrices(vp, speeds, n_cols, dt, (int64_t*)lm_ns, lm_frac, lm_mats, stream);
  if (rc) return rc;
  FusedArgs fa{w, v0, v2, xw, mom_part, rho_part};
  rc = SLDG_ERR_UNSUPPORTED;
  switch (vp->o * 10 + xp->o) {
#define CASE(A, B)                                                                          \
  case A * 10 + B:                                                                          \
    rc = launch_fused<A, B>(vp, xp, g, fin, fout, n_cols, speeds, bc, lm_ns, lm_mats, fa, st); \
    break;
    CASE(2, 2) CASE(2, 3) CASE(2, 4) CASE(3, 2) CASE(3, 3) CASE(3, 4) CASE(4, 2) CASE(4, 3)
    CASE(4, 4)
#undef CASE
  }
  if (rc) return rc;
  k_fold3<<<1, 96, 0, st>>>(mom_part, g.grid, mom_out3);
  SLDG_LAUNCH_CHECK("k_fold3");
  k_fold_cols<<<(unsigned)((n_cols * 32 + 255) / 256), 256, 0, st>>>(rho_part, g.grid, n_cols,
                                                                      rho_out);
  SLDG_LAUNCH_CHECK("k_fold_cols");
  return SLDG_OK;
}

}  // extern "C"
