// xfield.cu -- x-advection shift, charge density, velocity moments, 1D Poisson.
//
// Replaces xfield.precompute_x_matrices / advect_x (xfield.py:63-104),
// compute_rho (107-109), PoissonSolver.rhs/solve/electric_field (148-179),
// field_energy (192-195) and driver.moments (driver.py:139-146).
//
// All reductions are two-stage with a fixed partition that depends only on
// the problem shape, so results are bitwise reproducible run to run.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "sldg_common.cuh"
#include "plans.cuh"

namespace sldg {

template <int O>
__global__ void k_xmats(DevBasis b, const double* __restrict__ speeds, long long n, double dt,
                        double h, long long* __restrict__ ns, unsigned char* __restrict__ ident,
                        double* __restrict__ mats) {
  long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (u >= n) return;
  long long n_s;
  double a;
  split_shift(speeds[u], dt, h, &n_s, &a);
  double A[O * O], B[O * O];
  overlap_pair<O>(b, a, A, B);
  ns[u] = n_s;
  ident[u] = (n_s == 0 && a == 0.0) ? 1 : 0;
#pragma unroll
  for (int k = 0; k < O * O; ++k) {
    mats[u * 2 * O * O + k] = A[k];
    mats[u * 2 * O * O + O * O + k] = B[k];
  }
}

// One CTA handles ROWS rows.  The rows' input segments are staged in shared
// memory with coalesced loads, then each thread produces output DOFs
//   out[c*O+i] = sum_j A[i][j] u[(c-n)*O+j] + B[i][j] u[(c-n-1)*O+j]
// with periodic wrap (full rows) or halo offsets (slabs).
template <int O>
__global__ void __launch_bounds__(256)
k_advect_x(XPlanDev X, const double* __restrict__ fin, long long ld_in, double* __restrict__ fout,
           long long ld_out, long long n_rows, int in_cells, int out_cells, int halo_l,
           int periodic, int rows_per_cta) {
  extern __shared__ __align__(16) double srow[];
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  const int nr = (int)min((long long)rows_per_cta, n_rows - r0);
  const int in_len = in_cells * O, out_len = out_cells * O;
  // stage
  for (int k = threadIdx.x; k < nr * in_len; k += blockDim.x) {
    int r = k / in_len, j = k - r * in_len;
    srow[k] = fin[(r0 + r) * ld_in + j];
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nr * out_len; k += blockDim.x) {
    int r = k / out_len, j = k - r * out_len;
    int cell = j / O, i = j - cell * O;
    int g = X.row_speed[r0 + r];
    const double* u = srow + (long long)r * in_len;
    double y;
    if (X.ident[g]) {
      y = u[(cell + halo_l) * O + i];
    } else {
      long long n = X.ns[g];
      long long ca, cb;
      if (periodic) {
        ca = pymod(cell - n, in_cells);
        cb = pymod(cell - n - 1, in_cells);
      } else {
        ca = cell + halo_l - n;
        cb = ca - 1;
      }
      const double* A = X.mats + (long long)g * 2 * O * O;
      const double* B = A + O * O;
      const double* ua = u + ca * O;
      const double* ub = u + cb * O;
      double sa = A[i * O] * ua[0];
      double sb = B[i * O] * ub[0];
#pragma unroll
      for (int jj = 1; jj < O; ++jj) {
        sa = fma(A[i * O + jj], ua[jj], sa);
        sb = fma(B[i * O + jj], ub[jj], sb);
      }
      y = sa + sb;
    }
    fout[(r0 + r) * ld_out + j] = y;
  }
}

}  // namespace sldg


namespace sldg {

// rho stage 1: CTA (chunk, 32-column tile), 8 warps stride the chunk's rows;
// fixed-order smem combine -> partial[chunk][c]
__global__ void __launch_bounds__(256)
k_rho_partial(const double* __restrict__ f, long long ld, long long n_rows, long long n_cols,
              const double* __restrict__ w, long long chunk, double* __restrict__ partial) {
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const long long c = (long long)blockIdx.y * 32 + lane;
  const long long ra = (long long)blockIdx.x * chunk;
  const long long rb = min(ra + chunk, n_rows);
  double s0 = 0.0, s1 = 0.0;
  if (c < n_cols) {
    long long r = ra + wp;
    for (; r + 8 < rb; r += 16) {
      s0 = fma(__ldg(w + r), __ldg(f + r * ld + c), s0);
      s1 = fma(__ldg(w + r + 8), __ldg(f + (r + 8) * ld + c), s1);
    }
    for (; r < rb; r += 8) s0 = fma(__ldg(w + r), __ldg(f + r * ld + c), s0);
  }
  red[wp][lane] = s0 + s1;
  __syncthreads();
  if (wp == 0 && c < n_cols) {
    double s = red[0][lane];
#pragma unroll
    for (int k = 1; k < 8; ++k) s += red[k][lane];
    partial[(long long)blockIdx.x * n_cols + c] = s;
  }
}

// stage 2 column sum: one warp per column, lane-strided partial sums + butterfly
// (fixed order for a fixed n_chunks)
__global__ void k_colsum(const double* __restrict__ partial, long long n_chunks, long long n_cols,
                         double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long c = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (c >= n_cols) return;
  double s = 0.0;
  for (long long k = lane; k < n_chunks; k += 32) s += partial[k * n_cols + c];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[c] = s;
}

// moments stage 1: warp per row: col_r = sum_c f[r,c] xw[c]; per CTA fixed-order
// sums of w_r*col_r, w_r*v0_r*col_r, w_r*v2_r*col_r
__global__ void __launch_bounds__(256)
k_moments_partial(const double* __restrict__ f, long long ld, long long n_rows, long long n_cols,
                  const double* __restrict__ w, const double* __restrict__ v0,
                  const double* __restrict__ v2, const double* __restrict__ xw, long long chunk,
                  double* __restrict__ partial) {
  __shared__ double red[8][3];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const long long ra = (long long)blockIdx.x * chunk;
  const long long rb = min(ra + chunk, n_rows);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (long long r = ra + wp; r < rb; r += 8) {
    double s = 0.0;
    for (long long c = lane; c < n_cols; c += 32) s = fma(__ldg(f + r * ld + c), __ldg(xw + c), s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    double ws = __ldg(w + r) * s;
    a0 += ws;
    a1 = fma(__ldg(w + r) * __ldg(v0 + r), s, a1);
    a2 = fma(__ldg(w + r) * __ldg(v2 + r), s, a2);
  }
  if (lane == 0) {
    red[wp][0] = a0;
    red[wp][1] = a1;
    red[wp][2] = a2;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double s = 0.0;
    for (int k = 0; k < 8; ++k) s += red[k][threadIdx.x];
    partial[blockIdx.x * 3 + threadIdx.x] = s;
  }
}

// stage 2 of the moments: warp w sums component w (launch with 96 threads)
// the same sums added onto `out` when acc != 0 (row chunks of one pass, in chunk order)
__global__ void k_colsum_acc(const double* __restrict__ partial, long long n_chunks,
                             long long n_cols, double* __restrict__ out, int acc) {
  const int lane = threadIdx.x & 31;
  const long long c = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (c >= n_cols) return;
  double s = 0.0;
  for (long long k = lane; k < n_chunks; k += 32) s += partial[k * n_cols + c];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[c] = acc ? out[c] + s : s;
}

__global__ void k_sum3_acc(const double* __restrict__ partial, long long n,
                           double* __restrict__ out, int acc) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (w >= 3) return;
  double s = 0.0;
  for (long long k = lane; k < n; k += 32) s += partial[k * 3 + w];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[w] = acc ? out[w] + s : s;
}

__global__ void k_sum3(const double* __restrict__ partial, long long n, double* __restrict__ out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (w >= 3) return;
  double s = 0.0;
  for (long long k = lane; k < n; k += 32) s += partial[k * 3 + w];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[w] = s;
}

// Poisson rhs (xfield.py:148-155): rbar = (w.rho)/L; b[node] += w (rho - rbar) in
// np.add.at order (flat DOF order).  Single CTA.
__global__ void k_poisson_rhs(const double* __restrict__ rho, const double* __restrict__ xw,
                              long long n_cells, int p, double length, double* __restrict__ b) {
  __shared__ double red[1024];
  const int o = p + 1;
  const long long n_dofs = n_cells * o, n_nodes = n_cells * p;
  double s = 0.0;
  for (long long k = threadIdx.x; k < n_dofs; k += blockDim.x) s = fma(xw[k], rho[k], s);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  const double rbar = red[0] / length;
  for (long long node = threadIdx.x; node < n_nodes; node += blockDim.x) {
    long long cell = node / p;
    int j = (int)(node - cell * p);
    double v;
    if (j == 0) {
      // shared vertex: previous cell's last DOF (flat order first), then this cell's first;
      // node 0: cell 0 DOF 0 comes first, the wrapped last cell's DOF p second
      long long kprev = (cell == 0 ? n_cells - 1 : cell - 1) * o + p;
      long long kthis = cell * o;
      double cprev = __dmul_rn(xw[kprev], __dsub_rn(rho[kprev], rbar));
      double cthis = __dmul_rn(xw[kthis], __dsub_rn(rho[kthis], rbar));
      v = (cell == 0) ? __dadd_rn(cthis, cprev) : __dadd_rn(cprev, cthis);
    } else {
      long long k = cell * o + j;
      v = __dmul_rn(xw[k], __dsub_rn(rho[k], rbar));
    }
    b[node] = v;
  }
}

// phi = G b: warp per row, fixed lane-stride + butterfly order
__global__ void k_gemv(const double* __restrict__ G, const double* __restrict__ b, long long n,
                       double* __restrict__ phi) {
  const int lane = threadIdx.x & 31;
  const long long row = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  double s = 0.0;
  for (long long k = lane; k < n; k += 32) s = fma(__ldg(G + row * n + k), __ldg(b + k), s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) phi[row] = s;
}

// E = (-(2/h) phi_loc) @ D^T per element (xfield.py:170-179)
__global__ void k_efield(const double* __restrict__ phi, const double* __restrict__ D,
                         long long n_cells, int p, double h, double* __restrict__ e) {
  const int o = p + 1;
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n_cells * o) return;
  long long cell = k / o;
  int i = (int)(k - cell * o);
  const long long nn = n_cells * p;
  const double sc = -(2.0 / h);
  double s = 0.0;
  for (int j = 0; j < o; ++j) {
    long long node = (cell * p + j) % nn;
    s = fma(__dmul_rn(sc, phi[node]), D[i * o + j], s);
  }
  e[k] = s;
}

__global__ void k_field_diag(const double* __restrict__ e, const double* __restrict__ xw,
                             long long n, double* __restrict__ out2) {
  __shared__ double rm[1024], rs[1024];
  double m = 0.0, s = 0.0;
  for (long long k = threadIdx.x; k < n; k += blockDim.x) {
    double v = e[k];
    m = fmax(m, fabs(v));
    s = fma(xw[k], v * v, s);
  }
  rm[threadIdx.x] = m;
  rs[threadIdx.x] = s;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      rm[threadIdx.x] = fmax(rm[threadIdx.x], rm[threadIdx.x + st]);
      rs[threadIdx.x] += rs[threadIdx.x + st];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out2[0] = rm[0];
    out2[1] = 0.5 * rs[0];
  }
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// The row partition depends on n_rows only, so every column's rho is bitwise
// identical however the columns are sharded across ranks.
static long long rho_chunks(long long n_rows, long long n_cols) {
  (void)n_cols;
  long long chunk = std::max<long long>(64, (n_rows + 255) / 256);
  return (n_rows + chunk - 1) / chunk;
}

static long long moments_chunks(long long n_rows) {
  long long chunk = std::max<long long>(64, (n_rows + 148LL * 8 - 1) / (148LL * 8));
  return (n_rows + chunk - 1) / chunk;
}

template <int O>
static int launch_advect_x(const sldg_xplan* X, const double* fin, long long ld_in, double* fout,
                           long long ld_out, int in_cells, int out_cells, int halo_l, int periodic,
                           cudaStream_t st) {
  const int in_len = in_cells * O;
  // rows per CTA: stage about 24 KB of input
  int rows = std::max(1, (int)(3072 / std::max(1, in_len)));
  rows = std::min<long long>(rows, X->n_rows);
  size_t smem = sizeof(double) * (size_t)rows * in_len;
  if (smem > 200 * 1024) {
    set_error("x row too long for shared-memory staging");
    return SLDG_ERR_UNSUPPORTED;
  }
  SLDG_CUDA_TRY(smem_limit((const void*)k_advect_x<O>, (int)std::max<size_t>(smem, 48 * 1024)));
  long long blocks = (X->n_rows + rows - 1) / rows;
  k_advect_x<O><<<(unsigned)blocks, 256, smem, st>>>(X->dev, fin, ld_in, fout, ld_out, X->n_rows,
                                                     in_cells, out_cells, halo_l, periodic, rows);
  SLDG_LAUNCH_CHECK("k_advect_x");
  return SLDG_OK;
}

}  // namespace sldg

#include "xx_tiles.cuh"

namespace sldg {

// Geometry of k_xx_tiles: depends only on the problem shape (bitwise-stable sums).
// n_out: output cells per row (default: the periodic row); src_len: doubles staged
// per source row (default: the row itself; an x slab stages its margins too)
static XTGeom xt_geom(const sldg_xplan* X, long long n_out = -1, long long src_len = -1,
                      long long n_rows = -1) {
  XTGeom g{};
  g.ok = false;
  const int ov = X->vo, ox = X->o;
  const long long nxc = n_out < 0 ? X->n_cells : n_out;
  const long long rows = n_rows < 0 ? X->n_rows : n_rows;
  if (ov < 2 || ov > 4 || ox < 2 || ox > 4 || nxc > 512 || rows == 0) return g;
  const int nl = ov * ov, nloc = nl * ov;
  if (rows % nloc != 0) return g;
  g.tpc = (int)std::max<long long>(1, std::min<long long>(kXTMaxTpc, 512 / nxc));
  g.threads = (int)((g.tpc * nxc + 31) / 32 * 32);
  if (g.threads < 64) g.threads = 64;
  const long long row_len = src_len < 0 ? nxc * ox : src_len;
  g.n_out = (int)nxc;
  g.src_len = (int)row_len;
  const size_t table = sizeof(double) * X->n_speeds * 2 * ox * ox + 5 * X->n_speeds + 64;
  const size_t budget = 227 * 1024 - 1024;
  for (int nring : {3, 2}) {
    for (int rpt = nl; rpt >= 1 && !g.ok; --rpt) {
      if (nl % rpt) continue;
      const size_t slot = (size_t)g.tpc * rpt * row_len;
      const size_t smem = sizeof(double) * ((nring + 1) * slot + (size_t)nring * g.tpc * rpt * 3) + table;
      if (smem <= budget && sizeof(double) * nring * slot >= sizeof(double) * 3 * g.threads) {
        g.rpt = rpt;
        g.nring = nring;
        g.smem = smem;
        g.ok = true;
      }
    }
    if (g.ok) break;
  }
  if (!g.ok) return g;
  g.n_tiles = (rows / nloc) * (nl / g.rpt) * ov;
  if (g.n_tiles * g.tpc >= (1LL << 31)) {   // the kernel indexes tiles in 32 bits
    g.ok = false;
    return g;
  }
  g.n_groups = (g.n_tiles + g.tpc - 1) / g.tpc;
  const long long ctas_sm = std::max<long long>(1, std::min<long long>(
      (long long)(227 * 1024 / g.smem), 2048 / g.threads));
  g.n_groups = std::max<long long>(1, g.n_groups);
  g.grid_ = std::min<long long>(g.n_groups, 148LL * ctas_sm);
  return g;
}

template <int OV, int OX>
static int launch_xt_t(const sldg_xplan* X, const XTGeom& g, const double* fin, double* fout,
                       long long ld, int napply, bool mom, bool rho, const XEpi& epi,
                       cudaStream_t st, const XRowMap& rm) {
  auto k = k_xx_tiles<OV, OX, 0>;
  if constexpr (OV == 3) {
    if (g.rpt == 3) k = k_xx_tiles<OV, OX, 3>;
  }
  SLDG_CUDA_TRY(smem_limit((const void*)k, (int)g.smem));
  const long long rows = g.n_tiles / ((OV * OV / g.rpt) * OV) * (OV * OV * OV);
  k<<<(unsigned)g.grid_, g.threads, g.smem, st>>>(X->dev, fin, fout, ld, rows, g.n_out,
                                                  g.rpt, g.tpc, g.nring, (int)X->n_speeds, epi,
                                                  napply, mom ? 1 : 0, rho ? 1 : 0, rm);
  SLDG_LAUNCH_CHECK("k_xx_tiles");
  return SLDG_OK;
}

static int launch_xt(const sldg_xplan* X, const XTGeom& g, const double* fin, double* fout,
                     long long ld, int napply, bool mom, bool rho, const XEpi& epi,
                     cudaStream_t st, const XRowMap* rmap = nullptr) {
  // default: periodic rows, output in place of the input layout
  const XRowMap rm = rmap ? *rmap : XRowMap{g.src_len, 0, 0, 1, 0, ld, 0};
  switch (X->vo * 10 + X->o) {
#define CASE(A, B) \
  case A * 10 + B: return launch_xt_t<A, B>(X, g, fin, fout, ld, napply, mom, rho, epi, st, rm);
    CASE(2, 2) CASE(2, 3) CASE(2, 4) CASE(3, 2) CASE(3, 3) CASE(3, 4) CASE(4, 2) CASE(4, 3)
    CASE(4, 4)
#undef CASE
  }
  set_error("x tile kernel: unsupported degrees");
  return SLDG_ERR_UNSUPPORTED;
}

// X.X pass (moments of the intermediate, rho of the result) over the velocity cells
// cells[0 .. n_list), in place: the rows the one-pass AMR step does not finish
// (amr_fused.cuh).  xx_cells_grid: its CTA count (partials it writes), 0 when the
// tile kernel cannot run this plan.
long long xx_cells_grid(const sldg_xplan* X, long long n_list) {
  if (n_list <= 0) return 0;
  const long long nloc = (long long)X->vo * X->vo * X->vo;
  const XTGeom g = xt_geom(X, -1, -1, n_list * nloc);
  return g.ok ? g.grid_ : 0;
}

int xx_cells_run(const sldg_xplan* X, double* f, long long ld, const long long* cells,
                 long long n_list, const double* w, const double* v0, const double* v2,
                 const double* xw, double* mom_part, double* rho_part, cudaStream_t st) {
  if (n_list <= 0) return SLDG_OK;
  const long long nloc = (long long)X->vo * X->vo * X->vo;
  const XTGeom g = xt_geom(X, -1, -1, n_list * nloc);
  if (!g.ok) {
    set_error("cell-list x pass: unsupported geometry");
    return SLDG_ERR_UNSUPPORTED;
  }
  const XEpi epi{w, v0, v2, xw, mom_part, rho_part};
  const XRowMap rm{g.src_len, 0, 0, 1, 0, ld, 0, cells};
  return launch_xt(X, g, f, f, ld, 2, true, true, epi, st, &rm);
}

}  // namespace sldg

using namespace sldg;

extern "C" {

int sldg_xplan_create(const SldgXPlanDesc* d, sldg_xplan** out) {
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
  if (d->n_cells < 4 || !(d->h > 0.0) || !(d->dt > 0.0) || d->n_rows < 0 || d->n_speeds < 0 ||
      (d->n_rows > 0 && (!d->row_speed || !d->speeds))) {
    set_error("bad x plan description");
    return SLDG_ERR_ARG;
  }
  for (long long r = 0; r < d->n_rows; ++r)
    if (d->row_speed[r] < 0 || d->row_speed[r] >= d->n_speeds) {
      set_error("row speed index out of range");
      return SLDG_ERR_ARG;
    }
  const int o = basis.o;
  const long long S = std::max<long long>(d->n_speeds, 1), R = std::max<long long>(d->n_rows, 1);
  size_t off = 0;
  size_t o_ns = off; off = align_up(off + sizeof(long long) * S, 256);
  size_t o_id = off; off = align_up(off + S, 256);
  size_t o_m = off; off = align_up(off + sizeof(double) * 2 * o * o * S, 256);
  size_t o_rs = off; off = align_up(off + sizeof(int) * R, 256);
  size_t o_sp = off; off = align_up(off + sizeof(double) * S, 256);
  size_t o_nsm = off; off = align_up(off + sizeof(int) * S, 256);
  sldg_xplan* X = new sldg_xplan();
  cudaError_t ce = cudaMalloc(&X->block, off);
  if (ce != cudaSuccess) {
    delete X;
    return cuda_fail(ce, "cudaMalloc(xplan)");
  }
  unsigned char* base = (unsigned char*)X->block;
  X->dev.ns = (long long*)(base + o_ns);
  X->dev.ident = base + o_id;
  X->dev.mats = (double*)(base + o_m);
  X->dev.row_speed = (int*)(base + o_rs);
  X->dev.nsm = (int*)(base + o_nsm);
  double* dsp = (double*)(base + o_sp);
  if (d->n_rows > 0) {
    ce = cudaMemcpy((void*)X->dev.row_speed, d->row_speed, sizeof(int) * d->n_rows,
                    cudaMemcpyHostToDevice);
    if (ce == cudaSuccess)
      ce = cudaMemcpy(dsp, d->speeds, sizeof(double) * d->n_speeds, cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) {
      cudaFree(X->block);
      delete X;
      return cuda_fail(ce, "cudaMemcpy(xplan)");
    }
  }
  X->basis = basis;
  X->o = o;
  X->n_cells = d->n_cells;
  X->n_rows = d->n_rows;
  X->n_speeds = d->n_speeds;
  X->h = d->h;
  X->dt = d->dt;
  if (d->n_speeds > 0) {
    int threads = 128;
    int blocks = (int)((d->n_speeds + threads - 1) / threads);
    switch (o) {
#define CASE(O)                                                                               \
  case O:                                                                                     \
    k_xmats<O><<<blocks, threads>>>(basis, dsp, d->n_speeds, d->dt, d->h, (long long*)X->dev.ns, \
                                    (unsigned char*)X->dev.ident, (double*)X->dev.mats);      \
    break;
      CASE(2) CASE(3) CASE(4) CASE(5) CASE(6)
#undef CASE
    }
    count_launch();
    ce = cudaDeviceSynchronize();
    if (ce != cudaSuccess) {
      cudaFree(X->block);
      delete X;
      return cuda_fail(ce, "k_xmats");
    }
    // halo requirement from the integer shifts
    std::vector<long long> ns(d->n_speeds);
    cudaMemcpy(ns.data(), X->dev.ns, sizeof(long long) * d->n_speeds, cudaMemcpyDeviceToHost);
    std::vector<unsigned char> id(d->n_speeds);
    cudaMemcpy(id.data(), X->dev.ident, d->n_speeds, cudaMemcpyDeviceToHost);
    long long hl = 0, hr = 0;
    for (long long u = 0; u < d->n_speeds; ++u) {
      if (id[u]) continue;
      // sources: cell - n and cell - n - 1
      hl = std::max(hl, ns[u] + 1);
      hr = std::max(hr, -ns[u]);
    }
    X->halo_l = hl;
    X->halo_r = hr;
    std::vector<int> nsm(d->n_speeds);
    for (long long u = 0; u < d->n_speeds; ++u)
      nsm[u] = (int)(((ns[u] % d->n_cells) + d->n_cells) % d->n_cells);
    ce = cudaMemcpy((void*)X->dev.nsm, nsm.data(), sizeof(int) * d->n_speeds,
                    cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) {
      cudaFree(X->block);
      delete X;
      return cuda_fail(ce, "cudaMemcpy(xplan nsm)");
    }
  }
  *out = X;
  return SLDG_OK;
}

int sldg_xplan_destroy(sldg_xplan* X) {
  if (!X) return SLDG_OK;
  if (X->block) cudaFree(X->block);
  delete X;
  return SLDG_OK;
}

int sldg_xplan_halo(const sldg_xplan* X, int64_t* lr) {
  if (!X || !lr) {
    set_error("bad argument");
    return SLDG_ERR_ARG;
  }
  lr[0] = X->halo_l;
  lr[1] = X->halo_r;
  return SLDG_OK;
}

int sldg_xplan_set_vlayout(sldg_xplan* X, int32_t o_v) {
  if (!X || o_v < 1) {
    set_error("bad argument");
    return SLDG_ERR_ARG;
  }
  const long long nloc = (long long)o_v * o_v * o_v;
  if (X->n_rows % nloc != 0) {
    set_error("rows are not cells x o_v^3");
    return SLDG_ERR_ARG;
  }
  std::vector<int> rs(X->n_rows);
  cudaError_t ce = cudaMemcpy(rs.data(), X->dev.row_speed, sizeof(int) * X->n_rows,
                              cudaMemcpyDeviceToHost);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaMemcpy(row_speed)");
  // every row b = i + o j + o^2 k of a cell must share the speed of its v_x node i
  for (long long r = 0; r < X->n_rows; ++r) {
    const long long cell = r / nloc, b = r - cell * nloc;
    if (rs[r] != rs[cell * nloc + b % o_v]) {
      set_error("row speeds are not constant per (cell, v_x node)");
      return SLDG_ERR_ARG;
    }
  }
  X->vo = o_v;
  return SLDG_OK;
}

int sldg_advect_x(const sldg_xplan* X, const double* fin, double* fout, int64_t ld, void* stream) {
  if (!X || !fin || !fout || fin == fout || ld < X->n_cells * X->o) {
    set_error("bad advect_x arguments (f_in and f_out must be distinct device buffers)");
    return SLDG_ERR_ARG;
  }
  if (X->n_rows == 0) return SLDG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  XEpi epi{};
  {
    XTGeom tg = xt_geom(X);
    if (tg.ok) return launch_xt(X, tg, fin, fout, ld, 1, false, false, epi, st);
  }
  // rows without the velocity-cell layout (1V, or a plan built for arbitrary rows):
  // the generic row kernel
  switch (X->o) {
#define CASE(O) \
  case O: return launch_advect_x<O>(X, fin, ld, fout, ld, (int)X->n_cells, (int)X->n_cells, 0, 1, st);
    CASE(2) CASE(3) CASE(4) CASE(5) CASE(6)
#undef CASE
  }
  set_error("unsupported degree");
  return SLDG_ERR_UNSUPPORTED;
}

int sldg_xadv_scratch_bytes(const sldg_xplan* X, size_t* bytes) {
  if (!X || !bytes) {
    set_error("bad argument");
    return SLDG_ERR_ARG;
  }
  const XTGeom tg = xt_geom(X);
  const long long grid = tg.ok ? tg.grid_ : 1;
  *bytes = sizeof(double) * (size_t)grid * (3 + X->n_cells * X->o) + 256;
  return SLDG_OK;
}

int sldg_advect_x_fused(const sldg_xplan* X, const double* fin, double* fout, int64_t ld,
                        int32_t n_apply, const double* w, const double* v0, const double* v2,
                        const double* xw, double* mom_out3, double* rho_out, void* scratch,
                        void* stream) {
  const bool mom = mom_out3 != nullptr, rho = rho_out != nullptr;
  if (!X || !fin || !fout || fin == fout || ld < X->n_cells * X->o ||
      (n_apply != 1 && n_apply != 2) || (mom && (!w || !v0 || !v2 || !xw)) || (rho && !w) ||
      ((mom || rho) && !scratch)) {
    set_error("bad advect_x_fused arguments");
    return SLDG_ERR_ARG;
  }
  if (X->n_rows == 0) return SLDG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const XTGeom tg = xt_geom(X);
  if (!tg.ok) {   // the caller runs the separate passes (advect_x, rho, moments)
    set_error("fused x pass: needs the velocity-cell row layout (sldg_xplan_set_vlayout) "
              "and rows of at most 512 cells");
    return SLDG_ERR_UNSUPPORTED;
  }
  XEpi epi{w, v0, v2, xw, nullptr, nullptr};
  if (scratch) {
    epi.mom_part = (double*)scratch;
    epi.rho_part = (double*)scratch + 3 * (size_t)tg.grid_;
  }
  const int rc = launch_xt(X, tg, fin, fout, ld, n_apply, mom, rho, epi, st);
  if (rc) return rc;
  if (mom) {
    k_sum3<<<1, 96, 0, st>>>(epi.mom_part, tg.grid_, mom_out3);
    SLDG_LAUNCH_CHECK("k_sum3");
  }
  if (rho) {
    const long long row_len = X->n_cells * X->o;
    k_colsum<<<(unsigned)((row_len * 32 + 255) / 256), 256, 0, st>>>(epi.rho_part, tg.grid_,
                                                                row_len, rho_out);
    SLDG_LAUNCH_CHECK("k_colsum");
  }
  return SLDG_OK;
}

int sldg_advect_x_slab(const sldg_xplan* X, const double* fin, int64_t ld_in, int64_t halo_l,
                       int64_t halo_r, int64_t n_local, double* fout, int64_t ld_out,
                       void* stream) {
  if (!X || !fin || !fout || n_local < 1 || halo_l < X->halo_l || halo_r < X->halo_r ||
      ld_in < (halo_l + n_local + halo_r) * X->o || ld_out < n_local * X->o) {
    set_error("bad advect_x_slab arguments (halo too narrow?)");
    return SLDG_ERR_ARG;
  }
  if (X->n_rows == 0) return SLDG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int in_cells = (int)(halo_l + n_local + halo_r);
  switch (X->o) {
#define CASE(O)                                                                             \
  case O:                                                                                   \
    return launch_advect_x<O>(X, fin, ld_in, fout, ld_out, in_cells, (int)n_local, (int)halo_l, \
                              0, st);
    CASE(2) CASE(3) CASE(4) CASE(5) CASE(6)
#undef CASE
  }
  set_error("unsupported degree");
  return SLDG_ERR_UNSUPPORTED;
}

int sldg_advect_x_slab_tiles_scratch(const sldg_xplan* X, int64_t n_local, int64_t ld_in,
                                     size_t* bytes) {
  if (!X || !bytes || n_local < 1) {
    set_error("bad argument");
    return SLDG_ERR_ARG;
  }
  const XTGeom tg = xt_geom(X, n_local, ld_in);
  if (!tg.ok) {
    set_error("slab tile kernel: unsupported shape");
    return SLDG_ERR_UNSUPPORTED;
  }
  // the whole-plan launch has the largest grid of any row range
  *bytes = sizeof(double) * (size_t)tg.grid_ * (3 + n_local * X->o) + 256;
  return SLDG_OK;
}

int sldg_advect_x_slab_tiles(const sldg_xplan* X, const double* row_base, int64_t ld_in,
                             int64_t src_off, int64_t halo_l, int64_t halo_r, int64_t n_local,
                             double* fout, int64_t ld_out, int64_t out_off, int32_t n_apply,
                             int64_t row_begin, int64_t row_count, int32_t accumulate,
                             const double* w, const double* v0, const double* v2,
                             const double* xw_local, double* mom_out3, double* rho_out,
                             void* scratch, void* stream) {
  const bool mom = mom_out3 != nullptr, rho = rho_out != nullptr;
  if (!X) {
    set_error("null x plan");
    return SLDG_ERR_ARG;
  }
  const long long nloc = (long long)X->vo * X->vo * X->vo;
  // reach of the shifts: one application needs (halo_l, halo_r) >= the plan's, two need
  // twice that, and at least (2, 1) cells for the intermediate's halo cells
  const long long need_l = n_apply == 2 ? std::max<long long>(2, 2 * X->halo_l) : X->halo_l;
  const long long need_r = n_apply == 2 ? std::max<long long>(1, 2 * X->halo_r) : X->halo_r;
  if (!row_base || !fout || n_local < 1 || (n_apply != 1 && n_apply != 2) ||
      halo_l < need_l || halo_r < need_r || halo_l > n_local || halo_r > n_local ||
      src_off < 0 || src_off + (halo_l + n_local + halo_r) * X->o > ld_in || out_off < 0 ||
      out_off + n_local * X->o > ld_out || (mom && (!w || !v0 || !v2 || !xw_local)) ||
      (rho && !w) || ((mom || rho) && !scratch) || nloc == 0 || row_begin < 0 ||
      row_count < 0 || row_begin % nloc || row_count % nloc || row_begin + row_count > X->n_rows) {
    set_error("bad advect_x_slab_tiles arguments (halo too narrow? rows not whole cells?)");
    return SLDG_ERR_ARG;
  }
  if (row_count == 0) return SLDG_OK;
  // whole padded rows are staged (16-byte aligned bulk copies)
  const XTGeom tg = xt_geom(X, n_local, ld_in, row_count);
  if (!tg.ok || (ld_in & 1) || (((unsigned long long)row_base) & 15)) {
    set_error("slab tile kernel: unsupported shape (rows too long / unaligned)");
    return SLDG_ERR_UNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  XEpi epi{w, v0, v2, xw_local, nullptr, nullptr};
  if (scratch) {
    epi.mom_part = (double*)scratch;
    epi.rho_part = (double*)scratch + 3 * (size_t)tg.grid_;
  }
  const XRowMap rm{(int)ld_in, (int)src_off, (int)halo_l, 0, (int)out_off, ld_out, row_begin};
  int rc = launch_xt(X, tg, row_base, fout, ld_in, n_apply, mom, rho, epi, st, &rm);
  if (rc) return rc;
  if (mom) {
    k_sum3_acc<<<1, 96, 0, st>>>(epi.mom_part, tg.grid_, mom_out3, accumulate);
    SLDG_LAUNCH_CHECK("k_sum3");
  }
  if (rho) {
    const long long row_len = n_local * X->o;
    k_colsum_acc<<<(unsigned)((row_len * 32 + 255) / 256), 256, 0, st>>>(
        epi.rho_part, tg.grid_, row_len, rho_out, accumulate);
    SLDG_LAUNCH_CHECK("k_colsum");
  }
  return SLDG_OK;
}

int sldg_rho_scratch_bytes(int64_t n_rows, int64_t n_cols, size_t* bytes) {
  if (!bytes || n_rows < 0 || n_cols < 0) {
    set_error("bad argument");
    return SLDG_ERR_ARG;
  }
  *bytes = sizeof(double) * (size_t)std::max<long long>(1, rho_chunks(n_rows, n_cols)) *
           std::max<long long>(n_cols, 1);
  return SLDG_OK;
}

int sldg_rho(const double* f, int64_t ld, int64_t n_rows, int64_t n_cols, const double* w,
             double* rho, void* scratch, void* stream) {
  if (!f || !w || !rho || !scratch || n_rows < 1 || n_cols < 1 || ld < n_cols) {
    set_error("bad rho arguments");
    return SLDG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  long long nch = rho_chunks(n_rows, n_cols);
  long long chunk = (n_rows + nch - 1) / nch;
  nch = (n_rows + chunk - 1) / chunk;
  dim3 grid((unsigned)nch, (unsigned)((n_cols + 31) / 32));
  k_rho_partial<<<grid, 256, 0, st>>>(f, ld, n_rows, n_cols, w, chunk, (double*)scratch);
  SLDG_LAUNCH_CHECK("k_rho_partial");
  k_colsum<<<(unsigned)((n_cols * 32 + 255) / 256), 256, 0, st>>>((double*)scratch, nch, n_cols, rho);
  SLDG_LAUNCH_CHECK("k_colsum");
  return SLDG_OK;
}

int sldg_moments_scratch_bytes(int64_t n_rows, size_t* bytes) {
  if (!bytes || n_rows < 0) {
    set_error("bad argument");
    return SLDG_ERR_ARG;
  }
  *bytes = sizeof(double) * 3 * (size_t)std::max<long long>(1, moments_chunks(n_rows));
  return SLDG_OK;
}

int sldg_moments(const double* f, int64_t ld, int64_t n_rows, int64_t n_cols, const double* w,
                 const double* v0, const double* v2, const double* xw, double* out3,
                 void* scratch, void* stream) {
  if (!f || !w || !v0 || !v2 || !xw || !out3 || !scratch || n_rows < 1 || n_cols < 1 ||
      ld < n_cols) {
    set_error("bad moments arguments");
    return SLDG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  long long nch = moments_chunks(n_rows);
  long long chunk = (n_rows + nch - 1) / nch;
  nch = (n_rows + chunk - 1) / chunk;
  k_moments_partial<<<(unsigned)nch, 256, 0, st>>>(f, ld, n_rows, n_cols, w, v0, v2, xw, chunk,
                                                   (double*)scratch);
  SLDG_LAUNCH_CHECK("k_moments_partial");
  k_sum3<<<1, 96, 0, st>>>((double*)scratch, nch, out3);
  SLDG_LAUNCH_CHECK("k_sum3");
  return SLDG_OK;
}

int sldg_poisson_create(const SldgPoissonDesc* d, sldg_poisson** out) {
  if (!d || !out || d->degree < 1 || d->degree > SLDG_MAX_DEGREE || d->n_cells < 4 ||
      !d->dof_weights || !d->diff || !d->green || !(d->h > 0.0) || !(d->length > 0.0)) {
    set_error("bad Poisson description");
    return SLDG_ERR_ARG;
  }
  *out = nullptr;
  sldg_poisson* P = new sldg_poisson();
  P->p = d->degree;
  P->o = d->degree + 1;
  P->n_cells = d->n_cells;
  P->n_nodes = d->n_cells * d->degree;
  P->n_dofs = d->n_cells * P->o;
  P->h = d->h;
  P->length = d->length;
  size_t off = 0;
  size_t o_xw = off; off = align_up(off + sizeof(double) * P->n_dofs, 256);
  size_t o_d = off; off = align_up(off + sizeof(double) * P->o * P->o, 256);
  size_t o_g = off; off = align_up(off + sizeof(double) * P->n_nodes * P->n_nodes, 256);
  size_t o_w = off; off = align_up(off + sizeof(double) * (2 * P->n_nodes + 8), 256);
  cudaError_t ce = cudaMalloc(&P->block, off);
  if (ce != cudaSuccess) {
    delete P;
    return cuda_fail(ce, "cudaMalloc(poisson)");
  }
  unsigned char* base = (unsigned char*)P->block;
  P->xw = (double*)(base + o_xw);
  P->diff = (double*)(base + o_d);
  P->green = (double*)(base + o_g);
  P->work = (double*)(base + o_w);
  ce = cudaMemcpy(P->xw, d->dof_weights, sizeof(double) * P->n_dofs, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess)
    ce = cudaMemcpy(P->diff, d->diff, sizeof(double) * P->o * P->o, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess)
    ce = cudaMemcpy(P->green, d->green, sizeof(double) * P->n_nodes * P->n_nodes,
                    cudaMemcpyHostToDevice);
  if (ce != cudaSuccess) {
    cudaFree(P->block);
    delete P;
    return cuda_fail(ce, "cudaMemcpy(poisson)");
  }
  *out = P;
  return SLDG_OK;
}

int sldg_poisson_destroy(sldg_poisson* P) {
  if (!P) return SLDG_OK;
  if (P->block) cudaFree(P->block);
  delete P;
  return SLDG_OK;
}

int sldg_poisson_solve(const sldg_poisson* P, const double* rho, double* phi, double* e,
                       void* stream) {
  if (!P || !rho || (!e && !phi)) {
    set_error("bad Poisson solve arguments");
    return SLDG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  double* b = P->work;
  double* ph = phi ? phi : P->work + P->n_nodes;
  k_poisson_rhs<<<1, 1024, 0, st>>>(rho, P->xw, P->n_cells, P->p, P->length, b);
  SLDG_LAUNCH_CHECK("k_poisson_rhs");
  long long threads = P->n_nodes * 32;
  k_gemv<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(P->green, b, P->n_nodes, ph);
  SLDG_LAUNCH_CHECK("k_gemv");
  if (e) {
    k_efield<<<(unsigned)((P->n_dofs + 127) / 128), 128, 0, st>>>(ph, P->diff, P->n_cells, P->p,
                                                                  P->h, e);
    SLDG_LAUNCH_CHECK("k_efield");
  }
  return SLDG_OK;
}

int sldg_poisson_efield(const sldg_poisson* P, const double* phi, double* e, void* stream) {
  if (!P || !phi || !e) {
    set_error("bad electric_field arguments");
    return SLDG_ERR_ARG;
  }
  k_efield<<<(unsigned)((P->n_dofs + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      phi, P->diff, P->n_cells, P->p, P->h, e);
  SLDG_LAUNCH_CHECK("k_efield");
  return SLDG_OK;
}

int sldg_field_diag(const sldg_poisson* P, const double* e, double* out2, void* stream) {
  if (!P || !e || !out2) {
    set_error("bad field diag arguments");
    return SLDG_ERR_ARG;
  }
  k_field_diag<<<1, 1024, 0, (cudaStream_t)stream>>>(e, P->xw, P->n_dofs, out2);
  SLDG_LAUNCH_CHECK("k_field_diag");
  return SLDG_OK;
}

}  // extern "C"
