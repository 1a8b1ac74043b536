// pencil_ops.cu -- the reference's pure pencil-level functions on the device.
//
//   sldg_apply_update        apply_update (sldg1d.py:124-136): one uniform-pencil
//                            step out_i = A u_{i-n} + B u_{i-n-1}, batched
//   sldg_projection_oracle   projection_oracle (sldg1d.py:139-178): the brute-force
//                            exact-translation + 50-point Gauss L2 projection
//   sldg_weighted_writeback  weighted_writeback (vsweep.py:249-272): flat
//                            contribution arrays, numpy's assignment / bincount
//                            order (copies in flat order, then out += sum of
//                            w (v - f_in) in flat order)
// (generalized_overlap is sldg_generalized_overlap in vsweep.cu, next to the
// sweep's own block routine.)
#include <string>

#include "plans.cuh"
#include "sldg_common.cuh"

namespace sldg {

// thread = (batch, destination cell); the O outputs of the cell in registers
template <int O>
__global__ void k_apply_update(const double* __restrict__ v, long long n_batch, long long n,
                               long long n_shift, const double* __restrict__ A,
                               const double* __restrict__ B, int bc, double* __restrict__ out) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= n_batch * n) return;
  const long long bt = idx / n, i = idx - bt * n;
  long long qa = i - n_shift, qb = i - n_shift - 1;
  bool va = true, vb = true;
  if (bc == SLDG_BC_PERIODIC) {
    qa = pymod(qa, n);
    qb = pymod(qb, n);
  } else {
    va = qa >= 0 && qa < n;
    vb = qb >= 0 && qb < n;
  }
  double Ar[O * O], Br[O * O], ua[O], ub[O], y[O];
#pragma unroll
  for (int k = 0; k < O * O; ++k) {
    Ar[k] = A[k];
    Br[k] = B[k];
  }
  const double* row = v + bt * n * O;
#pragma unroll
  for (int j = 0; j < O; ++j) {
    ua[j] = va ? row[qa * O + j] : 0.0;
    ub[j] = vb ? row[qb * O + j] : 0.0;
  }
  two_cell<O>(Ar, Br, ua, ub, va, vb, y);
#pragma unroll
  for (int k = 0; k < O; ++k) out[idx * O + k] = y[k];
}

// thread = destination cell i: every source cell c and periodic image k whose
// translated support overlaps the foot [i w - d, (i+1) w - d) contributes a
// 50-point Gauss integral; the cell's rhs is then mapped by M^-1
template <int O>
__global__ void k_projection_oracle(DevBasis b, const double* __restrict__ v, long long n,
                                    double disp, double width, int n_images,
                                    const double* __restrict__ gq, const double* __restrict__ gw,
                                    int nq, double* __restrict__ out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double length = (double)n * width;
  const double foot_lo = (double)i * width - disp;
  double rhs[O];
#pragma unroll
  for (int k = 0; k < O; ++k) rhs[k] = 0.0;
  for (long long c = 0; c < n; ++c) {
    for (int im = -n_images; im <= n_images; ++im) {
      const double src_lo = (double)c * width + (double)im * length;
      const double vl = fmax(foot_lo, src_lo);
      const double vr = fmin(foot_lo + width, src_lo + width);
      if (vr <= vl) continue;
      double part[O];
#pragma unroll
      for (int k = 0; k < O; ++k) part[k] = 0.0;
      for (int q = 0; q < nq; ++q) {
        const double pt = 0.5 * (vl + vr) + 0.5 * (vr - vl) * gq[q];
        const double wt = 0.5 * (vr - vl) * gw[q];
        double ls[O], ld[O];
        lagrange_all<O>(b, 2.0 * (pt - src_lo) / width - 1.0, ls);
        lagrange_all<O>(b, 2.0 * (pt + disp - (double)i * width) / width - 1.0, ld);
        double sv = 0.0;
#pragma unroll
        for (int j = 0; j < O; ++j) sv = fma(ls[j], v[c * O + j], sv);
#pragma unroll
        for (int k = 0; k < O; ++k) part[k] = fma(wt * sv, ld[k], part[k]);
      }
#pragma unroll
      for (int k = 0; k < O; ++k) rhs[k] += (2.0 / width) * part[k];
    }
  }
#pragma unroll
  for (int k = 0; k < O; ++k) {   // out[i] = mass_inv @ rhs
    double y = 0.0;
#pragma unroll
    for (int j = 0; j < O; ++j) y = fma(b.minv[k * O + j], rhs[j], y);
    out[i * O + k] = y;
  }
}

// thread = element e; contributions of e are csr_idx[csr_off[e] .. csr_off[e+1]) in
// increasing flat order
__global__ void k_weighted_writeback(const double* __restrict__ f_in, long long n,
                                     const long long* __restrict__ csr_off,
                                     const long long* __restrict__ csr_idx,
                                     const double* __restrict__ w,
                                     const double* __restrict__ vals, double* __restrict__ out) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= n) return;
  const double f = f_in[e];
  double o = f, s = 0.0;
  for (long long k = csr_off[e]; k < csr_off[e + 1]; ++k) {
    const long long j = csr_idx[k];
    if (w[j] == 1.0) {
      o = vals[j];   // out[gather[is_copy]] = values[is_copy]: the last copy wins
    } else {
      s = __dadd_rn(s, __dmul_rn(w[j], __dsub_rn(vals[j], f)));
    }
  }
  out[e] = __dadd_rn(o, s);
}

}  // namespace sldg

using namespace sldg;

extern "C" {

int sldg_apply_update(const double* values, int64_t n_batch, int64_t n_cells, int32_t o,
                      int64_t n_shift, const double* A, const double* B, int32_t bc, double* out,
                      void* stream) {
  if (!values || !A || !B || !out || n_batch < 0 || n_cells <= 0 ||
      (bc != SLDG_BC_PERIODIC && bc != SLDG_BC_ABSORBING)) {
    set_error("bad apply_update arguments");
    return SLDG_ERR_ARG;
  }
  const long long total = n_batch * n_cells;
  if (total == 0) return SLDG_OK;
  const unsigned blocks = (unsigned)((total + 127) / 128);
  cudaStream_t st = (cudaStream_t)stream;
  switch (o) {
#define CASE(O)                                                                             \
  case O:                                                                                   \
    k_apply_update<O><<<blocks, 128, 0, st>>>(values, n_batch, n_cells, n_shift, A, B, bc, out); \
    break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6)
#undef CASE
    default:
      set_error("apply_update: degree 0..5");
      return SLDG_ERR_UNSUPPORTED;
  }
  SLDG_LAUNCH_CHECK("k_apply_update");
  return SLDG_OK;
}

int sldg_projection_oracle(const SldgBasis* basis, const double* values, int64_t n_cells,
                           double displacement, double width, int32_t bc, const double* gq,
                           const double* gw, int32_t nq, double* out, void* stream) {
  DevBasis b;
  std::string err;
  if (!basis || !make_dev_basis(*basis, &b, &err)) {
    set_error(basis ? err : "null basis");
    return SLDG_ERR_ARG;
  }
  if (!values || !gq || !gw || !out || n_cells <= 0 || nq <= 0 || !(width > 0.0) ||
      (bc != SLDG_BC_PERIODIC && bc != SLDG_BC_ABSORBING)) {
    set_error("bad projection_oracle arguments");
    return SLDG_ERR_ARG;
  }
  // periodic: images -n_images .. n_images of the source line (sldg1d.py:152-156)
  const double length = (double)n_cells * width;
  const int n_images = bc == SLDG_BC_PERIODIC ? (int)(fabs(displacement) / length) + 2 : 0;
  const unsigned blocks = (unsigned)((n_cells + 63) / 64);
  cudaStream_t st = (cudaStream_t)stream;
  switch (b.o) {
#define CASE(O)                                                                           \
  case O:                                                                                 \
    k_projection_oracle<O><<<blocks, 64, 0, st>>>(b, values, n_cells, displacement, width, \
                                                  n_images, gq, gw, nq, out);             \
    break;
    CASE(2) CASE(3) CASE(4) CASE(5) CASE(6)
#undef CASE
    default:
      set_error("projection_oracle: degree 1..5");
      return SLDG_ERR_UNSUPPORTED;
  }
  SLDG_LAUNCH_CHECK("k_projection_oracle");
  return SLDG_OK;
}

int sldg_weighted_writeback(const double* f_in, int64_t n, const int64_t* csr_off,
                            const int64_t* csr_idx, const double* weights, const double* values,
                            double* out, void* stream) {
  if (!f_in || !csr_off || !csr_idx || !weights || !values || !out || n < 0) {
    set_error("bad weighted_writeback arguments");
    return SLDG_ERR_ARG;
  }
  if (n == 0) return SLDG_OK;
  k_weighted_writeback<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      f_in, n, (const long long*)csr_off, (const long long*)csr_idx, weights, values, out);
  SLDG_LAUNCH_CHECK("k_weighted_writeback");
  return SLDG_OK;
}

}  // extern "C"
