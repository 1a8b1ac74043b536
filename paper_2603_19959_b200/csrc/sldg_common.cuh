// sldg_common.cuh -- shared device helpers for the SLDG transport kernels (sm_100a).
//
// Reference element math (basis.py:84-148), shift split (sldg1d.py:39-55) and
// overlap pair (sldg1d.py:72-100) restated for the device.  Everything is fp64
// with default IEEE division; the shift split uses _rn intrinsics so that it
// is bit-identical to Python's speed*dt/width.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "sldg_capi.h"

namespace sldg {

constexpr int kMaxO = SLDG_MAX_DEGREE + 1;
constexpr int kMaxQ = 2 * SLDG_MAX_DEGREE + 2;

// Basis constants passed by value as a kernel parameter (lives in the
// constant bank; every access below uses a warp-uniform index -> broadcast).
struct DevBasis {
  int p, o, nq;
  double nodes[kMaxO];
  double inv_denoms[kMaxO];
  double gq[kMaxQ];
  double gw[kMaxQ];
  double minv[kMaxO * kMaxO];
};

bool make_dev_basis(const SldgBasis& b, DevBasis* out, std::string* err);

// host-side error plumbing (capi.cu)
void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
void count_launch(int n = 1);
// Launch configuration without per-launch driver queries (so a launch sequence can be
// captured into a CUDA graph and replayed without host work): the dynamic shared
// memory limit of a kernel is only ever raised, the resident CTAs per SM and the SM
// count are memoised (capi.cu).
cudaError_t smem_limit(const void* kernel, int bytes);
cudaError_t resident_ctas(const void* kernel, int threads, int smem, int* per_sm);
int num_sms();

#define SLDG_CUDA_TRY(expr)                               \
  do {                                                    \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) return ::sldg::cuda_fail(_e, #expr); \
  } while (0)

#define SLDG_LAUNCH_CHECK(name)                                  \
  do {                                                           \
    ::sldg::count_launch();                                      \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::sldg::cuda_fail(_e, name);   \
  } while (0)

// ---------------------------------------------------------------------------
// device math
// ---------------------------------------------------------------------------
constexpr double kOneMinusUlp = 0.99999999999999988898;  // nextafter(1, 0)

// decompose_shift (sldg1d.py:39-55): r = speed*dt/width, n = floor(r), a = r-n,
// fold a >= nextafter(1,0) to (n+1, 0).
__device__ __forceinline__ void split_shift(double speed, double dt, double width,
                                            long long* n_out, double* a_out) {
  double r = __ddiv_rn(__dmul_rn(speed, dt), width);
  double n = floor(r);
  double a = __dsub_rn(r, n);
  if (a >= kOneMinusUlp) {
    n = n + 1.0;
    a = 0.0;
  }
  *n_out = (long long)n;
  *a_out = a;
}

// all Lagrange polynomials at x (basis.py:119-128): prod_{m != j}(x - x_m) * inv_denom_j,
// product taken in ascending m like numpy's prod over `_others[j]`.
template <int O>
__device__ __forceinline__ void lagrange_all(const DevBasis& b, double x, double* out) {
#pragma unroll
  for (int j = 0; j < O; ++j) {
    double prod = 1.0;
    bool first = true;
#pragma unroll
    for (int m = 0; m < O; ++m) {
      if (m == j) continue;
      double d = __dsub_rn(x, b.nodes[m]);
      prod = first ? d : __dmul_rn(prod, d);
      first = false;
    }
    out[j] = __dmul_rn(prod, b.inv_denoms[j]);
  }
}

// raw[j][k] = sum_q l_j(x_q) * (w_q * l_k(x_q + off)) over the 2p+2 Gauss rule
// mapped to [lo, hi]  (_interval_block, sldg1d.py:72-79)
template <int O>
__device__ __forceinline__ void interval_block(const DevBasis& b, double lo, double hi, double off,
                                               double* raw) {
  constexpr int NQ = 2 * O;
#pragma unroll
  for (int k = 0; k < O * O; ++k) raw[k] = 0.0;
  double half = 0.5 * (hi - lo);
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    double x = lo + half * (b.gq[q] + 1.0);
    double w = half * b.gw[q];
    double dv[O], sv[O];
    lagrange_all<O>(b, x, dv);
    lagrange_all<O>(b, x + off, sv);
#pragma unroll
    for (int j = 0; j < O; ++j)
#pragma unroll
      for (int k = 0; k < O; ++k) raw[j * O + k] = fma(dv[j], w * sv[k], raw[j * O + k]);
  }
}

// out = M^-1 raw
template <int O>
__device__ __forceinline__ void apply_minv(const DevBasis& b, const double* raw, double* out) {
#pragma unroll
  for (int i = 0; i < O; ++i)
#pragma unroll
    for (int k = 0; k < O; ++k) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < O; ++j) s = fma(b.minv[i * O + j], raw[j * O + k], s);
      out[i * O + k] = s;
    }
}

// overlap_pair (sldg1d.py:82-100): A acts on source cell i-n, B on i-n-1.
template <int O>
__device__ __forceinline__ void overlap_pair(const DevBasis& b, double a, double* A, double* B) {
  if (a == 0.0) {
#pragma unroll
    for (int i = 0; i < O; ++i)
#pragma unroll
      for (int k = 0; k < O; ++k) {
        A[i * O + k] = (i == k) ? 1.0 : 0.0;
        B[i * O + k] = 0.0;
      }
    return;
  }
  double raw[O * O];
  double split = 2.0 * a - 1.0;
  interval_block<O>(b, split, 1.0, -2.0 * a, raw);
  apply_minv<O>(b, raw, A);
  interval_block<O>(b, -1.0, split, 2.0 * (1.0 - a), raw);
  apply_minv<O>(b, raw, B);
}

// Python floor-mod for pencil/ring indices
__device__ __forceinline__ long long pymod(long long a, long long n) {
  long long r = a % n;
  return r < 0 ? r + n : r;
}

}  // namespace sldg
