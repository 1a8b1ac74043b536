// capi.cu -- error plumbing, basis upload and small utility entry points.
#include <atomic>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "sldg_common.cuh"

namespace sldg {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }

int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  return SLDG_ERR_CUDA;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

namespace {
std::mutex g_cfg_mu;
std::map<int, int> g_sms;                                  // dev -> SM count
std::map<std::pair<const void*, int>, int> g_smem_set;   // (k, dev) -> largest limit set
std::map<std::tuple<const void*, int, int, int>, int> g_resident;     // (k, dev, thr, smem)
int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
}  // namespace

cudaError_t smem_limit(const void* kernel, int bytes) {
  // the attribute is a per-function maximum: only ever raise it, so a smaller
  // request after a larger one cannot lower the limit under a cached larger key
  const auto key = std::make_pair(kernel, current_device());
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  auto it = g_smem_set.find(key);
  if (it != g_smem_set.end() && it->second >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) g_smem_set[key] = bytes;
  return e;
}

cudaError_t resident_ctas(const void* kernel, int threads, int smem, int* per_sm) {
  const int dev = current_device();
  const auto key = std::make_tuple(kernel, dev, threads, smem);
  {
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    auto it = g_resident.find(key);
    if (it != g_resident.end()) {
      *per_sm = it->second;
      return cudaSuccess;
    }
  }
  cudaError_t e = smem_limit(kernel, smem);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kernel, threads, (size_t)smem);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  g_resident[key] = *per_sm;
  return cudaSuccess;
}

int num_sms() {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  auto it = g_sms.find(dev);
  if (it != g_sms.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
    n = 148;
  g_sms[dev] = n;
  return n;
}

bool make_dev_basis(const SldgBasis& b, DevBasis* out, std::string* err) {
  if (b.degree < 1 || b.degree > SLDG_MAX_DEGREE) {
    *err = "degree " + std::to_string(b.degree) + " not compiled (1.." +
           std::to_string(SLDG_MAX_DEGREE) + ")";
    return false;
  }
  if (!b.nodes || !b.inv_denoms || !b.gauss_nodes || !b.gauss_weights || !b.mass_inv) {
    *err = "basis arrays must be non-null";
    return false;
  }
  DevBasis d{};
  d.p = b.degree;
  d.o = b.degree + 1;
  d.nq = 2 * b.degree + 2;
  for (int i = 0; i < d.o; ++i) {
    d.nodes[i] = b.nodes[i];
    d.inv_denoms[i] = b.inv_denoms[i];
  }
  for (int q = 0; q < d.nq; ++q) {
    d.gq[q] = b.gauss_nodes[q];
    d.gw[q] = b.gauss_weights[q];
  }
  for (int k = 0; k < d.o * d.o; ++k) d.minv[k] = b.mass_inv[k];
  *out = d;
  return true;
}

template <int O>
__global__ void k_overlap_pairs(DevBasis b, const double* __restrict__ fracs, long long n,
                                double* __restrict__ A, double* __restrict__ B) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a[O * O], bb[O * O];
  overlap_pair<O>(b, fracs[i], a, bb);
#pragma unroll
  for (int k = 0; k < O * O; ++k) {
    A[i * O * O + k] = a[k];
    B[i * O * O + k] = bb[k];
  }
}

// out[i, j] = a[i] * b[j]  (sample_initial, driver.py:132-136: gv[:, None] * gx[None, :])
__global__ void k_outer(const double* __restrict__ a, long long na, const double* __restrict__ b,
                        long long nb, double* __restrict__ out, long long ld) {
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= na * nb) return;
  long long i = idx / nb, j = idx - i * nb;
  out[i * ld + j] = a[i] * b[j];
}

}  // namespace sldg

using namespace sldg;

extern "C" {

const char* sldg_last_error(void) { return g_last_error.c_str(); }

int sldg_version(void) { return 10000; }

// bit 0: built with -DSLDG_FUZZ (schedule fuzzing, tests only)
int sldg_build_flags(void) {
#ifdef SLDG_FUZZ
  return 1;
#else
  return 0;
#endif
}

int64_t sldg_launch_count(void) { return (int64_t)g_launches.load(); }

int sldg_outer(const double* a, int64_t na, const double* b, int64_t nb, double* out, int64_t ld,
               void* stream) {
  if (!a || !b || !out || na < 0 || nb < 0 || ld < nb) {
    set_error("bad outer-product arguments");
    return SLDG_ERR_ARG;
  }
  long long n = na * nb;
  if (n == 0) return SLDG_OK;
  k_outer<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(a, na, b, nb, out, ld);
  SLDG_LAUNCH_CHECK("k_outer");
  return SLDG_OK;
}

int sldg_overlap_pairs(const SldgBasis* basis, const double* fracs, int64_t n, double* A,
                       double* B, void* stream) {
  DevBasis b;
  std::string err;
  if (!basis || !make_dev_basis(*basis, &b, &err)) {
    set_error(basis ? err : "null basis");
    return SLDG_ERR_ARG;
  }
  if (n <= 0) return SLDG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int threads = 128;
  int blocks = (int)((n + threads - 1) / threads);
  switch (b.o) {
#define CASE(O) \
  case O: k_overlap_pairs<O><<<blocks, threads, 0, s>>>(b, fracs, n, A, B); break;
    CASE(2) CASE(3) CASE(4) CASE(5) CASE(6)
#undef CASE
    default:
      set_error("unsupported degree");
      return SLDG_ERR_UNSUPPORTED;
  }
  SLDG_LAUNCH_CHECK("k_overlap_pairs");
  return SLDG_OK;
}

}  // extern "C"
