// halo.cu -- upwind-only x-halo pack / unpack for the x-slab sharded state
// (the paper's ghost exchange, without host staging).
//
// The x shift of a row (xfield.py:63-88 with the split of sldg1d.py:39-55) reads the
// source cells c - n and c - n - 1 of each output cell c, so a slab only needs cells
// on ONE side per row: n >= 0 reads n + 1 cells left of the slab (n_apply = 2: the
// trailing and the next leading half step in one pass, 2n + 2), n < 0 reads |n| cells
// right of it (2|n|); identity rows (n = 0, alpha = 0) read nothing.  Per row the widths
// are fixed by the row's speed, so every rank packs the same layout: a CSR over rows
// of the doubles each row sends right (its last w_l cells, the right neighbour's left
// halo) and left (its first w_r cells).  The exchange itself is the caller's (NCCL
// send/recv of the packed buffers); these kernels only gather and scatter, a few
// lanes per row.
#include <algorithm>
#include <vector>

#include "plans.cuh"

struct sldg_halo {
  int o;
  long long n_local, n_rows, n_speeds;
  int reach_l, reach_r;                 // widest left / right halo in cells
  int* wl;                              // device: per speed, left-halo cells
  int* wr;                              // device: per speed, right-halo cells
  long long* off_r;                     // device: per row + 1, doubles sent right
  long long* off_l;                     // device: per row + 1, doubles sent left
  const int* row_speed;                 // the plan's (device)
  std::vector<long long> h_off_r, h_off_l;
  void* block;
};

namespace sldg {

// rows [r0, r1): a group of L lanes (a power of two <= 32) per row copies its w cells
// (w*o doubles, contiguous in both places).  L follows the widest row (halo_launch):
// rows of a few cells (config 4L: <= 24 doubles) leave most of a warp idle behind the
// row's dependent table loads (row speed -> widths -> CSR offsets), so several rows share
// a warp; wide rows (config 5: up to 78 doubles) keep a warp each.
template <bool PACK>
__global__ void k_halo_copy(const int* __restrict__ row_speed, const int* __restrict__ wl,
                            const int* __restrict__ wr, const long long* __restrict__ off_r,
                            const long long* __restrict__ off_l, int o, long long n_local,
                            double* __restrict__ buf, long long ld, long long lw, long long r0,
                            long long r1, double* __restrict__ right, double* __restrict__ left,
                            int lanes) {
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  const int lane = (int)(t0 & (lanes - 1));
  const long long base_r = __ldg(off_r + r0), base_l = __ldg(off_l + r0);
  for (long long r = r0 + t0 / lanes; r < r1; r += nt / lanes) {
  const int g = __ldg(row_speed + r);
  double* row = buf + r * ld;
  const int nl = __ldg(wl + g) * o, nr = __ldg(wr + g) * o;
  // left-reaching row: my last nl doubles -> right neighbour; its data -> my left margin
  if (nl) {
    double* pr = right + (__ldg(off_r + r) - base_r);
    for (int k = lane; k < nl; k += lanes) {
      if (PACK)
        pr[k] = row[lw + n_local * o - nl + k];
      else
        row[lw - nl + k] = pr[k];
    }
  }
  // right-reaching row: my first nr doubles -> left neighbour; its data -> right margin
  if (nr) {
    double* pl = left + (__ldg(off_l + r) - base_l);
    for (int k = lane; k < nr; k += lanes) {
      if (PACK)
        pl[k] = row[lw + k];
      else
        row[lw + n_local * o + k] = pl[k];
    }
  }
  }
}

// out[i] = (((parts[0][i] + parts[1][i]) + parts[2][i]) + ...): a cross-rank sum in rank
// order, identical on every rank (never an unordered all-reduce)
__global__ void k_sum_parts(const double* __restrict__ parts, long long n_parts, long long n,
                            double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double s = parts[i];
    for (long long k = 1; k < n_parts; ++k) s += parts[k * n + i];
    out[i] = s;
  }
}

__global__ void k_gather_index(const double* __restrict__ src, const long long* __restrict__ idx,
                               long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = src[idx[i]];
}

}  // namespace sldg

using namespace sldg;

extern "C" {

int sldg_halo_create(const sldg_xplan* X, int64_t n_local, int32_t n_apply, sldg_halo** out) {
  if (!X || !out || n_local < 1 || (n_apply != 1 && n_apply != 2)) {
    set_error("bad sldg_halo_create arguments");
    return SLDG_ERR_ARG;
  }
  *out = nullptr;
  const long long S = X->n_speeds, R = X->n_rows;
  std::vector<long long> ns(std::max<long long>(S, 1));
  std::vector<unsigned char> id(std::max<long long>(S, 1));
  std::vector<int> rs(std::max<long long>(R, 1));
  cudaError_t ce = cudaSuccess;
  if (S > 0) {
    ce = cudaMemcpy(ns.data(), X->dev.ns, sizeof(long long) * S, cudaMemcpyDeviceToHost);
    if (ce == cudaSuccess)
      ce = cudaMemcpy(id.data(), X->dev.ident, S, cudaMemcpyDeviceToHost);
  }
  if (ce == cudaSuccess && R > 0)
    ce = cudaMemcpy(rs.data(), X->dev.row_speed, sizeof(int) * R, cudaMemcpyDeviceToHost);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaMemcpy(halo plan)");
  std::vector<int> wl(std::max<long long>(S, 1), 0), wr(std::max<long long>(S, 1), 0);
  int reach_l = 0, reach_r = 0;
  for (long long g = 0; g < S; ++g) {
    if (id[g]) continue;
    if (ns[g] >= 0)
      wl[g] = (int)(n_apply * (ns[g] + 1));
    else
      wr[g] = (int)(n_apply * -ns[g]);
    reach_l = std::max(reach_l, wl[g]);
    reach_r = std::max(reach_r, wr[g]);
  }
  if (reach_l > n_local || reach_r > n_local) {
    set_error("x halo wider than the slab: use fewer ranks");
    return SLDG_ERR_UNSUPPORTED;
  }
  sldg_halo* h = new sldg_halo();
  h->o = X->o;
  h->n_local = n_local;
  h->n_rows = R;
  h->n_speeds = S;
  h->reach_l = reach_l;
  h->reach_r = reach_r;
  h->row_speed = X->dev.row_speed;
  h->h_off_r.assign(R + 1, 0);
  h->h_off_l.assign(R + 1, 0);
  for (long long r = 0; r < R; ++r) {
    h->h_off_r[r + 1] = h->h_off_r[r] + (long long)wl[rs[r]] * X->o;
    h->h_off_l[r + 1] = h->h_off_l[r] + (long long)wr[rs[r]] * X->o;
  }
  const size_t sw = sizeof(int) * std::max<long long>(S, 1), so = sizeof(long long) * (R + 1);
  const size_t a0 = 0, a1 = (sw + 255) / 256 * 256, a2 = a1 + a1, a3 = a2 + (so + 255) / 256 * 256;
  ce = cudaMalloc(&h->block, a3 + so);
  if (ce != cudaSuccess) {
    delete h;
    return cuda_fail(ce, "cudaMalloc(halo plan)");
  }
  unsigned char* b = (unsigned char*)h->block;
  h->wl = (int*)(b + a0);
  h->wr = (int*)(b + a1);
  h->off_r = (long long*)(b + a2);
  h->off_l = (long long*)(b + a3);
  ce = cudaMemcpy(h->wl, wl.data(), sw, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess) ce = cudaMemcpy(h->wr, wr.data(), sw, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess) ce = cudaMemcpy(h->off_r, h->h_off_r.data(), so, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess) ce = cudaMemcpy(h->off_l, h->h_off_l.data(), so, cudaMemcpyHostToDevice);
  if (ce != cudaSuccess) {
    cudaFree(h->block);
    delete h;
    return cuda_fail(ce, "cudaMemcpy(halo plan)");
  }
  *out = h;
  return SLDG_OK;
}

int sldg_halo_destroy(sldg_halo* h) {
  if (!h) return SLDG_OK;
  cudaFree(h->block);
  delete h;
  return SLDG_OK;
}

static bool bad_rows(const sldg_halo* h, int64_t r0, int64_t r1) {
  return !h || r0 < 0 || r1 < r0 || r1 > h->n_rows;
}

int sldg_halo_extent(const sldg_halo* h, int64_t r0, int64_t r1, int64_t* out4) {
  if (bad_rows(h, r0, r1) || !out4) {
    set_error("bad sldg_halo_extent arguments");
    return SLDG_ERR_ARG;
  }
  out4[0] = h->h_off_r[r0];
  out4[1] = h->h_off_r[r1] - h->h_off_r[r0];
  out4[2] = h->h_off_l[r0];
  out4[3] = h->h_off_l[r1] - h->h_off_l[r0];
  return SLDG_OK;
}

int sldg_halo_reach(const sldg_halo* h, int64_t* out2) {
  if (!h || !out2) {
    set_error("null argument");
    return SLDG_ERR_ARG;
  }
  out2[0] = h->reach_l;
  out2[1] = h->reach_r;
  return SLDG_OK;
}

static int halo_launch(bool pack, const sldg_halo* h, double* buf, int64_t ld, int64_t lw,
                       int64_t r0, int64_t r1, double* right, double* left, void* stream) {
  if (bad_rows(h, r0, r1) || !buf || lw < h->reach_l * h->o ||
      ld < lw + (h->n_local + h->reach_r) * h->o ||
      ((h->h_off_r[r1] > h->h_off_r[r0]) && !right) ||
      ((h->h_off_l[r1] > h->h_off_l[r0]) && !left)) {
    set_error("bad halo pack/unpack arguments (margins narrower than the reach?)");
    return SLDG_ERR_ARG;
  }
  if (r1 == r0) return SLDG_OK;
  // lanes per row: about 4 doubles per lane of the widest row, a power of two <= 32
  const int widest = std::max(h->reach_l, h->reach_r) * h->o;
  int lanes = 1;
  while (lanes < 32 && lanes * 4 < widest) lanes *= 2;
  const long long threads = std::min<long long>((r1 - r0) * lanes, 148LL * 64 * 32);
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  cudaStream_t st = (cudaStream_t)stream;
  if (pack)
    k_halo_copy<true><<<blocks, 256, 0, st>>>(h->row_speed, h->wl, h->wr, h->off_r, h->off_l,
                                              h->o, h->n_local, buf, ld, lw, r0, r1, right, left,
                                              lanes);
  else
    k_halo_copy<false><<<blocks, 256, 0, st>>>(h->row_speed, h->wl, h->wr, h->off_r, h->off_l,
                                               h->o, h->n_local, buf, ld, lw, r0, r1, right, left,
                                               lanes);
  SLDG_LAUNCH_CHECK(pack ? "k_halo_pack" : "k_halo_unpack");
  return SLDG_OK;
}

int sldg_halo_pack(const sldg_halo* h, const double* buf, int64_t ld, int64_t lw, int64_t r0,
                   int64_t r1, double* to_right, double* to_left, void* stream) {
  return halo_launch(true, h, const_cast<double*>(buf), ld, lw, r0, r1, to_right, to_left,
                     stream);
}

int sldg_halo_unpack(const sldg_halo* h, double* buf, int64_t ld, int64_t lw, int64_t r0,
                     int64_t r1, const double* from_left, const double* from_right, void* stream) {
  return halo_launch(false, h, buf, ld, lw, r0, r1, const_cast<double*>(from_left),
                     const_cast<double*>(from_right), stream);
}

int sldg_sum_parts(const double* parts, int64_t n_parts, int64_t n, double* out, void* stream) {
  if (!parts || !out || n_parts < 1 || n < 0) {
    set_error("bad sldg_sum_parts arguments");
    return SLDG_ERR_ARG;
  }
  if (n == 0) return SLDG_OK;
  const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 148LL * 8);
  k_sum_parts<<<blocks, 256, 0, (cudaStream_t)stream>>>(parts, n_parts, n, out);
  SLDG_LAUNCH_CHECK("k_sum_parts");
  return SLDG_OK;
}

int sldg_gather_index(const double* src, const int64_t* idx, int64_t n, double* out,
                      void* stream) {
  if (!src || !idx || !out || n < 0) {
    set_error("bad sldg_gather_index arguments");
    return SLDG_ERR_ARG;
  }
  if (n == 0) return SLDG_OK;
  const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 148LL * 8);
  k_gather_index<<<blocks, 256, 0, (cudaStream_t)stream>>>(src, (const long long*)idx, n, out);
  SLDG_LAUNCH_CHECK("k_gather_index");
  return SLDG_OK;
}

}  // extern "C"
