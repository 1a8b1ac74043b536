// tma_util.cuh -- mbarrier + cp.async.bulk (TMA engine, 1-D and 2-D tensor) helpers for
// sm_100a.
#pragma once

#include <cuda.h>   // CUtensorMap (the type only; encoded through the runtime's entry point)
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

namespace sldg {

// Schedule fuzzing (the race check that stands in for compute-sanitizer, which the GPU
// pool does not allow): built with -DSLDG_FUZZ (tools/fuzz_build.sh -> libsldg_fuzz.so),
// every bulk-copy issue, cp.async issue, mbarrier wait and pipeline barrier first sleeps a
// pseudo-random 0-2 us on ~1 in 4 calls, so producers and consumers of each shared buffer
// run far out of their usual order; tests/test_gpu_schedule_fuzz.py then requires
// bit-identical results.  Compiles to nothing otherwise.
__device__ __forceinline__ void fuzz_delay() {
#ifdef SLDG_FUZZ
  unsigned long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  unsigned x = (unsigned)c ^ (threadIdx.x * 2654435761u) ^ (blockIdx.x * 40503u) ^
               (unsigned)(c >> 32);
  x ^= x >> 13;
  x *= 0x5bd1e995u;
  x ^= x >> 15;
  if ((x & 3u) == 0u) __nanosleep((x >> 4) & 2047u);
#endif
}
// __syncthreads with a fuzzed arrival (a pipeline barrier)
__device__ __forceinline__ void sync_fz() {
  fuzz_delay();
  __syncthreads();
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  fuzz_delay();
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA-engine bulk copy global -> shared (16-byte aligned, size % 16 == 0),
// completion counted in transaction bytes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  fuzz_delay();
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// TMA tensor copy of one 2-D box (coordinates: inner column, row) global -> shared,
// completion counted in transaction bytes on `bar` (the full box: out-of-range
// elements are zero-filled and counted)
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            unsigned long long* bar) {
  fuzz_delay();
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// TMA-engine bulk copy shared -> global (bulk async-group), and its completion:
// wait_read = the shared source may be reused, wait_all = the writes are done
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* src, unsigned bytes) {
  fuzz_delay();
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all0() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
// generic-proxy shared-memory writes -> visible to the async proxy (a bulk store)
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
// programmatic dependent launch: wait for the preceding grid (no-op when the kernel
// was not launched with programmatic stream serialization) / let the next grid start
__device__ __forceinline__ void grid_dep_wait() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}
__device__ __forceinline__ void grid_dep_launch() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
// per-thread asynchronous global -> shared copies (LDGSTS), completed by cp_async_wait_all
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  fuzz_delay();
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  fuzz_delay();
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  fuzz_delay();
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}
// arrive on `bar` once this thread's earlier cp.async copies have landed (counts as
// one of the barrier's expected arrivals)
__device__ __forceinline__ void cp_async_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

// Host: encode a 2-D tensor map over a row-major fp64 matrix (rows x ld doubles, the
// first `inner` columns addressed; columns past `inner` read as zeros), box
// box_rows x box_cols, no swizzle.  cuTensorMapEncodeTiled comes from the driver via
// the runtime's entry-point query, so nothing links against libcuda.  False when the
// driver or the geometry (16-byte aligned base and row pitch, box <= 256) refuses.
inline bool encode_tmap_2d(CUtensorMap* map, const double* base, long long inner,
                           long long rows, long long ld, int box_cols, int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000,
                                         cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }();
  if (!encode || ((unsigned long long)base & 15) || (ld * 8) % 16 || box_cols > 256 ||
      box_rows > 256 || rows >= (1ll << 31) || inner >= (1ll << 31) || (box_cols * 8) % 16)
    return false;
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace sldg
