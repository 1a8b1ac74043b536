// plans.cuh -- device plan structs and small device helpers shared by the
// translation units (vsweep.cu, xfield.cu, step_fused.cu).
#pragma once

#include "sldg_common.cuh"

namespace sldg {

struct VPlanDev {
  const long long* p_off;     // pencil -> first entry
  const int* p_n;             // pencil -> n cells
  const unsigned char* p_fast;// whole-pencil fast flag
  const int* e_pencil;        // entry -> pencil
  const long long* e_row0;    // entry -> cell_id * n_local
  const double* e_lower;
  const double* e_width;
  const int* e_level;
  const unsigned char* e_conf;
  const int* e_runs;          // 4 per entry: circular left/right, linear left/right
  const int* e_slot;          // -1 = direct store, else scratch slot
  const long long* t_row0;    // target -> first row
  const long long* t_off;     // target -> first contribution
  const int* c_slot;
  const int* c_group;
  const double* c_weight;
  const long long* walk_pencils;  // whole-fast pencils, for k_sweep_walk
  const long long* walk_desc;     // per walk position: {p_off, p_n | level << 32}
  const long long* gen_entries;   // entries of the per-cell worklist when walk is used
  // duplicate pencils (identical cell lists, whole-fast, every cell in exactly those
  // pencils): the walk sweeps one representative and writes the weighted average of the
  // identical results directly (the write-back formula, no scratch slots)
  const int* e_dd;                // entry -> dedup weight list (-1: none)
  const long long* dd_off;        // dedup list -> first weight
  const double* dd_w;             // weights of the duplicates, plan order
  const long long* walk_dd;       // the walk without the skipped duplicates
  const long long* t_dd;          // targets the write-back still owns in dedup mode
  const long long* walk_dd_desc;  // per walk_dd position: {p_off, p_n | level << 32}
  // cells whose rows the walk does not write directly (per-cell worklist cells and the
  // write-back targets of dedup mode), ascending: the one-pass AMR step
  // (amr_fused.cuh) finishes them with a cell-list x pass
  const long long* rest_cells;
  long long n_entries, n_targets, n_walk, n_gen, n_walk_dd, n_targets_dd;
  int stride_d, stride_t0, stride_t1;
  int n_levels;
  double radius, base_width;
};

}  // namespace sldg

struct sldg_vplan {
  sldg::DevBasis basis;
  sldg::VPlanDev dev;
  int dim, direction, o, n_lines, n_local;
  long long n_cells, n_pencils, n_entries, n_slots, n_targets, n_walk, n_gen, n_dofs;
  long long n_dd_sets, n_walk_dd, n_targets_dd, n_rest;
  int max_pencil_cells, max_walk_cells;
  void* block;
};

namespace sldg {

struct XPlanDev {
  const long long* ns;     // per unique speed: integer shift
  const unsigned char* ident;  // per unique speed: n == 0 && alpha == 0
  const double* mats;      // per unique speed: A (o*o) then B (o*o)
  const int* row_speed;    // per row
  const int* nsm;          // per unique speed: n_shift mod n_cells (periodic rows)
};

}  // namespace sldg

struct sldg_xplan {
  sldg::DevBasis basis;
  sldg::XPlanDev dev;
  int o;
  long long n_cells, n_rows, n_speeds;
  long long halo_l, halo_r;
  int vo;          // velocity nodes per direction when rows are cells x o^3 with a
                   // per-(cell, v_x node) speed (sldg_xplan_set_vlayout); 0 = unknown
  double h, dt;
  void* block;
};

struct sldg_poisson {
  int p, o;
  long long n_cells, n_nodes, n_dofs;
  double h, length;
  double* xw;      // dof weights
  double* diff;    // o*o
  double* green;   // n_nodes^2
  double* work;    // b (n_nodes) + scalars
  void* block;
};

namespace sldg {

template <int O>
__device__ __forceinline__ void load_pair(const double* __restrict__ lm_mats, int lev,
                                          long long n_cols, long long c, double* A, double* B) {
#pragma unroll
  for (int k = 0; k < O * O; ++k) {
    A[k] = __ldg(lm_mats + ((long long)(lev * 2 + 0) * O * O + k) * n_cols + c);
    B[k] = __ldg(lm_mats + ((long long)(lev * 2 + 1) * O * O + k) * n_cols + c);
  }
}

// _fast_sources_ok (vsweep.py:125-146) in O(1) from precomputed same-level runs
__device__ __forceinline__ bool sources_ok(const int* runs, int s, long long ns, int n, int bc) {
  long long lo = min((long long)s, s - ns - 1);
  long long hi = max((long long)s, s - ns);
  if (bc == SLDG_BC_PERIODIC) {
    if (hi - lo + 1 >= n) return runs[0] >= n;   // whole pencil one level
    return (s - lo) <= runs[0] && (hi - s) <= runs[1];
  }
  long long i0 = max(lo, 0LL), i1 = min(hi, (long long)n - 1);
  return (s - i0) <= runs[2] && (i1 - s) <= runs[3];
}

template <int O, int DIM>
struct Lines {
  static constexpr int NL = (DIM == 3) ? O * O : 1;
  static constexpr int NLOC = NL * O;
  __device__ __forceinline__ static int row(const VPlanDev& P, int t, int i) {
    if (DIM == 1) return i;
    return (t % O) * P.stride_t0 + (t / O) * P.stride_t1 + i * P.stride_d;
  }
};

// out (O values) = A ua + B ub  (apply_update, sldg1d.py:124-136: src_same@A.T + src_nb@B.T)
template <int O>
__device__ __forceinline__ void two_cell(const double* A, const double* B, const double* ua,
                                         const double* ub, bool va, bool vb, double* y) {
#pragma unroll
  for (int i = 0; i < O; ++i) {
    double sa = 0.0, sb = 0.0;
    if (va) {
      sa = A[i * O] * ua[0];
#pragma unroll
      for (int j = 1; j < O; ++j) sa = fma(A[i * O + j], ua[j], sa);
    }
    if (vb) {
      sb = B[i * O] * ub[0];
#pragma unroll
      for (int j = 1; j < O; ++j) sb = fma(B[i * O + j], ub[j], sb);
    }
    y[i] = sa + sb;
  }
}

}  // namespace sldg
