/*
 * sldg_capi.h -- C ABI of the B200-native SLDG transport step (libsldg.so).
 *
 * Plain pointers and sizes only; no torch types.  Every entry point returns
 * an int status (SLDG_OK == 0); on failure sldg_last_error() returns a
 * thread-local message.  Device pointers are caller-owned (fp64, row-major,
 * row = one velocity DOF, x fastest, leading dimension `ld` in elements).
 * Per-step entry points never allocate, never synchronise the host and
 * enqueue on the given stream (a cudaStream_t passed as void*; NULL = legacy
 * default stream).  Plans own their device memory.
 *
 * Reference interfaces replaced (all /root/reference/pkg/src/sldg_vlasov/):
 *   sldg_vplan_create       <- vsweep.build_sweep_plan          vsweep.py:307-387
 *                              (+ pencil.extract_pencils/classify_conforming arrays,
 *                               pencil.py:60-168, uploaded once)
 *   sldg_advect_v           <- vsweep.advect_velocity            vsweep.py:413-441
 *                              (_sweep_column 390-410, sweep_pencil 173-246,
 *                               weighted_writeback 249-272, precompute_level_matrices 47-61)
 *   sldg_level_matrices     <- vsweep.precompute_level_matrices  vsweep.py:47-61
 *                              (decompose_shift sldg1d.py:39-55, overlap_pair sldg1d.py:82-100)
 *   sldg_xplan_create       <- xfield.precompute_x_matrices      xfield.py:63-79
 *   sldg_advect_x           <- xfield.advect_x                   xfield.py:82-104
 *   sldg_rho                <- xfield.compute_rho                xfield.py:107-109
 *   sldg_poisson_create     <- xfield.PoissonSolver.__init__     xfield.py:121-146
 *   sldg_poisson_solve      <- PoissonSolver.solve + electric_field  xfield.py:148-179
 *   sldg_moments            <- driver.moments                    driver.py:139-146
 *   sldg_field_diag         <- xfield.field_energy + max|E|      xfield.py:192-195, driver.py:220-229
 */
#ifndef SLDG_CAPI_H
#define SLDG_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLDG_OK 0
#define SLDG_ERR_ARG 1      /* bad argument / shape (SweepError / ValueError in Python) */
#define SLDG_ERR_CUDA 2     /* CUDA runtime failure */
#define SLDG_ERR_PLAN 3     /* inconsistent plan (uncovered DOFs, bad CSR) */
#define SLDG_ERR_UNSUPPORTED 4

#define SLDG_BC_PERIODIC 0
#define SLDG_BC_ABSORBING 1

#define SLDG_MAX_DEGREE 5   /* p <= 5 (o = p+1 <= 6) compiled */

/* Reference element constants (basis.DGBasis, basis.py:84-148). */
typedef struct SldgBasis {
  int32_t degree;             /* p */
  const double* nodes;        /* p+1 GLL nodes */
  const double* inv_denoms;   /* p+1 Lagrange denominators^-1 (basis.py:101-106) */
  const double* gauss_nodes;  /* 2p+2 */
  const double* gauss_weights;/* 2p+2 */
  const double* mass_inv;     /* (p+1)^2 row-major */
} SldgBasis;

/* ---------------------------------------------------------------- v-sweep */
typedef struct sldg_vplan sldg_vplan;

typedef struct SldgVPlanDesc {
  SldgBasis basis;
  int32_t dim;                /* 1 or 3 */
  int32_t direction;          /* sweep axis, < dim */
  int32_t n_levels;           /* max level + 1 */
  double radius;              /* domain half width R */
  double base_width;          /* 2R / n_base (VelocityMesh.base_width) */
  int64_t n_cells;            /* mesh cells; n_dofs = n_cells*(p+1)^dim */
  int64_t n_pencils;          /* pencils in PLAN ORDER: groups in plan order, pencils of a group in order */
  const int64_t* pencil_offsets;  /* n_pencils+1 CSR offsets into the entry arrays */
  const int64_t* pencil_group;    /* n_pencils: group index (write-back summation order) */
  const int64_t* cell_ids;        /* entries */
  const double* lowers;           /* entries: sweep-axis lower coordinate */
  const double* widths;           /* entries: sweep-axis width */
  const int64_t* levels;          /* entries */
  const uint8_t* conforming;      /* entries: +-2 same-level flag (classify_conforming) */
  const double* weights;          /* entries: 1/n_c */
} SldgVPlanDesc;

int sldg_vplan_create(const SldgVPlanDesc* desc, sldg_vplan** out);
int sldg_vplan_destroy(sldg_vplan* plan);
/* bytes of device scratch sldg_advect_v needs for n_cols columns */
int sldg_vplan_scratch_bytes(const sldg_vplan* plan, int64_t n_cols, size_t* bytes);
/* plan statistics: [n_entries, n_acc_slots, n_targets, n_whole_fast_pencils, n_dofs] */
int sldg_vplan_info(const sldg_vplan* plan, int64_t* info5);

/* f_out[:, c] = sweep(f_in[:, c], speeds[c]) for every column; columns with
 * speeds[c] == 0.0 are copied bit for bit.  f_in and f_out must not alias.
 * `scratch` is sldg_vplan_scratch_bytes() bytes of device memory. */
int sldg_advect_v(const sldg_vplan* plan, const double* f_in, double* f_out, int64_t ld,
                  int64_t n_cols, const double* speeds, double dt, int32_t bc,
                  int32_t force_slow, void* scratch, void* stream);

/* Per-column level matrices (debug / API mirror of precompute_level_matrices):
 * n_shift[l*n_cols+c], frac[l*n_cols+c], mats[((l*2+ab)*o*o + k)*n_cols + c]. */
int sldg_level_matrices(const sldg_vplan* plan, const double* speeds, int64_t n_cols, double dt,
                        int64_t* n_shift, double* frac, double* mats, void* stream);

/* Overlap pair for arbitrary fractional shifts (overlap_pair, sldg1d.py:82-100):
 * fracs[n] device -> A[n*o*o], B[n*o*o] device (row-major per pair). */
int sldg_overlap_pairs(const SldgBasis* basis, const double* fracs, int64_t n, double* A,
                       double* B, void* stream);

/* Pure pencil-level functions of the reference (all device pointers):
 * apply_update (sldg1d.py:124-136): values/out (n_batch, n_cells, o) row-major,
 *   out_i = A v_{i-n_shift} + B v_{i-n_shift-1} (periodic wrap / absorbing zero fill);
 * projection_oracle (sldg1d.py:139-178): brute-force projection of the translated
 *   piecewise polynomial, Gauss rule gq/gw (nq points, e.g. 50) on every overlap;
 * generalized_overlap (vsweep.py:98-122): o x o block M^-1 (2/w_d) int_vl^vr l_i l_j
 *   for the overlap [vl, vr] (vl < vr) of a foot with a source cell;
 * weighted_writeback (vsweep.py:249-272): flat contributions grouped per element in
 *   increasing flat order (csr_off[n+1], csr_idx): copies (w == 1) in order, then
 *   out += sum of w (v - f_in), as numpy's assignment + bincount. */
int sldg_apply_update(const double* values, int64_t n_batch, int64_t n_cells, int32_t o,
                      int64_t n_shift, const double* A, const double* B, int32_t bc, double* out,
                      void* stream);
int sldg_projection_oracle(const SldgBasis* basis, const double* values, int64_t n_cells,
                           double displacement, double width, int32_t bc, const double* gq,
                           const double* gw, int32_t nq, double* out, void* stream);
int sldg_generalized_overlap(const SldgBasis* basis, double vl, double vr, double dest_lo,
                             double dest_width, double src_lo, double src_width,
                             double displacement, double* matrix, void* stream);
int sldg_weighted_writeback(const double* f_in, int64_t n, const int64_t* csr_off,
                            const int64_t* csr_idx, const double* weights, const double* values,
                            double* out, void* stream);

/* ---------------------------------------------------------------- x side */
typedef struct sldg_xplan sldg_xplan;

/* One steady-state AMR Strang step body in one HBM pass (csrc/amr_fused.cuh):
 * f_out = X(X(V(f_in))) -- the v-sweep (as sldg_advect_v with speeds = E) followed by
 * the trailing half x-step of this step and the leading half x-step of the next --
 * with mom_out3 = [m0, m1, m2] of the state after the first x half step and
 * rho_out[n_cols] = rho of f_out.  Replaces the sldg_advect_v + sldg_advect_x_fused
 * (n_apply 2) pair of Simulation.advance (the reference's vsweep.py:413-441 then
 * xfield.py:91-104 twice, driver.py:220-240).  Velocity cells the whole-fast walk
 * does not write directly get the separate kernels.  Query: SLDG_OK and the scratch
 * size when the plans qualify (3V, direction 0, the x plan's velocity layout,
 * sldg_xplan_set_vlayout), SLDG_ERR_UNSUPPORTED otherwise. */
int sldg_amr_step_query(const sldg_vplan* vplan, const sldg_xplan* xplan, int64_t n_cols,
                        int64_t ld, size_t* scratch_bytes);
int sldg_amr_step(const sldg_vplan* vplan, const sldg_xplan* xplan, const double* f_in,
                  double* f_out, int64_t ld, int64_t n_cols, const double* speeds, double dt,
                  int32_t bc, const double* w, const double* v0, const double* v2,
                  const double* xw, double* mom_out3, double* rho_out, void* scratch,
                  void* stream);


typedef struct SldgXPlanDesc {
  SldgBasis basis;            /* degree_x basis */
  int64_t n_cells;            /* global x cells (periodic) */
  double h;                   /* x cell width */
  double dt;                  /* shift time (dt/2 for a Strang half step) */
  int64_t n_rows;             /* velocity DOFs */
  int64_t n_speeds;           /* unique speeds (np.unique order) */
  const double* speeds;       /* n_speeds unique speeds (host) */
  const int32_t* row_speed;   /* n_rows: index into speeds (host) */
} SldgXPlanDesc;

int sldg_xplan_create(const SldgXPlanDesc* desc, sldg_xplan** out);
int sldg_xplan_destroy(sldg_xplan* plan);
/* Declare the velocity layout of the rows: n_rows = cells x o_v^3 and every row
 * b = i + o_v j + o_v^2 k of a cell has the speed of its v_x node i (true for the
 * driver's v_x speeds).  Verified on the host; enables the same-speed row-tile x
 * kernel (csrc/xx_tiles.cuh). */
int sldg_xplan_set_vlayout(sldg_xplan* plan, int32_t o_v);
/* max |n_shift| and max n_shift+1 over rows: halo cells needed [left, right] */
int sldg_xplan_halo(const sldg_xplan* plan, int64_t* left_right);

/* Periodic full-row update of rows [0, n_rows): f_out = X(f_in); rows with a
 * zero shift are copied bit for bit.  f_in/f_out must not alias. */
int sldg_advect_x(const sldg_xplan* plan, const double* f_in, double* f_out, int64_t ld,
                  void* stream);

/* Fused pass (csrc/xfield.cu k_xadv): f_out = X^n_apply (f_in), n_apply in {1, 2}
 * (2 = trailing half step of step n + leading half step of step n+1, bit-identical
 * to two sldg_advect_x calls).  If mom_out3 != NULL: (m0, m1, m2) of the state
 * after the FIRST application (needs w, v0, v2, xw); if rho_out != NULL: rho of the
 * final output (needs w).  scratch: sldg_xadv_scratch_bytes(). */
int sldg_xadv_scratch_bytes(const sldg_xplan* plan, size_t* bytes);
int sldg_advect_x_fused(const sldg_xplan* plan, const double* f_in, double* f_out, int64_t ld,
                        int32_t n_apply, const double* w, const double* v0, const double* v2,
                        const double* xw, double* mom_out3, double* rho_out, void* scratch,
                        void* stream);

/* Sharded update: f_in holds, per row, halo_l + n_local + halo_r cells starting
 * at global cell (cell0 - halo_l) (ld_in elements per row); f_out gets n_local
 * cells (ld_out).  Requires halo_l/halo_r >= sldg_xplan_halo(). */
int sldg_advect_x_slab(const sldg_xplan* plan, const double* f_in, int64_t ld_in,
                       int64_t halo_l, int64_t halo_r, int64_t n_local, double* f_out,
                       int64_t ld_out, void* stream);
/* The same slab update with the row-tile kernel (plans with a velocity layout,
 * sldg_xplan_set_vlayout) and the fused epilogues of sldg_advect_x_fused: the rows
 * of row_base (16-byte aligned, ld_in even) are staged whole; halo-relative cell 0
 * starts at double src_off, local cells at halo_l..; outputs go to out_off of rows
 * of f_out (ld_out).  rho_out: n_local*o columns; mom_out3 with xw_local (the local
 * x weights).  scratch: sldg_advect_x_slab_tiles_scratch bytes (NULL without
 * epilogues); SLDG_ERR_UNSUPPORTED when the plan or shape does not fit the kernel. */
int sldg_advect_x_slab_tiles_scratch(const sldg_xplan* plan, int64_t n_local, int64_t ld_in,
                                     size_t* bytes);
int sldg_advect_x_slab_tiles(const sldg_xplan* plan, const double* row_base, int64_t ld_in,
                             int64_t src_off, int64_t halo_l, int64_t halo_r, int64_t n_local,
                             double* f_out, int64_t ld_out, int64_t out_off, int32_t n_apply,
                             int64_t row_begin, int64_t row_count, int32_t accumulate,
                             const double* w, const double* v0, const double* v2,
                             const double* xw_local, double* mom_out3, double* rho_out,
                             void* scratch, void* stream);
/*   n_apply 2: trailing + leading half steps in one pass (halo_l, halo_r at least twice
 *   the plan's reach; the intermediate's moments over the local cells).  Rows
 *   [row_begin, row_begin + row_count) (whole velocity cells) only; accumulate != 0 adds
 *   this range's rho and moments onto rho_out / mom_out3 (row chunks of one pass, summed
 *   in call order on one stream). */

/* ---- x-slab halo exchange (upwind-only, per row) --------------------------------
 * A row with x shift n >= 0 reads n_apply*(n+1) cells left of its slab, a row with n < 0
 * n_apply*|n| cells right of it (identity rows none).  sldg_halo_pack gathers, for rows
 * [row_begin, row_end), the cells the right neighbour needs (this slab's last cells of
 * the left-reaching rows) into to_right and the cells the left neighbour needs into
 * to_left; sldg_halo_unpack writes the neighbours' data into this slab's margins.  Every
 * rank has the same rows and speeds, so the packed layouts match across ranks.
 * Buffers: [left margin lw | n_local*o local | right margin] per row, stride ld. */
typedef struct sldg_halo sldg_halo;
int sldg_halo_create(const sldg_xplan* plan, int64_t n_local, int32_t n_apply, sldg_halo** out);
int sldg_halo_destroy(sldg_halo* h);
/* out4 = {offset, count} of the to_right / from_left data, then of to_left / from_right,
 * in doubles, for rows [row_begin, row_end). */
int sldg_halo_extent(const sldg_halo* h, int64_t row_begin, int64_t row_end, int64_t* out4);
/* out2 = widest left / right halo in cells */
int sldg_halo_reach(const sldg_halo* h, int64_t* out2);
int sldg_halo_pack(const sldg_halo* h, const double* buf, int64_t ld, int64_t lw,
                   int64_t row_begin, int64_t row_end, double* to_right, double* to_left,
                   void* stream);
int sldg_halo_unpack(const sldg_halo* h, double* buf, int64_t ld, int64_t lw,
                     int64_t row_begin, int64_t row_end, const double* from_left,
                     const double* from_right, void* stream);
/* out[i] = parts[0][i] + parts[1][i] + ... in part (rank) order; parts is n_parts x n. */
int sldg_sum_parts(const double* parts, int64_t n_parts, int64_t n, double* out, void* stream);
/* out[i] = src[idx[i]] (compacts an all-gathered, padded rank-major buffer). */
int sldg_gather_index(const double* src, const int64_t* idx, int64_t n, double* out,
                      void* stream);

/* rho[c] = sum_r w[r] f[r, c]  (deterministic two-stage column reduction).
 * scratch: sldg_rho_scratch_bytes(). */
int sldg_rho_scratch_bytes(int64_t n_rows, int64_t n_cols, size_t* bytes);
int sldg_rho(const double* f, int64_t ld, int64_t n_rows, int64_t n_cols, const double* w,
             double* rho, void* scratch, void* stream);

/* (m0, m1, m2) = sum_r w_r {1, v0_r, v2_r} (sum_c f[r,c] xw[c])  -> out3 (device). */
int sldg_moments_scratch_bytes(int64_t n_rows, size_t* bytes);
int sldg_moments(const double* f, int64_t ld, int64_t n_rows, int64_t n_cols, const double* w,
                 const double* v0, const double* v2, const double* xw, double* out3,
                 void* scratch, void* stream);

/* ---------------------------------------------------------------- Poisson */
typedef struct sldg_poisson sldg_poisson;

typedef struct SldgPoissonDesc {
  int32_t degree;             /* p_x */
  int64_t n_cells;            /* x cells */
  double h, length;
  const double* dof_weights;  /* n_cells*(p+1) GLL quadrature weights */
  const double* diff;         /* (p+1)^2 differentiation matrix */
  const double* green;        /* n_nodes^2: (augmented matrix)^-1 leading block, row-major */
} SldgPoissonDesc;

int sldg_poisson_create(const SldgPoissonDesc* desc, sldg_poisson** out);
int sldg_poisson_destroy(sldg_poisson* p);
/* rho (n_cells*(p+1)) -> phi (n_nodes; NULL = internal) and E (n_cells*(p+1); NULL = skip). */
int sldg_poisson_solve(const sldg_poisson* p, const double* rho, double* phi, double* e,
                       void* stream);
/* E = -phi' at the DG nodes from a nodal FE potential (electric_field, xfield.py:170-179). */
int sldg_poisson_efield(const sldg_poisson* p, const double* phi, double* e, void* stream);
/* out2 = [max|E|, 0.5 * w.E^2]  (driver.py:220-229, xfield.py:192-195) */
int sldg_field_diag(const sldg_poisson* p, const double* e, double* out2, void* stream);

/* ------------------------------------------------ fused Strang step (one HBM pass) */
/* Steady-state step of Simulation.advance (csrc/step_fused.cu): from the state after the
 * leading half x-step, f_out = X(X(V(f_in; speeds = E, dt))) with the moments of
 * X(V(f_in)) (the step's diagnostics) in mom_out3 and rho of f_out in rho_out (the next
 * step's field source).  Replaces advect_velocity + advect_x + moments + advect_x +
 * compute_rho (vsweep.py:413-441, xfield.py:91-109, driver.py:139-146) in one pass.
 * _query returns SLDG_ERR_UNSUPPORTED (with the reason) for plans it does not cover. */
int sldg_step_fused_query(const sldg_vplan* vplan, const sldg_xplan* xplan, int64_t n_cols,
                          int64_t ld, size_t* scratch_bytes);
/* *profitable = 1 when the one-pass step is expected to beat the separate passes on
 * this device (its kernel keeps two CTAs per SM without register spills). */
int sldg_step_fused_advice(const sldg_vplan* vplan, const sldg_xplan* xplan, int64_t n_cols,
                           int64_t ld, int32_t* profitable);
int sldg_step_fused(const sldg_vplan* vplan, const sldg_xplan* xplan, const double* f_in,
                    double* f_out, int64_t ld, int64_t n_cols, const double* speeds, double dt,
                    int32_t bc, const double* w, const double* v0, const double* v2,
                    const double* xw, double* mom_out3, double* rho_out, void* scratch,
                    void* stream);
/* Pipelined form used by Simulation.advance: two launches per step.
 * sldg_field_chain does a step's field work in one launch -- [fold the previous
 * sldg_step_fused_deferred's partials into rho and its moments into mom_prev3
 * (when rho_in is NULL)] -> Poisson solve (phi, e; as sldg_poisson_solve) ->
 * diag2 = [max|E|, field energy] (as sldg_field_diag) -> the v-sweep level
 * matrices for speeds = e into `scratch`; rho_in != NULL uses that rho instead.
 * sldg_step_fused_deferred is sldg_step_fused with those level matrices and with
 * the moment / rho partials left in `scratch` for the next sldg_field_chain
 * (mom_out3 != NULL folds the moments right away).  mode 0 = steady state;
 * mode 1 = the last step of a run: f_out = X(V(f_in)), the state after the full
 * step (no next leading half step, no rho); mode 2 = the first (leading) half
 * x-step alone, f_out = X(f_in) with rho partials (speeds unused) -- the same tile
 * distribution, for pencil sharding.  Modes 1 and 2 give the separate calls' f
 * bit for bit; mode 0 applies the two half x-steps as one composed stencil
 * (A A, A B + B A, B B), equal to the separate calls to ~1e-16 relative.  The
 * x weights `xw` are the x DOF weights of the plan's uniform grid (every cell's
 * weights equal cell 0's, xfield.py XGrid.dof_weights). */
int sldg_field_chain(const sldg_vplan* vplan, const sldg_xplan* xplan, const sldg_poisson* p,
                     int64_t n_cols, int64_t ld, double dt, const double* rho_in, double* rho,
                     double* phi, double* e, double* diag2, double* mom_prev3, void* scratch,
                     void* stream);
int sldg_step_fused_deferred(const sldg_vplan* vplan, const sldg_xplan* xplan,
                             const double* f_in, double* f_out, int64_t ld, int64_t n_cols,
                             const double* speeds, int32_t bc, const double* w, const double* v0,
                             const double* v2, const double* xw, int32_t mode,
                             double* mom_out3, int64_t tile_begin, int64_t tile_count,
                             void* scratch, void* stream);
/* Pencil sharding: the work of one fused step is n_tiles tiles (pencil x line
 * group x cell, in plan walk order); tile_begin/tile_count of the deferred step
 * restrict it to one rank's contiguous share (tile_count = -1: all).  Rows outside
 * the share are not touched.  sldg_step_fused_tiles: info[4] = {n_tiles, rows per
 * tile, line groups per cell, cells per pencil}; tile t is cell t % cells of item
 * t / cells, item = walk pencil x line groups + line group.  sldg_step_fused_fold
 * folds the partials of the last deferred step (modes 0 and 2) into rho_out
 * (n_cols) / mom_out3 (either may be NULL), in sldg_field_chain's fold order. */
int sldg_step_fused_tiles(const sldg_vplan* vplan, const sldg_xplan* xplan, int64_t n_cols,
                          int64_t ld, int64_t* info);
int sldg_step_fused_fold(const sldg_vplan* vplan, const sldg_xplan* xplan, int64_t n_cols,
                         int64_t ld, double* rho_out, double* mom_out3, void* scratch,
                         void* stream);

/* ---------------------------------------------------------------- misc */
/* out[i*ld + j] = a[i] * b[j]: the separable initial condition sampled on the
 * device (sample_initial, driver.py:132-136), bit-identical to numpy's product. */
int sldg_outer(const double* a, int64_t na, const double* b, int64_t nb, double* out, int64_t ld,
               void* stream);
const char* sldg_last_error(void);
int sldg_version(void);
/* bit 0: schedule-fuzzing build (-DSLDG_FUZZ, libsldg_fuzz.so; tests only) */
int sldg_build_flags(void);
/* number of kernel launches enqueued by this library since load (for bench) */
int64_t sldg_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SLDG_CAPI_H */
