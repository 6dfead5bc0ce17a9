/*
 * enkf_mc.h -- C-ABI of the B200-native EnKF-MC analysis hot path (libenkfmc.so).
 *
 * The reference (/root/reference/pkg/src/mcholkf) is pure Python and has no FFI of
 * its own; these entry points are what a ctypes binding of its analysis step would
 * call.  Each function names the reference code it replaces.
 *
 * Conventions: plain pointers and sizes only; float64 ("f64") and int64 host arrays
 * are C-order; the ensemble is X[nstate][nens] with the member index fastest
 * (kernels.py:28-33); state label = field*(nx*ny) + 2-D label (field stacking is this
 * library's extension, nfields = 1 is exactly the reference).  Every function returns
 * 0 on success or a negative ENKFMC_E_* code; enkfmc_last_error() gives the message
 * of the calling thread's last failure.  "d_" parameters are device pointers on the
 * current CUDA device; "stream" is a cudaStream_t passed as void*.
 *
 * There is no CPU fallback: compute entry points fail with ENKFMC_E_CUDA when no
 * sm_100 device is usable.
 */
#ifndef ENKF_MC_H
#define ENKF_MC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ENKFMC_OK 0
#define ENKFMC_E_CONFIG   (-1)  /* ConfigurationError (errors.py:8)  */
#define ENKFMC_E_VALUE    (-2)  /* ValueError                        */
#define ENKFMC_E_NUMERIC  (-3)  /* NumericalError (errors.py:16)     */
#define ENKFMC_E_CUDA     (-4)  /* CUDA runtime / no device          */
#define ENKFMC_E_CAPACITY (-5)  /* CapacityError (errors.py:12)      */

typedef struct enkfmc_plan enkfmc_plan;   /* opaque: index maps on host + device */

const char *enkfmc_version(void);
const char *enkfmc_last_error(void);

/* ---- index maps (integer, bit-exact) ------------------------------------------- */

/* `periodic`: 0 clipped, 1 periodic on both axes (the reference's boundary flag, geometry.py:43),
 * 2 periodic along x only (columns: longitude periodic, latitude clipped), 3 along y only.  Codes 2
 * and 3 apply the reference's per-axis window / band rules (geometry.py:132-142) with one flag per
 * axis; the reference itself cannot express them. */

/* Near-square block grid pr x pc of `delta` tiles: geometry.py:179-193. */
int enkfmc_tiling(int64_t nx, int64_t ny, int64_t delta, int64_t *pr, int64_t *pc);

/* Box members / predecessors of one cell, ascending labels: geometry.py:145-162.
 * out must hold (2*zeta+1)^2 entries; *count receives the number written. */
int enkfmc_local_box(int64_t nx, int64_t ny, int row_major, int periodic, int64_t center,
                     int64_t zeta, int64_t *out, int64_t *count);
int enkfmc_predecessors(int64_t nx, int64_t ny, int row_major, int periodic, int64_t center,
                        int64_t zeta, int64_t *out, int64_t *count);

/* Plan over decompose(geometry, delta, zeta): tiles, interiors, zeta-ring halos,
 * local_order, interior positions (geometry.py:165-222) and the per-row local
 * predecessor lists of fit_factors (estimator.py:123-131), shared by all fields. */
int enkfmc_plan_create(int64_t nx, int64_t ny, int row_major, int periodic, int64_t nfields,
                       int64_t delta, int64_t zeta, enkfmc_plan **plan);

/* The same plan for vertically coupled fields (extension, no reference counterpart: BASELINE.json configs 3 and 5,
 * "vertical r = 1"): every field is nlev stacked 2-D levels (row = level * nx * ny + 2-D label, the reference's
 * ascending-label convention of geometry.py:145-162 carried to the third axis), a component's box is its 2-D box on
 * every level within zeta_v of its own (clipped), its predecessors the box members with a smaller label, and a
 * sub-domain is a 2-D tile of decompose() (geometry.py:165-222) with its zeta-ring halo on every level.  Host integer
 * code only: the kernels see longer local predecessor lists (up to (2 zeta + 1)^2 (zeta_v + 1) - ... <= 128) and wider
 * bands.  nlev = 1 is enkfmc_plan_create. */
int enkfmc_plan_create_levels(int64_t nx, int64_t ny, int row_major, int periodic, int64_t nlev, int64_t zeta_v,
                              int64_t nfields, int64_t delta, int64_t zeta, enkfmc_plan **plan);

/* Single-tile plan over an explicit strictly increasing local_order (the
 * fit_factors(U, geometry, zeta, local_order) call, estimator.py:64-131).  State rows
 * are local positions 0..n_local-1; every row is "interior". */
int enkfmc_plan_create_local(int64_t nx, int64_t ny, int row_major, int periodic, int64_t zeta,
                             int64_t n_local, const int64_t *local_order, enkfmc_plan **plan);

/* Single-tile plan over an arbitrary strictly-lower CSR pattern (analysis_primal on
 * caller-supplied PrecisionFactors, kernels.py:163-218 / factors.py:39-64). */
int enkfmc_plan_create_csr(int64_t n, const int64_t *indptr, const int64_t *indices,
                           enkfmc_plan **plan);

void enkfmc_plan_destroy(enkfmc_plan *plan);

/* restrict_network for every (field, tile): kernels.py:90-113.  obs_indices are
 * sorted global state labels. */
int enkfmc_plan_set_observations(enkfmc_plan *plan, int64_t nobs, const int64_t *obs_indices);

/* Sizes: what = 0 ntiles, 1 sum n_local, 2 nnz(T pattern), 3 sum interior, 4 sum halo,
 * 5 nobs, 6 sum restricted obs, 7 pr, 8 pc, 9 max n_local, 10 max predecessors,
 * 11 max half-bandwidth, 12 nfields, 13 n2d, 14 distinct regressions among the owned local rows
 * (halo rows shared by several tiles with the same predecessor list are regressed once and copied),
 * 15 owned local rows. */
int64_t enkfmc_plan_size(const enkfmc_plan *plan, int what);

/* Copy-out of the maps (for parity tests / the Python shim).  what = 0 tile_ptr[ntiles+1],
 * 1 local_order, 2 interior_ptr[ntiles+1], 3 interior, 4 interior_pos, 5 halo_ptr, 6 halo,
 * 7 row_ptr[sum n_local + 1], 8 col_idx[nnz] (local positions), 9 obs_ptr[nfields*ntiles+1],
 * 10 obs_pos, 11 obs_row, 12 half-bandwidth per tile, 13 physical order per local row,
 * 14 per local row the local row whose regression it shares (itself, or -1 outside the owned tiles). */
int enkfmc_plan_get(const enkfmc_plan *plan, int what, int64_t *out, int64_t capacity);

/* ---- device-resident stages ------------------------------------------------------ */

/* U = center_rows(X): validation.py:35-39 (means removed twice).  d_X, d_U: [nrows][nens]. */
int enkfmc_center_rows(const double *d_X, double *d_U, int64_t nrows, int64_t nens, void *stream);

/* K2: T values (-beta, in the plan's CSR order, per field) and floored D for every local
 * row of every tile: estimator.py:46-61,133-159 + factors.py:60.
 * d_U [nstate][nens] centred; d_T [nfields][nnz]; d_D [nfields][sum n_local];
 * d_flags [nfields][sum n_local] (may be NULL): bit0 = singular values were examined beyond the
 * certificate (deflation or fallback), bit1 = truncation active, bit2 = Jacobi sweep cap hit,
 * bit3 = D on the variance floor, bit4 = Jacobi-SVD fallback taken, bits 5-7 = why (1 zero pivot or
 * p > N, 2 certificate inconclusive, 3 out of deflation slots, 4 refined value above the threshold,
 * 5 cond(R) beyond the fast path's limit or certificate lost to cancellation, 6 block iteration not
 * converged, 7 kept direction inside the block); diagnostics: bits 8-15 inverse-iteration steps,
 * bits 16-21 Jacobi sweeps. */
int enkfmc_regress(enkfmc_plan *plan, const double *d_U, int64_t nens, double rank_tol,
                   double variance_floor, double *d_T, double *d_D, int32_t *d_flags, void *stream);

/* K3: per tile assemble A = T^T D^-1 T + H^T R^-1 H (factors.py:136-145, kernels.py:189-191),
 * banded Cholesky, solve all members, Xa = Xb + dx (kernels.py:182-218) and write the
 * interior rows into d_Xa (merge_interiors, driver.py:99-125).  d_X/d_Xa [nstate][nens];
 * d_rdiag [nobs]; d_Ys [nobs][nens]; d_status [nfields*ntiles]: 0 ok, 1 non-positive pivot,
 * 2 non-finite.  Tiles without observations copy Xb exactly (kernels.py:179-180). */
int enkfmc_local_solve(enkfmc_plan *plan, const double *d_X, const double *d_T, const double *d_D,
                       const double *d_rdiag, const double *d_Ys, int64_t nens, double *d_Xa,
                       int32_t *d_status, void *stream);

/* center -> regress -> local solve on device-resident inputs (the timed "value" path).
 * Workspace (U, T, D, scratch) lives in the plan and is reused across calls. */
int enkfmc_analysis_device(enkfmc_plan *plan, const double *d_X, const double *d_rdiag,
                           const double *d_Ys, int64_t nens, double rank_tol,
                           double variance_floor, double *d_Xa, void *stream);

/* Outcome of the last analysis on this plan (either entry point): synchronises, reads the per-tile
 * status words and the clamped-pivot count (enkfmc_plan_counter(plan, 5)); a failed tile returns
 * ENKFMC_E_NUMERIC naming the sub-domain, as analysis_primal raises NumericalError when the
 * factorisation fails (kernels.py:192-195).  enkfmc_analysis_device is asynchronous and
 * does not look at the status itself; callers check here once the step is done. */
int enkfmc_plan_check_status(enkfmc_plan *plan);

/* ---- host-buffer entry point (what assimilate_parallel binds; driver.py:159-253) -- */

/* Copies X, r_diag, Ys to the device, runs the analysis, copies Xa back.  The fields (independent
 * 2-D problems) are processed in up to five groups: a copy stream uploads group g+1 and downloads the
 * analysis of group g-1 under the kernels of group g (pinned host buffers make the copies asynchronous;
 * ENKFMC_HOST_GROUPS overrides the group count).  timings_ms[4] (may be NULL) receives the busy time of
 * h2d, estimation (K0+K2), analysis (K3), d2h from CUDA events, summed over the groups.
 * Fails with ENKFMC_E_NUMERIC naming the first failing (field, tile). */
int enkfmc_analysis_host(enkfmc_plan *plan, const double *X, const double *r_diag, const double *Ys,
                         int64_t nens, double rank_tol, double variance_floor, double *Xa,
                         double *timings_ms);

/* Counters of the last device run: what = 0 kernels launched, 1 regressions on the SVD path,
 * 2 regressions with truncation, 3 rows at the variance floor (filled only when the call
 * collected flags), 4 first failing work item (field*ntiles+tile) or -1, 5 Cholesky pivots clamped at the
 * rounding level in the last enkfmc_analysis_host call (A is positive semi-definite by construction). */
int64_t enkfmc_plan_counter(const enkfmc_plan *plan, int what);

/* Device pointers of the plan's workspace after enkfmc_analysis_device/_host:
 * what = 0 U, 1 T, 2 D, 3 flags, 4 status.  NULL if not allocated. */
void *enkfmc_plan_device_buffer(const enkfmc_plan *plan, int what);

/* Synchronise and copy `bytes` of that workspace buffer to host memory (parity tests). */
int enkfmc_plan_read_buffer(const enkfmc_plan *plan, int what, void *host_out, int64_t bytes);

/* ---- sharding and measurement ------------------------------------------------------- */

/* Restrict the plan's work to tiles [tile_begin, tile_end) (one rank's share; tiles are
 * independent units, driver.py:196-204).  Maps and state arrays stay global-sized; only rows
 * of owned tiles are regressed and only owned interiors are written to d_Xa. */
int enkfmc_plan_set_tile_range(enkfmc_plan *plan, int64_t tile_begin, int64_t tile_end);

/* Per-stage CUDA-event timing of enkfmc_analysis_device on its launching stream.
 * enable != 0 starts recording (and clears the log); stage_times synchronises and returns the
 * number of recorded calls and the SUMMED milliseconds of ms4 = {K0 centre, K2a QR, K2b probe/solve,
 * K3 assemble + local solve} (with field chunking the K2a/K2b split is that of the last chunk). */
int enkfmc_plan_profile(enkfmc_plan *plan, int enable);
int enkfmc_plan_stage_times(enkfmc_plan *plan, int64_t *ncalls, double *ms4);

/* Algorithmic work of one analysis with the current tile range (SURVEY 8d definitions):
 * flops3[0] = sum over owned local rows of 2*N*p^2 - (2/3)*p^3 + 4*N*p (Householder-QR least squares; the
 *             reference's work: one regression per local row of every sub-domain),
 * flops3[1] = sum over owned tiles with observations of n*b^2 + 4*n*b*N (banded Cholesky + two sweeps),
 * flops3[2] = as [0] over the distinct regressions only: what the regression kernels execute,
 * each times the number of fields. */
int enkfmc_plan_work(const enkfmc_plan *plan, int64_t nens, double *flops3);

/* FP64 DFMA peak of the current device, measured with a register-resident FMA-chain kernel
 * (MEASURED_PEAKS.json has no FP64 figure).  Returns TFLOP/s in *tflops. */
int enkfmc_fp64_peak(double *tflops, void *stream);

/* FP64 tensor-core (mma.sync m8n8k4 f64) peak of the current device, TFLOP/s. */
int enkfmc_fp64_mma_peak(double *tflops, void *stream);

/* ---- small device helpers behind the remaining reference callables ------------------ */

/* dst[dst_rows[k]][:] = src[src_rows[k]][:]  -- merge_interiors, driver.py:116. */
int enkfmc_scatter_rows(double *d_dst, const int64_t *d_dst_rows, const double *d_src,
                        const int64_t *d_src_rows, int64_t nrows, int64_t nens, void *stream);

/* Lower band of T^T D^-1 T (no observation term) of a single-tile plan, row form:
 * d_band[n][Wr], Wr = 8 (Wb + 1), Wb = floor((bw + 7) / 8); entry e of row I is column
 * 8 (I/8 - Wb) + e -- PrecisionFactors.dense_precision, factors.py:136-145. */
int enkfmc_assemble_band(enkfmc_plan *plan, const double *d_T, const double *d_D, int64_t tile,
                         double *d_band, void *stream);

/* d_out = T^T D^-1 T d_V for a single-tile plan; d_V, d_tmp, d_out are [n][ncols] --
 * PrecisionFactors.precision_apply, factors.py:86-96. */
int enkfmc_precision_apply(enkfmc_plan *plan, const double *d_T, const double *d_D, const double *d_V,
                           int64_t ncols, double *d_tmp, double *d_out, void *stream);

/* Unit-triangular solves with many right-hand sides on a single-tile plan, in place on d_B [n][ncols]:
 *   transposed = 0: (I + L) X = diag(d_scale_in) B    -- PrecisionFactors.sqrt_solve (factors.py:116-134, scale_in =
 *                   sqrt(D)) and the second half of covariance_apply (factors.py:98-114);
 *   transposed = 1: (I + L)^T X = B, X *= d_scale_out -- the first half of covariance_apply (scale_out = D).
 * Either scale may be NULL. */
int enkfmc_unit_tri_solve(enkfmc_plan *plan, const double *d_T, int transposed, const double *d_scale_in,
                          const double *d_scale_out, double *d_B, int64_t ncols, void *stream);

/* One explicit step of the periodic advection-diffusion forecast model on a device-resident ensemble
 * ([nfields*nx*ny][nens], d_in != d_out): upwind advection, centred diffusion, unit grid -- the
 * propagate hook of the device-resident cycle loop (models.py:114-132, driver.py:256-310).  Bit-identical
 * to the reference's numpy expression. */
int enkfmc_advdiff_step(const double *d_in, double *d_out, int64_t nx, int64_t ny, int row_major,
                        int64_t nfields, int64_t nens, double ux, double uy, double dt, double kappa,
                        void *stream);

/* LETKF baseline at every grid component -- letkf_analysis_global / letkf_analysis_point (kernels.py:251-335), the
 * paper's comparison method; a decomposed run gives the same rows (driver.py:128-156).  d_X, d_U (workspace), d_Xa:
 * [nfields*nx*ny][nens]; d_mean: workspace [nfields*nx*ny]; d_obs_of_state: observation row of each state row or -1;
 * *first_bad receives the first component whose weight matrix lost positive definiteness (-1: none; the call then
 * returns ENKFMC_E_NUMERIC like the reference raises NumericalError).  Synchronises the stream. */
int enkfmc_letkf_device(const double *d_X, double *d_U, double *d_mean, double *d_Xa,
                        const int32_t *d_obs_of_state, const double *d_rdiag, const double *d_y,
                        int64_t nx, int64_t ny, int row_major, int periodic, int64_t nfields,
                        int64_t nens, int64_t zeta, double inflation, int64_t *first_bad, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* ENKF_MC_H */
