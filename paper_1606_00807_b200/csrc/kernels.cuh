// Kernel parameter blocks and launchers (kernels.cu) used by api.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define ENKFMC_MAX_NENS 256

struct RegressParams {
    const double *U;           // [nfields * nstate2d][N] centred anomalies
    int N, ld;                 // ensemble size, odd column pitch of the per-warp workspace
    int pmax;                  // largest predecessor count in the plan
    int nfields;
    int64_t nloc, nnz, nstate2d, nwork;
    const int64_t *row_ptr;    // [nloc + 1]
    const int32_t *pred_state; // [nnz] state row of each predecessor
    const int32_t *state_row;  // [nloc]
    const int32_t *work_order; // distinct regressions (plan.h regress_order), most predecessors first
    double rank_tol, variance_floor, fast_ratio;
    double *T;                 // [nfields][tstride] (-beta), indexed by the plan's global CSR position: the pointer is biased by the
    double *D;                 // [nfields][dstride] floored    first owned position when the workspace covers the owned tiles only
    int32_t *flags;            // [nfields][dstride] or null
    int64_t tstride, dstride;  // field strides of T and of D / flags (nnz / nloc, or the owned counts)
    unsigned int *counter;     // two work-fetch counters (zeroed by the launcher)
    unsigned int *lcounter;    // five words: list length, K2b-2 fetch counter, rows sent to the Jacobi fallback, second list length, its fetch counter
    unsigned int *worklist;    // [nwork] rows K2b-1 hands to K2b-2 (work item numbers)
    unsigned int *worklist2;   // [nwork] rows the first K2b-2 pass hands to the second (larger blocks)
    int bmax, bmax1, bmax2, level;   // block cap of this K2b-2 pass, of the first and second pass, and which pass this is (set by the launcher)
    int f0, f1;                // fields handled by this launch pair (scratch is sized for f1 - f0)
    double *Rq;                // packed QR output scratch [f1 - f0][rq_stride]
    int64_t rq_stride;
    const int64_t *rq_ptr;     // [nloc + 1] offsets of each row's packed block
};

struct SolveParams {
    const double *X, *T, *D, *rdiag, *Ys;
    double *Xa;
    int N, nfields, ntiles, ntiles_owned;   // ntiles: global count (indexing); owned: work items
    int64_t nloc, nnz, nstate2d;
    int64_t tstride, dstride;  // field strides of T and D (see RegressParams)
    const int64_t *tile_ptr, *row_ptr, *csc_ptr, *csc_src;
    const int32_t *col_idx, *csc_row, *phys, *iphys, *bw, *state_row, *obs_slot, *tile_nobs, *tile_order;
    const uint8_t *is_interior;
    const uint8_t *tile_mono;  // per tile: physical order == local order (may be null)
    double *scratch;           // per-CTA scratch
    int64_t scratch_stride;    // doubles per CTA
    int64_t off_z, off_win_a, off_win_r;  // offsets (doubles) inside a CTA's scratch
    int bmax;                  // largest half-bandwidth
    int a_in_smem, r_in_smem;  // window placement
    int64_t a_doubles;         // size of the A window / backward reduction buffer
    int rows_smem;             // rows the per-row source tables in shared memory hold (0: none)
    int nr_pitch;              // member pitch of the right-hand-side window (see solve_plan_scratch)
    int32_t *status;           // [nfields * ntiles]
    unsigned int *counter;
    int assemble_only;         // 1: K3a writes T^T D^-1 T without the observation term, for every owned tile
    int f0, f1;                // fields handled by this launch pair
    double *band;              // [f1 - f0][band_stride]: per tile [n][b+1] column-form lower band / L
    int64_t band_stride;
    const int64_t *band_ptr;   // [ntiles] offset of each tile's band
    const int32_t *row_tile;   // [nloc]
    const int32_t *work_order; // owned local rows
    int64_t nrows_owned;
    int asm_nmax, asm_nnzmax;  // largest tile (rows, T entries): shared-memory staging of the tile-cooperative K3a
    int all_mono;              // every tile's physical order is its local order: the tensor-core form of K3a applies
};

struct LetkfParams {
    const double *X;           // [nfields * nx * ny][N] background
    double *U, *mean;          // workspace: anomalies (same shape), row means
    double *Xa;                // analysis
    const int32_t *obs_of_state;   // [nfields * nx * ny] observation row of a state row, or -1
    const double *rdiag, *y;   // [nobs]
    int64_t nx, ny, nitems, zeta;
    int row_major, periodic, N, boxmax;
    double inflation, eig_floor;
    unsigned int *counter;         // work-fetch counter (zeroed by the caller)
    unsigned long long *first_bad; // smallest state row whose weight matrix lost positive definiteness (initialised to ~0)
};

size_t regress_warp_workspace_doubles(int N, int pmax);
cudaError_t launch_letkf(const LetkfParams &p, int sm_count, size_t smem_limit, cudaStream_t s);
cudaError_t launch_center_rows(const double *X, double *U, int64_t nrows, int N, cudaStream_t s);
// mid (may be null) is recorded between the QR kernel (K2a) and the probe/solve kernel (K2b)
cudaError_t launch_regress(const RegressParams &p, int sm_count, size_t smem_limit, cudaStream_t s, cudaEvent_t mid);
// T, D, flags of row alias_row[a] := those of alias_rep[a] (same regression), every field
cudaError_t launch_replicate_rows(const int32_t *alias_row, const int32_t *alias_rep, int64_t naliases,
                                  const int64_t *row_ptr, int64_t nfields, int64_t nnz, int64_t nloc, double *T,
                                  double *D, int32_t *flags, cudaStream_t s);
// Fills scratch layout fields of p given bmax/nmax; returns doubles per CTA.
int64_t solve_plan_scratch(SolveParams &p, int64_t nmax, size_t smem_limit);
cudaError_t launch_assemble_band(const SolveParams &p, int sm_count, size_t smem_limit, cudaStream_t s);
int solve_grid_size(int sm_count, const SolveParams &p, size_t smem_limit);
cudaError_t launch_local_solve(const SolveParams &p, int grid, size_t smem_limit, cudaStream_t s);
cudaError_t launch_scatter_rows(double *dst, const int64_t *dst_rows, const double *src, const int64_t *src_rows,
                                int64_t nrows, int N, cudaStream_t s);
// w = (v + L v) / D (phase 0), out = w + L^T w (phase 1); v, w, out: [n][ncols]
cudaError_t launch_precision_apply(const int64_t *row_ptr, const int32_t *col_idx, const int64_t *csc_ptr,
                                   const int32_t *csc_row, const int64_t *csc_src, const double *T, const double *D,
                                   const double *V, double *Wtmp, double *Out, int64_t n, int64_t ncols, cudaStream_t s);
// unit-triangular solves with the strictly-lower pattern of a single-tile plan (see unit_tri_solve_kernel)
cudaError_t launch_unit_tri_solve(int transposed, const int64_t *ptr, const int32_t *idx, const int64_t *src, const double *T,
                                  const double *scale_in, const double *scale_out, double *B, int64_t n, int64_t ncols,
                                  cudaStream_t s);
cudaError_t launch_advdiff_step(const double *in, double *out, int64_t nx, int64_t ny, int row_major, int64_t nfields, int N,
                                double ux, double uy, double dt, double kappa, int sm_count, cudaStream_t s);
cudaError_t launch_fp64_peak(double *out, int iters, int sm_count, cudaStream_t s);
cudaError_t launch_dmma_peak(double *out, int iters, int sm_count, cudaStream_t s);
