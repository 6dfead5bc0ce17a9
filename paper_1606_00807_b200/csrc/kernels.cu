// sm_100a kernels of the EnKF-MC analysis step.  FP64 throughout (the reference has no
// reduced precision anywhere).  The work is FP64-DFMA / shared-memory bound,
// not GEMM-shaped for tcgen05 (which has no FP64 kind), so these are SIMT kernels sized
// for 148 SMs with persistent CTAs that fetch work items from an atomic counter.
//
//   K0 center_rows_kernel   validation.py:35-39
//   K2 regress_kernel       estimator.py:46-61,133-150 + factors.py:60
//   K3 local_solve_kernel   factors.py:136-145, kernels.py:178-218, driver.py:99-125
//
// All results are deterministic run to run: no floating-point atomics, fixed reduction
// trees, work items are independent.

#include <cfloat>
#include <cmath>
#include <cstdio>

#include "kernels.cuh"

#define FULL 0xffffffffu

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

// sum over aligned groups of T adjacent lanes (T power of two)
__device__ __forceinline__ double group_sum(double v, int T) {
    for (int o = T >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// largest power of two T with count * T <= 32 (1 if count > 16)
__device__ __forceinline__ int lanes_per_item(int count) {
    int T = 1;
    while (T < 32 && count * (T << 1) <= 32) T <<= 1;
    return T;
}

}  // namespace

// ------------------------------------------------------------------------------------------
// K0: U = X - mean(X); U -= mean(U)   (one warp per row, row = N contiguous doubles)
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) center_rows_kernel(const double *__restrict__ X, double *__restrict__ U,
                                                          int64_t nrows, int N) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < nrows; row += warps) {
        const double *x = X + row * N;
        double v[ENKFMC_MAX_NENS / 32];
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < ENKFMC_MAX_NENS / 32; ++k) {
            const int i = lane + 32 * k;
            v[k] = (i < N) ? x[i] : 0.0;
            s += v[k];
        }
        const double mean = warp_sum(s) / (double)N;
        s = 0.0;
#pragma unroll
        for (int k = 0; k < ENKFMC_MAX_NENS / 32; ++k) {
            const int i = lane + 32 * k;
            v[k] = (i < N) ? v[k] - mean : 0.0;
            s += v[k];
        }
        const double mean2 = warp_sum(s) / (double)N;
#pragma unroll
        for (int k = 0; k < ENKFMC_MAX_NENS / 32; ++k) {
            const int i = lane + 32 * k;
            if (i < N) U[row * N + i] = v[k] - mean2;
        }
    }
}

cudaError_t launch_center_rows(const double *X, double *U, int64_t nrows, int N, cudaStream_t s) {
    if (nrows == 0) return cudaSuccess;
    int64_t blocks = (nrows + 7) / 8;
    if (blocks > 148 * 16) blocks = 148 * 16;
    center_rows_kernel<<<(unsigned)blocks, 256, 0, s>>>(X, U, nrows, N);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// K2: one warp per regression.
//
// Workspace W (shared memory, column-major, odd pitch ld >= N): column j < p is predecessor
// j's anomaly vector, column p is the target y.  Steps:
//   1. Householder QR with column pivoting of W[:, 0:p], reflectors also applied to y.
//   2. if rank is safely full (|r_KK| > fast_ratio |r_11|): back-substitution R b = Q^T y.
//   3. else one-sided Jacobi on the ROWS of [R | Q^T y] (J^T R = S Z^T, the rotations carry
//      Q^T y along so no rotation matrix is accumulated), truncate s < rank_tol * s_max exactly as
//      estimator.py:55-57, b = sum_k z_k (J^T c)_k / s_k.
//   4. undo the pivoting, T = -b; residual recomputed from the original rows (estimator.py:60),
//      D = max(|resid|^2 / (N-1), floor)  (estimator.py:148, factors.py:60).
// ------------------------------------------------------------------------------------------
__host__ __device__ inline size_t regress_ws_doubles(int N, int pmax) {
    const int ld = N | 1;
    size_t d = (size_t)ld * (pmax + 1) + 4 * (size_t)pmax + (size_t)(pmax + 2) / 2 + 2;
    return (d + 1) & ~(size_t)1;
}
size_t regress_warp_workspace_doubles(int N, int pmax) { return regress_ws_doubles(N, pmax); }

#define JACOBI_MAX_SWEEPS 30

__global__ void __launch_bounds__(512) regress_kernel(const RegressParams P) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31;
    const int N = P.N, ld = P.ld, pmax = P.pmax;
    double *W = smem + (size_t)(threadIdx.x >> 5) * regress_ws_doubles(N, pmax);
    double *rdiag = W + (size_t)ld * (pmax + 1);
    double *cn = rdiag + pmax;
    double *cnref = cn + pmax;
    double *aux = cnref + pmax;
    int *perm = reinterpret_cast<int *>(aux + pmax);
    const double denom = (double)(N - 1);

    for (;;) {
        unsigned int wk = 0;
        if (lane == 0) wk = atomicAdd(P.counter, 1u);
        wk = __shfl_sync(FULL, wk, 0);
        if ((int64_t)wk >= P.nwork) break;
        const int q = P.work_order[wk / (unsigned)P.nfields];
        const int f = (int)(wk % (unsigned)P.nfields);
        const int64_t r0 = P.row_ptr[q];
        const int p = (int)(P.row_ptr[q + 1] - r0);
        const double *Uf = P.U + (int64_t)f * P.nstate2d * N;
        const double *yrow = Uf + (int64_t)P.state_row[q] * N;
        const int32_t *pred = P.pred_state + r0;
        int flag = 0;

        if (p == 0) {  // estimator.py:139-144
            double s = 0.0;
            for (int i = lane; i < N; i += 32) { const double v = yrow[i]; s += v * v; }
            s = warp_sum(s) / denom;
            if (lane == 0) {
                P.D[(int64_t)f * P.nloc + q] = fmax(s, P.variance_floor);
                if (P.flags) P.flags[(int64_t)f * P.nloc + q] = (s < P.variance_floor) ? 8 : 0;
            }
            continue;
        }

        // ---- load [A^T | y] ----------------------------------------------------------
        for (int j = 0; j <= p; ++j) {
            const double *src = (j < p) ? Uf + (int64_t)pred[j] * N : yrow;
            double *dst = W + (size_t)j * ld;
            for (int i = lane; i < N; i += 32) dst[i] = src[i];
        }
        __syncwarp();
        for (int j = lane; j < p; j += 32) {
            const double *col = W + (size_t)j * ld;
            double s = 0.0;
            for (int i = 0; i < N; ++i) s += col[i] * col[i];
            cn[j] = s; cnref[j] = s; perm[j] = j;
        }
        __syncwarp();

        // ---- Householder QR with column pivoting --------------------------------------
        const int K = p < N ? p : N;
        for (int k = 0; k < K; ++k) {
            // pivot = remaining column of largest norm (ties to the smaller index)
            double best = -1.0; int bidx = k;
            for (int j = k + lane; j < p; j += 32) { const double v = cn[j]; if (v > best) { best = v; bidx = j; } }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(FULL, best, o);
                const int oi = __shfl_xor_sync(FULL, bidx, o);
                if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
            }
            if (bidx != k) {
                double *ca = W + (size_t)k * ld, *cb = W + (size_t)bidx * ld;
                for (int i = lane; i < N; i += 32) { const double t = ca[i]; ca[i] = cb[i]; cb[i] = t; }
                if (lane == 0) {
                    const int t = perm[k]; perm[k] = perm[bidx]; perm[bidx] = t;
                    cn[bidx] = cn[k]; cnref[bidx] = cnref[k];
                }
                __syncwarp();
            }
            // reflector from column k, rows k..N-1
            double *ck = W + (size_t)k * ld;
            double ss = 0.0;
            for (int i = k + lane; i < N; i += 32) ss += ck[i] * ck[i];
            ss = warp_sum(ss);
            const double x0 = ck[k];
            const double nrm = sqrt(ss);
            __syncwarp();
            if (nrm == 0.0) {           // nothing left in any remaining column
                if (lane == 0) rdiag[k] = 0.0;
                __syncwarp();
                continue;
            }
            const double alpha = (x0 >= 0.0) ? -nrm : nrm;
            const double tau = 1.0 / (nrm * (nrm + fabs(x0)));   // 2 / v^T v
            if (lane == 0) { ck[k] = x0 - alpha; rdiag[k] = alpha; }
            __syncwarp();
            // apply H = I - tau v v^T to columns k+1..p; T lanes share one column
            const int C = p - k;
            const int T = lanes_per_item(C);
            const int per = 32 / T, sub = lane % T;
            for (int c0 = 0; c0 < C; c0 += per) {
                const int cj = c0 + lane / T;
                const bool on = cj < C;
                double *col = W + (size_t)(k + 1 + (on ? cj : 0)) * ld;
                double w = 0.0;
                if (on) for (int i = k + sub; i < N; i += T) w += ck[i] * col[i];
                w = group_sum(w, T) * tau;
                if (on) for (int i = k + sub; i < N; i += T) col[i] -= w * ck[i];
            }
            __syncwarp();
            // downdate the remaining column norms; recompute on heavy cancellation
            for (int j = k + 1 + lane; j < p; j += 32) {
                const double *col = W + (size_t)j * ld;
                const double r = col[k];
                double v = cn[j] - r * r;
                if (!(v > 1e-6 * cnref[j])) {
                    v = 0.0;
                    for (int i = k + 1; i < N; ++i) v += col[i] * col[i];
                    cnref[j] = v;
                }
                cn[j] = v;
            }
            __syncwarp();
        }

        // ---- rank decision ------------------------------------------------------------
        double dmin = DBL_MAX, dmax = 0.0;
        for (int k = lane; k < K; k += 32) { const double a = fabs(rdiag[k]); dmin = fmin(dmin, a); dmax = fmax(dmax, a); }
        dmin = warp_min(dmin);
        dmax = warp_max(dmax);
        const bool fast = (K == p) && (dmin > P.fast_ratio * dmax) && (dmax > 0.0);
        double *cvec = W + (size_t)p * ld;   // Q^T y

        if (fast) {
            // back-substitution R b = c, column oriented
            for (int k = lane; k < p; k += 32) cn[k] = 1.0 / rdiag[k];
            __syncwarp();
            for (int k = p - 1; k >= 0; --k) {
                const double bk = cvec[k] * cn[k];
                const double *col = W + (size_t)k * ld;
                __syncwarp();
                for (int i = lane; i < k; i += 32) cvec[i] -= col[i] * bk;
                if (lane == 0) aux[k] = bk;
                __syncwarp();
            }
        } else {
            flag |= 1;
            // make the K x p block an explicit upper-trapezoidal R
            for (int j = lane; j < p; j += 32) {
                double *col = W + (size_t)j * ld;
                if (j < K) col[j] = rdiag[j];
                for (int i = j + 1; i < K; ++i) col[i] = 0.0;
            }
            __syncwarp();
            // one-sided Jacobi on rows 0..K-1 of [R | c]; round-robin pairs, T lanes per pair
            const int M = (K + 1) & ~1;
            const int npairs = M >> 1;
            const int T = lanes_per_item(npairs);
            const int per = 32 / T, sub = lane % T;
            const double tolj = DBL_EPSILON * sqrt((double)p);
            int sweep = 0;
            bool rotated = (K > 1);
            while (rotated && sweep < JACOBI_MAX_SWEEPS) {
                rotated = false;
                ++sweep;
                for (int r = 0; r < M - 1; ++r) {
                    for (int q0 = 0; q0 < npairs; q0 += per) {
                        const int qi = q0 + lane / T;
                        int a, b;
                        if (qi == 0) { a = M - 1; b = r; }
                        else { a = (r + qi) % (M - 1); b = (r - qi + (M - 1)) % (M - 1); }
                        const bool on = (qi < npairs) && (a < K) && (b < K);
                        if (!on) { a = 0; b = 0; }
                        const double *ra = W + a, *rb = W + b;
                        double g = 0.0, da = 0.0, db = 0.0;
                        if (on) for (int c = sub; c < p; c += T) {
                            const double x = ra[(size_t)c * ld], y = rb[(size_t)c * ld];
                            g += x * y; da += x * x; db += y * y;
                        }
                        g = group_sum(g, T); da = group_sum(da, T); db = group_sum(db, T);
                        const bool rot = on && (fabs(g) > tolj * sqrt(da * db)) && (g != 0.0);
                        if (rot) {
                            const double zeta = (db - da) / (2.0 * g);
                            const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                            const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
                            double *wa = W + a, *wb = W + b;
                            for (int c = sub; c <= p; c += T) {
                                const double x = wa[(size_t)c * ld], y = wb[(size_t)c * ld];
                                wa[(size_t)c * ld] = cs * x - sn * y;
                                wb[(size_t)c * ld] = sn * x + cs * y;
                            }
                        }
                        if (__any_sync(FULL, rot)) rotated = true;
                    }
                    __syncwarp();
                }
            }
            if (sweep >= JACOBI_MAX_SWEEPS && rotated) flag |= 4;
            // singular values = row norms; truncate as estimator.py:55-57
            double smax = 0.0;
            for (int k = lane; k < K; k += 32) {
                const double *row = W + k;
                double s2 = 0.0;
                for (int c = 0; c < p; ++c) { const double v = row[(size_t)c * ld]; s2 += v * v; }
                cn[k] = s2;
                smax = fmax(smax, s2);
            }
            smax = sqrt(warp_max(smax));
            __syncwarp();
            bool dropped = false;
            for (int k = lane; k < K; k += 32) {
                const double s = sqrt(cn[k]);
                const bool keep = (s >= P.rank_tol * smax) && (s > 0.0);
                cnref[k] = keep ? cvec[k] / cn[k] : 0.0;
                dropped |= !keep;
            }
            if (__any_sync(FULL, dropped)) flag |= 2;
            __syncwarp();
            for (int j = lane; j < p; j += 32) {
                const double *col = W + (size_t)j * ld;
                double b = 0.0;
                for (int k = 0; k < K; ++k) b += col[k] * cnref[k];
                aux[j] = b;
            }
            __syncwarp();
        }

        // ---- undo pivoting, write T = -beta --------------------------------------------
        double *Tout = P.T + (int64_t)f * P.nnz + r0;
        for (int j = lane; j < p; j += 32) {
            const double b = aux[j];
            const int o = perm[j];
            rdiag[o] = b;
            Tout[o] = -b;
        }
        __syncwarp();
        // ---- residual from the original rows, D ----------------------------------------
        double res[ENKFMC_MAX_NENS / 32];
#pragma unroll
        for (int s = 0; s < ENKFMC_MAX_NENS / 32; ++s) { const int i = lane + 32 * s; res[s] = (i < N) ? yrow[i] : 0.0; }
        for (int j = 0; j < p; ++j) {
            const double b = rdiag[j];
            const double *src = Uf + (int64_t)pred[j] * N;
#pragma unroll
            for (int s = 0; s < ENKFMC_MAX_NENS / 32; ++s) { const int i = lane + 32 * s; if (i < N) res[s] -= b * src[i]; }
        }
        double d = 0.0;
#pragma unroll
        for (int s = 0; s < ENKFMC_MAX_NENS / 32; ++s) d += res[s] * res[s];
        d = warp_sum(d) / denom;
        if (lane == 0) {
            if (d < P.variance_floor) flag |= 8;
            P.D[(int64_t)f * P.nloc + q] = fmax(d, P.variance_floor);
            if (P.flags) P.flags[(int64_t)f * P.nloc + q] = flag;
        }
        __syncwarp();
    }
}

cudaError_t launch_regress(const RegressParams &p, int sm_count, size_t smem_limit, cudaStream_t s) {
    if (p.nwork == 0) return cudaSuccess;
    const size_t ws = regress_ws_doubles(p.N, p.pmax) * sizeof(double);
    int warps = (int)(smem_limit / ws);
    if (warps < 1) return cudaErrorInvalidConfiguration;
    if (warps > 16) warps = 16;
    int ctas_per_sm = 1;
    if (warps == 16) {  // small workspaces: several CTAs per SM
        ctas_per_sm = (int)(smem_limit / (ws * 16));
        if (ctas_per_sm > 4) ctas_per_sm = 4;
        if (ctas_per_sm < 1) ctas_per_sm = 1;
    }
    const size_t smem = ws * warps;
    cudaError_t e = cudaFuncSetAttribute(regress_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(p.counter, 0, sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
    int64_t grid = (int64_t)sm_count * ctas_per_sm;
    const int64_t need = (p.nwork + warps - 1) / warps;
    if (grid > need) grid = need;
    regress_kernel<<<(unsigned)grid, warps * 32, smem, s>>>(p);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// K3: one CTA per (field, tile).
//
// A = T~^T D^-1 T~ + H^T R^-1 H with T~ = I + strictly-lower T (factors.py:136-145,
// kernels.py:189-191) is symmetric and banded (half-bandwidth b) in the tile's physical
// order.  Phase A assembles its lower band column by column into CTA scratch (L2-resident);
// phase B runs a right-looking banded Cholesky through a sliding (b+2)-row window, carrying
// the N right-hand sides rhs[obs] = (Ys - Xb[obs]) / r (kernels.py:182-186) along (forward
// substitution fused); phase C is the backward substitution and writes Xa = Xb + dx for the
// interior rows straight into the global analysis (kernels.py:218, driver.py:116).
// ------------------------------------------------------------------------------------------
#define SOLVE_THREADS 256

__global__ void __launch_bounds__(SOLVE_THREADS) local_solve_kernel(const SolveParams P) {
    extern __shared__ double smem[];
    __shared__ unsigned int s_item;
    __shared__ int s_fail;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nthreads = blockDim.x, nwarps = nthreads >> 5;
    const int N = P.N;
    double *scr = P.scratch + (int64_t)blockIdx.x * P.scratch_stride;
    double *Acol = scr;                 // [n][b+1]  column-form lower band, overwritten by L
    double *Z = scr + P.off_z;          // [n][N]    forward-substituted right-hand sides
    // shared layout: lk[2][bmax+2] | red[nthreads] | window A | window RHS
    const int bmax = P.bmax;
    double *lk = smem;
    double *red = lk + 2 * (bmax + 2);
    double *sm_rest = red + nthreads;
    const int WnMax = bmax + 2, PitchMax = WnMax | 1;
    double *Aw = P.a_in_smem ? sm_rest : scr + P.off_win_a;
    double *Rw = P.r_in_smem ? (P.a_in_smem ? sm_rest + (size_t)WnMax * PitchMax : sm_rest) : scr + P.off_win_r;
    const int total_items = P.nfields * P.ntiles;

    for (;;) {
        __syncthreads();
        if (tid == 0) { s_item = atomicAdd(P.counter, 1u); s_fail = 0; }
        __syncthreads();
        const unsigned int item = s_item;
        if ((int)item >= total_items) break;
        const int t = P.assemble_only ? P.tile_sel : P.tile_order[item / (unsigned)P.nfields];
        const int f = P.assemble_only ? 0 : (int)(item % (unsigned)P.nfields);
        if (P.assemble_only && item > 0) break;
        const int64_t base = P.tile_ptr[t];
        const int n = (int)(P.tile_ptr[t + 1] - base);
        const int b = P.bw[t];
        const int Wn = b + 2, pitch = Wn | 1, bw1 = b + 1;
        const double *Xf = P.X + (int64_t)f * P.nstate2d * N;
        double *Xaf = P.Xa + (int64_t)f * P.nstate2d * N;
        const double *Tf = P.T + (int64_t)f * P.nnz;
        const double *Df = P.D + (int64_t)f * P.nloc + base;
        const int32_t *slotf = P.obs_slot + (int64_t)f * P.nloc + base;
        const int32_t *phys = P.phys + base, *iphys = P.iphys + base, *srow = P.state_row + base;
        const uint8_t *inter = P.is_interior + base;

        if (!P.assemble_only && P.tile_nobs[(int64_t)f * P.ntiles + t] == 0) {   // kernels.py:179-180: exact copy
            for (int j = warp; j < n; j += nwarps) {
                if (!inter[j]) continue;
                const int64_t g = (int64_t)srow[j] * N;
                for (int m = lane; m < N; m += 32) Xaf[g + m] = Xf[g + m];
            }
            if (tid == 0) P.status[(int64_t)f * P.ntiles + t] = 0;
            continue;
        }

        // ---- phase A: assemble the band, one warp per column I (physical index) ---------
        {
            double *acc = sm_rest + (size_t)warp * (bmax + 1);   // aliases the window: not live yet
            for (int I = warp; I < n; I += nwarps) {
                for (int d = lane; d <= b; d += 32) acc[d] = 0.0;
                __syncwarp();
                const int i = iphys[I];
                const int64_t c0 = P.csc_ptr[base + i], c1 = P.csc_ptr[base + i + 1];
                for (int64_t e = c0 - 1; e < c1; ++e) {
                    int j; double tji;
                    if (e < c0) { j = i; tji = 1.0; } else { j = P.csc_row[e]; tji = Tf[P.csc_src[e]]; }
                    const double s = tji / Df[j];
                    const int64_t q0 = P.row_ptr[base + j];
                    const int cnt = (int)(P.row_ptr[base + j + 1] - q0);
                    for (int m = lane - 1; m < cnt; m += 32) {
                        int k; double tjk;
                        if (m < 0) { k = j; tjk = 1.0; } else { k = P.col_idx[q0 + m]; tjk = Tf[q0 + m]; }
                        const int Kp = phys[k];
                        if (Kp >= I) acc[Kp - I] += s * tjk;
                    }
                    __syncwarp();
                }
                if (lane == 0 && !P.assemble_only) { const int sl = slotf[i]; if (sl >= 0) acc[0] += 1.0 / P.rdiag[sl]; }
                __syncwarp();
                for (int d = lane; d <= b; d += 32) Acol[(int64_t)I * bw1 + d] = acc[d];
                __syncwarp();
            }
        }
        __syncthreads();
        if (P.assemble_only) {
            for (int64_t e = tid; e < (int64_t)n * bw1; e += nthreads) P.band_out[e] = Acol[e];
            continue;
        }

        // window accessors (circular in both indices)
#define AW(I, K) Aw[(size_t)((I) % Wn) * pitch + ((K) % Wn)]
#define RW(I, m) Rw[(size_t)((I) % Wn) * N + (m)]
        // load physical row R of the band and of the right-hand side into the window
        auto load_row = [&](int R) {
            const int klo = R - b > 0 ? R - b : 0;
            for (int K = klo + tid; K <= R; K += nthreads) AW(R, K) = Acol[(int64_t)K * bw1 + (R - K)];
            const int i = iphys[R];
            const int sl = slotf[i];
            if (sl >= 0) {
                const double rinv = 1.0 / P.rdiag[sl];
                const double *ys = P.Ys + (int64_t)sl * N;
                const double *xb = Xf + (int64_t)srow[i] * N;
                for (int m = tid; m < N; m += nthreads) RW(R, m) = (ys[m] - xb[m]) * rinv;
            } else {
                for (int m = tid; m < N; m += nthreads) RW(R, m) = 0.0;
            }
        };
        for (int R = 0; R <= b && R < n; ++R) load_row(R);
        __syncthreads();

        // ---- phase B: banded Cholesky + forward substitution ----------------------------
        const int ty = tid >> 4, tx = tid & 15;
        const int da = nthreads / N, dm = nthreads % N;
        for (int k = 0; k < n; ++k) {
            const int hi = (k + b < n - 1) ? k + b : n - 1;
            const int cnt = hi - k;
            const double piv = AW(k, k);
            if (!(piv > 0.0) || !(piv < DBL_MAX)) { if (tid == 0) s_fail = (piv == piv) ? 1 : 2; }
            const double lkk = sqrt(piv), inv = 1.0 / lkk;
            // column k of L -> lk[] and global; z_k -> window (scaled) and global
            for (int a = tid; a < cnt; a += nthreads) {
                const double v = AW(k + 1 + a, k) * inv;
                lk[a] = v;
                Acol[(int64_t)k * bw1 + 1 + a] = v;
            }
            if (tid == 0) Acol[(int64_t)k * bw1] = lkk;
            for (int m = tid; m < N; m += nthreads) {
                const double z = RW(k, m) * inv;
                RW(k, m) = z;
                Z[(int64_t)k * N + m] = z;
            }
            __syncthreads();
            if (s_fail) break;
            // trailing update of the (cnt x cnt) lower triangle (window indices wrap at Wn)
            const int k1 = (k + 1) % Wn, k0 = k % Wn;
            for (int a = ty; a < cnt; a += SOLVE_THREADS / 16) {
                const double la = lk[a];
                int ra = k1 + a; if (ra >= Wn) ra -= Wn;
                double *row = Aw + (size_t)ra * pitch;
                for (int c = tx; c <= a; c += 16) {
                    int cc = k1 + c; if (cc >= Wn) cc -= Wn;
                    row[cc] -= la * lk[c];
                }
            }
            // right-hand sides of rows k+1..hi
            {
                const double *zk = Rw + (size_t)k0 * N;
                int a = tid / N, m = tid % N;
                while (a < cnt) {
                    int ra = k1 + a; if (ra >= Wn) ra -= Wn;
                    Rw[(size_t)ra * N + m] -= lk[a] * zk[m];
                    a += da; m += dm;
                    if (m >= N) { m -= N; ++a; }
                }
            }
            // bring in the next row (its slot held row k-1, already retired)
            if (k + b + 1 < n) load_row(k + b + 1);
            __syncthreads();
        }
        if (s_fail) {
            if (tid == 0) P.status[(int64_t)f * P.ntiles + t] = s_fail;
            continue;
        }

        // ---- phase C: backward substitution, Xa = Xb + dx on interior rows -------------
        const int parts = nthreads / N > 0 ? nthreads / N : 1;
        {
            const int k = n - 1;
            for (int d = tid; d < 1; d += nthreads) lk[d] = Acol[(int64_t)k * bw1 + d];
        }
        __syncthreads();
        for (int k = n - 1; k >= 0; --k) {
            const int hi = (k + b < n - 1) ? k + b : n - 1;
            const int cnt = hi - k;
            const double *lcur = lk + ((n - 1 - k) & 1) * (bmax + 2);
            double *lnext = lk + ((n - k) & 1) * (bmax + 2);
            // partial dot products over the already-solved rows k+1..hi
            {
                const int m = tid % N, part = tid / N;
                double s = 0.0;
                if (part < parts) for (int d = 1 + part; d <= cnt; d += parts) s += lcur[d] * RW(k + d, m);
                if (part < parts) red[part * N + m] = s;
            }
            // prefetch column k-1 of L
            if (k > 0) {
                const int hi2 = (k - 1 + b < n - 1) ? k - 1 + b : n - 1;
                for (int d = tid; d <= hi2 - (k - 1); d += nthreads) lnext[d] = Acol[(int64_t)(k - 1) * bw1 + d];
            }
            __syncthreads();
            if (tid < N) {
                double s = Z[(int64_t)k * N + tid];
                for (int pt = 0; pt < parts; ++pt) s -= red[pt * N + tid];
                const double x = s / lcur[0];
                RW(k, tid) = x;
                const int i = iphys[k];
                if (inter[i]) {
                    const int64_t g = (int64_t)srow[i] * N + tid;
                    Xaf[g] = Xf[g] + x;
                }
            }
            __syncthreads();
        }
        if (tid == 0) P.status[(int64_t)f * P.ntiles + t] = 0;
#undef AW
#undef RW
    }
}

// Scratch / shared-memory layout chosen on the host.
int64_t solve_plan_scratch(SolveParams &p, int64_t max_band_doubles, int64_t nmax, size_t smem_limit) {
    const int64_t Wn = p.bmax + 2, pitch = Wn | 1;
    const size_t fixed = (size_t)(2 * (p.bmax + 2) + SOLVE_THREADS) * sizeof(double) + 64;
    const size_t a_bytes = (size_t)(Wn * pitch) * sizeof(double);
    const size_t r_bytes = (size_t)(Wn * p.N) * sizeof(double);
    const size_t acc_bytes = (size_t)(SOLVE_THREADS / 32) * (p.bmax + 1) * sizeof(double);
    p.a_in_smem = fixed + a_bytes <= smem_limit;
    p.r_in_smem = fixed + (p.a_in_smem ? a_bytes : 0) + r_bytes <= smem_limit;
    (void)acc_bytes;
    int64_t off = max_band_doubles;
    p.off_z = off; off += nmax * p.N;
    p.off_win_a = off; if (!p.a_in_smem) off += Wn * pitch;
    p.off_win_r = off; if (!p.r_in_smem) off += Wn * p.N;
    off = (off + 15) & ~(int64_t)15;
    p.scratch_stride = off;
    return off;
}

static size_t solve_smem_bytes(const SolveParams &p) {
    const int64_t Wn = p.bmax + 2, pitch = Wn | 1;
    size_t rest = 0;
    if (p.a_in_smem) rest += (size_t)(Wn * pitch);
    if (p.r_in_smem) rest += (size_t)(Wn * p.N);
    const size_t acc = (size_t)(SOLVE_THREADS / 32) * (p.bmax + 1);
    if (rest < acc) rest = acc;
    return (size_t)(2 * (p.bmax + 2) + SOLVE_THREADS + rest) * sizeof(double);
}

int solve_grid_size(int sm_count, const SolveParams &p, size_t smem_limit) {
    const size_t smem = solve_smem_bytes(p) + 1024;
    int per_sm = (int)((smem_limit + 1024) / smem);
    if (per_sm < 1) per_sm = 1;
    if (per_sm > 4) per_sm = 4;
    int64_t grid = (int64_t)sm_count * per_sm;
    const int64_t items = (int64_t)p.nfields * p.ntiles;
    if (grid > items) grid = items;
    return (int)(grid < 1 ? 1 : grid);
}

cudaError_t launch_local_solve(const SolveParams &p, int grid, size_t smem_limit, cudaStream_t s) {
    if (p.nfields * p.ntiles == 0) return cudaSuccess;
    const size_t smem = solve_smem_bytes(p);
    if (smem > smem_limit) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(local_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(p.counter, 0, sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
    local_solve_kernel<<<grid, SOLVE_THREADS, smem, s>>>(p);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// Row gather/scatter (merge_interiors, driver.py:116) and matrix-free T^T D^-1 T v
// (factors.py:86-96).  Bandwidth-bound helpers; one warp per row.
// ------------------------------------------------------------------------------------------
__global__ void scatter_rows_kernel(double *__restrict__ dst, const int64_t *__restrict__ dst_rows,
                                    const double *__restrict__ src, const int64_t *__restrict__ src_rows,
                                    int64_t nrows, int N) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < nrows; r += warps) {
        const double *s = src + src_rows[r] * N;
        double *d = dst + dst_rows[r] * N;
        for (int i = lane; i < N; i += 32) d[i] = s[i];
    }
}

cudaError_t launch_scatter_rows(double *dst, const int64_t *dst_rows, const double *src, const int64_t *src_rows,
                                int64_t nrows, int N, cudaStream_t s) {
    if (nrows == 0) return cudaSuccess;
    int64_t blocks = (nrows + 7) / 8;
    if (blocks > 148 * 16) blocks = 148 * 16;
    scatter_rows_kernel<<<(unsigned)blocks, 256, 0, s>>>(dst, dst_rows, src, src_rows, nrows, N);
    return cudaGetLastError();
}

__global__ void precision_apply_kernel(int phase, const int64_t *__restrict__ ptr, const int32_t *__restrict__ idx,
                                       const int64_t *__restrict__ src, const double *__restrict__ T,
                                       const double *__restrict__ D, const double *__restrict__ V,
                                       double *__restrict__ Out, int64_t n, int64_t ncols) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
        for (int64_t c = lane; c < ncols; c += 32) {
            double acc = V[r * ncols + c];
            for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
                const double t = T[src ? src[e] : e];
                acc += t * V[(int64_t)idx[e] * ncols + c];
            }
            Out[r * ncols + c] = phase == 0 ? acc / D[r] : acc;
        }
    }
}

cudaError_t launch_precision_apply(const int64_t *row_ptr, const int32_t *col_idx, const int64_t *csc_ptr,
                                   const int32_t *csc_row, const int64_t *csc_src, const double *T, const double *D,
                                   const double *V, double *Wtmp, double *Out, int64_t n, int64_t ncols, cudaStream_t s) {
    if (n == 0 || ncols == 0) return cudaSuccess;
    int64_t blocks = (n + 7) / 8;
    if (blocks > 148 * 16) blocks = 148 * 16;
    precision_apply_kernel<<<(unsigned)blocks, 256, 0, s>>>(0, row_ptr, col_idx, nullptr, T, D, V, Wtmp, n, ncols);
    precision_apply_kernel<<<(unsigned)blocks, 256, 0, s>>>(1, csc_ptr, csc_row, csc_src, T, D, Wtmp, Out, n, ncols);
    return cudaGetLastError();
}
