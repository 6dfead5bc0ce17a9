// sm_100a kernels of the EnKF-MC analysis step.  FP64 throughout (the reference has no
// reduced precision anywhere).  tcgen05 has no FP64 kind; wherever the work forms
// 8 x 8 blocks it runs on the FP64 tensor cores through mma.sync.m8n8k4.f64 (DMMA), the rest is
// SIMT.  Persistent CTAs (one per SM) fetch work items from an atomic counter.
//
//   K0  center_rows_kernel                       validation.py:35-39
//   K2a regress_qr_mma_kernel / regress_qr_kernel  estimator.py:46-61,133-150 (the QR half)
//   K2b regress_clean_kernel / regress_trunc_kernel (regress_solve.cuh)   estimator.py:46-61 (truncated-SVD semantics) + factors.py:60
//   K3a assemble_band_tile_kernel / assemble_band_kernel   factors.py:136-145, kernels.py:189-191
//   K3b local_solve_kernel                       kernels.py:178-218, driver.py:99-125
//
// All results are deterministic run to run: no floating-point atomics, fixed reduction
// trees, work items are independent.

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>

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
// K2: per-component regression (estimator.py:46-61,133-150 + factors.py:60), one warp per
// regression, in two kernels so that each phase runs at its own occupancy.
//
// K2a: Householder QR of [A^T | y] (N x (p + 1); column j < p is predecessor j's anomaly vector, the
//   last column the target y) without pivoting.  Output per regression, packed in global scratch:
//   R by columns (min(j+1, K) entries of column j), c = (Q^T y)[0:K] and e2 = |(Q^T y)[K:N]|^2 --
//   the squared residual of the full least-squares fit.  Two forms: regress_qr_mma_kernel (N <= 128:
//   column blocks in tensor-core fragment layout in registers, described at its definition) and
//   regress_qr_kernel (any N <= 256: W in shared memory, column-major, odd pitch; lanes own rows
//   in S = ceil(N / 32) register slots, two reflectors per sweep, eight columns share two
//   transposing warp reductions).
//
// K2b regress_clean_kernel + regress_trunc_kernel: regress_solve.cuh (certificate and plain solve; block inverse
//   iteration + Rayleigh-Ritz for the rows that truncate; one-sided Jacobi SVD as the general fallback).
// ------------------------------------------------------------------------------------------

__host__ __device__ inline size_t regress_qr_ws_doubles(int N, int pmax) {
    const size_t d = (size_t)(N | 1) * (pmax + 1) + (size_t)pmax + 2;   // W | rdiag
    return (d + 1) & ~(size_t)1;
}
size_t regress_warp_workspace_doubles(int N, int pmax) { return regress_qr_ws_doubles(N, pmax); }

namespace {

// All-reduce of four per-lane partial sums: every lane returns with the four warp totals.
__device__ __forceinline__ void warp_sum4(double &d0, double &d1, double &d2, double &d3, int lane) {
    const bool hi = lane & 16;
    double s0 = hi ? d0 : d2, s1 = hi ? d1 : d3;
    double k0 = hi ? d2 : d0, k1 = hi ? d3 : d1;
    k0 += __shfl_xor_sync(FULL, s0, 16);
    k1 += __shfl_xor_sync(FULL, s1, 16);
    const bool b8 = lane & 8;
    const double send = b8 ? k0 : k1;
    double t = (b8 ? k1 : k0) + __shfl_xor_sync(FULL, send, 8);
    t += __shfl_xor_sync(FULL, t, 4);
    t += __shfl_xor_sync(FULL, t, 2);
    t += __shfl_xor_sync(FULL, t, 1);
    d0 = __shfl_sync(FULL, t, 0);    // bit4 = 0, bit3 = 0
    d1 = __shfl_sync(FULL, t, 8);    // bit4 = 0, bit3 = 1
    d2 = __shfl_sync(FULL, t, 16);   // bit4 = 1, bit3 = 0
    d3 = __shfl_sync(FULL, t, 24);
}

// One Householder step on columns [jbeg, p] of W.  Rows below 32*S0 are final (all < k) and are
// skipped; rows in [32*S0, k) carry v = 0, so re-storing them is exact.  NB columns per batch.
template <int S, int S0, int NB>
__device__ __forceinline__ void qr_apply(double *Wl, int ld, int jbeg, int jend, const double (&v)[S], double tau,
                                         bool tail_ok, int lane) {
    // Wl = W + lane ; tail_ok: row lane + 32 (S-1) exists (< N)
    double *col = Wl + (size_t)jbeg * ld;
    for (int j0 = jbeg; j0 + NB <= jend; j0 += NB, col += (size_t)NB * ld) {
        double c[NB][S], d[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            d[b] = 0.0;
#pragma unroll
            for (int s = S0; s < S; ++s) {
                c[b][s] = (s < S - 1 || tail_ok) ? col[(size_t)b * ld + 32 * s] : 0.0;
                d[b] += v[s] * c[b][s];
            }
        }
#pragma unroll
        for (int b = 0; b < NB; b += 4) warp_sum4(d[b], d[b + 1], d[b + 2], d[b + 3], lane);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const double w = d[b] * tau;
#pragma unroll
            for (int s = S0; s < S; ++s)
                if (s < S - 1 || tail_ok) col[(size_t)b * ld + 32 * s] = c[b][s] - w * v[s];
        }
    }
}

template <int S, int S0>
__device__ __forceinline__ void qr_step(double *W, int ld, int N, int k, int p, double *rdiag, int lane) {
    const bool tail_ok = lane + 32 * (S - 1) < N;
    double *Wl = W + lane;
    const double *ck = Wl + (size_t)k * ld;
    double v[S];
    double ss = 0.0;
#pragma unroll
    for (int s = 0; s < S; ++s) v[s] = 0.0;
#pragma unroll
    for (int s = S0; s < S; ++s) {
        const int i = lane + 32 * s;
        v[s] = (i >= k && (s < S - 1 || tail_ok)) ? ck[32 * s] : 0.0;
        ss += v[s] * v[s];
    }
    ss = warp_sum(ss);
    const double x0 = W[(size_t)k * ld + k];
    const double nrm = sqrt(ss);
    if (nrm == 0.0) {
        if (lane == 0) rdiag[k] = 0.0;
        return;
    }
    const double alpha = (x0 >= 0.0) ? -nrm : nrm;
    const double tau = 1.0 / (nrm * (nrm + fabs(x0)));   // 2 / v^T v
#pragma unroll
    for (int s = S0; s < S; ++s) if (lane + 32 * s == k) v[s] = x0 - alpha;
    if (lane == 0) rdiag[k] = alpha;
    // columns k+1 .. p (p = the y column): batches of 8, then 4, then a clamped batch of 4
    const int jend = p + 1;
    int j = k + 1;
    const int n8 = (jend - j) & ~7;
    qr_apply<S, S0, 8>(Wl, ld, j, j + n8, v, tau, tail_ok, lane);
    j += n8;
    if (jend - j >= 4) { qr_apply<S, S0, 4>(Wl, ld, j, j + 4, v, tau, tail_ok, lane); j += 4; }
    if (j < jend) {
        double c[4][S], d[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const double *col = Wl + (size_t)(j + b < jend ? j + b : jend - 1) * ld;
            d[b] = 0.0;
#pragma unroll
            for (int s = S0; s < S; ++s) {
                c[b][s] = (s < S - 1 || tail_ok) ? col[32 * s] : 0.0;
                d[b] += v[s] * c[b][s];
            }
        }
        warp_sum4(d[0], d[1], d[2], d[3], lane);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            if (j + b >= jend) break;
            double *col = Wl + (size_t)(j + b) * ld;
            const double w = d[b] * tau;
#pragma unroll
            for (int s = S0; s < S; ++s)
                if (s < S - 1 || tail_ok) col[32 * s] = c[b][s] - w * v[s];
        }
    }
}

// Two Householder steps (k, k+1) in one sweep over the trailing columns: each column is read and
// written once for two reflectors (halves the shared-memory traffic of the one-step version).
//   c' = H1 c = c - w1 v1,  w1 = tau1 v1.c ;  c'' = H2 c' = c' - w2 v2,  w2 = tau2 (v2.c - w1 v2.v1)
template <int S, int S0, int NB>
__device__ __forceinline__ void qr_apply2(double *Wl, int ld, int jbeg, int jend, const double (&v1)[S],
                                          const double (&v2)[S], double tau1, double tau2, double g, bool tail_ok,
                                          int lane) {
    double *col = Wl + (size_t)jbeg * ld;
    for (int j0 = jbeg; j0 + NB <= jend; j0 += NB, col += (size_t)NB * ld) {
        double c[NB][S], d1[NB], d2[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            d1[b] = 0.0; d2[b] = 0.0;
#pragma unroll
            for (int s = S0; s < S; ++s) {
                c[b][s] = (s < S - 1 || tail_ok) ? col[(size_t)b * ld + 32 * s] : 0.0;
                d1[b] += v1[s] * c[b][s];
                d2[b] += v2[s] * c[b][s];
            }
        }
#pragma unroll
        for (int b = 0; b < NB; b += 4) {
            warp_sum4(d1[b], d1[b + 1], d1[b + 2], d1[b + 3], lane);
            warp_sum4(d2[b], d2[b + 1], d2[b + 2], d2[b + 3], lane);
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const double w1 = d1[b] * tau1;
            const double w2 = (d2[b] - w1 * g) * tau2;
#pragma unroll
            for (int s = S0; s < S; ++s)
                if (s < S - 1 || tail_ok) col[(size_t)b * ld + 32 * s] = c[b][s] - w1 * v1[s] - w2 * v2[s];
        }
    }
}

template <int S, int S0>
__device__ __forceinline__ void qr_step2(double *W, int ld, int N, int k, int p, double *rdiag, int lane) {
    const bool tail_ok = lane + 32 * (S - 1) < N;
    double *Wl = W + lane;
    // reflector 1 from column k
    double v1[S], v2[S], c[S];
    double ss = 0.0, x0 = 0.0;
#pragma unroll
    for (int s = 0; s < S; ++s) { v1[s] = 0.0; v2[s] = 0.0; c[s] = 0.0; }
    const double *ck = Wl + (size_t)k * ld, *ck1 = Wl + (size_t)(k + 1) * ld;
    double dc = 0.0;
#pragma unroll
    for (int s = S0; s < S; ++s) {
        const int i = lane + 32 * s;
        const bool live = (s < S - 1 || tail_ok);
        v1[s] = (i >= k && live) ? ck[32 * s] : 0.0;
        c[s] = live ? ck1[32 * s] : 0.0;
        ss += v1[s] * v1[s];
        if (i == k) x0 = v1[s];
        dc += v1[s] * c[s];                       // raw v1 . c, corrected below for the modified v1[k]
    }
    double ck_k = 0.0;                            // c at row k
#pragma unroll
    for (int s = S0; s < S; ++s) if (lane + 32 * s == k) ck_k = c[s];
    warp_sum4(ss, x0, dc, ck_k, lane);
    const double nrm1 = sqrt(ss);
    const double alpha1 = nrm1 == 0.0 ? 0.0 : ((x0 >= 0.0) ? -nrm1 : nrm1);
    const double tau1 = nrm1 == 0.0 ? 0.0 : 1.0 / (nrm1 * (nrm1 + fabs(x0)));
#pragma unroll
    for (int s = S0; s < S; ++s) if (lane + 32 * s == k) v1[s] = x0 - alpha1;
    // column k+1 through H1 (v1.c with the final v1[k] = x0 - alpha1: dc - alpha1 * c[k])
    const double w1c = (dc - alpha1 * ck_k) * tau1;
    double ss2 = 0.0, y0 = 0.0, graw = 0.0, v1k1 = 0.0;
#pragma unroll
    for (int s = S0; s < S; ++s) {
        const int i = lane + 32 * s;
        c[s] -= w1c * v1[s];
        if (i == k) Wl[(size_t)(k + 1) * ld + 32 * s] = c[s];         // R[k][k+1] is final
        v2[s] = (i >= k + 1) ? c[s] : 0.0;
        if (s == S - 1 && !tail_ok) v2[s] = 0.0;
        ss2 += v2[s] * v2[s];
        graw += v2[s] * v1[s];
        if (i == k + 1) { y0 = v2[s]; v1k1 = v1[s]; }
    }
    warp_sum4(ss2, y0, graw, v1k1, lane);
    const double nrm2 = sqrt(ss2);
    const double alpha2 = nrm2 == 0.0 ? 0.0 : ((y0 >= 0.0) ? -nrm2 : nrm2);
    const double tau2 = nrm2 == 0.0 ? 0.0 : 1.0 / (nrm2 * (nrm2 + fabs(y0)));
#pragma unroll
    for (int s = S0; s < S; ++s) if (lane + 32 * s == k + 1) v2[s] = y0 - alpha2;
    const double g = graw - alpha2 * v1k1;        // v2 . v1 with the final v2[k+1]
    if (lane == 0) { rdiag[k] = alpha1; rdiag[k + 1] = alpha2; }
    // remaining columns k+2 .. p
    const int jend = p + 1;
    int j = k + 2;
    const int n8 = (jend - j) & ~7;
    qr_apply2<S, S0, 8>(Wl, ld, j, j + n8, v1, v2, tau1, tau2, g, tail_ok, lane);
    j += n8;
    if (jend - j >= 4) { qr_apply2<S, S0, 4>(Wl, ld, j, j + 4, v1, v2, tau1, tau2, g, tail_ok, lane); j += 4; }
    if (j < jend) {
        double cc[4][S], d1[4], d2[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const double *col = Wl + (size_t)(j + b < jend ? j + b : jend - 1) * ld;
            d1[b] = 0.0; d2[b] = 0.0;
#pragma unroll
            for (int s = S0; s < S; ++s) {
                cc[b][s] = (s < S - 1 || tail_ok) ? col[32 * s] : 0.0;
                d1[b] += v1[s] * cc[b][s];
                d2[b] += v2[s] * cc[b][s];
            }
        }
        warp_sum4(d1[0], d1[1], d1[2], d1[3], lane);
        warp_sum4(d2[0], d2[1], d2[2], d2[3], lane);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            if (j + b >= jend) break;
            double *col = Wl + (size_t)(j + b) * ld;
            const double w1 = d1[b] * tau1;
            const double w2 = (d2[b] - w1 * g) * tau2;
#pragma unroll
            for (int s = S0; s < S; ++s)
                if (s < S - 1 || tail_ok) col[32 * s] = cc[b][s] - w1 * v1[s] - w2 * v2[s];
        }
    }
}

// Advances k by the number of reflectors applied (2 while two columns remain, else 1).
template <int S>
__device__ __forceinline__ int qr_step_dispatch(double *W, int ld, int N, int k, int K, int p, double *rdiag, int lane) {
    const bool two = k + 1 < K;
    if constexpr (S <= 4) {
        switch (k >> 5) {
            case 0: if (two) qr_step2<S, 0>(W, ld, N, k, p, rdiag, lane); else qr_step<S, 0>(W, ld, N, k, p, rdiag, lane); break;
            case 1: if constexpr (S > 1) { if (two) qr_step2<S, 1>(W, ld, N, k, p, rdiag, lane); else qr_step<S, 1>(W, ld, N, k, p, rdiag, lane); } break;
            case 2: if constexpr (S > 2) { if (two) qr_step2<S, 2>(W, ld, N, k, p, rdiag, lane); else qr_step<S, 2>(W, ld, N, k, p, rdiag, lane); } break;
            default: if constexpr (S > 3) { if (two) qr_step2<S, 3>(W, ld, N, k, p, rdiag, lane); else qr_step<S, 3>(W, ld, N, k, p, rdiag, lane); } break;
        }
    } else {
        if (two) qr_step2<S, 0>(W, ld, N, k, p, rdiag, lane); else qr_step<S, 0>(W, ld, N, k, p, rdiag, lane);
    }
    return two ? 2 : 1;
}

// p-vectors live in registers: element e <-> lane e & 31, slot e >> 5 (PS slots).
template <int PS>
struct Vec {
    double v[PS];
};

template <int PS>
__device__ __forceinline__ double vdot(const Vec<PS> &a, const Vec<PS> &b) {
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < PS; ++t) s += a.v[t] * b.v[t];
    return warp_sum(s);
}

template <int PS>
__device__ __forceinline__ Vec<PS> vload(const double *src, int p, int lane) {
    Vec<PS> r;
#pragma unroll
    for (int t = 0; t < PS; ++t) { const int e = lane + 32 * t; r.v[t] = e < p ? src[e] : 0.0; }
    return r;
}

template <int PS>
__device__ __forceinline__ void vstore(double *dst, const Vec<PS> &a, int p, int lane) {
#pragma unroll
    for (int t = 0; t < PS; ++t) { const int e = lane + 32 * t; if (e < p) dst[e] = a.v[t]; }
}

// x = R^-1 b  (R upper triangular in W, diagonal reciprocals in rinv); b is overwritten.
// (called, not inlined: several call sites)
template <int PS>
__device__ __noinline__ Vec<PS> solve_upper(Vec<PS> b, const double *W, const double *rinv, int ld, int p, int lane) {
    // element k is final when column k is reached and never touched again: x = b * rinv once at the end
    const Vec<PS> rv = vload<PS>(rinv, p, lane);
#pragma unroll
    for (int sk = PS - 1; sk >= 0; --sk) {
        const int ktop = (p - 32 * sk < 32 ? p - 32 * sk : 32) - 1;
        const double *col = W + (size_t)(32 * sk + ktop) * ld + lane;
        for (int kk = ktop; kk >= 0; --kk, col -= ld) {
            const int k = 32 * sk + kk;
            const double xk = __shfl_sync(FULL, b.v[sk] * rv.v[sk], kk);
#pragma unroll
            for (int t = 0; t <= sk; ++t)
                if (lane + 32 * t < k) b.v[t] -= col[32 * t] * xk;
        }
    }
#pragma unroll
    for (int t = 0; t < PS; ++t) b.v[t] *= rv.v[t];
    return b;
}

// u = R^-T z ; z is overwritten.
template <int PS>
__device__ __noinline__ Vec<PS> solve_upper_t(Vec<PS> z, const double *W, const double *rinv, int ld, int p, int lane) {
    const Vec<PS> rv = vload<PS>(rinv, p, lane);
#pragma unroll
    for (int sk = 0; sk < PS; ++sk) {
        const int kend = p - 32 * sk < 32 ? p - 32 * sk : 32;
        const double *row = W + 32 * sk + (size_t)lane * ld;   // R[k, lane + 32 t] = row[kk + 32 t ld]
        for (int kk = 0; kk < kend; ++kk) {
            const int k = 32 * sk + kk;
            const double uk = __shfl_sync(FULL, z.v[sk] * rv.v[sk], kk);
#pragma unroll
            for (int t = sk; t < PS; ++t) {
                const int j = lane + 32 * t;
                if (j > k && j < p) z.v[t] -= row[kk + (size_t)32 * t * ld] * uk;
            }
        }
    }
#pragma unroll
    for (int t = 0; t < PS; ++t) z.v[t] *= rv.v[t];
    return z;
}

// y = R v
template <int PS>
__device__ __noinline__ Vec<PS> mul_upper(const Vec<PS> v, const double *W, int ld, int p, int lane) {
    Vec<PS> y;
#pragma unroll
    for (int t = 0; t < PS; ++t) y.v[t] = 0.0;
#pragma unroll
    for (int sj = 0; sj < PS; ++sj) {
        const int jend = p - 32 * sj < 32 ? p - 32 * sj : 32;
        const double *col = W + (size_t)(32 * sj) * ld + lane;
        for (int jj = 0; jj < jend; ++jj, col += ld) {
            const int j = 32 * sj + jj;
            const double vj = __shfl_sync(FULL, v.v[sj], jj);
#pragma unroll
            for (int t = 0; t <= sj; ++t)
                if (lane + 32 * t <= j) y.v[t] += col[32 * t] * vj;
        }
    }
    return y;
}

// w = R^T y
template <int PS>
__device__ __noinline__ Vec<PS> mul_upper_t(const Vec<PS> y, const double *W, int ld, int p, int lane) {
    Vec<PS> w;
#pragma unroll
    for (int t = 0; t < PS; ++t) w.v[t] = 0.0;
#pragma unroll
    for (int si = 0; si < PS; ++si) {
        const int iend = p - 32 * si < 32 ? p - 32 * si : 32;
        const double *row = W + 32 * si + (size_t)lane * ld;
        for (int ii = 0; ii < iend; ++ii) {
            const int i = 32 * si + ii;
            const double yi = __shfl_sync(FULL, y.v[si], ii);
#pragma unroll
            for (int t = si; t < PS; ++t) {
                const int j = lane + 32 * t;
                if (j >= i && j < p) w.v[t] += row[ii + (size_t)32 * t * ld] * yi;
            }
        }
    }
    return w;
}

// Single reflector per call (column k keeps its tail below the diagonal: the reflector can be rebuilt later).
template <int S>
__device__ __forceinline__ void qr_step1_dispatch(double *W, int ld, int N, int k, int plast, double *rdiag, int lane) {
    if constexpr (S <= 4) {
        switch (k >> 5) {
            case 0: qr_step<S, 0>(W, ld, N, k, plast, rdiag, lane); break;
            case 1: if constexpr (S > 1) qr_step<S, 1>(W, ld, N, k, plast, rdiag, lane); break;
            case 2: if constexpr (S > 2) qr_step<S, 2>(W, ld, N, k, plast, rdiag, lane); break;
            default: if constexpr (S > 3) qr_step<S, 3>(W, ld, N, k, plast, rdiag, lane); break;
        }
    } else {
        qr_step<S, 0>(W, ld, N, k, plast, rdiag, lane);
    }
}

}  // namespace

#include "regress_solve.cuh"


// ---- K2a: load + Householder QR ------------------------------------------------------------
template <int S>
__global__ void __launch_bounds__(256, 1) regress_qr_kernel(const RegressParams P) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31;
    const int N = P.N, ld = P.ld, pmax = P.pmax;
    double *W = smem + (size_t)(threadIdx.x >> 5) * regress_qr_ws_doubles(N, pmax);
    double *rdiag = W + (size_t)ld * (pmax + 1);
    const double denom = (double)(N - 1);
    const unsigned nf = (unsigned)(P.f1 - P.f0);

    for (;;) {
        unsigned int wk = 0;
        if (lane == 0) wk = atomicAdd(P.counter, 1u);
        wk = __shfl_sync(FULL, wk, 0);
        if ((int64_t)wk >= P.nwork) break;
        const int q = P.work_order[wk / nf];
        const int fl = (int)(wk % nf), f = P.f0 + fl;
        const int64_t r0 = P.row_ptr[q];
        const int p = (int)(P.row_ptr[q + 1] - r0);
        const double *Uf = P.U + (int64_t)f * P.nstate2d * N;
        const double *yrow = Uf + (int64_t)P.state_row[q] * N;
        const int32_t *pred = P.pred_state + r0;

        if (p == 0) {  // estimator.py:139-144
            double s = 0.0;
            for (int i = lane; i < N; i += 32) { const double v = yrow[i]; s += v * v; }
            s = warp_sum(s) / denom;
            if (lane == 0) {
                P.D[(int64_t)f * P.dstride + q] = fmax(s, P.variance_floor);
                if (P.flags) P.flags[(int64_t)f * P.dstride + q] = (s < P.variance_floor) ? 8 : 0;
            }
            continue;
        }
        for (int j = 0; j <= p; ++j) {
            const double *src = (j < p) ? Uf + (int64_t)pred[j] * N : yrow;
            double *dst = W + (size_t)j * ld;
#pragma unroll
            for (int s = 0; s < S; ++s) { const int i = lane + 32 * s; if (i < N) dst[i] = src[i]; }
        }
        __syncwarp();
        const int K = p < N ? p : N;
        for (int k = 0; k < K;) {
            k += qr_step_dispatch<S>(W, ld, N, k, K, p, rdiag, lane);
            __syncwarp();
        }
        // packed output: R by columns, then c[0:K], then e2
        double *out = P.Rq + (int64_t)fl * P.rq_stride + P.rq_ptr[q];
        for (int j = 0; j < p; ++j) {
            const int h = j + 1 < K ? j + 1 : K;
            const double *col = W + (size_t)j * ld;
            double *dst = out + packed_col_offset(j, K);
            for (int i = lane; i < h; i += 32) dst[i] = (i == j) ? rdiag[j] : col[i];
        }
        double *cdst = out + packed_col_offset(p, K);
        const double *ycol = W + (size_t)p * ld;
        double e2 = 0.0;
        for (int i = lane; i < N; i += 32) {
            const double yv = ycol[i];
            if (i < K) cdst[i] = yv; else e2 += yv * yv;
        }
        e2 = warp_sum(e2);
        if (lane == 0) cdst[K] = e2;
        __syncwarp();
    }
}

// ---- K2a, tensor-core form ---------------------------------------------------------------------
// Blocked Householder QR of [A^T | y] with the block of eight columns in registers in mma.m8n8k4 fragment
// layout: lane (g8, t4) = (lane >> 2, lane & 3) owns column g8 of the block and the rows 8 mt + 4 u + t4
// (m-tile mt, u in {0, 1}).  Earlier reflectors are applied eight at a time in compact WY form,
//     C <- C - V T^T (V^T C),
// as three chains of FP64 tensor-core products whose operands are the column registers themselves and
// fragments of V (reflectors, shared memory) and T (8 x 8 per block, shared memory): with the row <-> n and
// reflector <-> k index maps chosen below, the accumulator fragment of each product is exactly the A fragment
// of the next, so no shuffles or transposes are needed.  The block itself is then factored in registers:
// each reflector is broadcast by shuffles within the lanes sharing t4, one dot product per lane group gives
// the column updates (groups right of the pivot) and the V^T V entries of the T recurrence (groups left of it).
#define QRM_TP 12      // pitch of a T block: B-fragment loads (2 t4 + h) * 12 + g8 are conflict-free

__host__ __device__ constexpr int qrm_vp(int N) {            // reflector pitch: >= 8 ceil(N / 8), = 4 mod 16
    int v = (N + 7) / 8 * 8;
    while (v % 16 != 4) ++v;
    return v;
}
// Reflector block i (reflectors 8 i .. 8 i + 7) is zero above row 8 i: only rows >= 8 i are stored, with a pitch of
// its own (same bank rule).  Offset of block i's storage and its pitch, for rows padded to 8 nt:
__host__ __device__ constexpr int qrm_block_vp(int nt, int i) { return qrm_vp(8 * (nt - i > 1 ? nt - i : 1)); }
__host__ __device__ constexpr int qrm_block_off(int nt, int i) {
    int off = 0;
    for (int k = 0; k < i; ++k) off += 8 * qrm_block_vp(nt, k);
    return off;
}
__host__ __device__ inline size_t regress_qrm_ws_doubles(int nt, int pmax) {
    const int nblk = pmax / 8 > 0 ? pmax / 8 : 1;         // reflector blocks that a later column block can need
    return (size_t)qrm_block_off(nt, nblk) + (size_t)nblk * 8 * QRM_TP;
}

template <int NT>
__global__ void __launch_bounds__(256, 1) regress_qr_mma_kernel(const RegressParams P) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, g8 = lane >> 2, t4 = lane & 3;
    const int N = P.N, pmax = P.pmax;
    const int nblk_cap = pmax / 8 > 0 ? pmax / 8 : 1;      // rows are padded to 8 NT (zeros beyond N)
    double *Vs = smem + (size_t)(threadIdx.x >> 5) * regress_qrm_ws_doubles(NT, pmax);
    double *Ts = Vs + qrm_block_off(NT, nblk_cap);
    const double denom = (double)(N - 1);
    const unsigned nf = (unsigned)(P.f1 - P.f0);
    const int pig = 4 * (g8 & 1) + (g8 >> 1);              // row (within an m-tile) of accumulator column n = g8
    __shared__ int s_voff[16], s_vp[16];                   // offset and pitch of every reflector block (p <= 128)
    if (threadIdx.x < 16) { s_voff[threadIdx.x] = qrm_block_off(NT, threadIdx.x); s_vp[threadIdx.x] = qrm_block_vp(NT, threadIdx.x); }
    __syncthreads();

    for (;;) {
        unsigned int wk = 0;
        if (lane == 0) wk = atomicAdd(P.counter, 1u);
        wk = __shfl_sync(FULL, wk, 0);
        if ((int64_t)wk >= P.nwork) break;
        const int q = P.work_order[wk / nf];
        const int fl = (int)(wk % nf), f = P.f0 + fl;
        const int64_t r0 = P.row_ptr[q];
        const int p = (int)(P.row_ptr[q + 1] - r0);
        const double *Uf = P.U + (int64_t)f * P.nstate2d * N;
        const double *yrow = Uf + (int64_t)P.state_row[q] * N;
        const int32_t *pred = P.pred_state + r0;

        if (p == 0) {  // estimator.py:139-144
            double s = 0.0;
            for (int i = lane; i < N; i += 32) { const double v = yrow[i]; s += v * v; }
            s = warp_sum(s) / denom;
            if (lane == 0) {
                P.D[(int64_t)f * P.dstride + q] = fmax(s, P.variance_floor);
                if (P.flags) P.flags[(int64_t)f * P.dstride + q] = (s < P.variance_floor) ? 8 : 0;
            }
            continue;
        }
        const int K = p < N ? p : N;                     // reflectors
        const int ncols = p + 1;                         // the last column is y
        double *out = P.Rq + (int64_t)fl * P.rq_stride + P.rq_ptr[q];
        double *yout = out + packed_col_offset(p, K);

        // column block starting at column o0, in fragment layout (zeros beyond N rows / ncols columns)
        auto load_block = [&](int o0, auto &dst) {
            const int jc = o0 + g8;
            const double *src = jc < p ? Uf + (int64_t)pred[jc < p ? jc : 0] * N : yrow;
#pragma unroll
            for (int mt = 0; mt < NT; ++mt) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int row = 8 * mt + 4 * u + t4;
                    dst[mt][u] = (jc < ncols && row < N) ? src[row] : 0.0;
                }
            }
        };
        constexpr bool PREFETCH = NT <= 10;            // 16 m-tiles: the second block would spill
        double cn[PREFETCH ? NT : 1][2];
        if constexpr (PREFETCH) load_block(0, cn);
        for (int o = 0; o < ncols; o += 8) {
            const int m0 = o >> 3;                       // m-tile holding the diagonal rows of this block
            const bool stored = o + 8 < ncols;           // a later block will need these reflectors
            const int j_own = o + g8;                    // this lane group's column
            const bool isy = j_own == p;
            double *dst = out + packed_col_offset(j_own < p ? j_own : p, K);
            const int h = j_own < p ? (j_own + 1 < K ? j_own + 1 : K) : 0;    // R entries of my column (0: y or padding)
            double c[NT][2];
            if constexpr (PREFETCH) {
#pragma unroll
                for (int mt = 0; mt < NT; ++mt) { c[mt][0] = cn[mt][0]; c[mt][1] = cn[mt][1]; }
                if (o + 8 < ncols) load_block(o + 8, cn);  // the next block's columns: in flight during this block's work
            } else {
                load_block(o, c);
            }
            // ---- earlier reflector blocks: C <- C - V T^T (V^T C) ----
            for (int ob = 0; ob < o && ob < K; ob += 8) {
                const int mb = ob >> 3;
                const int VP = s_vp[mb];
                const double *Vblk = Vs + s_voff[mb] - 8 * mb;                 // row r of reflector k: Vblk[k * VP + r]
                const double *Vb = Vblk + (size_t)g8 * VP + 2 * (g8 >> 2) + t4;
                double wa0 = 0.0, wa1 = 0.0, wb0 = 0.0, wb1 = 0.0, wc0 = 0.0, wc1 = 0.0, wd0 = 0.0, wd1 = 0.0;
#pragma unroll
                for (int mt = 0; mt < NT; ++mt) {
                    if (mt >= mb) {
                        if (mt & 1) { mma_f64(wc0, wc1, c[mt][0], Vb[8 * mt]); mma_f64(wd0, wd1, c[mt][1], Vb[8 * mt + 4]); }
                        else { mma_f64(wa0, wa1, c[mt][0], Vb[8 * mt]); mma_f64(wb0, wb1, c[mt][1], Vb[8 * mt + 4]); }
                    }
                }
                const double w0 = (wa0 + wb0) + (wc0 + wd0), w1 = (wa1 + wb1) + (wc1 + wd1);   // (C^T V)[g8][2 t4 + {0, 1}]
                const double *Tb = Ts + (size_t)mb * 8 * QRM_TP;
                double z0 = 0.0, z1 = 0.0;                                                    // (C^T V T)[g8][2 t4 + {0, 1}]
                mma_f64(z0, z1, w0, Tb[(2 * t4) * QRM_TP + g8]);
                mma_f64(z0, z1, w1, Tb[(2 * t4 + 1) * QRM_TP + g8]);
                const double *V3 = Vblk + (size_t)(2 * t4) * VP + 2 * (t4 >> 1) + pig;   // reflectors 2 t4, 2 t4 + 1 share the skew
                z0 = -z0; z1 = -z1;
#pragma unroll
                for (int mt = 0; mt < NT; ++mt) {
                    if (mt >= mb) {
                        mma_f64(c[mt][0], c[mt][1], z0, V3[8 * mt]);
                        mma_f64(c[mt][0], c[mt][1], z1, V3[VP + 8 * mt]);
                    }
                }
            }
            // ---- rows above the block are final: write them out and clear them, so that the panel below runs over
            //      all m-tiles without masks (cleared rows contribute nothing) ----
            double dt[2] = {0.0, 0.0};                   // the diagonal m-tile of this lane's column
#pragma unroll
            for (int mt = 0; mt < NT; ++mt) {
                if (mt < m0) {
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int row = 8 * mt + 4 * u + t4;
                        if (row < h) dst[row] = c[mt][u];
                        if (isy && row < K) yout[row] = c[mt][u];
                        c[mt][u] = 0.0;
                    }
                } else if (mt == m0) { dt[0] = c[mt][0]; dt[1] = c[mt][1]; c[mt][0] = 0.0; c[mt][1] = 0.0; }
            }
            // ---- factor the block in registers ----
            const int VPown = s_vp[m0 & 15];
            double *Vown = Vs + s_voff[m0 & 15] - 8 * m0;                     // this block's reflectors, if stored
            double Trow[8];                              // row g8 of the block's T
            double vdiag = 0.0;                          // v[j] of this lane's column (lane holding row j), 0 without a reflector
#pragma unroll
            for (int k = 0; k < 8; ++k) Trow[k] = 0.0;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                const int j = o + jj;
                if (j < p && j < K) {                    // warp-uniform
                    const int src = 4 * jj + t4;
                    double vd[2], vv[NT][2];
                    const double s0 = (t4 >= jj) ? dt[0] : 0.0;                // rows o + t4 and o + 4 + t4 against row j = o + jj
                    const double s1 = (4 + t4 >= jj) ? dt[1] : 0.0;
                    vd[0] = __shfl_sync(FULL, s0, src);
                    vd[1] = __shfl_sync(FULL, s1, src);
#pragma unroll
                    for (int mt = 0; mt < NT; ++mt) {
                        vv[mt][0] = __shfl_sync(FULL, c[mt][0], src);
                        vv[mt][1] = __shfl_sync(FULL, c[mt][1], src);
                    }
                    double a0 = vd[0] * dt[0], a1 = vd[1] * dt[1], a2 = 0.0, a3 = 0.0;
#pragma unroll
                    for (int mt = 0; mt < NT; ++mt) {
                        if (mt & 1) { a2 = fma(vv[mt][0], c[mt][0], a2); a3 = fma(vv[mt][1], c[mt][1], a3); }
                        else { a0 = fma(vv[mt][0], c[mt][0], a0); a1 = fma(vv[mt][1], c[mt][1], a1); }
                    }
                    double d = (a0 + a1) + (a2 + a3);                          // raw v . (my column), over my rows
                    d += __shfl_xor_sync(FULL, d, 1);
                    d += __shfl_xor_sync(FULL, d, 2);
                    const double ss = __shfl_sync(FULL, d, 4 * jj);            // |raw v|^2
                    const double x0 = __shfl_sync(FULL, dt[jj >> 2], 4 * jj + (jj & 3));
                    const double cj = __shfl_sync(FULL, dt[jj >> 2], (lane & ~3) | (jj & 3));   // my column at row j
                    // nrm = sqrt(ss), tau = 2 / v^T v = 1 / (ss + nrm |x0|): rsqrt + reciprocal instead of sqrt + division
                    const bool zero = !(ss > 0.0);
                    const double nrm = zero ? 0.0 : ss * rsqrt(ss);
                    const double alpha = (x0 >= 0.0) ? -nrm : nrm;
                    const double tj = zero ? 0.0 : __drcp_rn(fma(nrm, fabs(x0), ss));
                    const double gfin = d - alpha * cj;                        // v . (my column) with v[j] = x0 - alpha
                    if (t4 == (jj & 3)) vd[jj >> 2] = x0 - alpha;
                    const double w = (g8 > jj) ? gfin * tj : 0.0;
                    dt[0] = fma(-w, vd[0], dt[0]);
                    dt[1] = fma(-w, vd[1], dt[1]);
#pragma unroll
                    for (int mt = 0; mt < NT; ++mt) { c[mt][0] = fma(-w, vv[mt][0], c[mt][0]); c[mt][1] = fma(-w, vv[mt][1], c[mt][1]); }
                    if (g8 == jj && t4 == (jj & 3)) dt[jj >> 2] = alpha;      // R[j][j]; the rows below keep v
                    // T[:, jj] = -tau T[:, :jj] (V^T v)[:jj], T[jj][jj] = tau; (V^T v)[k] sits in lane group k
                    {
                        double sA = 0.0, sB = 0.0;
#pragma unroll
                        for (int k = 0; k < jj; ++k) {
                            const double gk = __shfl_sync(FULL, gfin, 4 * k);
                            if (k & 1) sB = fma(Trow[k], gk, sB); else sA = fma(Trow[k], gk, sA);
                        }
                        Trow[jj] = (g8 < jj) ? -tj * (sA + sB) : (g8 == jj ? tj : 0.0);
                    }
                    if (g8 == jj && t4 == (jj & 3)) vdiag = x0 - alpha;       // v[j]: kept for the block's store below
                }
            }
            // ---- the block's reflectors, all eight at once: column g8 of the registers holds reflector g8 below its
            //      diagonal (later steps of the panel never touch a finished column), v[j] was kept aside, zero above ----
            if (stored) {
                double *vdst = Vown + (size_t)g8 * VPown + 2 * (g8 >> 2) + t4;
#pragma unroll
                for (int mt = 1; mt < NT; ++mt)
                    if (mt > m0) { vdst[8 * mt] = c[mt][0]; vdst[8 * mt + 4] = c[mt][1]; }
                vdst[8 * m0] = t4 > g8 ? dt[0] : (t4 == g8 ? vdiag : 0.0);
                vdst[8 * m0 + 4] = 4 + t4 > g8 ? dt[1] : (4 + t4 == g8 ? vdiag : 0.0);
            }
            if (stored && t4 == 0) {
                double *tdst = Ts + (size_t)m0 * 8 * QRM_TP + g8 * QRM_TP;
#pragma unroll
                for (int k = 0; k < 8; ++k) tdst[k] = Trow[k];
            }
            // ---- the block's own rows of R; for y: rows < K are Q^T y, the rest gives e2 ----
            {
                double e2 = 0.0;
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int row = o + 4 * u + t4;
                    if (row < h) dst[row] = dt[u];
                    if (isy) { if (row < K) yout[row] = dt[u]; else e2 = fma(dt[u], dt[u], e2); }
                }
                if (o + 8 >= ncols) {                    // last block (uniform): the y column is here
#pragma unroll
                    for (int mt = 0; mt < NT; ++mt) {
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const int row = 8 * mt + 4 * u + t4;
                            if (isy && mt > m0) { if (row < K) yout[row] = c[mt][u]; else e2 = fma(c[mt][u], c[mt][u], e2); }
                        }
                    }
                    e2 += __shfl_xor_sync(FULL, e2, 1);
                    e2 += __shfl_xor_sync(FULL, e2, 2);
                    if (isy && t4 == 0) yout[K] = e2;
                }
            }
            __syncwarp();
        }
    }
}

template <int S>
static cudaError_t launch_qr_t(const RegressParams &p, int grid, int warps, size_t smem, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(regress_qr_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    regress_qr_kernel<S><<<grid, warps * 32, smem, s>>>(p);
    return cudaGetLastError();
}

template <int NT>
static cudaError_t launch_qrm_t(const RegressParams &p, int grid, int warps, size_t smem, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(regress_qr_mma_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    regress_qr_mma_kernel<NT><<<grid, warps * 32, smem, s>>>(p);
    return cudaGetLastError();
}

template <int PS>
static cudaError_t launch_clean_t(const RegressParams &p, int grid, int warps, size_t smem, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(regress_clean_kernel<PS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    regress_clean_kernel<PS><<<grid, warps * 32, smem, s>>>(p);
    return cudaGetLastError();
}

template <int PS>
static cudaError_t launch_trunc_t(const RegressParams &p, int grid, int warps, size_t smem, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(regress_trunc_kernel<PS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    regress_trunc_kernel<PS><<<grid, warps * 32, smem, s>>>(p);
    return cudaGetLastError();
}

// Launches K2a + K2b-1 + K2b-2 for fields [p.f0, p.f1).  p.counter: two words, p.lcounter: five words (zeroed here).
cudaError_t launch_regress(const RegressParams &p_in, int sm_count, size_t smem_limit, cudaStream_t s, cudaEvent_t mid) {
    if (p_in.nwork == 0) return cudaSuccess;
    if (p_in.pmax > 128) return cudaErrorInvalidConfiguration;
    RegressParams p = p_in;
    cudaError_t e = cudaMemsetAsync(p.counter, 0, 2 * sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(p.lcounter, 0, 5 * sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
    // K2a
    const int S = (p.N + 31) / 32;
    // ensembles of up to 128 members: tensor-core form; larger ones (or ENKFMC_QR=smem, for comparisons): the
    // shared-memory SIMT form
#ifdef ENKFMC_TUNING
    const char *qr_sel = getenv("ENKFMC_QR");
#else
    const char *qr_sel = nullptr;      // run-time knobs exist in tuning builds only (-DENKFMC_TUNING)
#endif
    if (p.N <= 128 && !qr_sel) {
        const int nt = (p.N + 7) / 8;
        const int NTc = nt <= 4 ? 4 : nt <= 6 ? 6 : nt <= 10 ? 10 : 16;      // the instantiation used below
        const size_t ws = regress_qrm_ws_doubles(NTc, p.pmax) * sizeof(double);
        int warps = (int)(smem_limit / ws);
        if (warps < 1) return cudaErrorInvalidConfiguration;
        if (warps > 8) warps = 8;
#ifdef ENKFMC_TUNING
        if (const char *wenv = getenv("ENKFMC_QR_WARPS")) { const int wv = atoi(wenv); if (wv >= 1 && wv < warps) warps = wv; }
#endif
        int64_t grid = sm_count;
        const int64_t need = (p.nwork + warps - 1) / warps;
        if (grid > need) grid = need;
        if (nt <= 4) e = launch_qrm_t<4>(p, (int)grid, warps, ws * warps, s);
        else if (nt <= 6) e = launch_qrm_t<6>(p, (int)grid, warps, ws * warps, s);
        else if (nt <= 10) e = launch_qrm_t<10>(p, (int)grid, warps, ws * warps, s);
        else e = launch_qrm_t<16>(p, (int)grid, warps, ws * warps, s);
        if (e != cudaSuccess) return e;
    } else {
        const size_t ws = regress_qr_ws_doubles(p.N, p.pmax) * sizeof(double);
        int warps = (int)(smem_limit / ws);
        if (warps < 1) return cudaErrorInvalidConfiguration;
        if (warps > 8) warps = 8;                      // <= 256 threads: the kernel may use up to 255 registers
        int ctas = (int)(smem_limit / (ws * warps + 1024));
        if (ctas > 2) ctas = 2;
        if (ctas < 1) ctas = 1;
        int64_t grid = (int64_t)sm_count * ctas;
        const int64_t need = (p.nwork + warps - 1) / warps;
        if (grid > need) grid = need;
        switch (S) {
            case 1: e = launch_qr_t<1>(p, (int)grid, warps, ws * warps, s); break;
            case 2: e = launch_qr_t<2>(p, (int)grid, warps, ws * warps, s); break;
            case 3: e = launch_qr_t<3>(p, (int)grid, warps, ws * warps, s); break;
            case 4: e = launch_qr_t<4>(p, (int)grid, warps, ws * warps, s); break;
            case 5: e = launch_qr_t<5>(p, (int)grid, warps, ws * warps, s); break;   // the row guards assume S = ceil(N / 32) exactly
            case 6: e = launch_qr_t<6>(p, (int)grid, warps, ws * warps, s); break;
            case 7: e = launch_qr_t<7>(p, (int)grid, warps, ws * warps, s); break;
            default: e = launch_qr_t<8>(p, (int)grid, warps, ws * warps, s); break;
        }
        if (e != cudaSuccess) return e;
    }
    if (mid) { e = cudaEventRecord(mid, s); if (e != cudaSuccess) return e; }
    // K2b-1: certificate + plain solve; rows that (may) truncate are listed for K2b-2
    {
        const size_t ws = regress_clean_ws_doubles(p.pmax) * sizeof(double);
        int warps = (int)(smem_limit / ws);
        if (warps < 1) return cudaErrorInvalidConfiguration;
        if (warps > 16) warps = 16;
        int64_t grid = sm_count;
        const int64_t need = (p.nwork + warps - 1) / warps;
        if (grid > need) grid = need;
        if (p.pmax <= 32) e = launch_clean_t<1>(p, (int)grid, warps, ws * warps, s);
        else if (p.pmax <= 64) e = launch_clean_t<2>(p, (int)grid, warps, ws * warps, s);
        else if (p.pmax <= 96) e = launch_clean_t<3>(p, (int)grid, warps, ws * warps, s);
        else e = launch_clean_t<4>(p, (int)grid, warps, ws * warps, s);
        if (e != cudaSuccess) return e;
    }
    // K2b-2, two passes: small blocks at high occupancy first; rows whose block has to grow beyond that are handed to a
    // second pass with room for up to 32 vectors (the number of sub-threshold singular values grows with the predecessor
    // count).  The list lengths are known on the device only: both passes are always launched.
    {
        const int b1 = p.pmax < 8 ? 0 : p.pmax <= 48 ? 8 : 16;
        int b2 = p.pmax < 8 ? 0 : p.pmax <= 16 ? 8 : p.pmax <= 64 ? 24 : 32;
#ifdef ENKFMC_TUNING
        if (const char *benv = getenv("ENKFMC_K2B_BMAX")) { const int bv = atoi(benv); if (bv >= 8 && bv <= 32) b2 = bv & ~7; }
#endif
        while (b2 > 8 && regress_trunc_ws_doubles(p.pmax, b2) * sizeof(double) > smem_limit) b2 -= 8;
        for (int level = 0; level < 2; ++level) {
            p.level = level;
            p.bmax = level == 0 ? std::min(b1, b2) : b2;
            p.bmax1 = std::min(b1, b2);
            p.bmax2 = b2;
            if (level == 1 && b2 <= std::min(b1, b2)) break;     // nothing is ever escalated
            const size_t ws = regress_trunc_ws_doubles(p.pmax, p.bmax) * sizeof(double);
            int warps = (int)(smem_limit / ws);
            if (warps < 1) return cudaErrorInvalidConfiguration;
            if (warps > 8) warps = 8;
#ifdef ENKFMC_TUNING
            if (const char *wenv = getenv("ENKFMC_K2B_WARPS")) { const int wv = atoi(wenv); if (wv >= 1 && wv < warps) warps = wv; }
#endif
            const int64_t grid = sm_count;
            if (p.pmax <= 32) e = launch_trunc_t<1>(p, (int)grid, warps, ws * warps, s);
            else if (p.pmax <= 64) e = launch_trunc_t<2>(p, (int)grid, warps, ws * warps, s);
            else if (p.pmax <= 96) e = launch_trunc_t<3>(p, (int)grid, warps, ws * warps, s);
            else e = launch_trunc_t<4>(p, (int)grid, warps, ws * warps, s);
            if (e != cudaSuccess) return e;
        }
    }
    return e;
}

// Copies a finished regression to its aliases: one warp per (alias row, field).
__global__ void __launch_bounds__(256) replicate_rows_kernel(const int32_t *__restrict__ alias_row,
                                                             const int32_t *__restrict__ alias_rep, int64_t naliases,
                                                             const int64_t *__restrict__ row_ptr, int64_t nfields,
                                                             int64_t nnz, int64_t nloc, double *__restrict__ T,
                                                             double *__restrict__ D, int32_t *__restrict__ flags) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= naliases * nfields) return;
    const int64_t a = w % naliases, f = w / naliases;
    const int q = alias_row[a], r = alias_rep[a];
    const int64_t dst = row_ptr[q], src = row_ptr[r];
    const int p = (int)(row_ptr[q + 1] - dst);
    double *Tf = T + f * nnz;
    for (int j = lane; j < p; j += 32) Tf[dst + j] = Tf[src + j];
    if (lane == 0) {
        D[f * nloc + q] = D[f * nloc + r];
        if (flags) flags[f * nloc + q] = flags[f * nloc + r];
    }
}

cudaError_t launch_replicate_rows(const int32_t *alias_row, const int32_t *alias_rep, int64_t naliases,
                                  const int64_t *row_ptr, int64_t nfields, int64_t nnz, int64_t nloc, double *T,
                                  double *D, int32_t *flags, cudaStream_t s) {
    const int64_t warps = naliases * nfields;
    if (warps == 0) return cudaSuccess;
    replicate_rows_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(alias_row, alias_rep, naliases, row_ptr, nfields,
                                                                       nnz, nloc, T, D, flags);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// K3: local analysis of every (field, tile), in two kernels.
//
// A = T~^T D^-1 T~ + H^T R^-1 H with T~ = I + strictly-lower T (factors.py:136-145,
// kernels.py:189-191) is symmetric and banded (half-bandwidth b) in the tile's physical order.
// Rows are grouped in blocks of 8; Wb = floor((b+7)/8) block sub-diagonals can be non-zero.
//
// K3a: A[I, K] = sum_j T~[j,i] T~[j,k] / D_j over the rows j holding both i and k, accumulated in
//   ascending j in a per-warp shared buffer (deterministic), stored in row form:
//   band[tile][I][e] = A[I, 8 (I/8 - Wb) + e], e < Wr = 8 (Wb + 1), zeros elsewhere.
//   assemble_band_tile_kernel (one CTA per (field, tile), the tile's T staged in shared memory)
//   whenever the tile fits, else assemble_band_kernel (one warp per row, from global memory).
// K3b local_solve_kernel: one CTA per (field, tile).  Right-looking blocked banded Cholesky
//   through a sliding window of Wb+1 block rows in shared memory, carrying the N right-hand sides
//   rhs[obs] = (Ys - Xb[obs]) / r (kernels.py:182-186) along (forward substitution fused).
//   Per block column: warp 0 factors and inverts the next 8 x 8 diagonal block in registers while
//   the other warps run the trailing update and the right-hand-side update as 8 x 8 tensor-core
//   tiles; panel and right-hand-side solves are tensor-core products with the stored inverse.
//   L (with the inverse of each diagonal block in that block's upper triangle) overwrites the
//   band block by block.  The backward substitution runs blockwise the same way and writes
//   Xa = Xb + dx for the interior rows straight into the global analysis (kernels.py:218,
//   driver.py:116).
// ------------------------------------------------------------------------------------------
#define SOLVE_THREADS 512
#define ASM_WARPS 8
#define LP_PITCH 10   // doubles per panel row: 16-byte aligned, conflict-free for 128-bit loads

__host__ __device__ inline int solve_wb(int b) { return (b + 7) >> 3; }

__global__ void __launch_bounds__(ASM_WARPS * 32) assemble_band_kernel(const SolveParams P) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *acc = smem + (size_t)warp * (8 * (solve_wb(P.bmax) + 1));
    const int nf = P.f1 - P.f0;
    const int64_t nrows = P.nrows_owned;
    const int64_t total = nrows * nf;
    const int64_t stride = (int64_t)gridDim.x * ASM_WARPS;
    for (int64_t w = (int64_t)blockIdx.x * ASM_WARPS + warp; w < total; w += stride) {
        const int fl = (int)(w / nrows), f = P.f0 + fl;
        const int q = P.work_order[w % nrows];
        const int t = P.row_tile[q];
        if (!P.assemble_only && P.tile_nobs[(int64_t)f * P.ntiles + t] == 0) continue;
        const int64_t base = P.tile_ptr[t];
        const int i = (int)(q - base);
        const int Wb = solve_wb(P.bw[t]), Wr = 8 * (Wb + 1);
        const int32_t *phys = P.phys + base;
        const int I = phys[i];
        const int col0 = 8 * ((I >> 3) - Wb);          // column of band entry e = 0
        const double *Tf = P.T + (int64_t)f * P.tstride;
        const double *Df = P.D + (int64_t)f * P.dstride + base;
        for (int e = lane; e < Wr; e += 32) acc[e] = 0.0;
        __syncwarp();
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
                if (Kp <= I) acc[Kp - col0] += s * tjk;
            }
            __syncwarp();
        }
        if (lane == 0 && !P.assemble_only) {
            const int sl = P.obs_slot[(int64_t)f * P.nloc + q];
            if (sl >= 0) acc[I - col0] += 1.0 / P.rdiag[sl];
        }
        __syncwarp();
        double *dst = P.band + (int64_t)fl * P.band_stride + P.band_ptr[t] + (int64_t)I * Wr;
        for (int e = lane; e < Wr; e += 32) dst[e] = acc[e];
        __syncwarp();
    }
}

// Tile-cooperative form of K3a: one CTA per (field, tile).  The tile's T values, the physical column of every
// entry, D and the row pointers are staged in shared memory once, so the index chase of every row of A runs at
// shared-memory latency; each warp then assembles rows as assemble_band_kernel does (same order of additions; 1/D is
// formed once per row instead of one division per term).  Used whenever the staging fits (launch_assemble_band decides).
#define ASMT_THREADS 512

__host__ __device__ inline size_t asm_tile_smem_bytes(int nmax, int nnzmax, int bmax) {
    size_t b = (size_t)nnzmax * 8 + (size_t)nmax * 8 + (size_t)(ASMT_THREADS / 32) * 8 * (solve_wb(bmax) + 1) * 8;
    b += (size_t)(nmax + 1) * 4;
    b += (size_t)nnzmax * 2 + (size_t)nmax * 2;
    return (b + 15) & ~(size_t)15;
}

__global__ void __launch_bounds__(ASMT_THREADS) assemble_band_tile_kernel(const SolveParams P) {
    extern __shared__ double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nf = P.f1 - P.f0;
    const int t = P.tile_order[blockIdx.x / nf];
    const int fl = (int)(blockIdx.x % nf), f = P.f0 + fl;
    if (!P.assemble_only && P.tile_nobs[(int64_t)f * P.ntiles + t] == 0) return;
    const int64_t base = P.tile_ptr[t];
    const int n = (int)(P.tile_ptr[t + 1] - base);
    const int64_t e0 = P.row_ptr[base];
    const int nz = (int)(P.row_ptr[base + n] - e0);
    const int Wb = solve_wb(P.bw[t]), Wr = 8 * (Wb + 1);
    const int accw = 8 * (solve_wb(P.bmax) + 1);

    double *sT = smem;
    double *sD = sT + P.asm_nnzmax;
    double *accs = sD + P.asm_nmax;
    int32_t *sRow = reinterpret_cast<int32_t *>(accs + (size_t)(ASMT_THREADS / 32) * accw);
    uint16_t *sK = reinterpret_cast<uint16_t *>(sRow + P.asm_nmax + 1);
    uint16_t *sPhys = sK + P.asm_nnzmax;

    const double *Tf = P.T + (int64_t)f * P.tstride + e0;
    const double *Df = P.D + (int64_t)f * P.dstride + base;
    const int32_t *phys = P.phys + base;
    for (int i = tid; i < n; i += ASMT_THREADS) { sD[i] = 1.0 / Df[i]; sPhys[i] = (uint16_t)phys[i]; }
    for (int i = tid; i <= n; i += ASMT_THREADS) sRow[i] = (int32_t)(P.row_ptr[base + i] - e0);
    for (int e = tid; e < nz; e += ASMT_THREADS) { sT[e] = Tf[e]; sK[e] = (uint16_t)phys[P.col_idx[e0 + e]]; }
    __syncthreads();

    const bool mono = P.tile_mono != nullptr && P.tile_mono[t] != 0;
    double *acc = accs + (size_t)warp * accw;
    for (int i = warp; i < n; i += ASMT_THREADS / 32) {
        const int I = sPhys[i];
        const int col0 = 8 * ((I >> 3) - Wb);
        for (int e = lane; e < Wr; e += 32) acc[e] = 0.0;
        const int64_t c0 = P.csc_ptr[base + i];
        const int ncsc = (int)(P.csc_ptr[base + i + 1] - c0);
        __syncwarp();
        // rows j > i holding column i: lists are short (<= 96), fetched 32 at a time and broadcast by shuffle
        for (int eb = -1; eb < ncsc; eb = (eb < 0 ? 0 : eb + 32)) {
            int jl = 0, sl = 0, cnt_e = 1;
            if (eb >= 0) {
                cnt_e = ncsc - eb < 32 ? ncsc - eb : 32;
                if (lane < cnt_e) { jl = P.csc_row[c0 + eb + lane]; sl = (int)(P.csc_src[c0 + eb + lane] - e0); }
            }
            for (int ee = 0; ee < cnt_e; ++ee) {
                int j; double tji;
                if (eb < 0) { j = i; tji = 1.0; }
                else { j = __shfl_sync(FULL, jl, ee); tji = sT[__shfl_sync(FULL, sl, ee)]; }
                const double sc = tji * sD[j];
                const int q0 = sRow[j];
                int cnt = sRow[j + 1] - q0, mfirst = lane - 1;
                if (mono && eb >= 0) {              // sorted columns: nothing right of the pivot entry (column i) is wanted
                    cnt = __shfl_sync(FULL, sl, ee) - q0 + 1;
                    mfirst = lane;                  // nor is the diagonal of a later row
                }
                for (int m = mfirst; m < cnt; m += 32) {
                    int Kp; double tjk;
                    if (m < 0) { Kp = sPhys[j]; tjk = 1.0; } else { Kp = sK[q0 + m]; tjk = sT[q0 + m]; }
                    if (Kp <= I) acc[Kp - col0] += sc * tjk;
                }
                __syncwarp();
            }
        }
        if (lane == 0 && !P.assemble_only) {
            const int sl = P.obs_slot[(int64_t)f * P.nloc + base + i];
            if (sl >= 0) acc[I - col0] += 1.0 / P.rdiag[sl];
        }
        __syncwarp();
        double *dst = P.band + (int64_t)fl * P.band_stride + P.band_ptr[t] + (int64_t)I * Wr;
        for (int e = lane; e < Wr; e += 32) dst[e] = acc[e];
        __syncwarp();
    }
}

// Tensor-core form of K3a: A = T~^T D^-1 T~ as a banded SYRK of 8 x 8 tiles, one CTA per (field, tile).  For tiles whose
// physical order is the local order (every clipped tile) T~ is lower triangular with its entries inside the band, so
//     A[I, K] = sum_{J = I}^{K + Wb} C[J, I]^T C[J, K],  C = D^-1/2 T~   (8 x 8 blocks, K <= I <= K + Wb).
// Block rows of C are scattered from the CSR values into a ring of Wb + 2 dense 8 x Wr slots in shared memory (zeros where
// the pattern has no entry); block row I of A then takes (Wb + 1)(Wb + 2) / 2 tile products of two mma.m8n8k4 each: warp d
// accumulates tile (I, I - d) over its J in ascending order (two interleaved accumulator chains, added at the end: a fixed
// order, results are deterministic), while the warps with the short chains scatter block row I + Wb + 1 into the free slot --
// one barrier per block row.  Same band layout as the gather forms; the sums run over the same terms in the same order of
// rows j, grouped four at a time by the tensor-core product.
#define ASMM_THREADS 512
__host__ __device__ inline int asmm_pitch(int Wr) { int v = Wr + 4; while (v % 16 != 4) ++v; return v; }   // fragment loads t4 * pitch + g8: conflict-free
__host__ __device__ inline size_t asmm_smem_bytes(int bmax) {
    const int Wr = 8 * (solve_wb(bmax) + 1);
    return (size_t)(Wr + 8) * asmm_pitch(Wr) * sizeof(double);
}

__global__ void __launch_bounds__(ASMM_THREADS) assemble_band_mma_kernel(const SolveParams P) {
    extern __shared__ double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = ASMM_THREADS / 32;
    const int g8 = lane >> 2, t4 = lane & 3;
    const int nf = P.f1 - P.f0;
    const int t = P.tile_order[blockIdx.x / nf];
    const int fl = (int)(blockIdx.x % nf), f = P.f0 + fl;
    if (!P.assemble_only && P.tile_nobs[(int64_t)f * P.ntiles + t] == 0) return;
    const int64_t base = P.tile_ptr[t];
    const int n = (int)(P.tile_ptr[t + 1] - base), nb = (n + 7) >> 3;
    const int Wb = solve_wb(P.bw[t]), Wr = 8 * (Wb + 1), pitch = asmm_pitch(Wr), nslot = Wb + 2;
    double *ring = smem;                                   // [nslot][8][pitch]
    const double *Tf = P.T + (int64_t)f * P.tstride;
    const double *Df = P.D + (int64_t)f * P.dstride + base;
    double *band = P.band + (int64_t)fl * P.band_stride + P.band_ptr[t];

    // row jr of block row J into its ring slot (one warp): zeros, then the row's entries at column - 8 (J - Wb)
    auto load_row = [&](int J, int jr) {
        const int sl = J % nslot, j = 8 * J + jr;
        double *S = ring + ((size_t)sl * 8 + jr) * pitch;
        for (int e = lane; e < Wr; e += 32) S[e] = 0.0;
        __syncwarp();
        if (j < n) {
            const int c0 = 8 * (J - Wb);
            const int64_t q0 = P.row_ptr[base + j];
            const int cnt = (int)(P.row_ptr[base + j + 1] - q0);
            const double sc = rsqrt(Df[j]);              // row j of D^-1/2 T~ (factors.py:140-143 forms the same matrix)
            for (int m = lane - 1; m < cnt; m += 32) {
                if (m < 0) S[j - c0] = sc;
                else S[P.col_idx[q0 + m] - c0] = Tf[q0 + m] * sc;
            }
        }
    };
    for (int idx = warp; idx < 8 * (Wb + 1); idx += nwarps)
        if ((idx >> 3) < nb) load_row(idx >> 3, idx & 7);
    __syncthreads();

    // The warps with the short chains (the last eight) fill the slot that is free during a step with block row I + Wb + 1,
    // one row each.  The row's values travel through registers: its CSR range is read one step ahead and the values / columns
    // at the top of the step, so that both global latencies pass under the tile products; the slot is written at the end.
    const bool loader = warp >= nwarps - 8;
    const int ljr = warp - (nwarps - 8);
    int64_t nq0 = 0;
    int ncnt = -1;                                          // CSR range of this warp's row of the next block row (-1: none)
    auto peek_row = [&](int J) {
        const int j = 8 * J + ljr;
        ncnt = -1;
        if (J < nb && j < n) { nq0 = P.row_ptr[base + j]; ncnt = (int)(P.row_ptr[base + j + 1] - nq0); }
    };
    if (loader) peek_row(Wb + 1);
    int sI = 0;                                             // ring slot of block row I
    for (int I = 0; I < nb; ++I) {
        const int Jn = I + Wb + 1;
        double tv0 = 0.0, tv1 = 0.0, dvn = 0.0;
        int tc0 = 0, tc1 = 0;
        const int64_t q0c = nq0;
        const int cntc = ncnt;
        if (loader && cntc >= 0) {
            const int m0 = lane - 1, m1 = lane + 31;
            if (m0 >= 0 && m0 < cntc) { tv0 = Tf[q0c + m0]; tc0 = P.col_idx[q0c + m0]; }
            if (m1 < cntc) { tv1 = Tf[q0c + m1]; tc1 = P.col_idx[q0c + m1]; }
            dvn = rsqrt(Df[8 * Jn + ljr]);
            peek_row(Jn + 1);
        }
        for (int d = warp; d <= Wb; d += nwarps) {
            const int K = I - d;
            double p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0;
            if (K >= 0) {
                const int Jend = (I + Wb - d < nb - 1) ? I + Wb - d : nb - 1;
                // slot of block row J walks the ring from the slot of row I; the tile columns move left by 8 per block row
                int sl = sI, oi = 8 * Wb + g8, ok = 8 * (Wb - d) + g8;
                for (int J = I; J <= Jend; ++J) {
                    const double *S = ring + ((size_t)sl * 8 + t4) * pitch;
                    const double a0 = S[oi], a1 = S[(size_t)4 * pitch + oi];
                    const double b0 = S[ok], b1 = S[(size_t)4 * pitch + ok];
                    if ((J - I) & 1) { mma_f64(q0, q1, a0, b0); mma_f64(q0, q1, a1, b1); }
                    else { mma_f64(p0, p1, a0, b0); mma_f64(p0, p1, a1, b1); }
                    sl = sl + 1 == nslot ? 0 : sl + 1;
                    oi -= 8; ok -= 8;
                }
            }
            double v0 = p0 + q0, v1 = p1 + q1;              // A[8 I + g8, 8 K + 2 t4 + {0, 1}]
            const int i = 8 * I + g8;
            if (d == 0) {
                if (2 * t4 > g8) v0 = 0.0;                   // row form keeps the lower triangle of the diagonal block
                if (2 * t4 + 1 > g8) v1 = 0.0;
                if (!P.assemble_only && i < n && (g8 >> 1) == t4) {
                    const int sl = P.obs_slot[(int64_t)f * P.nloc + base + i];
                    if (sl >= 0) { const double ri = 1.0 / P.rdiag[sl]; if (g8 & 1) v1 += ri; else v0 += ri; }
                }
            }
            if (i < n) *reinterpret_cast<double2 *>(band + (int64_t)i * Wr + 8 * (Wb - d) + 2 * t4) = make_double2(v0, v1);
        }
        if (loader && Jn < nb) {
            const int sl = sI == 0 ? nslot - 1 : sI - 1;     // slot of row I + Wb + 1 = slot of row I - 1 (Wb + 2 slots)
            const int j = 8 * Jn + ljr, c0 = 8 * (Jn - Wb);
            double *S = ring + ((size_t)sl * 8 + ljr) * pitch;
            for (int e = lane; e < Wr; e += 32) S[e] = 0.0;
            __syncwarp();
            if (cntc >= 0) {
                if (lane == 0) S[j - c0] = dvn;
                else if (lane - 1 < cntc) S[tc0 - c0] = tv0 * dvn;
                if (lane + 31 < cntc) S[tc1 - c0] = tv1 * dvn;
                for (int m = lane + 63; m < cntc; m += 32) S[P.col_idx[q0c + m] - c0] = Tf[q0c + m] * dvn;   // (more than 63 predecessors)
            }
        }
        __syncthreads();
        sI = sI + 1 == nslot ? 0 : sI + 1;
    }
}

__host__ __device__ inline size_t solve_strip_doubles(int Wb) { return (((4 * (size_t)Wb * (Wb + 1) * 2 + 7) / 8 + 1) & ~(size_t)1); }
__host__ __device__ inline size_t solve_rowsrc_doubles(int rows) { return ((3 * (size_t)rows * 4 + 15) / 16) * 2; }

#ifdef ENKFMC_K3B_TIMING
__device__ unsigned long long g_k3b_t[24];
#define K3T(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) { const long long now_ = clock64(); atomicAdd(&g_k3b_t[i], (unsigned long long)(now_ - tmark_)); tmark_ = now_; } } while (0)
extern "C" int enkfmc_debug_k3b_times(unsigned long long *out24) {
    cudaMemcpyFromSymbol(out24, g_k3b_t, sizeof(g_k3b_t));
    unsigned long long z[24] = {0};
    cudaMemcpyToSymbol(g_k3b_t, z, sizeof(z));
    return 0;
}
#else
#define K3T(i) do { } while (0)
#endif

__global__ void __launch_bounds__(SOLVE_THREADS) local_solve_kernel(const SolveParams P) {
#ifdef ENKFMC_K3B_TIMING
    long long tmark_ = clock64();
#endif
    extern __shared__ double smem[];
    __shared__ unsigned int s_item;
    __shared__ int s_fail;
    __shared__ double s_red[SOLVE_THREADS / 32];
    const int tid = threadIdx.x, lane = tid & 31;
    const int nthreads = SOLVE_THREADS;
    const int N = P.N;
    double *scr = P.scratch + (int64_t)blockIdx.x * P.scratch_stride;
    double *Z = scr + P.off_z;                 // [nbp][N] forward-substituted right-hand sides
    // shared layout: Lp[2][WrMax][LP_PITCH] | Zb[8][NR] | invd[2][8] | rinv[2][8] | tile table | row sources | window A | window RHS
    const int WbMax = solve_wb(P.bmax), WrMax = 8 * (WbMax + 1);
    const int NR = P.nr_pitch;                 // member pitch of Zb / the RHS window / red: >= 8 ceil(N/8), = 8 mod 16
    double *Lp0 = smem;
    double *Zb = Lp0 + 2 * (size_t)WrMax * LP_PITCH;
    double *invd0 = Zb + 8 * (size_t)NR;
    double *rinv0 = invd0 + 16;
    unsigned short *strips = reinterpret_cast<unsigned short *>(rinv0 + 16);
    int32_t *rsl = reinterpret_cast<int32_t *>(rinv0 + 16 + solve_strip_doubles(WbMax));   // [nmax8] obs slot or -1
    int32_t *rxr = rsl + P.rows_smem;                                                      // [nmax8] state row
    int32_t *rxi = rxr + P.rows_smem;                                                      // [nmax8] state row if interior, else -1
    double *sm_rest = rinv0 + 16 + solve_strip_doubles(WbMax) + solve_rowsrc_doubles(P.rows_smem);
    double *Aw = P.a_in_smem ? sm_rest : scr + P.off_win_a;
    double *Rw = P.r_in_smem ? (P.a_in_smem ? sm_rest + P.a_doubles : sm_rest) : scr + P.off_win_r;
    const unsigned nf = (unsigned)(P.f1 - P.f0);
    const int total_items = (int)nf * P.ntiles_owned;
    const int warp = tid >> 5, nwarps = nthreads >> 5;
    const int g8 = lane >> 2, t4 = lane & 3;                  // mma.m8n8k4 fragment coordinates of this lane
    const int nct = (N + 7) >> 3;                             // 8-member column tiles

    for (;;) {
        __syncthreads();
        if (tid == 0) { s_item = atomicAdd(P.counter, 1u); s_fail = 0; }
        __syncthreads();
        const unsigned int item = s_item;
        if ((int)item >= total_items) break;
        K3T(0);
        const int t = P.tile_order[item / nf];
        const int fl = (int)(item % nf), f = P.f0 + fl;
        const int64_t base = P.tile_ptr[t];
        const int n = (int)(P.tile_ptr[t + 1] - base);
        const int Wb = solve_wb(P.bw[t]), nslot = Wb + 1, Wr = 8 * nslot, pitch = Wr + 2;
        const int nb = (n + 7) >> 3;
        const double *Xf = P.X + (int64_t)f * P.nstate2d * N;
        double *Xaf = P.Xa + (int64_t)f * P.nstate2d * N;
        const int32_t *slotf = P.obs_slot + (int64_t)f * P.nloc + base;
        const int32_t *iphys = P.iphys + base, *srow = P.state_row + base;
        const uint8_t *inter = P.is_interior + base;
        double *band = P.band + (int64_t)fl * P.band_stride + P.band_ptr[t];   // [8 nb][Wr]: A rows, then L blocks

        if (P.tile_nobs[(int64_t)f * P.ntiles + t] == 0) {   // kernels.py:179-180: exact copy
            for (int j = tid >> 5; j < n; j += nthreads >> 5) {
                if (!inter[j]) continue;
                const int64_t g = (int64_t)srow[j] * N;
                for (int m = lane; m < N; m += 32) Xaf[g + m] = Xf[g + m];
            }
            if (tid == 0) P.status[(int64_t)f * P.ntiles + t] = 0;
            continue;
        }

        // largest diagonal entry of A over the tile (the scale a negative pivot is judged against, see factor_diag)
        double gmax = 0.0;
        {
            for (int i = tid; i < n; i += nthreads) gmax = fmax(gmax, band[(int64_t)i * Wr + 8 * Wb + (i & 7)]);
            gmax = warp_max(gmax);
            if (lane == 0) s_red[warp] = gmax;
            __syncthreads();
            gmax = 0.0;
            for (int k = 0; k < nwarps; ++k) gmax = fmax(gmax, s_red[k]);
        }
        // 8x8 tiles (rb, cb <= rb) of the trailing update, ordered by rb: the live ones are a prefix
        for (int s = tid; s < Wb * (Wb + 1) / 2; s += nthreads) {
            int rb = 0, rem = s;
            while (rem > rb) { rem -= rb + 1; ++rb; }
            strips[s] = (unsigned short)((rb << 8) | rem);
        }
        // where each physical row's right-hand side and analysis row live (resolves the index chain once)
        const bool rows_cached = 8 * nb <= P.rows_smem;
        if (rows_cached) {
            for (int i = tid; i < 8 * nb; i += nthreads) {
                int sl = -1, xr = 0, xi = -1;
                if (i < n) {
                    const int il = iphys[i];
                    sl = slotf[il]; xr = srow[il]; xi = inter[il] ? xr : -1;
                }
                rsl[i] = sl; rxr[i] = xr; rxi[i] = xi;
            }
            __syncthreads();
        }
        // block row R (8 rows of A and of the right-hand side): fetch into registers, commit to its window slot
        const bool pf = rows_cached && 8 * Wr <= 2 * nthreads && 8 * N <= 2 * nthreads;
        double fa[2], fy[2], fx[2], fr[2];
        int ea_r[2], ea_e[2], er_r[2], er_m[2];     // this thread's (row, entry) of the A part and (row, member) of the RHS part
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int e = tid + k * nthreads;
            ea_r[k] = e / Wr; ea_e[k] = e - ea_r[k] * Wr;
            er_r[k] = e / N; er_m[k] = e - er_r[k] * N;
        }
        auto rhs_value = [&](int i, int m) {
            double v = 0.0;
            if (i < n) {
                const int il = iphys[i];
                const int sl = slotf[il];
                if (sl >= 0) v = (P.Ys[(int64_t)sl * N + m] - Xf[(int64_t)srow[il] * N + m]) * (1.0 / P.rdiag[sl]);
            }
            return v;
        };
        auto fetch_block_row = [&](int R) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                fa[k] = 0.0; fy[k] = 0.0; fx[k] = 0.0; fr[k] = 0.0;
                if (ea_r[k] < 8) {
                    const int i = 8 * R + ea_r[k];
                    fa[k] = (i < n) ? band[(int64_t)i * Wr + ea_e[k]] : ((ea_e[k] == 8 * Wb + ea_r[k]) ? 1.0 : 0.0);   // padding row: identity
                }
                if (er_r[k] < 8) {
                    const int i = 8 * R + er_r[k];
                    const int sl = rsl[i];
                    if (sl >= 0) {
                        fy[k] = P.Ys[(int64_t)sl * N + er_m[k]]; fx[k] = Xf[(int64_t)rxr[i] * N + er_m[k]]; fr[k] = P.rdiag[sl];
                    }
                }
            }
        };
        // rs: window slot (row offset) of block row R; rot: window column of its band entry 0
        auto commit_block_row = [&](int rs, int rot) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (ea_r[k] < 8) {
                    int cc = rot + ea_e[k]; if (cc >= Wr) cc -= Wr;
                    Aw[(size_t)(rs + ea_r[k]) * pitch + cc] = fa[k];
                    if (ea_e[k] == 8 * Wb + ea_r[k]) Aw[(size_t)(rs + ea_r[k]) * pitch + Wr] = fa[k];   // the row's original diagonal (pitch padding)
                }
                if (er_r[k] < 8)
                    Rw[(size_t)(rs + er_r[k]) * NR + er_m[k]] = (fr[k] != 0.0) ? (fy[k] - fx[k]) * (1.0 / fr[k]) : 0.0;
            }
        };
        auto load_block_row = [&](int R) {
            const int rs = (R % nslot) * 8;
            const int rot = (((R - Wb) % nslot) + nslot) % nslot * 8;
            if (pf) { fetch_block_row(R); commit_block_row(rs, rot); return; }
            for (int e = tid; e < 8 * Wr; e += nthreads) {
                const int rr = e / Wr, ee = e - rr * Wr, i = 8 * R + rr;
                const double v = (i < n) ? band[(int64_t)i * Wr + ee] : ((ee == 8 * Wb + rr) ? 1.0 : 0.0);
                int cc = rot + ee; if (cc >= Wr) cc -= Wr;
                Aw[(size_t)(rs + rr) * pitch + cc] = v;
                if (ee == 8 * Wb + rr) Aw[(size_t)(rs + rr) * pitch + Wr] = v;
            }
            for (int e = tid; e < 8 * N; e += nthreads) {
                const int rr = e / N, m = e - rr * N;
                Rw[(size_t)(rs + rr) * NR + m] = rhs_value(8 * R + rr, m);
            }
        };
        K3T(1);
        for (int R = 0; R <= Wb && R < nb; ++R) load_block_row(R);
        __syncthreads();
        K3T(2);

        // ---- forward: blocked Cholesky + forward substitution --------------------------------
        // Everything but the 8x8 diagonal factorisation runs as 8x8 tiles on the FP64 tensor cores (mma.m8n8k4, two
        // k-steps per tile).  Panel buffer J & 1 holds, in rows 0..7, L_JJ (lower) and the strict lower part of
        // L_JJ^-1 transposed into the upper triangle (diagonal of the inverse in invd); rows 8.. hold the panel.
        double pivmax = 0.0;                         // largest pivot so far (warp 0 tracks it redundantly per lane)
        // Diagonal block J (warp 0): lane r (mod 8) keeps row r of the block and of the running inverse in registers;
        // right-looking Cholesky with the same eliminations applied to the identity.
        auto factor_diag = [&](int sJ, int buf) {
            double *Lp = Lp0 + (size_t)buf * WrMax * LP_PITCH;
            double *invd = invd0 + 8 * buf;
            const double *Dg = Aw + (size_t)sJ * pitch + sJ;
            const int r = lane & 7;
            double a[8], v[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) { a[c] = (c <= r) ? Dg[(size_t)r * pitch + c] : 0.0; v[c] = (c == r) ? 1.0 : 0.0; }
            double og[8];                                                // A_cc before any elimination (uniform loads: kept out of the chain)
#pragma unroll
            for (int c = 0; c < 8; ++c) og[c] = Aw[(size_t)(sJ + c) * pitch + Wr];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                double piv = __shfl_sync(FULL, a[c], c);
                double inv = rsqrt(piv);                                 // issued before the pivot test: replaced below in the rare cases
                const double orig = og[c];
                // A = T~^T D^-1 T~ + H^T R^-1 H is positive (semi-)definite by construction.
                bool pin = false;
                // The scale a pivot is judged against: the largest pivot so far, or the row's own diagonal before
                // elimination (row scales differ by up to 1e10 when some D sit on the variance floor).  At or below the
                // rounding level of that scale the pivot is cancellation noise of either sign: pinned.  A clearly negative
                // pivot means the matrix handed in is indefinite (bad factors): fail like the reference's Cholesky
                // (kernels.py:192-195).  "Clearly" is judged against the largest diagonal entry of the whole tile as well
                // (gmax): the elimination error of a pivot scales with |A|, which the entries met so far underestimate when
                // the large rows come later (deep levels of a vertically coupled tile: |A| 1e15 against 1e12).  NaN / inf fail.
                const double scale = fmax(pivmax, orig);
                if (!(piv > 1e-13 * scale) || !(piv < DBL_MAX)) {        // rare and warp-uniform: NaN / inf, noise-level or negative pivot
                    if (!(piv == piv) || !(fabs(piv) < DBL_MAX)) { if (lane == 0 && s_fail == 0) s_fail = 2; }
                    else if ((pivmax == 0.0 && !(piv > 0.0)) || piv < -1e-8 * fmax(scale, gmax)) { if (lane == 0 && s_fail == 0) s_fail = 1; }
                    else { pin = true; if (lane == 0) atomicAdd(P.counter + 1, 1u); }
                    // a pinned variable gets the pivot +infinity: column of L zero, unit diagonal, zero increment -- no
                    // element growth, unlike a tiny positive pivot
                    if (pin) inv = 0.0;
                }
                pivmax = fmax(pivmax, piv);
                a[c] = (r == c) ? (pin ? 1.0 : piv * inv) : a[c] * inv;   // column c of L
#pragma unroll
                for (int k = 0; k <= c; ++k) if (r == c) v[k] *= inv; // row c of L^-1 is final
#pragma unroll
                for (int c2 = c + 1; c2 < 8; ++c2) {
                    const double lc2 = __shfl_sync(FULL, a[c], c2);
                    if (r >= c2) a[c2] -= a[c] * lc2;
                }
#pragma unroll
                for (int k = 0; k <= c; ++k) {
                    const double vk = __shfl_sync(FULL, v[k], c);
                    if (r > c) v[k] -= a[c] * vk;
                }
            }
            if (lane < 8) {
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    if (c <= r) Lp[r * LP_PITCH + c] = a[c];          // L[r][c]
                    if (c < r) Lp[c * LP_PITCH + r] = v[c];           // (L^-1)[r][c] at the transposed place
                }
                invd[r] = v[r];
            }
        };
        // (L_JJ^-1)[i][j] from a panel buffer
        auto linv = [&](const double *Lp, const double *dg, int i, int j) {
            return i == j ? dg[i] : (i > j ? Lp[j * LP_PITCH + i] : 0.0);
        };
        if (warp == 0) factor_diag(0, 0);
        __syncthreads();
        K3T(3);
        int sJ = 0;                                    // window slot of block row J
        for (int J = 0; J < nb; ++J) {
            if (s_fail) break;
            double *Lp = Lp0 + (size_t)(J & 1) * WrMax * LP_PITCH;
            const double *invd = invd0 + 8 * (J & 1);
            int s1 = sJ + 8; if (s1 >= Wr) s1 = 0;     // window row of panel row r is wrap(s1 + r)
            const int below = (nb - 1 - J < Wb ? nb - 1 - J : Wb) * 8;     // panel rows under the diagonal block
            const int nbl = below >> 3;
            // (e) the next block row will go into the slot of block row J: its global loads are issued first thing, into
            // registers, and committed at the end of the step
            const bool more = J + Wb + 1 < nb;
            if (more && pf) fetch_block_row(J + Wb + 1);
            // (b) panel X = A_panel L_JJ^-T (one 8-row block per unit) and right-hand sides Z_J = L_JJ^-1 B_J (one
            // 8-member tile per unit)
            {
                const double li0 = linv(Lp, invd, g8, t4), li1 = linv(Lp, invd, g8, 4 + t4);
                for (int u = warp; u < nbl + nct; u += nwarps) {
                    double c0 = 0.0, c1 = 0.0;
                    if (u < nbl) {
                        int wr0 = s1 + 8 * u; if (wr0 >= Wr) wr0 -= Wr;
                        const double *ar = Aw + (size_t)(wr0 + g8) * pitch + sJ + t4;
                        mma_f64(c0, c1, ar[0], li0);
                        mma_f64(c0, c1, ar[4], li1);
                        *reinterpret_cast<double2 *>(Lp + (8 + 8 * u + g8) * LP_PITCH + 2 * t4) = make_double2(c0, c1);
                    } else {
                        const int ct = u - nbl;
                        const double *br = Rw + (size_t)(sJ + t4) * NR + 8 * ct + g8;
                        mma_f64(c0, c1, li0, br[0]);
                        mma_f64(c0, c1, li1, br[(size_t)4 * NR]);
                        const int col = 8 * ct + 2 * t4;
                        *reinterpret_cast<double2 *>(Zb + (size_t)g8 * NR + col) = make_double2(c0, c1);
                        double *zg = Z + (int64_t)(8 * J + g8) * N + col;
                        if (col < N) zg[0] = c0;
                        if (col + 1 < N) zg[1] = c1;
                    }
                }
            }
            __syncthreads();
            K3T(4);
            // (e) block row J of the window (A rows and right-hand sides) was consumed by (b): the next block row goes into its slot
            // now, which also ends the life of the prefetch registers before the serial factorisation below
            if (more) { if (pf) commit_block_row(sJ, s1); else load_block_row(J + Wb + 1); }
            // L block -> global (overwrites the A rows of block J, already consumed)
            for (int e = tid; e < (8 + below) * 8; e += nthreads)
                band[(int64_t)8 * J * Wr + e] = Lp[(e >> 3) * LP_PITCH + (e & 7)];
            // (c) trailing update A[rb, cb] -= L_rb L_cb^T and (d) right-hand sides B[rb, :] -= L_rb Z_J.  Warp 0 owns
            // tile (0, 0) = the next diagonal block and (a) factors it right away; the other warps share the rest.
            {
                const int nC = nbl * (nbl + 1) / 2;
                auto l_frag = [&](int blk, double &a0, double &a1) {
                    const double *l = Lp + (8 + 8 * blk + g8) * LP_PITCH + t4;
                    a0 = l[0]; a1 = l[4];
                };
                auto c_tile = [&](int rb, int cb) {
                    double a0, a1, b0, b1;
                    l_frag(rb, a0, a1);
                    l_frag(cb, b0, b1);
                    int wr0 = s1 + 8 * rb; if (wr0 >= Wr) wr0 -= Wr;
                    int wc0 = s1 + 8 * cb; if (wc0 >= Wr) wc0 -= Wr;
                    double2 *cp = reinterpret_cast<double2 *>(Aw + (size_t)(wr0 + g8) * pitch + wc0 + 2 * t4);
                    double2 c = *cp;
                    mma_f64(c.x, c.y, -a0, b0);
                    mma_f64(c.x, c.y, -a1, b1);
                    *cp = c;
                };
                // The FP64 pipe of a sub-partition serves DFMA and DMMA alike: the serial factorisation of warp 0 would
                // queue behind the tile products of the warps sharing its sub-partition (warps 4, 8, 12), so those sit
                // this phase out when the next block has to be factored; the other twelve share the tiles.
                const bool spare = (J + 1 < nb) && nwarps >= 8;
                const int nwork = spare ? nwarps - (nwarps >> 2) : nwarps - 1;
                const int widx = spare ? ((warp & 3) ? warp - 1 - (warp >> 2) : -1) : warp - 1;
                if (warp == 0) {
                    K3T(12);
                    if (nbl > 0) c_tile(0, 0);
                    K3T(13);
#ifdef ENKFMC_K3B_TWICE
                    if (J + 1 < nb) {     // (timing experiment: the second pass through the same code is the hot-instruction-cache cost)
#pragma unroll 1
                        for (int rep = 0; rep < 2; ++rep) { __syncwarp(); factor_diag(s1, (J + 1) & 1); if (rep == 0) K3T(14); else K3T(15); }
                    }
#else
                    if (J + 1 < nb) { __syncwarp(); factor_diag(s1, (J + 1) & 1); }
                    K3T(14);
#endif
                } else if (widx >= 0) {
                    for (int u = 1 + widx; u < nC; u += nwork) {
                        const int rc = strips[u];
                        c_tile(rc >> 8, rc & 255);
                    }
                    // (d): units (rb, ct), rb-major, continuing the round-robin where (c) stopped
                    int u = nC > 0 ? widx - (nC - 1) % nwork : widx;
                    if (u < 0) u += nwork;
                    int rb = 0, ct = u;
                    while (ct >= nct) { ct -= nct; ++rb; }
                    while (rb < nbl) {
                        double a0, a1;
                        l_frag(rb, a0, a1);
                        int wr0 = s1 + 8 * rb; if (wr0 >= Wr) wr0 -= Wr;
                        double2 *cp = reinterpret_cast<double2 *>(Rw + (size_t)(wr0 + g8) * NR + 8 * ct + 2 * t4);
                        double2 c = *cp;
                        mma_f64(c.x, c.y, -a0, Zb[(size_t)t4 * NR + 8 * ct + g8]);
                        mma_f64(c.x, c.y, -a1, Zb[(size_t)(4 + t4) * NR + 8 * ct + g8]);
                        *cp = c;
                        ct += nwork;
                        while (ct >= nct) { ct -= nct; ++rb; }
                    }
                }
            }
            K3T(5);
            K3T(6);
            __syncthreads();
            K3T(7);
            sJ = s1;
        }
        if (s_fail) {
            if (tid == 0) P.status[(int64_t)f * P.ntiles + t] = s_fail;
            continue;
        }

        // ---- backward: L^T x = z blockwise, Xa = Xb + dx on interior rows --------------------
        // One warp per 8-member tile: S = L_below^T x (chain of tensor-core products over the rows below), then
        // x_J = L_JJ^-T (z_J - S) with the stored inverse; one barrier per block.
        double *red = Aw;                       // [8][NR] staging of z_J - S (the A window is dead now)
        const bool pfb = 8 * Wr <= 2 * nthreads;
        double fl2[2];
        auto fetch_panel = [&](int J) {
            const int below = (nb - 1 - J < Wb ? nb - 1 - J : Wb) * 8;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int e = tid + k * nthreads;
                fl2[k] = (e < (8 + below) * 8) ? band[(int64_t)8 * J * Wr + e] : 0.0;
            }
        };
        auto commit_panel = [&](int J, double *dst, double *rinv) {
            const int below = (nb - 1 - J < Wb ? nb - 1 - J : Wb) * 8;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int e = tid + k * nthreads;
                if (e < (8 + below) * 8) {
                    dst[(e >> 3) * LP_PITCH + (e & 7)] = fl2[k];
                    if (e < 64 && (e >> 3) == (e & 7)) rinv[e & 7] = 1.0 / fl2[k];
                }
            }
        };
        auto load_panel = [&](int J, double *dst, double *rinv) {
            if (pfb) { fetch_panel(J); commit_panel(J, dst, rinv); return; }
            const int below = (nb - 1 - J < Wb ? nb - 1 - J : Wb) * 8;
            for (int e = tid; e < (8 + below) * 8; e += nthreads) {
                const double v = band[(int64_t)8 * J * Wr + e];
                dst[(e >> 3) * LP_PITCH + (e & 7)] = v;
                if (e < 64 && (e >> 3) == (e & 7)) rinv[e & 7] = 1.0 / v;
            }
        };
        load_panel(nb - 1, Lp0, rinv0);
        __syncthreads();
        K3T(8);
        int sB = ((nb - 1) % nslot) * 8;                // window slot of block row J
        for (int J = nb - 1; J >= 0; --J) {
            const int cur = (nb - 1 - J) & 1;
            const double *Lc = Lp0 + (size_t)cur * WrMax * LP_PITCH;
            const double *rinvc = rinv0 + 8 * cur;
            double *Ln = Lp0 + (size_t)(cur ^ 1) * WrMax * LP_PITCH;
            const int below = (nb - 1 - J < Wb ? nb - 1 - J : Wb) * 8;
            int s1 = sB + 8; if (s1 >= Wr) s1 = 0;
            // this warp's first tile of z_J (B-fragment layout) and the next panel: issued now, used after the sums
            double zf0 = 0.0, zf1 = 0.0;
            if (warp < nct) {
                const int col = 8 * warp + g8;
                if (col < N) { zf0 = Z[(int64_t)(8 * J + t4) * N + col]; zf1 = Z[(int64_t)(8 * J + 4 + t4) * N + col]; }
            }
            // the background values of the interior rows this lane will write (first tile), likewise
            int xi0 = -1;
            double xb0 = 0.0, xb1 = 0.0;
            if (warp < nct) {
                const int i = 8 * J + g8;
                if (rows_cached) xi0 = rxi[i];
                else if (i < n) { const int il = iphys[i]; if (inter[il]) xi0 = srow[il]; }
                const int col = 8 * warp + 2 * t4;
                if (xi0 >= 0) {
                    if (col < N) xb0 = Xf[(int64_t)xi0 * N + col];
                    if (col + 1 < N) xb1 = Xf[(int64_t)xi0 * N + col + 1];
                }
            }
            K3T(16);
            if (J > 0 && pfb) fetch_panel(J - 1);
            K3T(17);
            const double lt0 = linv(Lc, rinvc, t4, g8), lt1 = linv(Lc, rinvc, 4 + t4, g8);   // (L_JJ^-T)[g8][k]
            for (int ct = warp; ct < nct; ct += nwarps) {
                double p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll 4
                for (int k0 = 0; k0 < below; k0 += 8) {
                    int w = s1 + k0; if (w >= Wr) w -= Wr;
                    const double *lk = Lc + (8 + k0 + t4) * LP_PITCH + g8;
                    const double *xk = Rw + (size_t)(w + t4) * NR + 8 * ct + g8;
                    mma_f64(p0, p1, lk[0], xk[0]);
                    mma_f64(q0, q1, lk[4 * LP_PITCH], xk[(size_t)4 * NR]);
                }
                K3T(18);
                // S (C-fragment layout) -> shared -> B fragments of z_J - S, within the warp
                double *rd = red + 8 * ct;
                *reinterpret_cast<double2 *>(rd + (size_t)g8 * NR + 2 * t4) = make_double2(p0 + q0, p1 + q1);
                __syncwarp();
                if (ct != warp) {
                    const int col = 8 * ct + g8;
                    zf0 = zf1 = 0.0;
                    if (col < N) { zf0 = Z[(int64_t)(8 * J + t4) * N + col]; zf1 = Z[(int64_t)(8 * J + 4 + t4) * N + col]; }
                }
                const double w0 = zf0 - rd[(size_t)t4 * NR + g8], w1 = zf1 - rd[(size_t)(4 + t4) * NR + g8];
                K3T(19);
                double x0 = 0.0, x1 = 0.0;
                mma_f64(x0, x1, lt0, w0);
                mma_f64(x0, x1, lt1, w1);
                const int col = 8 * ct + 2 * t4;
                if (col < N && (!(fabs(x0) < DBL_MAX) || (col + 1 < N && !(fabs(x1) < DBL_MAX)))) s_fail = 3;   // benign race
                *reinterpret_cast<double2 *>(Rw + (size_t)(sB + g8) * NR + col) = make_double2(x0, x1);
                if (xi0 >= 0) {
                    const int64_t gidx = (int64_t)xi0 * N + col;
                    if (ct != warp) {
                        if (col < N) xb0 = Xf[gidx];
                        if (col + 1 < N) xb1 = Xf[gidx + 1];
                    }
                    if (col < N) Xaf[gidx] = xb0 + x0;
                    if (col + 1 < N) Xaf[gidx + 1] = xb1 + x1;
                }
                __syncwarp();
                K3T(20);
            }
            K3T(9);
            if (J > 0) { if (pfb) commit_panel(J - 1, Ln, rinv0 + 8 * (cur ^ 1)); else load_panel(J - 1, Ln, rinv0 + 8 * (cur ^ 1)); }
            K3T(10);
            __syncthreads();
            K3T(11);
            sB = sB == 0 ? Wr - 8 : sB - 8;
        }
        if (tid == 0) P.status[(int64_t)f * P.ntiles + t] = s_fail;
    }
}

// Scratch / shared-memory layout chosen on the host.
static size_t solve_fixed_doubles(const SolveParams &p) {
    const int Wb = solve_wb(p.bmax), Wr = 8 * (Wb + 1);
    return 2 * (size_t)Wr * LP_PITCH + 8 * (size_t)p.nr_pitch + 32 + solve_strip_doubles(Wb) + solve_rowsrc_doubles(p.rows_smem);
}

int64_t solve_plan_scratch(SolveParams &p, int64_t nmax, size_t smem_limit) {
    const int64_t Wb = solve_wb(p.bmax), Wr = 8 * (Wb + 1), pitch = Wr + 2;
    // member pitch: covers the padded 8-member tiles and is 8 mod 16, so fragment loads of consecutive rows fall
    // into different bank halves
    p.nr_pitch = (p.N + 7) / 8 * 8;
    if (p.nr_pitch % 16 == 0) p.nr_pitch += 8;
    // per-row source tables in shared memory (3 x int32 per row) for tiles of up to 4096 rows
    p.rows_smem = nmax <= 4096 ? (int)((nmax + 7) / 8 * 8) : 0;
    const size_t fixed = solve_fixed_doubles(p) * sizeof(double) + 64;
    // the A window doubles as the [8][nr_pitch] buffer of the backward pass
    const size_t a_doubles = std::max<size_t>((size_t)(Wr * pitch), (size_t)8 * p.nr_pitch);
    const size_t r_bytes = (size_t)(Wr * p.nr_pitch) * sizeof(double);
    p.a_doubles = (int64_t)a_doubles;
    p.a_in_smem = fixed + a_doubles * sizeof(double) <= smem_limit;
    p.r_in_smem = fixed + (p.a_in_smem ? a_doubles * sizeof(double) : 0) + r_bytes <= smem_limit;
    int64_t off = 0;
    p.off_z = off; off += ((nmax + 7) / 8 * 8) * p.N;
    p.off_win_a = off; if (!p.a_in_smem) off += (int64_t)a_doubles;
    p.off_win_r = off; if (!p.r_in_smem) off += Wr * p.nr_pitch;
    off = (off + 15) & ~(int64_t)15;
    p.scratch_stride = off;
    return off;
}

static size_t solve_smem_bytes(const SolveParams &p) {
    const int64_t Wb = solve_wb(p.bmax), Wr = 8 * (Wb + 1), pitch = Wr + 2;
    size_t rest = 0;
    if (p.a_in_smem) rest += (size_t)p.a_doubles;
    if (p.r_in_smem) rest += (size_t)(Wr * p.nr_pitch);
    (void)pitch;
    return (solve_fixed_doubles(p) + rest) * sizeof(double);
}

int solve_grid_size(int sm_count, const SolveParams &p, size_t smem_limit) {
    const size_t smem = solve_smem_bytes(p) + 1024;
    int per_sm = (int)((smem_limit + 1024) / smem);
    if (per_sm < 1) per_sm = 1;
    if (per_sm > 4) per_sm = 4;
    int64_t grid = (int64_t)sm_count * per_sm;
    const int64_t items = (int64_t)p.nfields * p.ntiles_owned;
    if (grid > items) grid = items;
    return (int)(grid < 1 ? 1 : grid);
}

cudaError_t launch_assemble_band(const SolveParams &p, int sm_count, size_t smem_limit, cudaStream_t s) {
    const int64_t total = p.nrows_owned * (p.f1 - p.f0);
    if (total == 0) return cudaSuccess;
    const size_t tile_smem = asm_tile_smem_bytes(p.asm_nmax, p.asm_nnzmax, p.bmax);
    // (ENKFMC_K3A=rows forces the warp-per-row form that large tiles fall back to: tests compare the two)
    const char *k3a_sel = getenv("ENKFMC_K3A");
    // tensor-core form: every tile in its local order and a ring that fits (ENKFMC_K3A=tile / rows force the gather forms)
    if (p.all_mono && !k3a_sel && asmm_smem_bytes(p.bmax) + 2048 <= smem_limit) {
        const size_t smem = asmm_smem_bytes(p.bmax);
        cudaError_t e = cudaFuncSetAttribute(assemble_band_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        assemble_band_mma_kernel<<<(unsigned)((int64_t)p.ntiles_owned * (p.f1 - p.f0)), ASMM_THREADS, smem, s>>>(p);
        return cudaGetLastError();
    }
    if (p.asm_nmax > 0 && p.asm_nmax < 65536 && p.asm_nnzmax < 65536 && tile_smem + 2048 <= smem_limit &&   // 1 KB is reserved per CTA
        !(k3a_sel && k3a_sel[0] == 'r')) {
        cudaError_t e = cudaFuncSetAttribute(assemble_band_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)tile_smem);
        if (e != cudaSuccess) return e;
        assemble_band_tile_kernel<<<(unsigned)((int64_t)p.ntiles_owned * (p.f1 - p.f0)), ASMT_THREADS, tile_smem, s>>>(p);
        return cudaGetLastError();
    }
    int64_t grid = (total + ASM_WARPS - 1) / ASM_WARPS;
    if (grid > (int64_t)sm_count * 8) grid = (int64_t)sm_count * 8;
    const size_t smem = (size_t)ASM_WARPS * 8 * (solve_wb(p.bmax) + 1) * sizeof(double);
    if (smem + 2048 > smem_limit) return cudaErrorInvalidConfiguration;     // band too wide for a shared-memory row
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(assemble_band_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    assemble_band_kernel<<<(unsigned)grid, ASM_WARPS * 32, smem, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_local_solve(const SolveParams &p, int grid, size_t smem_limit, cudaStream_t s) {
    if ((p.f1 - p.f0) * p.ntiles_owned == 0) return cudaSuccess;
    const size_t smem = solve_smem_bytes(p);
    if (smem > smem_limit) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(local_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(p.counter, 0, sizeof(unsigned int), s);   // p.counter[1] counts clamped pivots (caller zeroes)
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

// ------------------------------------------------------------------------------------------
// Unit-triangular solves with many right-hand sides (factors.py:98-134: sqrt_solve, covariance_apply).
// One thread per right-hand-side column walks the rows in dependency order; the row's sparse entries
// are shared by all columns (broadcast loads), B is [n][ncols] (column index fastest: coalesced).
//   transposed = 0:  (I + L) X = diag(scale_in) B          forward substitution over CSR rows
//   transposed = 1:  (I + L)^T X = B, then X *= scale_out   backward substitution over CSC columns
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(128) unit_tri_solve_kernel(int transposed, const int64_t *__restrict__ ptr,
                                                            const int32_t *__restrict__ idx, const int64_t *__restrict__ src,
                                                            const double *__restrict__ T, const double *__restrict__ scale_in,
                                                            const double *__restrict__ scale_out, double *__restrict__ B,
                                                            int64_t n, int64_t ncols) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncols) return;
    for (int64_t k = 0; k < n; ++k) {
        const int64_t r = transposed ? n - 1 - k : k;
        double acc = B[r * ncols + c];
        if (scale_in) acc *= scale_in[r];
        for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e)
            acc = fma(-T[src ? src[e] : e], B[(int64_t)idx[e] * ncols + c], acc);
        B[r * ncols + c] = acc;
    }
    if (scale_out)
        for (int64_t r = 0; r < n; ++r) B[r * ncols + c] *= scale_out[r];
}

cudaError_t launch_unit_tri_solve(int transposed, const int64_t *ptr, const int32_t *idx, const int64_t *src, const double *T,
                                  const double *scale_in, const double *scale_out, double *B, int64_t n, int64_t ncols,
                                  cudaStream_t s) {
    if (n == 0 || ncols == 0) return cudaSuccess;
    unit_tri_solve_kernel<<<(unsigned)((ncols + 127) / 128), 128, 0, s>>>(transposed, ptr, idx, src, T, scale_in, scale_out, B, n, ncols);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// Forecast step of the periodic advection-diffusion toy model (models.py:114-132) on the device-resident ensemble:
// first-order upwind advection, centred diffusion, unit grid.  One thread per (cell, member); the member index is the
// fastest, so the five neighbour rows are read coalesced.  The operation order is the reference's and nothing is
// contracted into FMAs (round-to-nearest intrinsics), so a step is bit-identical to the numpy expression.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) advdiff_step_kernel(const double *__restrict__ in, double *__restrict__ out, int64_t nx,
                                                          int64_t ny, int row_major, int64_t nfields, int N, double ux,
                                                          double uy, double dt, double kappa) {
    const int64_t total = nx * ny * nfields * (int64_t)N;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int m = (int)(i % N);
        const int64_t cell = i / N, f = cell / (nx * ny), lab = cell % (nx * ny);
        const int64_t r = row_major ? lab / nx : lab % ny, c = row_major ? lab % nx : lab / ny;
        auto at = [&](int64_t rr, int64_t cc) {
            rr = (rr + ny) % ny; cc = (cc + nx) % nx;
            const int64_t l = row_major ? rr * nx + cc : cc * ny + rr;
            return in[((f * nx * ny) + l) * N + m];
        };
        const double u = at(r, c), un = at(r - 1, c), us = at(r + 1, c), uw = at(r, c - 1), ue = at(r, c + 1);
        const double ddx = ux >= 0.0 ? __dsub_rn(u, uw) : __dsub_rn(ue, u);
        const double ddy = uy >= 0.0 ? __dsub_rn(u, un) : __dsub_rn(us, u);
        const double lap = __dsub_rn(__dadd_rn(__dadd_rn(__dadd_rn(un, us), uw), ue), __dmul_rn(4.0, u));
        const double tend = __dadd_rn(__dsub_rn(__dmul_rn(-ux, ddx), __dmul_rn(uy, ddy)), __dmul_rn(kappa, lap));
        out[i] = __dadd_rn(u, __dmul_rn(dt, tend));
    }
}

cudaError_t launch_advdiff_step(const double *in, double *out, int64_t nx, int64_t ny, int row_major, int64_t nfields, int N,
                                double ux, double uy, double dt, double kappa, int sm_count, cudaStream_t s) {
    const int64_t total = nx * ny * nfields * (int64_t)N;
    if (total == 0) return cudaSuccess;
    int64_t blocks = (total + 255) / 256;
    if (blocks > (int64_t)sm_count * 16) blocks = (int64_t)sm_count * 16;
    advdiff_step_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, out, nx, ny, row_major, nfields, N, ux, uy, dt, kappa);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// LETKF baseline (kernels.py:251-335), the paper's comparison method: at every grid point the ensemble-space weights
// from the observations inside its local box,
//     M = Z^T R^-1 Z + (N-1)/inflation I = Q Lambda Q^T,   wa = Q Lambda^-1 Q^T Z^T R^-1 (y - H xb_mean),
//     Wa = Q sqrt((N-1)/Lambda) Q^T,                        xa_row = mean + U_c (wa 1^T + Wa).
// One CTA per (field, grid point): M and Q (N x N each) live in shared memory; the symmetric eigendecomposition is a
// cyclic two-sided Jacobi with a round-robin ordering (N/2 disjoint rotations per round; rows, then columns of M and
// Q, updated by all threads).  Points without observations in their box keep the background row (bit for bit when
// inflation = 1: kernels.py:328-329).
// ------------------------------------------------------------------------------------------
#define LETKF_THREADS 256
#define LETKF_MAX_SWEEPS 30

__global__ void __launch_bounds__(256) mean_anomaly_kernel(const double *__restrict__ X, double *__restrict__ U, double *__restrict__ mean,
                                                          int64_t nrows, int N) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < nrows; row += warps) {
        double s = 0.0;
        for (int i = lane; i < N; i += 32) s += X[row * N + i];
        const double m = warp_sum(s) / (double)N;
        for (int i = lane; i < N; i += 32) U[row * N + i] = X[row * N + i] - m;
        if (lane == 0) mean[row] = m;
    }
}

__global__ void __launch_bounds__(LETKF_THREADS) letkf_kernel(const LetkfParams P) {
    extern __shared__ double smem[];
    const int N = P.N, ld = N | 1, tid = threadIdx.x, nth = blockDim.x;
    const int M2 = (N + 1) & ~1, npairs = M2 >> 1;
    double *Ms = smem;                        // [N][ld]
    double *Qs = Ms + (size_t)N * ld;         // [N][ld]
    double *zb = Qs + (size_t)N * ld;         // [N] current observation row / scratch
    double *zri = zb + N;                     // [N]
    double *lamv = zri + N;                   // [N]
    double *tv = lamv + N;                    // [N]
    double *gv = tv + N;                      // [N]
    double *cs = gv + N;                      // [npairs]
    double *sn = cs + npairs;                 // [npairs]
    int *ip = reinterpret_cast<int *>(sn + npairs);   // [npairs] p, [npairs] q
    int *iq = ip + npairs;
    int *box_state = iq + npairs;             // [(2 zeta + 1)^2] state rows of the observed box members
    int *box_slot = box_state + P.boxmax;     // their observation rows
    __shared__ int s_item, s_m, s_rot, s_rows[64], s_cols[64], s_nr, s_nc;
    const double alpha = (double)(N - 1) / P.inflation;
    const int64_t n2d = P.nx * P.ny;

    for (;;) {
        if (tid == 0) s_item = (int)atomicAdd(P.counter, 1u);
        __syncthreads();
        const int64_t item = s_item;
        if (item >= P.nitems) break;
        const int64_t f = item / n2d, lab = item % n2d;
        const int64_t r0 = P.row_major ? lab / P.nx : lab % P.ny, c0 = P.row_major ? lab % P.nx : lab / P.ny;
        const int64_t srow = f * n2d + lab;
        // ---- box members (geometry.py:132-156) with an observation, in ascending label order ----
        if (tid == 0) {
            auto window = [&](int64_t ctr, int64_t n, bool per, int *out) {
                int cnt = 0;
                if (per) {
                    for (int64_t d = -P.zeta; d <= P.zeta; ++d) {
                        const int v = (int)(((ctr + d) % n + n) % n);
                        int k = cnt;
                        bool dup = false;
                        for (int e = 0; e < cnt; ++e) if (out[e] == v) dup = true;
                        if (dup) continue;
                        while (k > 0 && out[k - 1] > v) { out[k] = out[k - 1]; --k; }
                        out[k] = v;
                        ++cnt;
                    }
                } else {
                    const int64_t lo = ctr - P.zeta < 0 ? 0 : ctr - P.zeta, hi = ctr + P.zeta + 1 > n ? n : ctr + P.zeta + 1;
                    for (int64_t v = lo; v < hi; ++v) out[cnt++] = (int)v;
                }
                return cnt;
            };
            s_nr = window(r0, P.ny, P.periodic == 1 || P.periodic == 3, s_rows);
            s_nc = window(c0, P.nx, P.periodic == 1 || P.periodic == 2, s_cols);
            int m = 0;
            const int na = P.row_major ? s_nr : s_nc, nb = P.row_major ? s_nc : s_nr;
            for (int a = 0; a < na; ++a)
                for (int b = 0; b < nb; ++b) {
                    const int64_t rr = P.row_major ? s_rows[a] : s_rows[b], cc = P.row_major ? s_cols[b] : s_cols[a];
                    const int64_t l = P.row_major ? rr * P.nx + cc : cc * P.ny + rr;
                    const int slot = P.obs_of_state[f * n2d + l];
                    if (slot >= 0) { box_state[m] = (int)(f * n2d + l); box_slot[m] = slot; ++m; }
                }
            s_m = m;
        }
        __syncthreads();
        const int m = s_m;
        double *xa = P.Xa + srow * N;
        const double *ub = P.U + srow * N;
        if (m == 0) {
            if (P.inflation == 1.0) { for (int i = tid; i < N; i += nth) xa[i] = P.X[srow * N + i]; }
            else { const double sq = sqrt(P.inflation), mc = P.mean[srow]; for (int i = tid; i < N; i += nth) xa[i] = mc + sq * ub[i]; }
            __syncthreads();
            continue;
        }
        // ---- M = alpha I + sum_o z_o z_o^T / r_o,  zri = sum_o z_o (y_o - mean_o) / r_o ----
        for (int e = tid; e < N * ld; e += nth) { const int i = e / ld, j = e - i * ld; Ms[e] = (i == j) ? alpha : 0.0; Qs[e] = (i == j) ? 1.0 : 0.0; }
        for (int i = tid; i < N; i += nth) zri[i] = 0.0;
        __syncthreads();
        for (int o = 0; o < m; ++o) {
            const int st = box_state[o], sl = box_slot[o];
            const double rinv = 1.0 / P.rdiag[sl];
            for (int i = tid; i < N; i += nth) zb[i] = P.U[(int64_t)st * N + i];
            __syncthreads();
            const double w = (P.y[sl] - P.mean[st]) * rinv;
            for (int e = tid; e < N * N; e += nth) { const int i = e / N, j = e - i * N; Ms[i * ld + j] = fma(zb[i] * rinv, zb[j], Ms[i * ld + j]); }
            for (int i = tid; i < N; i += nth) zri[i] = fma(zb[i], w, zri[i]);
            __syncthreads();
        }
        // ---- cyclic two-sided Jacobi: M <- J^T M J, Q <- Q J ----
        double dmax = 0.0;
        for (int k = 0; k < N; ++k) dmax = fmax(dmax, Ms[k * ld + k]);        // (every thread: N broadcast reads)
        const double thr = 4.0 * sqrt((double)N) * DBL_EPSILON * dmax;
        int sweep = 0;
        for (; sweep < LETKF_MAX_SWEEPS; ++sweep) {
            if (tid == 0) s_rot = 0;
            __syncthreads();
            for (int rr = 0; rr < M2 - 1; ++rr) {
                if (tid < npairs) {
                    int a, b;
                    if (tid == 0) { a = M2 - 1; b = rr; }
                    else { a = (rr + tid) % (M2 - 1); b = (rr - tid + (M2 - 1)) % (M2 - 1); }
                    if (a > b) { const int t = a; a = b; b = t; }
                    double c = 1.0, s = 0.0;
                    if (b < N) {
                        const double app = Ms[a * ld + a], aqq = Ms[b * ld + b], apq = Ms[a * ld + b];
                        // classical criterion: an off-diagonal entry at the rounding level of the largest diagonal entry is
                        // converged (the rotations that involve the large eigenvalues regenerate such entries every sweep)
                        if (fabs(apq) > thr) {
                            const double tau = (aqq - app) / (2.0 * apq);
                            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                            c = 1.0 / sqrt(1.0 + t * t);
                            s = t * c;
                            s_rot = 1;
                        }
                    } else { b = a; }                       // the dummy index of an odd N: nothing to do
                    cs[tid] = c; sn[tid] = s; ip[tid] = a; iq[tid] = b;
                }
                __syncthreads();
                for (int e = tid; e < npairs * N; e += nth) {          // rows p, q of M
                    const int k = e / N, j = e - k * N;
                    const double s = sn[k];
                    if (s != 0.0) {
                        const double c = cs[k];
                        const int a = ip[k], b = iq[k];
                        const double x = Ms[a * ld + j], y = Ms[b * ld + j];
                        Ms[a * ld + j] = c * x - s * y;
                        Ms[b * ld + j] = s * x + c * y;
                    }
                }
                __syncthreads();
                for (int e = tid; e < npairs * N; e += nth) {          // columns p, q of M and of Q
                    const int k = e / N, i = e - k * N;
                    const double s = sn[k];
                    if (s != 0.0) {
                        const double c = cs[k];
                        const int a = ip[k], b = iq[k];
                        const double x = Ms[i * ld + a], y = Ms[i * ld + b];
                        Ms[i * ld + a] = c * x - s * y;
                        Ms[i * ld + b] = s * x + c * y;
                        const double u = Qs[i * ld + a], v = Qs[i * ld + b];
                        Qs[i * ld + a] = c * u - s * v;
                        Qs[i * ld + b] = s * u + c * v;
                    }
                }
                __syncthreads();
            }
            const int rotated = s_rot;      // (read by every thread before thread 0 clears it for the next sweep)
            __syncthreads();
            if (!rotated) break;
        }
        // ---- weights and the analysis row ----
        double lmin = DBL_MAX;
        for (int k = tid; k < N; k += nth) { lamv[k] = Ms[k * ld + k]; lmin = fmin(lmin, lamv[k]); }
        if (!(lmin >= P.eig_floor) || sweep >= LETKF_MAX_SWEEPS) atomicMin(P.first_bad, (unsigned long long)srow);   // kernels.py:295-298
        __syncthreads();
        for (int k = tid; k < N; k += nth) {
            double a = 0.0, g = 0.0;
            for (int i = 0; i < N; ++i) { a = fma(Qs[i * ld + k], zri[i], a); g = fma(Qs[i * ld + k], ub[i], g); }
            tv[k] = a / lamv[k];                                      // (Q^T zri) / lambda
            gv[k] = g * sqrt((double)(N - 1) / lamv[k]);              // (U_c Q) sqrt((N-1)/lambda)
        }
        __syncthreads();
        {
            // U_c . wa with wa = Q t
            double part = 0.0;
            for (int i = tid; i < N; i += nth) {
                double wa = 0.0;
                for (int k = 0; k < N; ++k) wa = fma(Qs[i * ld + k], tv[k], wa);
                part = fma(ub[i], wa, part);
            }
            zb[tid < N ? tid : 0] = 0.0;
            __syncthreads();
            if (tid < N) zb[tid] = part;
            __syncthreads();
            if (tid == 0) { double t = 0.0; for (int i = 0; i < N && i < nth; ++i) t += zb[i]; zb[0] = t; }
            __syncthreads();
        }
        const double base = P.mean[srow] + zb[0];
        for (int j = tid; j < N; j += nth) {
            double acc = 0.0;
            for (int k = 0; k < N; ++k) acc = fma(gv[k], Qs[j * ld + k], acc);
            xa[j] = base + acc;
        }
        __syncthreads();
    }
}

size_t letkf_smem_bytes(int N, int boxmax) {
    const int ld = N | 1, npairs = ((N + 1) & ~1) >> 1;
    return ((size_t)2 * N * ld + 5 * (size_t)N + 2 * (size_t)npairs) * sizeof(double) + ((size_t)2 * npairs + 2 * (size_t)boxmax) * sizeof(int) + 16;
}

cudaError_t launch_letkf(const LetkfParams &p, int sm_count, size_t smem_limit, cudaStream_t s) {
    if (p.nitems == 0) return cudaSuccess;
    const size_t smem = letkf_smem_bytes(p.N, p.boxmax);
    if (smem > smem_limit || 2 * p.zeta + 1 > 64) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(letkf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t nrows = p.nitems;
    int64_t blocks = (nrows + 7) / 8;
    if (blocks > (int64_t)sm_count * 16) blocks = (int64_t)sm_count * 16;
    mean_anomaly_kernel<<<(unsigned)blocks, 256, 0, s>>>(p.X, p.U, p.mean, nrows, p.N);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    int per_sm = (int)(smem_limit / (smem + 1024));
    if (per_sm < 1) per_sm = 1;
    if (per_sm > 4) per_sm = 4;
    int64_t grid = (int64_t)sm_count * per_sm;
    if (grid > p.nitems) grid = p.nitems;
    letkf_kernel<<<(unsigned)grid, LETKF_THREADS, smem, s>>>(p);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// FP64 DFMA peak: 8 independent FMA chains per thread, register resident.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) fp64_peak_kernel(double *out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-3, x1 = x0 + 1.0, x2 = x0 + 2.0, x3 = x0 + 3.0, x4 = x0 + 4.0, x5 = x0 + 5.0,
           x6 = x0 + 6.0, x7 = x0 + 7.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 123.456) out[0] = s;   // never true; keeps the chains alive
}

// FP64 tensor-core peak: mma.sync m8n8k4 f64, 8 independent accumulator tiles per warp.
__global__ void __launch_bounds__(256) dmma_peak_kernel(double *out, int iters, double a, double b) {
    double c[8][2];
#pragma unroll
    for (int u = 0; u < 8; ++u) { c[u][0] = threadIdx.x * 1e-3 + u; c[u][1] = c[u][0] + 0.5; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[u][0]), "+d"(c[u][1]) : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1];
    if (s == 123.456) out[0] = s;
}

cudaError_t launch_dmma_peak(double *out, int iters, int sm_count, cudaStream_t s) {
    dmma_peak_kernel<<<sm_count * 8, 256, 0, s>>>(out, iters, 0.999999, 1e-7);
    return cudaGetLastError();
}

cudaError_t launch_fp64_peak(double *out, int iters, int sm_count, cudaStream_t s) {
    fp64_peak_kernel<<<sm_count * 8, 256, 0, s>>>(out, iters, 0.999999, 1e-7);
    return cudaGetLastError();
}
