// K2b: truncated-SVD semantics of the per-component regression (estimator.py:46-61) on the packed QR output of K2a.
// Included by kernels.cu (inside its translation unit, after the warp-level helpers and K2a).
//
// Two kernels, one warp per regression:
//
//  regress_clean_kernel (K2b-1, small workspace, high occupancy).  R | c unpacked to shared memory.  X = R^-1 by 8 x 8
//    blocks on the FP64 tensor cores gives sum 1/s_i^2 = |X|_F^2, a rigorous lower bound of the smallest singular
//    value: if it clears rank_tol * |R|_F nothing is truncated and beta = R^-1 c by back-substitution.  Otherwise one
//    inverse-iteration probe looks for a single, well separated sub-threshold value (the common case on smooth
//    ensembles with p < N / 2): if it converges and |X|_F^2 - 1/s_1^2 proves every other value above the threshold, the
//    pair is deflated here.  Everything else (several small values, slow convergence, a pivot far below the threshold,
//    more predecessors than members) is appended to a work list.
//
//  regress_trunc_kernel (K2b-2).  For the listed rows the singular values below the threshold are found together by
//    block inverse iteration: an orthonormal block Z (p x b, b = 8, 16, ...; pseudo-random start) is iterated as
//        Y = orth(R^-T Z),  Z G = R^-1 Y  (Z orthonormal, G upper triangular),
//    the triangular solves running eight right-hand sides at a time as tensor-core tile products with the scalar
//    substitution order kept inside each 8 x 8 diagonal tile (an explicit inverse, or inverted diagonal blocks, lose a
//    factor 3-6 in accuracy at cond(R) ~ 1e12).  The block grows by eight vectors until its largest Ritz value is
//    well above the threshold (the smallest |G_kk| bounds it), so that every truncated direction converges at least
//    as fast as (threshold / that value)^2 per sweep; the number of sweeps follows from that ratio.  Rayleigh-Ritz:
//    one-sided Jacobi on the rows of [G | I] gives G = P S Q^T, the Ritz values 1 / S_k of R and the left / right
//    Ritz vectors Y Q, Z P.  With T the set of values below rank_tol * s_max (s_max bracketed by the Frobenius norm
//    and a power iteration that is refined only when a Ritz value falls inside the bracket),
//        beta = (I - Z_T Z_T^T) R^-1 (I - U_T U_T^T) c
//    is the reference's truncated-SVD minimum-norm answer.  Rows with more predecessors than members (R is K x p,
//    K < p) are first reduced by a second Householder QR, R^T = Q2 R2, to the K x K problem R2^T g = c, beta = Q2 g
//    (the roles of the left and right vectors swap).  What cannot be settled this way -- a Ritz value within 1e-6 of
//    the threshold, more small values than the block holds, breakdown -- goes to the general fallback: one-sided
//    Jacobi SVD of the rows of [R | c] with the same rule.
//
//  T = -beta;  D = max((e2 + |c - R beta|^2) / (N - 1), floor): |y - A^T beta|^2 of estimator.py:60,148 in the QR
//  basis (orthogonal invariance), the second term only when something was truncated.
//
// flag bits: 1 row went to K2b-2, 2 truncated, 8 D floored, 16 Jacobi fallback, 5-7 with bit 16: fallback reason (1
// non-finite / breakdown, 2 block too small, 3 Ritz value at the threshold, 4 sweep cap), bit 5 without bit 16: single pair
// deflated in K2b-1, 8-15 block sweeps / probe steps, 16-21 Jacobi sweeps, 22-24 block size / 8.
#pragma once

#define JACOBI_MAX_SWEEPS 30
#define TRUNC_MAX_SWEEPS 16
#define UNPACK_COLS 8          // columns of the packed R fetched together by unpack_rc
#define REG_PROBE_TOL 1e-10    // K2b-1 probe: predicted distance of the iterate to the singular vector at which it stops

__host__ __device__ inline int trunc_zp(int pmax) { return 8 * ((pmax + 7) / 8) + 4; }   // block pitch: = 4 mod 8
__host__ __device__ inline size_t regress_clean_ws_doubles(int pmax) {
    // R | c (pitch pmax|1, pmax+1 columns) | rinv | mma staging
    const size_t d = (size_t)(pmax | 1) * (pmax + 1) + (size_t)pmax + 64;
    return (d + 1) & ~(size_t)1;
}
__host__ __device__ inline size_t regress_trunc_ws_doubles(int pmax, int bmax) {
    // R | c | rinv | aux | tmp | x0 | alpha | Z block | Y block | [G | P] (pitch bmax|1, 2 bmax columns)
    const size_t d = (size_t)(pmax | 1) * (pmax + 1) + (size_t)5 * pmax + (size_t)2 * bmax * trunc_zp(pmax) +
                     (size_t)(bmax | 1) * 2 * bmax;
    return (d + 1) & ~(size_t)1;
}

namespace {

// ---- tensor-core helpers ----------------------------------------------------------------------------------------
__device__ __forceinline__ void mma_f64(double &d0, double &d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// R[r, c] (upper triangular incl. diagonal, column-major in W) with zero padding beyond p
__device__ __forceinline__ double r_elem(const double *W, int ld, int p, int r, int c) {
    return (r <= c && c < p) ? W[(size_t)c * ld + r] : 0.0;
}
// X = R^-1: strictly upper part stored transposed in the strict lower triangle of W, diagonal = rinv
__device__ __forceinline__ double x_elem(const double *W, const double *rinv, int ld, int p, int r, int c) {
    if (r > c || c >= p) return 0.0;
    return r == c ? rinv[r] : W[(size_t)r * ld + c];
}

// |X|_F^2 = sum 1/s_i^2 of X = R^-1, by 8 x 8 blocks on the FP64 tensor cores (mma.sync m8n8k4): X_jj by
// back-substitution (one lane per column), X_ij = -X_ii sum_k R_ik X_kj.  X^T is left in the strict lower triangle
// of W; stage = 64 doubles of per-warp scratch.
__device__ __noinline__ double inverse_norm2_mma(double *W, const double *rinv, int ld, int p, double *stage, int lane) {
    const int t4 = lane & 3, m = lane >> 2;
    const int nbk = (p + 7) >> 3;
    double f2 = 0.0;
    // diagonal blocks, four at a time: lanes 8 g .. 8 g + 7 own the columns of block jb0 + g.  Column c of X_jj by
    // back-substitution held in registers (x[i] = 0 below the diagonal, so every lane runs the same unrolled sums):
    // x_c = 1 / r_cc, x_k = -(sum_{i > k} r_ki x_i) / r_kk.  The block of R is read with block-uniform addresses.
    for (int jb0 = 0; jb0 < nbk; jb0 += 4) {
        const int j = jb0 + (lane >> 3), l8 = lane & 7;
        const int c = 8 * j + l8;
        const bool act = c < p;
        const int j8 = 8 * (j < nbk ? j : nbk - 1);              // (lanes beyond the last block read a valid one; nothing is stored)
        double x[8];
#pragma unroll
        for (int kk = 7; kk >= 0; --kk) {
            const int k = j8 + kk;
            const double rk = k < p ? rinv[k] : 0.0;
            double acc = 0.0;
#pragma unroll
            for (int i = kk + 1; i < 8; ++i) {
                const int ci = j8 + i;
                acc = fma(ci < p ? W[(size_t)ci * ld + k] : 0.0, x[i], acc);        // R[k, ci] X[ci, c]
            }
            x[kk] = kk == l8 ? rk : (kk < l8 ? -rk * acc : 0.0);
        }
        if (act) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                if (kk < l8) W[(size_t)(j8 + kk) * ld + c] = x[kk];                  // X[k, c] at (row c, column k)
                if (kk <= l8) f2 = fma(x[kk], x[kk], f2);
            }
        }
    }
    __syncwarp();
    // blocks above the diagonal, column block by column block: X_ij = -X_ii sum_{i<k<=j} R_ik X_kj.  Only X_jj, X_ii and the
    // last (possibly partial) block column need the guarded element access.
    for (int j = 1; j < nbk; ++j) {
        const bool jfull = 8 * j + 8 <= p;
        for (int i = j - 1; i >= 0; --i) {
            double s0 = 0.0, s1 = 0.0;
            for (int k = i + 1; k < j; ++k) {                                   // dense R_ik (8 k + 7 < p) and dense X_kj
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double a = W[(size_t)(8 * k + 4 * h + t4) * ld + 8 * i + m];
                    const double b = jfull ? W[(size_t)(8 * k + 4 * h + t4) * ld + 8 * j + m]
                                           : x_elem(W, rinv, ld, p, 8 * k + 4 * h + t4, 8 * j + m);
                    mma_f64(s0, s1, a, b);
                }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {                                       // k = j: R_ij may be partial, X_jj is triangular
                const double a = r_elem(W, ld, p, 8 * i + m, 8 * j + 4 * h + t4);
                const double b = x_elem(W, rinv, ld, p, 8 * j + 4 * h + t4, 8 * j + m);
                mma_f64(s0, s1, a, b);
            }
            stage[m * 8 + 2 * t4] = s0;                     // S (8 x 8, row-major) -> B fragments of the next product
            stage[m * 8 + 2 * t4 + 1] = s1;
            __syncwarp();
            double x0 = 0.0, x1 = 0.0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double a = x_elem(W, rinv, ld, p, 8 * i + m, 8 * i + 4 * h + t4);
                mma_f64(x0, x1, a, stage[(4 * h + t4) * 8 + m]);
            }
            const int row = 8 * i + m, c0 = 8 * j + 2 * t4;
            if (c0 < p) W[(size_t)row * ld + c0] = -x0;     // X[row, c0] at (row c0, column row); row < 8 j <= c0
            if (c0 + 1 < p) W[(size_t)row * ld + c0 + 1] = -x1;
            f2 += x0 * x0 + x1 * x1;                        // padded entries are exactly zero
            __syncwarp();
        }
    }
    return warp_sum(f2);
}

// ---- block triangular solves: NS slabs of eight right-hand sides, in place ----------------------------------------
// Blocks are column-major (vector v at B + v * ZP), rows [0, 8 ceil(p / 8)), rows >= p zero.  Accumulator tile of
// block row i and slab s: lane (g8, t4) holds row 8 i + g8 of vectors 8 s + 2 t4 + {0, 1}.  The products with the
// off-diagonal tiles are tensor-core products; inside the diagonal tile the substitution runs row by row (the row
// just finished is broadcast by shuffles), so the arithmetic is that of the scalar substitution.
// R x = b (back substitution).
template <int NS>
__device__ __noinline__ void blk_solve_upper(double *B, int ZP, const double *W, const double *rinv, int ld, int p, int lane) {
    const int t4 = lane & 3, g8 = lane >> 2;
    const int nbk = (p + 7) >> 3;
    for (int i = nbk - 1; i >= 0; --i) {
        const int row = 8 * i + g8;
        double a0[NS], a1[NS], n0[NS], n1[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            a0[s] = B[(size_t)(8 * s + 2 * t4) * ZP + row];
            a1[s] = B[(size_t)(8 * s + 2 * t4 + 1) * ZP + row];
            n0[s] = 0.0; n1[s] = 0.0;
        }
        for (int k = i + 1; k < nbk; ++k) {
            const bool full = 8 * k + 8 <= p;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = 8 * k + 4 * h + t4;
                const double a = (full || col < p) ? W[(size_t)col * ld + row] : 0.0;       // R[row, col], row < col
#pragma unroll
                for (int s = 0; s < NS; ++s) mma_f64(n0[s], n1[s], a, B[(size_t)(8 * s + g8) * ZP + col]);
            }
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) { a0[s] -= n0[s]; a1[s] -= n1[s]; }
#pragma unroll
        for (int c = 7; c >= 0; --c) {
            const int r = 8 * i + c;
            if (r < p) {                                      // warp-uniform
                const double rin = rinv[r];
                const double rr = (g8 < c) ? W[(size_t)r * ld + row] : 0.0;                // R[row, r]
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    const double x0 = __shfl_sync(FULL, a0[s] * rin, 4 * c + t4);
                    const double x1 = __shfl_sync(FULL, a1[s] * rin, 4 * c + t4);
                    if (g8 == c) { a0[s] = x0; a1[s] = x1; }
                    else { a0[s] = fma(-rr, x0, a0[s]); a1[s] = fma(-rr, x1, a1[s]); }
                }
            }
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            B[(size_t)(8 * s + 2 * t4) * ZP + row] = row < p ? a0[s] : 0.0;
            B[(size_t)(8 * s + 2 * t4 + 1) * ZP + row] = row < p ? a1[s] : 0.0;
        }
        __syncwarp();
    }
}

// R^T y = b (forward substitution).
template <int NS>
__device__ __noinline__ void blk_solve_upper_t(double *B, int ZP, const double *W, const double *rinv, int ld, int p, int lane) {
    const int t4 = lane & 3, g8 = lane >> 2;
    const int nbk = (p + 7) >> 3;
    for (int i = 0; i < nbk; ++i) {
        const int row = 8 * i + g8;                          // unknown index = column of R
        const bool live = row < p;
        double a0[NS], a1[NS], n0[NS], n1[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            a0[s] = B[(size_t)(8 * s + 2 * t4) * ZP + row];
            a1[s] = B[(size_t)(8 * s + 2 * t4 + 1) * ZP + row];
            n0[s] = 0.0; n1[s] = 0.0;
        }
        const double *colp = W + (size_t)(live ? row : 0) * ld;
        for (int k = 0; k < i; ++k) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int rr_ = 8 * k + 4 * h + t4;          // < 8 i <= row
                const double a = live ? colp[rr_] : 0.0;     // R[rr_, row]
#pragma unroll
                for (int s = 0; s < NS; ++s) mma_f64(n0[s], n1[s], a, B[(size_t)(8 * s + g8) * ZP + rr_]);
            }
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) { a0[s] -= n0[s]; a1[s] -= n1[s]; }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int r = 8 * i + c;
            if (r < p) {
                const double rin = rinv[r];
                const double rr = (g8 > c && live) ? colp[r] : 0.0;                         // R[r, row]
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    const double x0 = __shfl_sync(FULL, a0[s] * rin, 4 * c + t4);
                    const double x1 = __shfl_sync(FULL, a1[s] * rin, 4 * c + t4);
                    if (g8 == c) { a0[s] = x0; a1[s] = x1; }
                    else { a0[s] = fma(-rr, x0, a0[s]); a1[s] = fma(-rr, x1, a1[s]); }
                }
            }
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            B[(size_t)(8 * s + 2 * t4) * ZP + row] = live ? a0[s] : 0.0;
            B[(size_t)(8 * s + 2 * t4 + 1) * ZP + row] = live ? a1[s] : 0.0;
        }
        __syncwarp();
    }
}

// dst = op(R)^-1 src for a block of b = 8 nsl vectors (src may equal dst)
__device__ __forceinline__ void blk_copy(double *dst, const double *src, int ZP, int b, int lane) {
    if (dst == src) return;
    for (int e = lane; e < b * ZP; e += 32) dst[e] = src[e];
    __syncwarp();
}
__device__ __forceinline__ void blk_solve(bool transposed, double *B, int ZP, int b, const double *W, const double *rinv,
                                          int ld, int p, int lane) {
    for (int c0 = 0; c0 < b;) {                               // slabs in groups of up to three (instruction-level parallelism)
        const int left = (b - c0) >> 3;
        double *Bs = B + (size_t)c0 * ZP;
        if (left >= 3 && left != 4) {
            if (transposed) blk_solve_upper_t<3>(Bs, ZP, W, rinv, ld, p, lane); else blk_solve_upper<3>(Bs, ZP, W, rinv, ld, p, lane);
            c0 += 24;
        } else if (left >= 2) {
            if (transposed) blk_solve_upper_t<2>(Bs, ZP, W, rinv, ld, p, lane); else blk_solve_upper<2>(Bs, ZP, W, rinv, ld, p, lane);
            c0 += 16;
        } else {
            if (transposed) blk_solve_upper_t<1>(Bs, ZP, W, rinv, ld, p, lane); else blk_solve_upper<1>(Bs, ZP, W, rinv, ld, p, lane);
            c0 += 8;
        }
    }
}

// Orthonormalises columns [c0, b) of the block against all earlier columns and each other: classical Gram-Schmidt
// in batches of four with one re-orthogonalisation pass ("twice is enough").  G (may be null): b x b upper
// triangular, element (l, k) at G[k * GP + l], with B_in[:, k] = sum_l G[l, k] B_out[:, l].  Returns false on
// breakdown (a column vanished or is not finite).
template <int PS>
__device__ __noinline__ bool orth_block(double *B, int ZP, int c0, int b, int p, double *G, int GP, int lane, int passes = 2) {
    for (int k = c0; k < b; ++k) {
        Vec<PS> v = vload<PS>(B + (size_t)k * ZP, p, lane);
#pragma unroll 1
        for (int pass = 0; pass < passes; ++pass) {
            for (int l0 = 0; l0 < k; l0 += 4) {
                Vec<PS> q[4];
                double d[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    d[j] = 0.0;
                    const bool on = l0 + j < k;
                    const double *src = B + (size_t)(on ? l0 + j : 0) * ZP;
#pragma unroll
                    for (int t = 0; t < PS; ++t) {
                        const int e = lane + 32 * t;
                        q[j].v[t] = (on && e < p) ? src[e] : 0.0;
                        d[j] = fma(q[j].v[t], v.v[t], d[j]);
                    }
                }
                warp_sum4(d[0], d[1], d[2], d[3], lane);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
#pragma unroll
                    for (int t = 0; t < PS; ++t) v.v[t] = fma(-d[j], q[j].v[t], v.v[t]);
                }
                if (G && lane < 4 && l0 + lane < k) {
                    const double dj = lane == 0 ? d[0] : lane == 1 ? d[1] : lane == 2 ? d[2] : d[3];
                    double *g = G + (size_t)k * GP + l0 + lane;
                    *g = pass ? *g + dj : dj;
                }
            }
        }
        const double n2 = vdot<PS>(v, v);
        if (!(n2 > 0.0) || !(n2 < 1e300)) return false;
        const double nrm = sqrt(n2), inv = 1.0 / nrm;
#pragma unroll
        for (int t = 0; t < PS; ++t) v.v[t] *= inv;
        vstore<PS>(B + (size_t)k * ZP, v, p, lane);
        if (G && lane == 0) G[(size_t)k * GP + k] = nrm;
        __syncwarp();
    }
    return true;
}

// Rotation (cs, sn) that orthogonalises the row pair x, y with x.y = g, |x|^2 = da, |y|^2 = db:
// x' = cs x - sn y, y' = sn x + cs y.  tan = sgn(tau) g / (|tau| + sqrt(tau^2 + g^2)), tau = (db - da) / 2, evaluated with
// reciprocal square roots and one reciprocal (no division / square-root sequences).
__device__ __forceinline__ void jacobi_rotation(double g, double da, double db, double &cs, double &sn) {
    const double tau = 0.5 * (db - da);
    const double h2 = fma(tau, tau, g * g);
    const double r = h2 * rsqrt(h2);
    const double t = (tau >= 0.0 ? g : -g) * __drcp_rn(fabs(tau) + r);
    cs = rsqrt(fma(t, t, 1.0));
    sn = cs * t;
}

// The same on an 8 x 16 matrix held in registers: lane (r, t4) = (lane >> 2, lane & 3) owns M[r][t4 + 4 j], j < 4;
// the first eight columns enter the inner products.  Four disjoint row pairs rotate at a time (round robin).
__device__ __noinline__ int jacobi8_regs(double *W, int ld, int lane) {
    const int r = lane >> 2, t4 = lane & 3;
    double m[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) m[j] = W[(size_t)(t4 + 4 * j) * ld + r];
    const double tol2 = 8.0 * DBL_EPSILON * DBL_EPSILON;
    int sweep = 0;
    bool rotated = true;
    while (rotated && sweep < JACOBI_MAX_SWEEPS) {
        rotated = false;
        ++sweep;
#pragma unroll 1
        for (int rr = 0; rr < 7; ++rr) {
            int partner;
            if (r == 7) partner = rr;
            else if (r == rr) partner = 7;
            else {
                const int d = (r - rr + 7) % 7;
                partner = d <= 3 ? (rr - d + 7) % 7 : (rr + 7 - d) % 7;
            }
            const bool isx = r < partner;                   // the pair's lower row plays x
            double pm[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) pm[j] = __shfl_sync(FULL, m[j], 4 * partner + t4);
            double g = fma(m[1], pm[1], m[0] * pm[0]);
            double dm = fma(m[1], m[1], m[0] * m[0]);
            double dp = fma(pm[1], pm[1], pm[0] * pm[0]);
            g += __shfl_xor_sync(FULL, g, 1); dm += __shfl_xor_sync(FULL, dm, 1); dp += __shfl_xor_sync(FULL, dp, 1);
            g += __shfl_xor_sync(FULL, g, 2); dm += __shfl_xor_sync(FULL, dm, 2); dp += __shfl_xor_sync(FULL, dp, 2);
            const double da = isx ? dm : dp, db = isx ? dp : dm;
            const bool rot = (g * g > tol2 * da * db) && (g != 0.0);
            if (rot) {
                double cs, sn;
                jacobi_rotation(g, da, db, cs, sn);
                const double sg = isx ? -sn : sn;          // x' = cs x - sn y ; y' = cs y + sn x
#pragma unroll
                for (int j = 0; j < 4; ++j) m[j] = fma(sg, pm[j], cs * m[j]);
            }
            if (__any_sync(FULL, rot)) rotated = true;
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) W[(size_t)(t4 + 4 * j) * ld + r] = m[j];
    __syncwarp();
    return (sweep >= JACOBI_MAX_SWEEPS && rotated) ? JACOBI_MAX_SWEEPS + 1 : sweep;
}

// One-sided Jacobi on the rows of a K x na matrix (column-major, pitch ld): plane rotations of row pairs until the
// first nd columns of all rows are mutually orthogonal; the rotations act on all na columns.  Returns the sweeps
// used (JACOBI_MAX_SWEEPS + 1 if not converged).
__device__ __noinline__ int jacobi_rows(double *W, int ld, int K, int nd, int na, int lane) {
    const int M = (K + 1) & ~1;
    const int npairs = M >> 1;
    const int T = lanes_per_item(npairs);
    const int per = 32 / T, sub = lane % T;
    const double tolj = DBL_EPSILON * sqrt((double)nd);
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
                if (on) for (int c = sub; c < nd; c += T) {
                    const double x = ra[(size_t)c * ld], y = rb[(size_t)c * ld];
                    g += x * y; da += x * x; db += y * y;
                }
                g = group_sum(g, T); da = group_sum(da, T); db = group_sum(db, T);
                const bool rot = on && (g * g > tolj * tolj * da * db) && (g != 0.0);
                if (rot) {
                    double cs, sn;
                    jacobi_rotation(g, da, db, cs, sn);
                    double *wa = W + a, *wb = W + b;
                    for (int c = sub; c < na; c += T) {
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
    return (sweep >= JACOBI_MAX_SWEEPS && rotated) ? JACOBI_MAX_SWEEPS + 1 : sweep;
}

// General fallback: one-sided Jacobi SVD on the rows of [R | c] (K x (p+1), explicit zeros below
// the diagonal), truncation as estimator.py:55-57.  Writes beta to out[0..p); returns flag bits and
// the squared norm of the truncated part of c in *dropped2.
__device__ __noinline__ int jacobi_solve(double *W, int ld, int K, int p, double rank_tol, double *s2buf, double *coef,
                            double *out, double *dropped2, int lane) {
    int flag = 0;
    const int sweeps = jacobi_rows(W, ld, K, p, p + 1, lane);
    if (sweeps > JACOBI_MAX_SWEEPS) flag |= 4;
    flag |= (sweeps > 63 ? 63 : sweeps) << 16;         // sweeps used (diagnostics, flag bits 16-21)
    const double *cvec = W + (size_t)p * ld;
    double smax = 0.0;
    for (int k = lane; k < K; k += 32) {
        const double *row = W + k;
        double s2 = 0.0;
        for (int c = 0; c < p; ++c) { const double v = row[(size_t)c * ld]; s2 += v * v; }
        s2buf[k] = s2;
        smax = fmax(smax, s2);
    }
    smax = sqrt(warp_max(smax));
    __syncwarp();
    bool dropped = false;
    double d2 = 0.0;
    for (int k = lane; k < K; k += 32) {
        const double s = sqrt(s2buf[k]);
        const bool keep = (s >= rank_tol * smax) && (s > 0.0);
        coef[k] = keep ? cvec[k] / s2buf[k] : 0.0;
        if (!keep) d2 += cvec[k] * cvec[k];
        dropped |= !keep;
    }
    *dropped2 = warp_sum(d2);
    if (__any_sync(FULL, dropped)) flag |= 2;
    __syncwarp();
    for (int j = lane; j < p; j += 32) {
        const double *col = W + (size_t)j * ld;
        double b = 0.0;
        for (int k = 0; k < K; ++k) b += col[k] * coef[k];
        out[j] = b;
    }
    __syncwarp();
    return flag;
}

// offset of column j inside a packed R with K rows: sum_{i<j} min(i+1, K)
__device__ __forceinline__ int packed_col_offset(int j, int K) {     // (j, K <= 256: 32-bit arithmetic)
    return j <= K ? (j * (j + 1)) >> 1 : ((K * (K + 1)) >> 1) + (j - K) * K;
}

// Packed block -> dense [R | c] with p rows (rows >= K and the strict lower part are zero); p <= 32 PS.
// *fro2 (if asked for) = |R|_F^2.
template <int PS>
__device__ __forceinline__ void unpack_rc(const double *in, double *W, int ld, int p, int K, int lane,
                                          double *fro2 = nullptr) {
    double f2 = 0.0;
    for (int j0 = 0; j0 <= p; j0 += UNPACK_COLS) {     // several columns in flight: the loads are latency-bound (DRAM: K2a's output is far larger than L2)
        double v[UNPACK_COLS][PS];
#pragma unroll
        for (int b = 0; b < UNPACK_COLS; ++b) {
            const int j = j0 + b <= p ? j0 + b : p;
            const int h = j < p ? (j + 1 < K ? j + 1 : K) : K;
            const double *src = in + packed_col_offset(j, K);
#pragma unroll
            for (int t = 0; t < PS; ++t) { const int i = lane + 32 * t; v[b][t] = i < h ? src[i] : 0.0; }
        }
#pragma unroll
        for (int b = 0; b < UNPACK_COLS; ++b) {
            const int j = j0 + b;
            if (j > p) break;
            double *col = W + (size_t)j * ld;
#pragma unroll
            for (int t = 0; t < PS; ++t) {
                const int i = lane + 32 * t;
                if (i < p) col[i] = v[b][t];
                if (j < p) f2 = fma(v[b][t], v[b][t], f2);
            }
        }
    }
    if (fro2) *fro2 = warp_sum(f2);
}

// Packed K x p block (K < p) -> W = R^T as a p x K column-major matrix (column j = row j of R, zero above row j and in
// the padding rows [p, ld)), c -> column K.  *fro2 = |R|_F^2.
template <int PS>
__device__ __forceinline__ void unpack_rc_wide(const double *in, double *W, int ld, int p, int K, int lane, double *fro2) {
    for (int j = 0; j <= K; ++j) {
        double *col = W + (size_t)j * ld;
        for (int i = lane; i < ld; i += 32) col[i] = 0.0;
    }
    __syncwarp();
    double f2 = 0.0;
    for (int i = 0; i < p; ++i) {                       // column i of R: rows 0 .. min(i, K - 1)
        const int h = i + 1 < K ? i + 1 : K;
        const double *src = in + packed_col_offset(i, K);
        for (int j = lane; j < h; j += 32) { const double v = src[j]; W[(size_t)j * ld + i] = v; f2 = fma(v, v, f2); }
    }
    const double *csrc = in + packed_col_offset(p, K);
    for (int j = lane; j < K; j += 32) W[(size_t)K * ld + j] = csrc[j];
    *fro2 = warp_sum(f2);
    __syncwarp();
}

// x -= B C_T (C_T^T (B^T x)): removes from x its components along the Ritz vectors B C[:, k], k in mask.  B: p x b
// orthonormal block; C: b x b orthogonal, element (j, k) at Cm[j * GP + k] * (scale ? scale[k] : 1).
template <int PS>
__device__ __noinline__ void project_out(Vec<PS> &x, const double *B, int ZP, int b, int p, const double *Cm, int GP,
                                         const double *scale, unsigned mask, int lane) {
    double w = 0.0;                                      // lane j: (B^T x)_j
    for (int j0 = 0; j0 < b; j0 += 4) {
        double d[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            d[j] = 0.0;
            const double *src = B + (size_t)(j0 + j) * ZP;
#pragma unroll
            for (int t = 0; t < PS; ++t) { const int e = lane + 32 * t; d[j] = fma(e < p ? src[e] : 0.0, x.v[t], d[j]); }
        }
        warp_sum4(d[0], d[1], d[2], d[3], lane);
#pragma unroll
        for (int j = 0; j < 4; ++j) if (lane == j0 + j) w = d[j];
    }
    double h = 0.0;                                      // lane j: coefficient of B[:, j] to remove
    for (unsigned mk = mask; mk; mk &= mk - 1) {
        const int k = __ffs(mk) - 1;
        const double sc = scale ? scale[k] : 1.0;
        const double cjk = lane < b ? Cm[(size_t)lane * GP + k] * sc : 0.0;
        const double alpha = warp_sum(cjk * w);
        h = fma(alpha, cjk, h);
    }
    for (int j = 0; j < b; ++j) {
        const double hj = __shfl_sync(FULL, h, j);
        const double *src = B + (size_t)j * ZP;
#pragma unroll
        for (int t = 0; t < PS; ++t) { const int e = lane + 32 * t; if (e < p) x.v[t] = fma(-hj, src[e], x.v[t]); }
    }
}

}  // namespace

// ---- K2b-1: certificate + plain solve; everything else goes to the work list ------------------------------------------
template <int PS>
__global__ void __launch_bounds__(512, 1) regress_clean_kernel(const RegressParams P) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31;
    const int N = P.N, pmax = P.pmax, ld = pmax | 1;
    double *W = smem + (size_t)(threadIdx.x >> 5) * regress_clean_ws_doubles(pmax);
    double *rinv = W + (size_t)ld * (pmax + 1);
    double *stage = rinv + pmax;
    const double denom = (double)(N - 1);
    const unsigned nf = (unsigned)(P.f1 - P.f0);

    for (;;) {
        unsigned int wk = 0;
        if (lane == 0) wk = atomicAdd(P.counter + 1, 1u);
        wk = __shfl_sync(FULL, wk, 0);
        if ((int64_t)wk >= P.nwork) break;
        const int q = P.work_order[wk / nf];
        const int fl = (int)(wk % nf), f = P.f0 + fl;
        const int64_t r0 = P.row_ptr[q];
        const int p = (int)(P.row_ptr[q + 1] - r0);
        if (p == 0) continue;                    // done in K2a
        const int K = p < N ? p : N;
        const double *in = P.Rq + (int64_t)fl * P.rq_stride + P.rq_ptr[q];
        bool clean = false, single = false;          // single: exactly one singular value below the threshold, deflated here
        double e2 = 0.0, sv = 0.0;
        int nsteps = 0;
        if (K == p) {
            double dmin = DBL_MAX, dmax = 0.0, fro2 = 0.0;
            unpack_rc<PS>(in, W, ld, p, K, lane, &fro2);
            __syncwarp();
            int jmin = 0;                                // column of the smallest pivot (smallest index among ties)
            for (int j = lane; j < K; j += 32) {
                const double v = W[(size_t)j * ld + j];
                rinv[j] = 1.0 / v;
                if (fabs(v) < dmin) { dmin = fabs(v); jmin = j; }
                dmax = fmax(dmax, fabs(v));
            }
            {
                const double mine = dmin;
                dmin = warp_min(dmin);
                const unsigned who = __ballot_sync(FULL, mine == dmin);
                jmin = __shfl_sync(FULL, jmin, __ffs(who) - 1);
            }
            dmax = warp_max(dmax);
            e2 = in[packed_col_offset(p, K) + K];
            __syncwarp();
            // a pivot ratio far below the threshold (s_min <= min |r_jj|, s_max >= max |r_jj|) means several small values in
            // practice: straight to the block kernel
            if (dmin > 1e-3 * P.rank_tol * dmax && fro2 < 1e300) {
                const double fro = sqrt(fro2);
                const double tail2 = inverse_norm2_mma(W, rinv, ld, p, stage, lane);   // sum 1 / s_i^2 >= 1 / s_min^2
                clean = tail2 > 0.0 && 1.0 / sqrt(tail2) >= P.rank_tol * fro * (1.0 + 1e-3);
                if (!clean && tail2 > 0.0 && p >= 2) {
                    // One inverse-iteration probe (two scalar triangular solves per step) from a pseudo-random start.  If it
                    // converges to a value s_1 that is provably below the threshold and the rest of the spectrum is provably
                    // above it -- sum_{i>=2} 1/s_i^2 = |X|_F^2 - 1/s_1^2 bounds s_2 from below -- the row is finished here
                    // with the single pair deflated; anything else goes to the block kernel.
                    // Start: column jmin of X = R^-1 (the certificate left X in W), i.e. half an inverse-iteration step from the
                    // unit vector of the smallest pivot -- the direction in which R is nearly singular is already amplified by
                    // 1 / s_1 in it.  (X[r, c] for r < c sits at W[r ld + c], the diagonal in rinv, zero below.)
                    Vec<PS> z, yt;
#pragma unroll
                    for (int t = 0; t < PS; ++t) {
                        const int e = lane + 32 * t;
                        z.v[t] = e < jmin ? W[(size_t)e * ld + jmin] : (e == jmin ? rinv[jmin] : 0.0);
                    }
                    {
                        const double inv = rsqrt(vdot<PS>(z, z));
#pragma unroll
                        for (int t = 0; t < PS; ++t) z.v[t] *= inv;
                    }
                    double dz_old = 1.0;
                    bool conv = false;
                    for (int it = 0; it < 12 && !conv; ++it) {
                        ++nsteps;
                        Vec<PS> zz = solve_upper_t<PS>(z, W, rinv, ld, p, lane);
                        yt = zz;                                       // R^-T z: the left singular direction
                        zz = solve_upper<PS>(zz, W, rinv, ld, p, lane);
                        const double zMz = vdot<PS>(zz, z);
                        const double inv = rsqrt(vdot<PS>(zz, zz));
                        const double sg = zMz >= 0.0 ? 1.0 : -1.0;
                        double dz = 0.0;
#pragma unroll
                        for (int t = 0; t < PS; ++t) {
                            const double zn = zz.v[t] * inv;
                            const double df = zn - sg * z.v[t];
                            dz = fma(df, df, dz);
                            z.v[t] = zn;
                        }
                        dz = sqrt(warp_sum(dz));
                        if ((dz < 1e-6 && dz > 0.9 * dz_old) || dz < 1e-12) conv = true;          // at the rounding floor
                        // linear convergence with ratio q = dz / dz_old: the iterate just computed is within dz q / (1 - q) of
                        // the limit -- stop once that is at the 1e-10 level.  The vector enters T to first order, so this is
                        // a relative 1e-10 in T: a tenth of the north_star gate and a tenth of the distance of the reference's
                        // own LAPACK answer from the exact one on these inputs (1.1e-9, oracle/noise_floor.py); measured T / D /
                        // Xa errors against the oracle are unchanged from the 5e-14 level used before.
                        else if (it >= 2 && dz < 0.25 * dz_old && dz * dz < REG_PROBE_TOL * dz_old) conv = true;
                        else if (it >= 3 && dz > 0.3 * dz_old) break;                                // close values: a block is the better tool
                        dz_old = dz;
                    }
                    if (conv) {
                        // s_1 = 1 / |R^-T z| (an upper bound of the singular value, tight to second order in the error of z),
                        // u = R^-T z / |R^-T z| from the last step (z moved by less than the stopping level since)
                        const double ny = sqrt(vdot<PS>(yt, yt));
                        sv = 1.0 / ny;
                        double smax_lo = dmax;
                        bool pw_used = false;
                        if (!(sv < P.rank_tol * smax_lo * (1.0 - 1e-3))) {       // sharpen the lower bound of s_max: two power steps
                            pw_used = true;
                            Vec<PS> v;
                            const double v0 = rsqrt((double)p);
#pragma unroll
                            for (int t = 0; t < PS; ++t) v.v[t] = (lane + 32 * t < p) ? v0 : 0.0;
                            // every half step gives a lower bound (|R v| <= sqrt |R^T R v| <= s_max for unit v); on smooth
                            // ensembles the first one, |R 1| / sqrt(p), is already within a few per cent: stop as soon as the
                            // bound settles the question
                            for (int pw = 0; pw < 2; ++pw) {
                                const Vec<PS> y = mul_upper<PS>(v, W, ld, p, lane);
                                smax_lo = fmax(smax_lo, sqrt(vdot<PS>(y, y)));
                                if (sv < P.rank_tol * smax_lo * (1.0 - 1e-3)) break;
                                v = mul_upper_t<PS>(y, W, ld, p, lane);
                                const double nv = sqrt(vdot<PS>(v, v));
                                smax_lo = fmax(smax_lo, sqrt(nv));
                                if (sv < P.rank_tol * smax_lo * (1.0 - 1e-3)) break;
                                const double inv = 1.0 / nv;
#pragma unroll
                                for (int t = 0; t < PS; ++t) v.v[t] *= inv;
                            }
                        }
                        // X carries a relative error of at most about c eps cond(R): added to what is left, so that the bound
                        // stays a lower bound
                        const double noise = 2.2e-14 * (fro * ny);
                        const double rem = tail2 - ny * ny;
                        const double up2 = fmax(rem, 0.0) + noise * tail2;
                        single = sv < P.rank_tol * smax_lo * (1.0 - 1e-3) && rem > -noise * tail2 && noise < 0.25 &&
                                 1.0 / sqrt(up2) >= P.rank_tol * fro * (1.0 + 1e-3);
                        if (single) {
#pragma unroll
                            for (int t = 0; t < PS; ++t) yt.v[t] *= sv;
                            Vec<PS> b = vload<PS>(W + (size_t)p * ld, p, lane);
                            const double pr = vdot<PS>(b, yt);                    // c -= u u^T c
#pragma unroll
                            for (int t = 0; t < PS; ++t) b.v[t] = fma(-pr, yt.v[t], b.v[t]);
                            b = solve_upper<PS>(b, W, rinv, ld, p, lane);
                            const double pz = vdot<PS>(b, z);                     // beta -= z z^T beta
#pragma unroll
                            for (int t = 0; t < PS; ++t) b.v[t] = fma(-pz, z.v[t], b.v[t]);
                            double *Tout = P.T + (int64_t)f * P.tstride + r0;
#pragma unroll
                            for (int t = 0; t < PS; ++t) { const int e = lane + 32 * t; if (e < p) Tout[e] = -b.v[t]; }
                            // |c - R beta|^2
                            const Vec<PS> rb = mul_upper<PS>(b, W, ld, p, lane);
                            const Vec<PS> c0 = vload<PS>(W + (size_t)p * ld, p, lane);
                            double rest2 = 0.0;
#pragma unroll
                            for (int t = 0; t < PS; ++t) { const double df = c0.v[t] - rb.v[t]; rest2 = fma(df, df, rest2); }
                            rest2 = warp_sum(rest2);
                            if (lane == 0) {
                                const double d = (e2 + rest2) / denom;
                                P.D[(int64_t)f * P.dstride + q] = fmax(d, P.variance_floor);
                                if (P.flags) P.flags[(int64_t)f * P.dstride + q] = 2 | 32 | (pw_used ? 64 : 0) | (d < P.variance_floor ? 8 : 0) | ((nsteps < 255 ? nsteps : 255) << 8);
                            }
                            __syncwarp();
                            continue;
                        }
                    }
                }
            }
        }
        if (!clean) {
            if (lane == 0) P.worklist[atomicAdd(P.lcounter, 1u)] = wk;
            continue;
        }
        Vec<PS> b = vload<PS>(W + (size_t)p * ld, p, lane);
        b = solve_upper<PS>(b, W, rinv, ld, p, lane);
        double *Tout = P.T + (int64_t)f * P.tstride + r0;
#pragma unroll
        for (int t = 0; t < PS; ++t) { const int e = lane + 32 * t; if (e < p) Tout[e] = -b.v[t]; }
        if (lane == 0) {
            const double d = e2 / denom;
            P.D[(int64_t)f * P.dstride + q] = fmax(d, P.variance_floor);
            if (P.flags) P.flags[(int64_t)f * P.dstride + q] = d < P.variance_floor ? 8 : 0;
        }
        __syncwarp();
    }
}

// ---- K2b-2: block inverse iteration + Rayleigh-Ritz for the listed rows --------------------------------------------------
template <int PS>
__global__ void __launch_bounds__(256, 1) regress_trunc_kernel(const RegressParams P) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31;
    const int N = P.N, pmax = P.pmax, ld = pmax | 1, bmax = P.bmax;
    const int ZP = trunc_zp(pmax), GP = bmax | 1;
    double *W = smem + (size_t)(threadIdx.x >> 5) * regress_trunc_ws_doubles(pmax, bmax);
    double *rinv = W + (size_t)ld * (pmax + 1);
    double *aux = rinv + pmax;
    double *tmp = aux + pmax;
    double *x0s = tmp + pmax;                   // wide rows: heads x0 and pivots alpha of the second QR's reflectors
    double *alphas = x0s + pmax;
    double *Zs = alphas + pmax;
    double *Ys = Zs + (size_t)bmax * ZP;
    double *Gs = Ys + (size_t)bmax * ZP;        // [G | P]: bmax x 2 bmax, pitch GP
    const double denom = (double)(N - 1);
    const unsigned nf = (unsigned)(P.f1 - P.f0);
    const unsigned nlist = P.lcounter[P.level ? 3 : 0];
    const unsigned int *list = P.level ? P.worklist2 : P.worklist;

    for (;;) {
        unsigned int it = 0;
        if (lane == 0) it = atomicAdd(P.lcounter + (P.level ? 4 : 1), 1u);
        it = __shfl_sync(FULL, it, 0);
        if (it >= nlist) break;
        const unsigned wk = list[it];
        const int q = P.work_order[wk / nf];
        const int fl = (int)(wk % nf), f = P.f0 + fl;
        const int64_t r0 = P.row_ptr[q];
        const int p = (int)(P.row_ptr[q + 1] - r0);
        const int K = p < N ? p : N;
        const bool wide = K < p;
        const int pe = K;                        // order of the triangular problem
        const double *in = P.Rq + (int64_t)fl * P.rq_stride + P.rq_ptr[q];
        const double e2 = in[packed_col_offset(p, K) + K];
        int flag = 1, why = 0, sweeps = 0;
        int b = P.level ? P.bmax1 + 8 : 8;          // second pass: the first one found bmax1 vectors too few
        bool escalate = false;
        unsigned tmask = 0;                      // Ritz values below the threshold
        double fro2 = 0.0, smax_lo = 0.0;

        if (!wide) {
            unpack_rc<PS>(in, W, ld, p, K, lane, &fro2);
            __syncwarp();
        } else {
            unpack_rc_wide<PS>(in, W, ld, p, K, lane, &fro2);
            // s_max (lower bound, within ~1e-6 on smooth ensembles): four power steps on R^T R from the all-ones vector (predecessor rows are positively
            // correlated, the dominant right vector is close to uniform)
            {
                Vec<PS> v;
#pragma unroll
                for (int t = 0; t < PS; ++t) v.v[t] = (lane + 32 * t < p) ? 1.0 : 0.0;
                for (int pw = 0; pw < 4; ++pw) {
                    Vec<PS> acc;
#pragma unroll
                    for (int t = 0; t < PS; ++t) acc.v[t] = 0.0;
                    for (int j = 0; j < K; ++j) {
                        const Vec<PS> cj = vload<PS>(W + (size_t)j * ld, p, lane);
                        const double yj = vdot<PS>(cj, v);
#pragma unroll
                        for (int t = 0; t < PS; ++t) acc.v[t] = fma(yj, cj.v[t], acc.v[t]);
                    }
                    const double nv = sqrt(vdot<PS>(acc, acc));
                    if (pw > 0) smax_lo = sqrt(nv);
                    const double inv = nv > 0.0 ? 1.0 / nv : 0.0;
#pragma unroll
                    for (int t = 0; t < PS; ++t) v.v[t] = acc.v[t] * inv;
                }
            }
            // second QR: R^T (p x K) = Q2 R2; R2 stays in the upper triangle, the reflectors below it
            for (int k = 0; k < K; ++k) {            // one reflector per sweep: column k keeps its tail below the diagonal
                qr_step1_dispatch<PS>(W, ld, p, k, K - 1, alphas, lane);
                __syncwarp();
            }
            for (int j = lane; j < K; j += 32) { x0s[j] = W[(size_t)j * ld + j]; W[(size_t)j * ld + j] = alphas[j]; }
            __syncwarp();
        }
        const double *cvec = W + (size_t)pe * ld;   // right-hand side of the triangular problem
        double dmax = 0.0;
        for (int j = lane; j < pe; j += 32) dmax = fmax(dmax, fabs(W[(size_t)j * ld + j]));
        dmax = warp_max(dmax);
        const double fro = sqrt(fro2);
        bool fallback = !(dmax > 0.0) || !(fro < 1e150);
        if (fallback) why = 1;
        if (!fallback && (pe < 8 || bmax < 8)) { fallback = true; why = 2; }   // too small for a block of eight
        if (!fallback) {
            // pivots below 1e-20 of the largest are set to that size (a perturbation far below the rounding of R), so
            // that every quantity stays finite
            for (int j = lane; j < pe; j += 32) {
                double v = W[(size_t)j * ld + j];
                if (!(fabs(v) >= 1e-20 * dmax)) { v = (v < 0.0 ? -1e-20 : 1e-20) * dmax; W[(size_t)j * ld + j] = v; }
                rinv[j] = 1.0 / v;
            }
            __syncwarp();
            smax_lo = fmax(smax_lo, dmax);
            const double thr_hi = P.rank_tol * fro;
            // ---- block inverse iteration ----
            const unsigned seed0 = (unsigned)P.state_row[q] * 7919u + (unsigned)p * 104729u;
            auto fill_random = [&](int c0, int c1) {
                for (int k = c0; k < c1; ++k) {
                    double *dst = Zs + (size_t)k * ZP;
                    for (int e = lane; e < ZP; e += 32) {
                        unsigned h = (unsigned)(e + 1) * 2654435761u ^ ((seed0 + (unsigned)k) * 40503u + 0x9e3779b9u);
                        h ^= h >> 15; h *= 2246822519u; h ^= h >> 13; h *= 3266489917u; h ^= h >> 16;
                        dst[e] = e < pe ? (double)(h >> 8) * (1.0 / 8388608.0) - 1.0 : 0.0;
                    }
                }
                __syncwarp();
            };
            const int bcap = bmax < (pe & ~7) ? bmax : (pe & ~7);
            if (b > bcap) b = bcap;
            fill_random(0, b);
            int need = 2;
            bool final_done = false, wide_span = true;
            for (;;) {
                ++sweeps;
                // one Gram-Schmidt pass keeps the block well conditioned as long as its Ritz values span less than ~1e6 (what a
                // single pass leaves of the dominant direction is amplified by that ratio in the next solve); the first sweep
                // (span unknown) and the predicted last one (the accurate one) take two
                const int passes = (sweeps >= need || sweeps == 1 || wide_span) ? 2 : 1;
                blk_copy(Ys, Zs, ZP, b, lane);
                blk_solve(true, Ys, ZP, b, W, rinv, ld, pe, lane);                    // Y = R^-T Z
                if (!orth_block<PS>(Ys, ZP, 0, b, pe, nullptr, GP, lane, passes)) { fallback = true; why = 1; break; }
                blk_copy(Zs, Ys, ZP, b, lane);
                blk_solve(false, Zs, ZP, b, W, rinv, ld, pe, lane);                   // Z G = R^-1 Y
                if (!orth_block<PS>(Zs, ZP, 0, b, pe, Gs, GP, lane, passes)) { fallback = true; why = 1; break; }
                final_done = passes == 2;
                // 1 / |G_kk| estimate the Ritz values of the block; the largest is at least 1 / min |G_kk|
                double gk = lane < b ? fabs(Gs[(size_t)lane * GP + lane]) : DBL_MAX;
                const double top = 1.0 / warp_min(gk);
                wide_span = warp_max(lane < b ? gk : 0.0) * top > 1e6;
                if (top < 8.0 * thr_hi) {                                            // the block does not reach far enough
                    if (b + 8 > bcap) {
                        if (b == pe) break;                                           // the block is the whole space
                        if (P.level == 0 && b + 8 <= (pe & ~7) && P.bmax2 > bmax) {    // the second pass has room for it
                            if (lane == 0) P.worklist2[atomicAdd(P.lcounter + 3, 1u)] = wk;
                            escalate = true;
                            break;
                        }
                        fallback = true; why = 2; break;
                    }
                    fill_random(b, b + 8);
                    if (!orth_block<PS>(Zs, ZP, b, b + 8, pe, nullptr, GP, lane)) { fallback = true; why = 1; break; }
                    b += 8;
                    need = sweeps + 2;
                    final_done = false;
                    continue;
                }
                const double est = lane < b ? 1.0 / gk : 0.0;
                const double marg = warp_max(est < 2.0 * thr_hi ? est : 0.0);         // largest estimate near / below the threshold
                if (marg > 0.0) {
                    const double lr = 2.0 * log(marg / top);                          // log of the contraction per sweep (< 0)
                    int n = lr < -2.5 ? (int)ceil(-23.0 / lr) : TRUNC_MAX_SWEEPS;     // 1e-10 after n sweeps
                    if (n > TRUNC_MAX_SWEEPS) n = TRUNC_MAX_SWEEPS;
                    if (n > need) need = n;
                }
                if (sweeps >= need && final_done) break;
                if (sweeps >= TRUNC_MAX_SWEEPS + 4) { fallback = true; why = 4; break; }
            }
        }
        if (escalate) continue;
        double sig = 0.0;                            // lane k: Ritz value k
        if (!fallback) {
            // ---- Rayleigh-Ritz: G = P S Q^T by one-sided Jacobi on the rows of [G | I] ----
            for (int e = lane; e < 2 * b * GP; e += 32) {
                const int c = e / GP, r = e - c * GP;
                if (c < b) { if (r > c) Gs[e] = 0.0; }                               // strict lower part of G
                else Gs[e] = (r == c - b) ? 1.0 : 0.0;
            }
            __syncwarp();
            const int js = b == 8 ? jacobi8_regs(Gs, GP, lane) : jacobi_rows(Gs, GP, b, b, 2 * b, lane);
            flag |= (js > 63 ? 63 : js) << 16;
            if (js > JACOBI_MAX_SWEEPS) { fallback = true; why = 1; }
            double s2 = 0.0;
            if (lane < b) for (int c = 0; c < b; ++c) { const double v = Gs[(size_t)c * GP + lane]; s2 = fma(v, v, s2); }
            sig = lane < b ? 1.0 / sqrt(s2) : DBL_MAX;
            if (lane < b) tmp[lane] = sqrt(s2) > 0.0 ? 1.0 / sqrt(s2) : 0.0;         // scale of row k: q_k = row / S_k  (tmp reused)
            __syncwarp();
            if (!(warp_min(sig) > 0.0)) { fallback = true; why = 1; }
        }
        if (!fallback) {
            // ---- which Ritz values are below rank_tol * s_max?  s_max in [smax_lo, smax_hi] ----
            double smax_hi = fro;
            const double guard = 1e-6;
            auto ambiguous = [&]() -> bool {
                const bool amb = lane < b && sig >= P.rank_tol * smax_lo * (1.0 - guard) && sig <= P.rank_tol * smax_hi * (1.0 + guard);
                return __any_sync(FULL, amb);
            };
            if (ambiguous()) {
                // power iteration on R^T R (p_e-vector) from the normalised all-ones vector: every Rayleigh estimate is a
                // lower bound of s_max and they rise monotonically
                Vec<PS> v;
                const double v0 = rsqrt((double)pe);
#pragma unroll
                for (int t = 0; t < PS; ++t) v.v[t] = (lane + 32 * t < pe) ? v0 : 0.0;
                double prev = 0.0, inc_old = 0.0;
                for (int round = 0; round < 60; ++round) {
                    Vec<PS> y = wide ? mul_upper_t<PS>(v, W, ld, pe, lane) : mul_upper<PS>(v, W, ld, pe, lane);
                    v = wide ? mul_upper<PS>(y, W, ld, pe, lane) : mul_upper_t<PS>(y, W, ld, pe, lane);
                    const double nv = sqrt(vdot<PS>(v, v));
                    const double cur = sqrt(nv);
                    const double inv = 1.0 / nv;
#pragma unroll
                    for (int t = 0; t < PS; ++t) v.v[t] *= inv;
                    smax_lo = fmax(smax_lo, cur);
                    const double inc = cur - prev;
                    prev = cur;
                    // with ratio qq per step the tail of the increments is inc qq / (1 - qq)
                    const double qq = inc_old > 0.0 ? inc / inc_old : 1.0;
                    if (round >= 2 && qq < 0.9) smax_hi = fmin(fro, smax_lo * (1.0 + 1e-7) + 10.0 * inc * qq / (1.0 - qq));
                    if (!ambiguous()) break;
                    if (round >= 2 && qq < 0.9 && inc <= 1e-10 * cur) break;          // converged: what is still inside is at the threshold
                    inc_old = inc;
                }
                if (ambiguous()) { fallback = true; why = 3; }
            }
            tmask = __ballot_sync(FULL, lane < b && sig < P.rank_tol * smax_lo);
        }

        if (!fallback) {
            if (tmask) flag |= 2;
            flag |= (b >> 3) << 22;
            // left / right Ritz vectors of the triangular matrix: U = Y Q (q_k = row k of the left half / S_k), V = Z P
            // (p_k = row k of the right half).  Upper problem R x = c:  x = (I - V V^T) R^-1 (I - U U^T) c;  the wide
            // rows solve R2^T g = c: the roles swap.
            const double *Cq = Gs, *Cp = Gs + (size_t)b * GP;
            Vec<PS> x = vload<PS>(cvec, pe, lane);
            if (tmask) {
                if (!wide) project_out<PS>(x, Ys, ZP, b, pe, Cq, GP, tmp, tmask, lane);
                else project_out<PS>(x, Zs, ZP, b, pe, Cp, GP, nullptr, tmask, lane);
            }
            x = wide ? solve_upper_t<PS>(x, W, rinv, ld, pe, lane) : solve_upper<PS>(x, W, rinv, ld, pe, lane);
            if (tmask) {
                if (!wide) project_out<PS>(x, Zs, ZP, b, pe, Cp, GP, nullptr, tmask, lane);
                else project_out<PS>(x, Ys, ZP, b, pe, Cq, GP, tmp, tmask, lane);
            }
            // |c - R x|^2 (wide: |c - R2^T g|^2)
            double rest2 = 0.0;
            if (tmask) {
                const Vec<PS> rb = wide ? mul_upper_t<PS>(x, W, ld, pe, lane) : mul_upper<PS>(x, W, ld, pe, lane);
                const Vec<PS> c0 = vload<PS>(cvec, pe, lane);
#pragma unroll
                for (int t = 0; t < PS; ++t) { const double df = c0.v[t] - rb.v[t]; rest2 = fma(df, df, rest2); }
                rest2 = warp_sum(rest2);
            }
            vstore<PS>(aux, x, pe, lane);
            __syncwarp();
            if (wide) {
                // beta = Q2 [g; 0]: reflectors of the second QR, last to first.  v_k = (x0 - alpha, column k below the
                // diagonal), tau = 1 / (|alpha| (|alpha| + |x0|))
                Vec<PS> bt = vload<PS>(aux, pe, lane);       // zero beyond K
                for (int k = K - 1; k >= 0; --k) {
                    const double alpha = alphas[k], x0 = x0s[k];
                    const double an = fabs(alpha);
                    if (an == 0.0) continue;
                    const double tau = 1.0 / (an * (an + fabs(x0)));
                    Vec<PS> v;
                    const double *col = W + (size_t)k * ld;
                    double d = 0.0;
#pragma unroll
                    for (int t = 0; t < PS; ++t) {
                        const int e = lane + 32 * t;
                        v.v[t] = e == k ? x0 - alpha : ((e > k && e < p) ? col[e] : 0.0);
                        d = fma(v.v[t], bt.v[t], d);
                    }
                    const double wv = warp_sum(d) * tau;
#pragma unroll
                    for (int t = 0; t < PS; ++t) bt.v[t] = fma(-wv, v.v[t], bt.v[t]);
                }
                vstore<PS>(aux, bt, p, lane);
                __syncwarp();
            }
            double *Tout = P.T + (int64_t)f * P.tstride + r0;
            for (int j = lane; j < p; j += 32) Tout[j] = -aux[j];
            if (lane == 0) {
                const double d = (e2 + rest2) / denom;
                if (d < P.variance_floor) flag |= 8;
                P.D[(int64_t)f * P.dstride + q] = fmax(d, P.variance_floor);
                if (P.flags) P.flags[(int64_t)f * P.dstride + q] = flag | ((sweeps < 255 ? sweeps : 255) << 8);
            }
            __syncwarp();
            continue;
        }

        // ---- general fallback ----
        flag |= 16 | (why << 5);
        unpack_rc<PS>(in, W, ld, p, K, lane);
        __syncwarp();
        double dropped2;
        flag |= jacobi_solve(W, ld, K, p, P.rank_tol, rinv, tmp, aux, &dropped2, lane);
        double *Tout = P.T + (int64_t)f * P.tstride + r0;
        for (int j = lane; j < p; j += 32) Tout[j] = -aux[j];
        unpack_rc<PS>(in, W, ld, p, K, lane);
        __syncwarp();
        double rest2 = 0.0;
        {
            // |c - R beta|^2 over the K rows of R (K x p)
            for (int r = lane; r < K; r += 32) {
                double acc = W[(size_t)p * ld + r];
                for (int c = r; c < p; ++c) acc = fma(-W[(size_t)c * ld + r], aux[c], acc);
                rest2 = fma(acc, acc, rest2);
            }
            rest2 = warp_sum(rest2);
        }
        if (lane == 0) {
            const double d = (e2 + rest2) / denom;
            if (d < P.variance_floor) flag |= 8;
            P.D[(int64_t)f * P.dstride + q] = fmax(d, P.variance_floor);
            if (P.flags) P.flags[(int64_t)f * P.dstride + q] = flag | ((sweeps < 255 ? sweeps : 255) << 8);
            atomicAdd(P.lcounter + 2, 1u);
        }
        __syncwarp();
    }
}
