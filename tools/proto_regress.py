"""Numerical prototype of the K2 regression kernel (research tool, not on any product path).

Restates in numpy the algorithm the CUDA kernel runs per component -- Householder QR with
column pivoting, a diagonal-ratio test that picks the back-substitution fast path, else a
one-sided Jacobi SVD on the rows of [R | Q^T y] with the reference's 1e-8*s_max truncation --
and reports its distance from the oracle's LAPACK truncated SVD on golden / synthetic tiles.
"""

from __future__ import annotations

import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from oracle import enkf_mc_oracle as orc  # noqa: E402

EPS = np.finfo(float).eps


def qrcp(M, p):
    """In-place Householder QRCP of the first p columns of M (N x (p+1)); returns perm, K."""
    N = M.shape[0]
    K = min(p, N)
    perm = np.arange(p)
    cn = np.einsum("ij,ij->j", M[:, :p], M[:, :p])
    for k in range(K):
        cn[k:] = np.einsum("ij,ij->j", M[k:, k:p], M[k:, k:p])  # recomputed (kernel downdates + refresh)
        j = k + int(np.argmax(cn[k:]))
        if j != k:
            M[:, [k, j]] = M[:, [j, k]]
            perm[[k, j]] = perm[[j, k]]
        x = M[k:, k]
        nrm = np.sqrt(x @ x)
        if nrm == 0.0:
            continue
        alpha = -np.copysign(nrm, x[0])
        v = x.copy()
        v[0] -= alpha
        tau = 2.0 / (v @ v)
        M[k:, k:] -= np.outer(v, tau * (v @ M[k:, k:]))
        M[k + 1:, k] = 0.0
    return perm, K


def jacobi_rows(W, p, max_sweeps=40, tol=None):
    """One-sided Jacobi on the rows of W[:, :p] (rotations also applied to column p)."""
    K = W.shape[0]
    tol = tol or EPS * np.sqrt(p)
    sweeps = 0
    for sweeps in range(1, max_sweeps + 1):
        rotated = 0
        for i in range(K - 1):
            for j in range(i + 1, K):
                di = W[i, :p] @ W[i, :p]
                dj = W[j, :p] @ W[j, :p]
                g = W[i, :p] @ W[j, :p]
                if abs(g) <= tol * np.sqrt(di * dj) or g == 0.0:
                    continue
                rotated += 1
                zeta = (dj - di) / (2.0 * g)
                t = np.copysign(1.0, zeta) / (abs(zeta) + np.sqrt(1.0 + zeta * zeta))
                cs = 1.0 / np.sqrt(1.0 + t * t)
                sn = cs * t
                wi = cs * W[i] - sn * W[j]
                W[j] = sn * W[i] + cs * W[j]
                W[i] = wi
        if rotated == 0:
            break
    return sweeps


def regress(A, y, rank_tol=1e-8, fast_ratio=1e-6, stats=None):
    p, N = A.shape
    M = np.empty((N, p + 1))
    M[:, :p] = A.T
    M[:, p] = y
    perm, K = qrcp(M, p)
    R = M[:K, :p + 1].copy()
    diag = np.abs(np.diag(R[:, :K]))
    betap = np.zeros(p)
    if K == p and diag[-1] > fast_ratio * diag[0]:
        c = R[:, p].copy()
        for k in range(p - 1, -1, -1):
            betap[k] = c[k] / R[k, k]
            c[:k] -= R[:k, k] * betap[k]
        if stats is not None:
            stats["fast"] += 1
    else:
        sw = jacobi_rows(R, p)
        s2 = np.einsum("ij,ij->i", R[:, :p], R[:, :p])
        s = np.sqrt(s2)
        keep = (s >= rank_tol * s.max()) & (s > 0)
        for k in np.flatnonzero(keep):
            betap += R[k, :p] * (R[k, p] / s2[k])
        if stats is not None:
            stats["slow"] += 1
            stats["sweeps"].append(sw)
            stats["trunc"] += int((~keep).any())
    beta = np.empty(p)
    beta[perm] = betap
    resid = y - A.T @ beta
    return beta, resid @ resid / (N - 1)


def compare_tile(U, grid, zeta, local_order, fast_ratio=1e-6):
    ip, ii = orc.predecessor_csr(grid, zeta, local_order)
    ref = orc.fit_factors(U, grid, zeta, local_order)
    stats = {"fast": 0, "slow": 0, "trunc": 0, "sweeps": []}
    data = np.zeros_like(ref.data)
    d = np.empty(ref.n)
    for j in range(ref.n):
        a, b = ip[j], ip[j + 1]
        if a == b:
            d[j] = U[j] @ U[j] / (U.shape[1] - 1)
            continue
        beta, d[j] = regress(U[ii[a:b]], U[j], fast_ratio=fast_ratio, stats=stats)
        data[a:b] = -beta
    terr = np.linalg.norm(data - ref.data) / np.linalg.norm(ref.data)
    rowerr = max((np.linalg.norm(data[ip[j]:ip[j + 1]] - ref.data[ip[j]:ip[j + 1]]) /
                  max(np.linalg.norm(ref.data[ip[j]:ip[j + 1]]), 1e-300)) for j in range(ref.n) if ip[j + 1] > ip[j])
    derr = np.max(np.abs(np.maximum(d, 1e-10) - ref.d) / ref.d)
    return terr, rowerr, derr, stats


if __name__ == "__main__":
    from paper_1606_00807_b200 import synthetic
    cases = [
        ("golden a3 (nugget)", dict(nx=32, ny=20, nens=56, corr_len=4.0, zeta=3, delta=6, obs="random", obs_arg=0.3, r_rel=None, r_abs=0.1, seed=14, nugget=0.01)),
        ("golden a5 (trunc)", dict(nx=32, ny=20, nens=56, corr_len=8.0, zeta=3, delta=6, obs="random", obs_arg=0.3, r_rel=None, r_abs=0.1, seed=16)),
    ]
    for name, kw in cases:
        w = synthetic.make_workload("x", **kw)
        grid = orc.grid_for(w.nx, w.ny, w.boundary)
        t = orc.decompose(grid, w.delta, w.zeta)[0]
        U = orc.center_rows(w.X[t.local_order])
        terr, rowerr, derr, st = compare_tile(U, grid, w.zeta, t.local_order)
        print(f"{name}: T normwise {terr:.2e}  worst row {rowerr:.2e}  D max rel {derr:.2e}  fast {st['fast']} slow {st['slow']} "
              f"trunc {st['trunc']} sweeps {np.bincount(st['sweeps']) if st['sweeps'] else '-'}")
