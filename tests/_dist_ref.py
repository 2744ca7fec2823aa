"""Row-partitioned NetMF+ schedule in fp64 numpy on CPU, with
torch.distributed (gloo) collectives at exactly the points where the CUDA
library (paper_2110_12782_b200/csrc/pipeline.cu, dist.cu) issues NCCL calls:

  * before every SpMM: all-gather of the input block's rows (dist_gather_rows)
  * after every Gram (CholeskyQR, Rayleigh–Ritz S, Eq. 3's K): all-reduce
  * the sketch's gathered rows F_{r_{c,t}} (Ψ, Π) and FC_{r_{c',t'}}: all-reduce
    of zero-padded buffers (each row lives on one rank)
  * Πᵀ Q: all-reduce of the per-rank partial sums
  * vol(G): all-reduce of the local nnz
  * small fp64 problems (Cholesky, eig, core solve, SVD): replicated

Each rank owns rows [b_r, b_{r+1}).  Test infrastructure only (oracle/ is used
for the per-rank arithmetic); tests/test_dist_cpu.py checks that the schedule
reproduces the single-process oracle."""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

import oracle as O


def _allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def _gather_rows(Xl, bounds):
    """all-gather of every rank's rows into the full n × c block."""
    ws = dist.get_world_size()
    rows = [bounds[r + 1] - bounds[r] for r in range(ws)]
    mx = max(rows)
    pad = np.zeros((mx, Xl.shape[1]))
    pad[:Xl.shape[0]] = Xl
    outs = [torch.zeros(mx, Xl.shape[1], dtype=torch.float64) for _ in range(ws)]
    dist.all_gather(outs, torch.from_numpy(pad))
    return np.concatenate([o.numpy()[:rows[r]] for r, o in enumerate(outs)], axis=0)


def _dpow(deg, e):
    """row scale d^-e (0 for d = 0), the library's convention"""
    return O.deg_pow(deg, -e)


def dist_netmf_plus(n, src, dst, bounds, *, alpha, k, s1, q, T, b, d, s2, s3, z, prop_order, mu, theta,
                    seed, logmode=0):
    rank = dist.get_rank()
    b0, b1 = int(bounds[rank]), int(bounds[rank + 1])
    rp, col, deg = O.build_csr(n, src, dst)        # CSR rows of this rank (global column ids)
    lrp = rp[b0:b1 + 1] - rp[b0]
    lcol = col[rp[b0]:rp[b1]]
    ldeg = deg[b0:b1]
    vol = float(_allreduce(np.array([lcol.size], dtype=np.float64))[0])

    def spmm(Xfull, a):                              # y_u = d_u^-a Σ_{v ∈ N(u)} X_v (pre-scaled basis)
        Y = np.zeros((b1 - b0, Xfull.shape[1]))
        for u in range(b1 - b0):
            Y[u] = Xfull[lcol[lrp[u]:lrp[u + 1]]].sum(axis=0)
        return _dpow(ldeg, a)[:, None] * Y

    def gram(A, B):
        return _allreduce(A.T @ B)

    def cholqr(Y, rexp, passes):                     # CholeskyQR(2) with all-reduced Grams [R7]
        cur = Y
        for _ in range(passes):
            G = gram(cur, cur)
            R = np.linalg.cholesky(G).T
            cur = cur @ np.linalg.inv(R)
        return _dpow(ldeg, rexp)[:, None] * cur if rexp is not None else cur

    # ---- Alg. 2 freigs with P = D^-α Q
    l = k + s1
    Omega = O.gaussian_matrix(n, l, seed)[b0:b1]
    P = _dpow(ldeg, alpha)[:, None] * Omega
    Y = spmm(_gather_rows(P, bounds), alpha)
    P = cholqr(Y, alpha, 2 if q == 0 else 1)
    for it in range(q):
        Tm = spmm(_gather_rows(P, bounds), 2 * alpha)
        Y = spmm(_gather_rows(Tm, bounds), alpha)
        P = cholqr(Y, alpha, 2 if it + 1 == q else 1)
    Tm = spmm(_gather_rows(P, bounds), 0.0)
    S = gram(P, Tm)
    S = 0.5 * (S + S.T)
    lam, V = O.sym_eig_abs_sorted(S)
    lam = lam[:k]
    U = _dpow(ldeg, -alpha)[:, None] * (P @ V[:, :k])
    # ---- Eq. 3
    K = gram(U * _dpow(ldeg, 1.0 - 2.0 * alpha)[:, None], U) @ np.diag(lam)
    acc, Pw = np.eye(k), np.eye(k)
    for _ in range(2, T + 1):
        Pw = Pw @ K
        acc = acc + Pw
    Cm = np.diag(lam) @ acc
    F = _dpow(ldeg, 1.0 - alpha)[:, None] * U
    # ---- Alg. 4, Eq. 5 grouped by sparse-sign column [R9]
    scale = vol / (b * T)
    FC = F @ Cm
    h2, h3 = d + s2, d + s3

    def rows_at(M, rows):                            # M's rows at global ids (zero when not local), all-reduced
        out = np.zeros((rows.size, M.shape[1]))
        loc = (rows >= b0) & (rows < b1)
        out[loc] = M[rows[loc] - b0]
        return _allreduce(out)

    rows_psi, sg_psi, _ = O.gen_sparse_sign(n, h2, z, seed, O.TAG_PSI)
    Bpsi = rows_at(F, rows_psi.reshape(-1))          # (h2·z) × k
    G = O.elementwise_log(scale * (FC @ Bpsi.T), logmode)
    Yl = (G.reshape(b1 - b0, h2, z) * sg_psi[None, :, :]).sum(axis=2)
    Q = cholqr(Yl, None, 2)
    rows_pi, sg_pi, _ = O.gen_sparse_sign(n, h3, z, seed, O.TAG_PI)
    Api = rows_at(FC, rows_pi.reshape(-1))
    Bpi = rows_at(F, rows_pi.reshape(-1))
    H = O.elementwise_log(scale * (Api @ Bpi.T), logmode)       # replicated
    Z = (sg_pi[:, :, None, None] * H.reshape(h3, z, h3, z) * sg_pi[None, None, :, :]).sum(axis=(1, 3))
    PtQ = np.zeros((h3, h2))
    for j in range(h3):
        for t in range(z):
            r = rows_pi[j, t]
            if b0 <= r < b1:
                PtQ[j] += sg_pi[j, t] * Q[r - b0]
    PtQ = _allreduce(PtQ)
    Sc = O.core_solve(PtQ, Z)
    Uh, sig, _ = np.linalg.svd(Sc)
    sig = sig[:d]
    E = (Q @ Uh[:, :d]) * np.sqrt(np.maximum(sig, 0.0))[None, :]
    # ---- spectral propagation with L~ = -D^-1 A
    if prop_order > 0:
        c = O.cheb_coeffs(prop_order, mu, theta)
        Lt = lambda Xl: -spmm(_gather_rows(Xl, bounds), 1.0)
        Z0, Z1 = E, Lt(E)
        out = c[0] * Z0 + c[1] * Z1
        for r in range(2, prop_order + 1):
            Z2 = 2.0 * Lt(Z1) - Z0
            out = out + c[r] * Z2
            Z0, Z1 = Z1, Z2
        E = out
    return dict(lam=lam, sigma=sig, E=E, vol=vol)
