"""Brute-force dense references used to PIN the oracle (tests only).

These deliberately take a different route from oracle/: dense n x n matrices
built by explicit Python loops over edges, matrix powers of D^-1 A (Eq. 1
directly), dense sign matrices.  Only for tiny n.
"""
import numpy as np


def dense_adjacency(n, src, dst):
    A = np.zeros((n, n))
    for u, v in zip(np.asarray(src).tolist(), np.asarray(dst).tolist()):
        if u != v:
            A[u, v] = 1.0
            A[v, u] = 1.0
    return A


def csr_from_dense(A):
    n = A.shape[0]
    rowptr = [0]
    col = []
    for u in range(n):
        for v in range(n):
            if A[u, v] != 0:
                col.append(v)
        rowptr.append(len(col))
    return np.array(rowptr, dtype=np.int64), np.array(col, dtype=np.int32)


def dinv_pow(d, e):
    out = np.zeros(len(d))
    for i, x in enumerate(d):
        if x > 0:
            out[i] = float(x) ** e
    return out


def netmf_dense(A, T, b, logmode=0):
    """Eq. 1 by dense matrix powers."""
    d = A.sum(axis=1)
    Dinv = np.diag(dinv_pow(d, -1.0))
    P = Dinv @ A
    M = np.zeros_like(A)
    Pr = np.eye(A.shape[0])
    for _ in range(T):
        Pr = Pr @ P
        M = M + Pr @ Dinv
    X = d.sum() / (b * T) * M
    if logmode == 0:
        out = np.zeros_like(X)
        for i in range(X.shape[0]):
            for j in range(X.shape[1]):
                out[i, j] = np.log(X[i, j]) if X[i, j] > 1.0 else 0.0
        return out
    return np.log1p(np.maximum(X, 0.0))


def dense_sign_matrix(n, rows, signs):
    h, z = rows.shape
    P = np.zeros((n, h))
    for j in range(h):
        for t in range(z):
            P[rows[j, t], j] = signs[j, t]
    return P


def connected_er(n, p, seed):
    rng = np.random.default_rng(seed)
    while True:
        A = (rng.random((n, n)) < p).astype(float)
        A = np.triu(A, 1)
        A = A + A.T
        # connectivity via BFS
        seen = {0}
        frontier = [0]
        while frontier:
            u = frontier.pop()
            for v in np.nonzero(A[u])[0]:
                if v not in seen:
                    seen.add(int(v))
                    frontier.append(int(v))
        if len(seen) == n:
            src, dst = np.nonzero(np.triu(A, 1))
            return A, src.astype(np.int32), dst.astype(np.int32)
