"""NetMF+ oracle (TEST INFRASTRUCTURE — see oracle/__init__.py).

Every function restates one passage of PAPER.md (arxiv 2110.12782) in plain
fp64 numpy, in the paper's order and notation; "PAPER.md:L" is a line of
/root/reference/PAPER.md.  Readings where the paper is silent or garbled are
listed in DESIGN.md §3 and referenced here as [R#].

Nothing here is blocked, fused or reordered beyond what the cited passage
states.  Library primitives used as single steps: numpy matmul, numpy.linalg
eigh / svd / pinv, scipy.sparse CSR products, numpy.unique / lexsort.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

__all__ = [
    "philox4x32_10", "gaussian_matrix", "gen_sparse_sign", "TAG_OMEGA", "TAG_PSI", "TAG_PI",
    "build_csr", "deg_pow", "spmm_scaled", "spmm_scaled_rows", "normalized_spmm",
    "eig_svd", "orth_range", "freigs", "factor_pair", "trunc_log", "log1p_trunc", "elementwise_log",
    "sketch_y", "sketch_z", "sparse_sign_apply_T", "core_solve", "single_pass_svd", "embedding_from_svd",
    "cheb_coeffs", "spectral_propagate", "netmf_plus", "sym_eig_abs_sorted",
]

MASK32 = np.uint64(0xFFFFFFFF)

# ---------------------------------------------------------------------------
# Counter-based generator for the random draws of Alg. 2 (randn) and
# Alg. 3 (randperm / sign(randn)).  The paper does not name a generator
# (PAPER.md:204, :256-257); both this oracle and the CUDA library implement
# Philox4x32-10 (Salmon et al., SC'11) independently [R1].
# ---------------------------------------------------------------------------
_PM0 = np.uint64(0xD2511F53)
_PM1 = np.uint64(0xCD9E8D57)
_PW0 = np.uint64(0x9E3779B9)
_PW1 = np.uint64(0xBB67AE85)

TAG_OMEGA = 0x4F4D4547   # Gaussian test matrix Omega of Alg. 2 step 2
TAG_PSI = 0x50534931     # sparse-sign Psi of Alg. 4 step 2
TAG_PI = 0x50493132      # sparse-sign Pi of Alg. 4 step 5


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32 with 10 rounds on uint32 lanes (held in uint64 arrays)."""
    c0 = np.asarray(c0, dtype=np.uint64) & MASK32
    c1 = np.asarray(c1, dtype=np.uint64) & MASK32
    c2 = np.asarray(c2, dtype=np.uint64) & MASK32
    c3 = np.asarray(c3, dtype=np.uint64) & MASK32
    k0 = np.asarray(k0, dtype=np.uint64) & MASK32
    k1 = np.asarray(k1, dtype=np.uint64) & MASK32
    for _ in range(10):
        p0 = _PM0 * c0
        p1 = _PM1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & MASK32, lo1, (hi0 ^ c3 ^ k1) & MASK32, lo0
        k0 = (k0 + _PW0) & MASK32
        k1 = (k1 + _PW1) & MASK32
    return c0, c1, c2, c3


def gaussian_matrix(n: int, cols: int, seed: int, tag: int = TAG_OMEGA) -> np.ndarray:
    """Omega = randn(n, cols) of Alg. 2 step 2 [R1].

    Entries (i, 4q .. 4q+3): Philox4x32-10 on counter (q, i mod 2^32, i >> 32,
    tag), key (seed mod 2^32, seed >> 32); u_t = (w_t + 1/2) 2^-32 and
    Box–Muller with both outputs of each word pair:
      g(i, 4q)   = r_0 cos(2 pi u_1),  g(i, 4q+1) = r_0 sin(2 pi u_1),
      g(i, 4q+2) = r_2 cos(2 pi u_3),  g(i, 4q+3) = r_2 sin(2 pi u_3),
    r_t = sqrt(-2 ln u_t)."""
    nq = (cols + 3) // 4
    i = np.repeat(np.arange(n, dtype=np.uint64), nq)
    q = np.tile(np.arange(nq, dtype=np.uint64), n)
    w0, w1, w2, w3 = philox4x32_10(q, i & MASK32, i >> np.uint64(32), tag,
                                   seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    u0, u1, u2, u3 = ((w.astype(np.float64) + 0.5) * 2.0 ** -32 for w in (w0, w1, w2, w3))
    r0 = np.sqrt(-2.0 * np.log(u0))
    r2 = np.sqrt(-2.0 * np.log(u2))
    g = np.stack([r0 * np.cos(2.0 * np.pi * u1), r0 * np.sin(2.0 * np.pi * u1),
                  r2 * np.cos(2.0 * np.pi * u3), r2 * np.sin(2.0 * np.pi * u3)], axis=-1)
    return g.reshape(n, 4 * nq)[:, :cols]


def gen_sparse_sign(n: int, h: int, z: int, seed: int, tag: int):
    """Alg. 3 gen_sparse_sign_matrix(n, h, z).

    For column j: p((z(j-1)+1):zj) = randperm(n, z) and
    Psi(p(...), j) = sign(randn(z,1)).  randperm(n, z) is realised as
    sequential rejection sampling of uniform rows from the counter stream
    (j, r, 0, tag), r = 0, 1, ...: row = floor(w0 * n / 2^32), sign =
    +1 if w1 is even else -1; a repeated row is rejected [R1].

    Returns (rows[h, z] int64, signs[h, z] float64, p) with p = unique(rows)
    sorted (step 7)."""
    if not (2 <= z <= n):
        raise ValueError("need 2 <= z <= n")
    rows = np.empty((h, z), dtype=np.int64)
    signs = np.empty((h, z), dtype=np.float64)
    for j in range(h):
        chosen: list[int] = []
        sg: list[float] = []
        r = 0
        while len(chosen) < z:
            w0, w1, _, _ = philox4x32_10(j, r, 0, tag, seed & 0xFFFFFFFF,
                                         (seed >> 32) & 0xFFFFFFFF)
            r += 1
            row = int((int(w0) * n) >> 32)
            if row in chosen:
                continue
            chosen.append(row)
            sg.append(1.0 if (int(w1) & 1) == 0 else -1.0)
        rows[j] = chosen
        signs[j] = sg
    p = np.unique(rows)
    return rows, signs, p


def _dense_sparse_sign(rows, signs, p):
    """Psi(p, :) as a dense v x h matrix (row i <-> coordinate p[i])."""
    h, z = rows.shape
    pos = np.searchsorted(p, rows)
    M = np.zeros((p.size, h))
    for j in range(h):
        M[pos[j], j] = signs[j]
    return M


# ---------------------------------------------------------------------------
# Graph (PAPER.md:124 problem statement; :151 "The element in A corresponding
# to each edge is 1"; D = diag(degrees); vol(G) = 2m)
# ---------------------------------------------------------------------------

def build_csr(n: int, src, dst):
    """Undirected simple graph G = (V, E, A) in CSR form.

    Input edges are symmetrised, self-loops dropped, duplicates collapsed
    (A is 0/1), neighbour lists sorted ascending.  Returns
    (rowptr int64[n+1], col int32[nnz], deg int32[n]); vol(G) = nnz = 2m."""
    s = np.asarray(src, dtype=np.int64)
    t = np.asarray(dst, dtype=np.int64)
    keep = s != t
    s, t = s[keep], t[keep]
    u = np.concatenate([s, t])
    v = np.concatenate([t, s])
    key = np.unique(u * n + v)
    u = key // n
    v = key % n
    deg = np.bincount(u, minlength=n).astype(np.int32)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg, out=rowptr[1:])
    return rowptr, v.astype(np.int32), deg


def deg_pow(deg, e: float):
    """d_i^e with the convention d^e := 0 for isolated vertices (d = 0) [R2]."""
    d = np.asarray(deg, dtype=np.float64)
    out = np.zeros_like(d)
    nz = d > 0
    out[nz] = d[nz] ** e
    return out


def _adj(rowptr, col, n):
    return sp.csr_matrix((np.ones(col.size), col.astype(np.int64), rowptr), shape=(n, n))


def spmm_scaled(rowptr, col, deg, X, a: float, b: float):
    """Y = D^-a A D^-b X (PAPER.md:217 modified Laplacian with a = b = alpha;
    :171 D^-1 A with a = 1, b = 0).  scipy CSR product as the matmul step."""
    n = rowptr.size - 1
    A = _adj(rowptr, col, n)
    X = np.asarray(X, dtype=np.float64)
    return deg_pow(deg, -a)[:, None] * (A @ (deg_pow(deg, -b)[:, None] * X))


def spmm_scaled_rows(rowptr, col, deg, X, rows, a: float, b: float):
    """Rows `rows` of D^-a A D^-b X, one row at a time (for sampled parity)."""
    rs = deg_pow(deg, -a)
    out = np.empty((len(rows), X.shape[1]))
    for t, u in enumerate(rows):
        nb = col[rowptr[u]:rowptr[u + 1]].astype(np.int64)
        cs = deg_pow(deg[nb], -b)
        out[t] = rs[u] * (cs[:, None] * X[nb].astype(np.float64)).sum(axis=0)
    return out


def normalized_spmm(rowptr, col, deg, X, alpha: float):
    """D^-alpha A D^-alpha X (alpha = 1/2 is the normalized
    adjacency of Eq. 2)."""
    return spmm_scaled(rowptr, col, deg, X, alpha, alpha)


# ---------------------------------------------------------------------------
# Alg. 2: fast randomized eigen-decomposition
# ---------------------------------------------------------------------------

def eig_svd(Y):
    """eigSVD ("compared with qr, eigSVD is much faster", after
    frPCA): B = Y^T Y, [V, D] = eig(B), S = sqrt(D), Q = Y V S^-1.
    Returns (Q, S, V) with S descending."""
    Y = np.asarray(Y, dtype=np.float64)
    B = Y.T @ Y
    D, V = np.linalg.eigh(B)
    order = np.argsort(D)[::-1]
    D, V = D[order], V[:, order]
    if D[-1] <= 1e-12 * D[0]:
        raise np.linalg.LinAlgError("eigSVD: input not of full column rank (PAPER.md:215)")
    S = np.sqrt(D)
    Q = Y @ (V / S[None, :])
    return Q, S, V


def orth_range(Y, rtol: float = 1e-12):
    """Q = orth(Y) of Alg. 4 step 4 ("Q = orth(Y)"; :305 realises
    it with eigSVD).  With full column rank this IS eigSVD (same steps, same Q).
    PAPER.md:215 notes eigSVD's numerical issue when Y lacks full column rank;
    then orth(Y) is an orthonormal basis of range(Y): the eigen-directions of
    B = Y^T Y with D_i <= rtol * D_1 are dropped (DESIGN.md [R10]; e.g. a Psi
    column whose z rows are all isolated vertices gives an exactly-zero column
    of Y).  Returns Q with rank(Y) columns."""
    Y = np.asarray(Y, dtype=np.float64)
    B = Y.T @ Y
    D, V = np.linalg.eigh(B)
    order = np.argsort(D)[::-1]
    D, V = D[order], V[:, order]
    r = int(np.sum(D > rtol * D[0])) if D[0] > 0 else 0
    if r == 0:
        raise np.linalg.LinAlgError("orth: Y is zero")
    S = np.sqrt(D[:r])
    return Y @ (V[:, :r] / S[None, :])


def sym_eig_abs_sorted(S):
    """[U, Lambda] = eig(S) for symmetric S, ordered by descending |lambda|
    (ties: descending signed value) [R3]."""
    lam, U = np.linalg.eigh(S)
    order = np.lexsort((-lam, -np.abs(lam)))
    return lam[order], U[:, order]


def freigs(apply_X, n: int, k: int, s1: int, q: int, seed: int):
    """Alg. 2 freigs(X, k, s1, q), X applied as a callable.

    step 2: Omega = randn(n, k+s1), Y = X Omega
    step 3: [Q,~,~] = eigSVD(Y)
    steps 4-6: for i = 1..q: [Q,~,~] = eigSVD(X X Q)
    step 7: S = Q^T X Q
    step 8: [U^, Lambda] = eig(S)
    step 9: U = Q U^
    step 10: return U(:, 1:k), Lambda(1:k, 1:k)"""
    l = k + s1
    if l > n:
        raise ValueError("k + s1 must not exceed n")
    Omega = gaussian_matrix(n, l, seed, TAG_OMEGA)
    Y = apply_X(Omega)
    Q, _, _ = eig_svd(Y)
    for _ in range(q):
        Q, _, _ = eig_svd(apply_X(apply_X(Q)))
    S = Q.T @ apply_X(Q)
    S = 0.5 * (S + S.T)
    lam, Uh = sym_eig_abs_sorted(S)
    U = Q @ Uh
    return U[:, :k], lam[:k]


# ---------------------------------------------------------------------------
# Eq. 3-4 and Alg. 5 steps 2-3
# ---------------------------------------------------------------------------

def factor_pair(U, lam, deg, alpha: float, T: int):
    """K = U_k^T D^(-1+2a) U_k Lambda_k;  F = D^(-1+a) U_k;
    C = Lambda_k sum_{r=1}^T K^(r-1)  (Alg. 5 steps 2-3)."""
    U = np.asarray(U, dtype=np.float64)
    lam = np.asarray(lam, dtype=np.float64)
    K = (U.T * deg_pow(deg, -1.0 + 2.0 * alpha)[None, :]) @ U @ np.diag(lam)
    F = deg_pow(deg, -1.0 + alpha)[:, None] * U
    k = lam.size
    acc = np.eye(k)
    P = np.eye(k)
    for _ in range(2, T + 1):
        P = P @ K
        acc = acc + P
    C = np.diag(lam) @ acc
    return K, F, C


def trunc_log(x):
    """trunc_log(x) = max(0, log x); max(0, log x) = log(max(x,1))
    so non-positive arguments map to 0 [R4]."""
    return np.log(np.maximum(np.asarray(x, dtype=np.float64), 1.0))


def log1p_trunc(x):
    """The optional log1p(x) = log(1+x) of PAPER.md:158, with arguments
    clamped at 0 (the exact M is non-negative) [R4]."""
    return np.log1p(np.maximum(np.asarray(x, dtype=np.float64), 0.0))


def elementwise_log(x, logmode: int):
    return trunc_log(x) if logmode == 0 else log1p_trunc(x)


# ---------------------------------------------------------------------------
# §4.2: sketches and Alg. 4
# ---------------------------------------------------------------------------

def sketch_y(F, C, scale: float, rows, signs, p, logmode: int = 0, batch_rows: int = 4096):
    """Eq. 5 / Alg. 4 step 3:
    Y = trunc_log(vol/(bT) F C F(p,:)^T) Psi, with Psi(p,:) the only non-zero
    rows; computed in row batches r as in §4.4."""
    F = np.asarray(F, dtype=np.float64)
    Psi_p = _dense_sparse_sign(rows, signs, p)
    FpT = F[p].T
    n = F.shape[0]
    Y = np.empty((n, Psi_p.shape[1]))
    for r0 in range(0, n, batch_rows):
        r1 = min(n, r0 + batch_rows)
        G = scale * (F[r0:r1] @ C @ FpT)
        Y[r0:r1] = elementwise_log(G, logmode) @ Psi_p
    return Y


def sketch_z(F, C, scale: float, rows, signs, p, logmode: int = 0):
    """Alg. 4 step 6:
    Z = Pi^T trunc_log(vol/(bT) F(p,:) C F(p,:)^T) Pi (only rows p of Pi)."""
    F = np.asarray(F, dtype=np.float64)
    Pi_p = _dense_sparse_sign(rows, signs, p)
    Fp = F[p]
    G = scale * (Fp @ C @ Fp.T)
    return Pi_p.T @ elementwise_log(G, logmode) @ Pi_p


def sparse_sign_apply_T(rows, signs, X):
    """Pi^T X for a sparse-sign Pi (n x h) and dense X (n x c): row j of the
    result is sum_t signs[j,t] X[rows[j,t]] ("Pi^T Q")."""
    return (signs[:, :, None] * np.asarray(X, dtype=np.float64)[rows]).sum(axis=1)


def core_solve(PtQ, Z):
    """S = (Pi^T Q)^dagger Z (Q^T Pi)^dagger (Alg. 4 step 7)."""
    Pinv = np.linalg.pinv(PtQ)
    S = Pinv @ Z @ Pinv.T
    return S


def single_pass_svd(F, C, scale: float, d: int, s2: int, s3: int, z: int, seed: int,
                    logmode: int = 0):
    """Alg. 4 sparse_sign_rand_single_pass_SVD(F, C, d, s2, s3, z).

    Returns (U, Sigma, V, Q): steps 2-9 with Sigma = Sigma^(1:d,1:d) [R5]."""
    n = F.shape[0]
    rows_psi, sg_psi, p_psi = gen_sparse_sign(n, d + s2, z, seed, TAG_PSI)       # step 2
    Y = sketch_y(F, C, scale, rows_psi, sg_psi, p_psi, logmode)                  # step 3
    Q = orth_range(Y)                                                            # step 4 [R10]
    rows_pi, sg_pi, p_pi = gen_sparse_sign(n, d + s3, z, seed, TAG_PI)           # step 5
    Z = sketch_z(F, C, scale, rows_pi, sg_pi, p_pi, logmode)                     # step 6
    PtQ = sparse_sign_apply_T(rows_pi, sg_pi, Q)
    S = core_solve(PtQ, Z)                                                       # step 7
    Uh, sig, Vht = np.linalg.svd(S)                                              # step 8
    U = Q @ Uh[:, :d]                                                            # step 9
    V = Q @ Vht.T[:, :d]
    sig = sig[:d]
    if sig.size < d:  # rank(Y) < d [R10]: Sigma^(1:d,1:d) has zeros past the rank
        pad = d - sig.size
        sig = np.concatenate([sig, np.zeros(pad)])
        U = np.concatenate([U, np.zeros((U.shape[0], pad))], axis=1)
        V = np.concatenate([V, np.zeros((V.shape[0], pad))], axis=1)
    return U, sig, V, Q


def embedding_from_svd(U, sigma):
    """E = T sqrt(Sigma) (Alg. 5 step 5)."""
    return np.asarray(U) * np.sqrt(np.maximum(np.asarray(sigma), 0.0))[None, :]


# ---------------------------------------------------------------------------
# Spectral propagation (Alg. 5 step 6 :321) [R6]
# ---------------------------------------------------------------------------

def cheb_coeffs(order: int, mu: float, theta: float, nquad: int = 256):
    """Chebyshev coefficients c_0..c_order of the band-pass kernel
    g(lam) = exp(-((lam - mu)^2 - 1) theta / 2), lam in [0, 2], in the variable
    x = lam - 1, by N-point Gauss-Chebyshev quadrature:
        c_r = (2/N) sum_j g(x_j + 1) cos(r t_j),  t_j = pi (j+1/2)/N,  x_j = cos t_j,
    with c_0 halved; then normalised so c_0 = 1 [R6]."""
    j = np.arange(nquad)
    t = np.pi * (j + 0.5) / nquad
    x = np.cos(t)
    g = np.exp(-0.5 * ((x + 1.0 - mu) ** 2 - 1.0) * theta)
    c = np.array([(2.0 / nquad) * np.sum(g * np.cos(r * t)) for r in range(order + 1)])
    c[0] *= 0.5
    return c / c[0]


def spectral_propagate(rowptr, col, deg, E, order: int, mu: float, theta: float):
    """E <- sum_{r=0}^{p} c_r T_r(L~) E with L~ = L - I = -D^-1 A, L = I - D^-1 A
    (PAPER.md:171): Z_0 = E, Z_1 = L~ E, Z_{r+1} = 2 L~ Z_r - Z_{r-1} [R6]."""
    E = np.asarray(E, dtype=np.float64)
    c = cheb_coeffs(order, mu, theta)
    if order == 0:
        return c[0] * E
    Lt = lambda X: -spmm_scaled(rowptr, col, deg, X, 1.0, 0.0)
    Z0 = E
    Z1 = Lt(E)
    out = c[0] * Z0 + c[1] * Z1
    for r in range(2, order + 1):
        Z2 = 2.0 * Lt(Z1) - Z0
        out = out + c[r] * Z2
        Z0, Z1 = Z1, Z2
    return out


# ---------------------------------------------------------------------------
# Alg. 5 NetMF+ 
# ---------------------------------------------------------------------------

def netmf_plus(n, src, dst, *, alpha, k, s1, q, T, b, d, s2, s3, z, prop_order, mu, theta,
               seed, logmode=0):
    """Alg. 5: D = sum(A,1); [U_k, Lambda_k] = freigs(D^-a A D^-a, k, s1, q);
    K, F, C (steps 2-3); [T, Sigma, ~] = single-pass SVD (step 4);
    E = T sqrt(Sigma) (step 5); E = sum_r c_r L^r E (step 6)."""
    rowptr, col, deg = build_csr(n, src, dst)
    X = lambda M: normalized_spmm(rowptr, col, deg, M, alpha)
    U, lam = freigs(X, n, k, s1, q, seed)
    K, F, C = factor_pair(U, lam, deg, alpha, T)
    vol = float(col.size)
    scale = vol / (b * T)
    Ud, sig, _, _ = single_pass_svd(F, C, scale, d, s2, s3, z, seed, logmode)
    E = embedding_from_svd(Ud, sig)
    if prop_order > 0:
        E = spectral_propagate(rowptr, col, deg, E, prop_order, mu, theta)
    return dict(rowptr=rowptr, col=col, deg=deg, U=U, lam=lam, F=F, C=C, sigma=sig,
                E_raw=embedding_from_svd(Ud, sig), E=E)
