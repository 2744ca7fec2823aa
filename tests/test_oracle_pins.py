"""Pins of the CPU oracle against things other than itself.

Each test names the PAPER.md passage it pins and the independent fact used:
golden known-answer vectors, hand computations of Eq. 1, closed forms,
paper invariants, dense brute force, textbook library routines.
"""
import math
import os

import numpy as np
import pytest

import oracle as O
from tests import _brute as B

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- generator
def test_philox_known_answers():
    """[R1] Philox4x32-10 == Random123 KAT (tests/golden/philox4x32_10_kat.txt)."""
    for line in open(os.path.join(GOLD, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        t = [int(x, 16) for x in line.split()]
        out = O.philox4x32_10(*t[:6])
        assert [int(x) for x in out] == t[6:]


def test_gaussian_matrix_is_standard_normal():
    """Alg. 2 step 2 randn: moments + KS distance of N(0,1)."""
    from scipy.stats import kstest
    G = O.gaussian_matrix(2000, 50, seed=7)
    assert abs(G.mean()) < 0.01
    assert abs(G.var() - 1.0) < 0.02
    assert kstest(G.ravel(), "norm").statistic < 0.006
    # columns independent: sample correlation small
    C = np.corrcoef(G[:, :8].T)
    assert np.abs(C - np.eye(8)).max() < 0.1
    # deterministic in seed, different across seeds
    assert np.array_equal(G, O.gaussian_matrix(2000, 50, seed=7))
    assert not np.allclose(G, O.gaussian_matrix(2000, 50, seed=8))


def test_sparse_sign_structure():
    """Alg. 3: z distinct rows per column, signs +-1,
    p = sorted unique union of the supports."""
    n, h, z = 100, 10, 8
    rows, signs, p = O.gen_sparse_sign(n, h, z, seed=3, tag=O.TAG_PSI)
    for j in range(h):
        assert len(set(rows[j].tolist())) == z
    assert set(np.unique(signs).tolist()) <= {-1.0, 1.0}
    assert np.array_equal(p, np.array(sorted(set(rows.ravel().tolist()))))
    assert p.size <= z * h
    # z = n forces full support (SPEC example)
    r2, s2, p2 = O.gen_sparse_sign(4, 1, 4, seed=0, tag=O.TAG_PI)
    assert np.array_equal(np.sort(r2[0]), np.arange(4)) and np.array_equal(p2, np.arange(4))
    with pytest.raises(ValueError):
        O.gen_sparse_sign(4, 1, 5, seed=0, tag=O.TAG_PI)


def test_sparse_sign_uniform():
    """Alg. 3 randperm(n, z): rows uniform over [0, n) (chi-square) and signs
    balanced (binomial 3 sigma)."""
    from scipy.stats import chisquare
    n, h, z = 50, 400, 8
    rows, signs, _ = O.gen_sparse_sign(n, h, z, seed=11, tag=O.TAG_PSI)
    counts = np.bincount(rows.ravel(), minlength=n)
    assert chisquare(counts).pvalue > 1e-3
    npos = (signs > 0).sum()
    N = signs.size
    assert abs(npos - N / 2) < 3 * math.sqrt(N / 4)


# ---------------------------------------------------------------- graph
def test_build_csr_hand_examples():
    """PAPER.md:124/:151 simple undirected graph; SPEC examples."""
    rp, col, deg = O.build_csr(3, [0, 1, 2], [1, 2, 0])
    assert rp.tolist() == [0, 2, 4, 6] and col.tolist() == [1, 2, 0, 2, 0, 1]
    assert deg.tolist() == [2, 2, 2]
    rp, col, deg = O.build_csr(2, [0, 1, 0], [1, 0, 0])   # duplicate + self loop
    assert rp.tolist() == [0, 1, 2] and col.tolist() == [1, 0] and deg.tolist() == [1, 1]


@pytest.mark.parametrize("seed", range(5))
def test_build_csr_vs_dense_bruteforce(seed):
    rng = np.random.default_rng(seed)
    n = 37
    src = rng.integers(0, n, 200)
    dst = rng.integers(0, n, 200)
    A = B.dense_adjacency(n, src, dst)
    rp_b, col_b = B.csr_from_dense(A)
    rp, col, deg = O.build_csr(n, src, dst)
    assert np.array_equal(rp, rp_b) and np.array_equal(col, col_b)
    assert np.array_equal(deg, A.sum(1).astype(np.int32))
    assert col.size % 2 == 0   # vol(G) = 2m


# ---------------------------------------------------------------- SpMM
def test_spmm_hand_examples():
    """SPEC graph examples: triangle alpha=1/2 keeps constants; single edge permutes."""
    rp, col, deg = O.build_csr(3, [0, 1, 2], [1, 2, 0])
    assert np.allclose(O.normalized_spmm(rp, col, deg, np.ones((3, 1)), 0.5), 1.0)
    rp, col, deg = O.build_csr(2, [0], [1])
    assert np.allclose(O.normalized_spmm(rp, col, deg, np.array([[1.0], [0.0]]), 0.5),
                       [[0.0], [1.0]])
    # L = I - D^-1 A on the triangle: X=e0 -> [1, -1/2, -1/2]
    rp, col, deg = O.build_csr(3, [0, 1, 2], [1, 2, 0])
    X = np.array([[1.0], [0.0], [0.0]])
    LX = X - O.spmm_scaled(rp, col, deg, X, 1.0, 0.0)
    assert np.allclose(LX.ravel(), [1.0, -0.5, -0.5])


@pytest.mark.parametrize("alpha", [0.5, 0.4, 0.25])
def test_spmm_vs_dense_loops(alpha):
    rng = np.random.default_rng(1)
    n = 50
    src = rng.integers(0, n, 250)
    dst = rng.integers(0, n, 250)
    A = B.dense_adjacency(n, src, dst)
    d = A.sum(1)
    X = rng.standard_normal((n, 7))
    Y = np.zeros((n, 7))
    for u in range(n):
        for v in range(n):
            if A[u, v]:
                Y[u] += d[u] ** -alpha * d[v] ** -alpha * X[v]
    rp, col, deg = O.build_csr(n, src, dst)
    assert np.abs(O.normalized_spmm(rp, col, deg, X, alpha) - Y).max() < 1e-12
    rows = [0, 5, 17, n - 1]
    assert np.abs(O.spmm_scaled_rows(rp, col, deg, X, rows, alpha, alpha) - Y[rows]).max() < 1e-12


def test_normalized_adjacency_top_eigenvector_closed_form():
    """North-star invariant: D^-1/2 A D^-1/2 (D^1/2 1) = D^1/2 1 on any graph
    without isolated vertices."""
    A, s, t = B.connected_er(40, 0.15, 2)
    rp, col, deg = O.build_csr(40, s, t)
    x = np.sqrt(deg.astype(float))[:, None]
    assert np.allclose(O.normalized_spmm(rp, col, deg, x, 0.5), x)


# ---------------------------------------------------------------- eigSVD
def test_eig_svd_examples():
    """PAPER.md:215 eigSVD; SPEC examples: diagonal case, orthonormal input."""
    Q, S, V = O.eig_svd(np.array([[2.0, 0], [0, 1], [0, 0]]))
    assert np.allclose(S, [2, 1])
    Y = np.linalg.qr(np.random.default_rng(0).standard_normal((30, 5)))[0]
    Q, S, V = O.eig_svd(Y)
    assert np.allclose(S, 1.0) and np.allclose(Q @ Q.T, Y @ Y.T)
    with pytest.raises(np.linalg.LinAlgError):
        O.eig_svd(np.ones((10, 3)))


@pytest.mark.parametrize("seed", range(5))
def test_eig_svd_vs_textbook_svd(seed):
    Y = np.random.default_rng(seed).standard_normal((200, 16))
    Q, S, V = O.eig_svd(Y)
    assert np.allclose(S, np.linalg.svd(Y, compute_uv=False), rtol=1e-10)
    assert np.abs(Q.T @ Q - np.eye(16)).max() < 1e-10
    assert np.abs(Q @ np.diag(S) @ V.T - Y).max() < 1e-10
    Qr = np.linalg.qr(Y)[0]
    assert np.linalg.norm(Q @ Q.T - Qr @ Qr.T) < 1e-8


@pytest.mark.parametrize("seed", range(3))
def test_orth_range_rank_deficient(seed):
    """Alg. 4 step 4 orth(Y) [R10]: full rank -> exactly eigSVD's Q; with
    exactly-zero and repeated columns -> rank(Y) orthonormal columns whose
    projector equals the textbook one (numpy SVD of Y, left vectors of the
    nonzero singular values)."""
    rng = np.random.default_rng(seed)
    Y = rng.standard_normal((300, 20))
    assert np.array_equal(O.orth_range(Y), O.eig_svd(Y)[0])
    Y[:, [3, 11]] = 0.0                     # a Psi column drawing only isolated rows
    Y[:, 7] = 2.0 * Y[:, 5]                 # a dependent column
    Q = O.orth_range(Y)
    assert Q.shape[1] == 17
    assert np.abs(Q.T @ Q - np.eye(17)).max() < 1e-10
    U, s, _ = np.linalg.svd(Y, full_matrices=False)
    Ur = U[:, s > 1e-8 * s[0]]
    assert Ur.shape[1] == 17
    assert np.linalg.norm(Q @ Q.T - Ur @ Ur.T) < 1e-8
    with pytest.raises(np.linalg.LinAlgError):
        O.eig_svd(Y)                        # eigSVD itself needs full column rank


# ---------------------------------------------------------------- freigs
def _op(rp, col, deg, a):
    return lambda X: O.normalized_spmm(rp, col, deg, X, a)


def test_freigs_single_edge():
    """SPEC example: single edge, alpha=1/2, k=1 -> Lambda=[1], U=+-[1,1]/sqrt2.
    (k+s1 = n = 2 is the whole space.)"""
    rp, col, deg = O.build_csr(2, [0], [1])
    U, lam = O.freigs(_op(rp, col, deg, 0.5), 2, k=1, s1=1, q=2, seed=0)
    assert np.allclose(lam, [1.0])
    assert np.allclose(np.abs(U[:, 0]), [1 / math.sqrt(2)] * 2)


def test_freigs_complete_graph_top():
    """K4, alpha=1/2: spectrum {1, -1/3, -1/3, -1/3} (closed form)."""
    s, t = zip(*[(i, j) for i in range(4) for j in range(i + 1, 4)])
    rp, col, deg = O.build_csr(4, s, t)
    U, lam = O.freigs(_op(rp, col, deg, 0.5), 4, k=4, s1=0, q=1, seed=0)
    assert np.allclose(lam, [1.0, -1 / 3, -1 / 3, -1 / 3])


@pytest.mark.parametrize("alpha", [0.5, 0.4])
def test_freigs_full_rank_matches_dense_spectrum(alpha):
    """freigs with k+s1 = n reproduces the dense spectrum (np.linalg.eigh of
    the explicitly built D^-a A D^-a)."""
    A, s, t = B.connected_er(48, 0.12, 5)
    rp, col, deg = O.build_csr(48, s, t)
    d = A.sum(1)
    Xd = np.diag(d ** -alpha) @ A @ np.diag(d ** -alpha)
    ev = np.linalg.eigvalsh(Xd)
    ev = ev[np.lexsort((-ev, -np.abs(ev)))]
    U, lam = O.freigs(_op(rp, col, deg, alpha), 48, k=48, s1=0, q=1, seed=1)
    assert np.abs(lam - ev).max() < 1e-9
    assert np.abs(Xd @ U - U * lam[None, :]).max() < 1e-8


def test_freigs_paper_invariants():
    """North-star invariants: alpha = 1/2 eigenvalues in [-1, 1]; top eigenpair
    (1, D^1/2 1/sqrt(vol)) on a connected graph."""
    A, s, t = B.connected_er(120, 0.08, 9)
    rp, col, deg = O.build_csr(120, s, t)
    U, lam = O.freigs(_op(rp, col, deg, 0.5), 120, k=16, s1=10, q=8, seed=2)
    assert np.all(np.abs(lam) <= 1 + 1e-10)
    assert abs(lam[0] - 1.0) < 1e-8
    v = np.sqrt(deg / deg.sum())
    assert abs(abs(U[:, 0] @ v) - 1.0) < 1e-8


def test_freigs_theorem1_bound():
    """Theorem 1 with eps = 0.5 over 10 seeds (SPEC A2)."""
    A, s, t = B.connected_er(300, 0.05, 4)
    rp, col, deg = O.build_csr(300, s, t)
    d = A.sum(1)
    alpha = 0.4
    Xa = np.diag(d ** -alpha) @ A @ np.diag(d ** -alpha)
    ev = np.linalg.eigvalsh(Xa)
    tail = np.sqrt(np.sort(ev ** 2)[::-1][16:].sum())
    Nh = np.diag(d ** -0.5) @ A @ np.diag(d ** -0.5)
    ok = 0
    for seed in range(10):
        U, lam = O.freigs(_op(rp, col, deg, alpha), 300, k=16, s1=10, q=10, seed=seed)
        Dm = np.diag(d ** (-0.5 + alpha))
        lhs = np.linalg.norm(Nh - Dm @ U @ np.diag(lam) @ U.T @ Dm)
        ok += lhs <= 1.5 * tail
    assert ok >= 9


# ---------------------------------------------------------------- Eq. 3
def test_factor_pair_T1_and_scalar():
    rng = np.random.default_rng(0)
    U = np.linalg.qr(rng.standard_normal((20, 3)))[0]
    lam = np.array([0.9, -0.5, 0.3])
    deg = rng.integers(1, 6, 20)
    K, F, C = O.factor_pair(U, lam, deg, 0.4, T=1)
    assert np.allclose(C, np.diag(lam))                        # T=1: C = Lambda
    u = U[:, :1]
    K, F, C = O.factor_pair(u, lam[:1], deg, 0.4, T=7)          # k = 1 geometric series
    kap = float((u[:, 0] ** 2 * deg ** (-1 + 0.8)).sum() * lam[0])
    assert np.isclose(K[0, 0], kap)
    assert np.isclose(C[0, 0], lam[0] * (1 - kap ** 7) / (1 - kap))


@pytest.mark.parametrize("alpha,T", [(0.5, 10), (0.4, 5), (0.3, 3)])
def test_eq3_full_rank_equals_eq1_closed_form(alpha, T):
    """Eq. 3 with the exact full eigendecomposition equals Eq. 1's
    sum_{r=1}^T (D^-1 A)^r D^-1 built by dense matrix powers."""
    A, s, t = B.connected_er(30, 0.2, 3)
    rp, col, deg = O.build_csr(30, s, t)
    d = A.sum(1)
    lam, U = np.linalg.eigh(np.diag(d ** -alpha) @ A @ np.diag(d ** -alpha))
    K, F, C = O.factor_pair(U, lam, deg, alpha, T)
    P = np.diag(1 / d) @ A
    M = sum(np.linalg.matrix_power(P, r) @ np.diag(1 / d) for r in range(1, T + 1))
    assert np.abs(F @ C @ F.T - M).max() < 1e-10


def test_trunc_log_values():
    """trunc_log(x) = max(0, log x); SPEC examples."""
    assert O.trunc_log(1.0) == 0 and O.trunc_log(0.5) == 0 and O.trunc_log(0.0) == 0
    assert np.isclose(O.trunc_log(math.e), 1.0) and O.trunc_log(-3.0) == 0
    assert O.log1p_trunc(0.0) == 0 and np.isclose(O.log1p_trunc(math.e - 1), 1.0)


def test_netmf_hand_examples():
    """Eq. 1 hand computations (tests/golden/netmf_hand_examples.txt) through
    the oracle's Eq. 3-4 route with the exact eigendecomposition."""
    g = {}
    for line in open(os.path.join(GOLD, "netmf_hand_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, *vals = line.split()
        g[name] = [float(v) for v in vals]

    def mprime(n, s, t, T):
        rp, col, deg = O.build_csr(n, s, t)
        d = deg.astype(float)
        lam, U = np.linalg.eigh(B.dense_adjacency(n, s, t) / np.sqrt(np.outer(d, d)))
        K, F, C = O.factor_pair(U, lam, deg, 0.5, T)
        return O.trunc_log(col.size / T * (F @ C @ F.T))

    assert np.allclose(mprime(2, [0], [1], 1).ravel(), g["single_edge_T1"])
    M = mprime(3, [0, 1, 2], [1, 2, 0], 1)
    assert np.allclose(M[0, 1], g["triangle_T1_offdiag"]) and np.allclose(np.diag(M), 0)
    M = mprime(3, [0, 1, 2], [1, 2, 0], 2)
    assert np.allclose(M[0, 1], g["triangle_T2_offdiag"]) and np.allclose(np.diag(M), g["triangle_T2_diag"])


# ---------------------------------------------------------------- sketches
def _exact_setup(n=40, p=0.15, seed=3, alpha=0.45, T=10, b=1.0):
    A, s, t = B.connected_er(n, p, seed)
    rp, col, deg = O.build_csr(n, s, t)
    d = A.sum(1)
    lam, U = np.linalg.eigh(np.diag(d ** -alpha) @ A @ np.diag(d ** -alpha))
    K, F, C = O.factor_pair(U, lam, deg, alpha, T)
    scale = col.size / (b * T)
    Mp = B.netmf_dense(A, T, b)
    return A, rp, col, deg, F, C, scale, Mp


@pytest.mark.parametrize("logmode", [0, 1])
def test_sketch_y_equals_dense_eq1_times_psi(logmode):
    """Eq. 5 == dense M' (Eq. 1 by matrix powers) times dense Psi."""
    A, rp, col, deg, F, C, scale, _ = _exact_setup()
    Mp = B.netmf_dense(A, 10, 1.0, logmode)
    n = A.shape[0]
    rows, signs, p = O.gen_sparse_sign(n, 12, 8, seed=5, tag=O.TAG_PSI)
    Y = O.sketch_y(F, C, scale, rows, signs, p, logmode)
    assert np.abs(Y - Mp @ B.dense_sign_matrix(n, rows, signs)).max() < 1e-9


def test_sketch_y_batching_invariance():
    """SPEC A6 / PAPER.md:270 batching: batch_rows in {1, 7, 64, n} identical."""
    A, rp, col, deg, F, C, scale, _ = _exact_setup()
    rows, signs, p = O.gen_sparse_sign(40, 12, 8, seed=5, tag=O.TAG_PSI)
    Y0 = O.sketch_y(F, C, scale, rows, signs, p, batch_rows=40)
    for br in (1, 7, 64):
        assert np.abs(O.sketch_y(F, C, scale, rows, signs, p, batch_rows=br) - Y0).max() < 1e-10


def test_sketch_z_equals_dense_and_symmetric():
    """Alg. 4 step 6 == Pi^T M' Pi (dense) and symmetric."""
    A, rp, col, deg, F, C, scale, Mp = _exact_setup()
    rows, signs, p = O.gen_sparse_sign(40, 30, 8, seed=6, tag=O.TAG_PI)
    Z = O.sketch_z(F, C, scale, rows, signs, p)
    Pi = B.dense_sign_matrix(40, rows, signs)
    assert np.abs(Z - Pi.T @ Mp @ Pi).max() < 1e-9
    assert np.abs(Z - Z.T).max() < 1e-10
    assert np.abs(O.sparse_sign_apply_T(rows, signs, Mp) - Pi.T @ Mp).max() < 1e-12


def test_core_solve_plant_and_recover():
    """PAPER.md:281 S = (Pi^T Q)^+ Z (Q^T Pi)^+: exact recovery of a planted S0."""
    rng = np.random.default_rng(0)
    P = rng.standard_normal((96, 32))
    S0 = rng.standard_normal((32, 32))
    S0 = S0 + S0.T
    assert np.abs(O.core_solve(P, P @ S0 @ P.T) - S0).max() < 1e-8
    Z = rng.standard_normal((5, 5))
    assert np.allclose(O.core_solve(np.eye(5), Z), Z)


def test_single_pass_svd_exact_case():
    """Alg. 4 on an exactly representable target: with d + s2 >= n the range
    sketch spans R^n, so Sigma equals the exact top-d singular values of the
    dense M' (Eq. 1) and Q S Q^T reproduces M'."""
    A, rp, col, deg, F, C, scale, Mp = _exact_setup(n=30, seed=7)
    d = 6
    U, sig, V, Q = O.single_pass_svd(F, C, scale, d, s2=24, s3=60, z=8, seed=3)
    ex = np.linalg.svd(Mp, compute_uv=False)[:d]
    assert np.allclose(sig, ex, rtol=1e-7)
    # U, V span the same subspace (symmetric target) up to sign
    assert np.abs(np.abs(np.sum(U * V, axis=0)) - 1).max() < 1e-6
    E = O.embedding_from_svd(U, sig)
    assert np.allclose(E @ E.T, U @ np.diag(sig) @ U.T)


# ---------------------------------------------------------------- propagation
def test_cheb_coeffs_reproduce_kernel():
    """[R6] the Gauss-Chebyshev coefficients are a Chebyshev expansion of
    g(x+1)/c0: at order 40 sum_r c_r T_r(x) matches it (numpy chebval)."""
    from numpy.polynomial import chebyshev as Ch
    mu, th = 0.2, 0.5
    c = O.cheb_coeffs(40, mu, th)
    x = np.linspace(-1, 1, 101)
    g = np.exp(-0.5 * ((x + 1 - mu) ** 2 - 1) * th)
    # raw c0 = mean of g over Chebyshev nodes = (1/pi) int g / sqrt(1-x^2)
    t = np.pi * (np.arange(256) + 0.5) / 256
    c0raw = np.mean(np.exp(-0.5 * ((np.cos(t) + 1 - mu) ** 2 - 1) * th))
    assert np.abs(Ch.chebval(x, c) - g / c0raw).max() < 1e-10


def test_propagate_identity_and_constants():
    A, s, t = B.connected_er(30, 0.2, 1)
    rp, col, deg = O.build_csr(30, s, t)
    E = np.random.default_rng(0).standard_normal((30, 4))
    assert np.allclose(O.spectral_propagate(rp, col, deg, E, 0, 0.2, 0.5), E)
    ones = np.ones((30, 2))     # L 1 = 0 -> L~ 1 = -1 -> output = (sum_r c_r (-1)^r) 1
    c = O.cheb_coeffs(10, 0.2, 0.5)
    out = O.spectral_propagate(rp, col, deg, ones, 10, 0.2, 0.5)
    assert np.allclose(out, np.sum(c * (-1.0) ** np.arange(11)))


@pytest.mark.parametrize("order", [1, 2, 10])
def test_propagate_spectral_route(order):
    """Recurrence == spectral evaluation through the eigendecomposition of
    D^-1/2 A D^-1/2 with numpy's chebval (independent route)."""
    from numpy.polynomial import chebyshev as Ch
    A, s, t = B.connected_er(35, 0.2, 8)
    rp, col, deg = O.build_csr(35, s, t)
    d = A.sum(1)
    lam, V = np.linalg.eigh(np.diag(d ** -0.5) @ A @ np.diag(d ** -0.5))
    c = O.cheb_coeffs(order, 0.2, 0.5)
    h = Ch.chebval(-lam, c)        # L~ = -D^-1 A ~ -Lambda
    E = np.random.default_rng(1).standard_normal((35, 3))
    ref = np.diag(d ** -0.5) @ V @ np.diag(h) @ V.T @ np.diag(d ** 0.5) @ E
    assert np.abs(O.spectral_propagate(rp, col, deg, E, order, 0.2, 0.5) - ref).max() < 1e-10


# ---------------------------------------------------------------- Alg. 5
def test_netmf_plus_exact_regime():
    """Alg. 5 in its exact regime (k = n, q large, d + s2 >= n): singular values
    == exact SVD of the dense Eq. 1 matrix; E_raw E_raw^T == rank-d part."""
    A, s, t = B.connected_er(28, 0.2, 11)
    n = 28
    out = O.netmf_plus(n, s, t, alpha=0.5, k=n, s1=0, q=3, T=5, b=1.0, d=5, s2=23, s3=60,
                       z=8, prop_order=0, mu=0.2, theta=0.5, seed=0)
    Mp = B.netmf_dense(A, 5, 1.0)
    U, S, Vt = np.linalg.svd(Mp)
    assert np.allclose(out["sigma"], S[:5], rtol=1e-7)


def test_single_pass_svd_rank_below_d_pads_zeros():
    """Alg. 4 step 9 Sigma = Sigma^(1:d,1:d) [R5] with rank(Y) < d [R10]: the
    singular values past the rank are zero and their columns of U are zero;
    the leading ones equal the exact SVD of the (low-rank) Eq. 1 matrix."""
    rng = np.random.default_rng(3)
    n, k = 60, 3
    F = rng.standard_normal((n, k))
    C = np.diag([3.0, 2.0, 1.0])
    U, sig, V, Q = O.single_pass_svd(F, C, 1.0, 8, 4, 40, 4, 7, 1)   # log1p: rank(f(F C F^T)) can exceed k
    assert sig.shape == (8,) and U.shape == (n, 8)
    r = Q.shape[1]
    if r < 8:
        assert np.all(sig[r:] == 0.0) and np.all(U[:, r:] == 0.0)
    # a rank-2 matrix through trunc_log: Y has rank <= its nonzero pattern allows
    F2 = np.zeros((n, 2))
    F2[:5] = rng.uniform(1.0, 2.0, (5, 2))        # M = F2 F2^T > 1 only on a 5x5 block
    U2, sig2, _, Q2 = O.single_pass_svd(F2, np.eye(2), 10.0, 8, 4, 40, n, 7, 0)   # z = n: dense signs, exact regime
    M = O.trunc_log(10.0 * F2 @ F2.T)
    ex = np.linalg.svd(M, compute_uv=False)
    assert Q2.shape[1] <= 5 and np.all(sig2[Q2.shape[1]:] == 0.0)
    r2 = int((ex > 1e-6 * ex[0]).sum())          # orth_range keeps sigma > 1e-6 sigma_1 (eigenvalues > 1e-12)
    lead = int((ex > 1e-3 * ex[0]).sum())
    assert Q2.shape[1] == r2 and np.allclose(sig2[:lead], ex[:lead], rtol=1e-6)
