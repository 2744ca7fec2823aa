"""GPU parity of the dense steps of Alg. 2 / Alg. 4 exposed through the ABI:
the Gaussian draw Ω (Alg. 2 step 2, Philox [R1]), Gram (eigSVD's YᵀY), orth (CholeskyQR [R7]) and the symmetric eigensolver
(Alg. 2 step 8, Alg. 4 step 8) against numpy / the oracle."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
DEV = "cuda:0"


@pytest.fixture(scope="module")
def L():
    import __graft_entry__ as ge
    ge.build()
    from paper_2110_12782_b200 import _lib
    return _lib


@pytest.fixture(scope="module")
def ctx(L):
    return L.Context(0)


def padded(n, c):
    ld = (c + 31) // 32 * 32
    return torch.zeros(n, ld, dtype=torch.float32, device=DEV)[:, :c]


@pytest.mark.parametrize("n,l,seed", [(1, 1, 0), (7, 3, 5), (1001, 286, 2), (4099, 287, 2**40 + 3), (333, 5, 9),
                                      (50003, 128, 11)])
def test_gaussian_matches_oracle(L, ctx, n, l, seed):
    """Ω = randn(n, l): the same Philox counters as the oracle,
    Box–Muller in fp32 with MUFU log2 / sincos against the oracle's fp64.
    Bound: MUFU.LG2's absolute error (~2^-22) enters r² = -2 ln u, so where r
    is tiny (u -> 1) |Δr| <= sqrt(1.39 · 2^-22) ≈ 6e-4; elsewhere the error is
    ~1e-7 relative, so all but a handful of entries are within 1e-5."""
    ref = O.gaussian_matrix(n, l, seed)
    Om = padded(n, l)
    L.netmfp_gaussian(ctx, seed, Om)
    got = Om.cpu().numpy().astype(np.float64)
    err = np.abs(got - ref)
    assert err.max() <= 6e-4
    assert np.mean(err > 1e-5 * np.maximum(1.0, np.abs(ref))) <= 1e-4
    # host buffers take the same path (staged through a device block)
    Oh = torch.zeros(n, l, dtype=torch.float32)
    L.netmfp_gaussian(ctx, seed, Oh)
    assert np.array_equal(Oh.numpy(), Om.cpu().numpy())


@pytest.mark.parametrize("n,a,b,same", [(1000, 7, 7, True), (5000, 158, 158, True), (3000, 64, 37, False),
                                        (70000, 286, 286, True), (70001, 286, 286, False), (131, 40, 40, True),
                                        (100, 33, 33, True), (250007, 228, 228, True), (20000, 256, 100, False),
                                        (4099, 300, 300, True)])
def test_gram(L, ctx, n, a, b, same):
    rng = np.random.default_rng(a + n)
    A = rng.standard_normal((n, a)).astype(np.float32)
    B = A if same else rng.standard_normal((n, b)).astype(np.float32)
    Ad = padded(n, a); Ad.copy_(torch.from_numpy(A))
    Bd = Ad if same else padded(n, b)
    if not same:
        Bd.copy_(torch.from_numpy(B))
    G = torch.zeros(a, b, dtype=torch.float64, device=DEV)
    L.netmfp_gram(ctx, Ad, Bd, G)
    ref = A.astype(np.float64).T @ B.astype(np.float64)
    # 3xTF32 on tcgen05: the fp32 TMEM accumulation truncates, so each K-chain
    # of <= ~2k rows carries a relative bias of ~1e-8 per row
    assert np.abs(G.cpu().numpy() - ref).max() <= 1e-4 * np.abs(ref).max()


@pytest.mark.parametrize("passes", [1, 2])
@pytest.mark.parametrize("n,c", [(2000, 5), (20000, 158), (50000, 286)])
def test_orthonormalize(L, ctx, n, c, passes):
    rng = np.random.default_rng(c)
    Y = (rng.standard_normal((n, c)) * np.logspace(0, 2, c)[None, :]).astype(np.float32)
    Yd = padded(n, c); Yd.copy_(torch.from_numpy(Y))
    Qd = padded(n, c)
    L.netmfp_orthonormalize(ctx, Yd, Qd, passes)
    Q = Qd.cpu().numpy().astype(np.float64)
    assert np.abs(Q.T @ Q - np.eye(c)).max() <= (1e-5 if passes == 2 else 1e-3)
    Qo, _, _ = O.eig_svd(Y.astype(np.float64))          # span(Q) == span(eigSVD Q)  [R7]
    assert np.abs(Q.T @ Qo).sum(0).min() > 0            # not degenerate
    assert np.linalg.norm(Q @ (Q.T @ Qo) - Qo) <= 1e-4 * np.sqrt(c)


def _check_eig(L, ctx, S, abs_order=True):
    l = S.shape[0]
    lam = torch.zeros(l, dtype=torch.float64, device=DEV)
    V = torch.zeros(l, l, dtype=torch.float64, device=DEV)
    L.netmfp_sym_eig(ctx, torch.from_numpy(S).to(DEV), lam, V, abs_order)
    lg, Vg = lam.cpu().numpy(), V.cpu().numpy()
    ev = np.linalg.eigvalsh(S)
    nrm = np.abs(ev).max()
    # same multiset of eigenvalues; order non-increasing in |λ| (or λ) up to
    # rounding (exact ties such as +1 / -1 may come in either order)
    assert np.abs(np.sort(lg) - np.sort(ev)).max() <= 1e-10 * nrm
    key = np.abs(lg) if abs_order else lg
    assert np.all(np.diff(key) <= 1e-10 * nrm)
    assert np.abs(Vg.T @ Vg - np.eye(l)).max() <= 1e-9
    assert np.abs(S @ Vg - Vg * lg[None, :]).max() <= 1e-9 * nrm


@pytest.mark.parametrize("l", [1, 2, 3, 4, 5, 7, 13, 42, 158, 228, 255, 256, 257, 286, 287, 288, 289, 460])
def test_sym_eig_random(L, ctx, l):
    A = np.random.default_rng(l).standard_normal((l, l))
    _check_eig(L, ctx, (A + A.T) / 2)


@pytest.mark.parametrize("l", [40, 228])
def test_sym_eig_degenerate(L, ctx, l):
    """Exactly repeated eigenvalues (twin vertices give such spectra)."""
    rng = np.random.default_rng(1)
    Q = np.linalg.qr(rng.standard_normal((l, l)))[0]
    ev = np.resize(np.repeat(np.linspace(-1, 1, l // 8), 8), l)
    ev[: l // 4] = 0.5
    _check_eig(L, ctx, (Q * ev) @ Q.T)
    _check_eig(L, ctx, (Q * ev) @ Q.T, abs_order=False)


def test_sym_eig_graph_ritz(L, ctx):
    """A Rayleigh-quotient matrix of a power-law graph operator (the Alg. 2 step 8 input)."""
    from paper_2110_12782_b200 import inputs
    n, s, t = inputs.small_graph("rmat", 4096, 2, edge_factor=8)
    rp, col, deg = O.build_csr(n, s, t)
    Y = O.normalized_spmm(rp, col, deg, np.random.default_rng(0).standard_normal((n, 120)), 0.45)
    Q = np.linalg.qr(Y)[0]
    S = Q.T @ O.normalized_spmm(rp, col, deg, Q, 0.45)
    _check_eig(L, ctx, (S + S.T) / 2)


@pytest.mark.parametrize("l", [17, 228, 286, 460])
def test_sym_eig_repeatable(L, ctx, l):
    """The cluster tridiagonalisation exchanges data through other CTAs' shared
    memory with a fixed reduction order: repeated runs must agree bit for bit
    (a buffer overwritten before its last read shows up as run-to-run noise)."""
    A = np.random.default_rng(l + 1).standard_normal((l, l))
    S = torch.from_numpy((A + A.T) / 2).to(DEV)
    outs = []
    for _ in range(12):
        lam = torch.zeros(l, dtype=torch.float64, device=DEV)
        V = torch.zeros(l, l, dtype=torch.float64, device=DEV)
        L.netmfp_sym_eig(ctx, S.clone(), lam, V, True)
        outs.append((lam.cpu().numpy(), V.cpu().numpy()))
    for lam, V in outs[1:]:
        assert np.array_equal(lam, outs[0][0]) and np.array_equal(V, outs[0][1])


def test_gram_orth_repeatable(L, ctx):
    """Gram partials are reduced in a fixed order and the CholeskyQR tile
    dataflow publishes through release/acquire flags: repeated calls on the
    same input must agree bit for bit."""
    n, c = 90001, 286
    Y = (np.random.default_rng(5).standard_normal((n, c)) * np.logspace(0, 1, c)[None, :]).astype(np.float32)
    Yd = padded(n, c); Yd.copy_(torch.from_numpy(Y))
    G0 = Q0 = None
    for _ in range(6):
        G = torch.zeros(c, c, dtype=torch.float64, device=DEV)
        L.netmfp_gram(ctx, Yd, Yd, G)
        Qd = padded(n, c)
        L.netmfp_orthonormalize(ctx, Yd, Qd, 2)
        if G0 is None:
            G0, Q0 = G.clone(), Qd.clone()
        else:
            assert torch.equal(G, G0) and torch.equal(Qd, Q0)
