"""GPU parity: every C-ABI entry point vs the CPU oracle on the same seeded
inputs.  Tolerances (north_star): bit-exact for CSR/degrees/
partition; 1e-4 relative Frobenius on SpMM and sketch outputs; 1e-3 on
leading eigenvalues and singular values."""
import numpy as np
import pytest

import oracle as O
from paper_2110_12782_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def relf(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def L():
    import __graft_entry__ as ge
    ge.build()
    from paper_2110_12782_b200 import _lib
    assert torch.cuda.is_available()
    return _lib


@pytest.fixture(scope="module")
def ctx(L):
    return L.Context(0)


DEV = "cuda:0"


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def padded(n, c, dtype=torch.float32, ld=None):
    ld = ld or ((c + 31) // 32 * 32)
    return torch.zeros(n, ld, dtype=dtype, device=DEV)[:, :c]


# ---------------------------------------------------------------- graphs
GRAPHS = {
    "er600": lambda: inputs.small_graph("er", 600, 3, avg_deg=10.0),
    "star1500": lambda: inputs.small_graph("star", 1500, 0),
    "rmat_s13": lambda: inputs.small_graph("rmat", 8192, 4, edge_factor=16),
    "cfg0": lambda: inputs.make_graph(inputs.CONFIGS[0].graph),
}


@pytest.fixture(scope="module")
def graphs(L, ctx):
    out = {}
    for name, mk in GRAPHS.items():
        n, s, t = mk()
        g = L.netmfp_build_csr(ctx, n, dev(s), dev(t))
        out[name] = (n, s, t, g, O.build_csr(n, s, t))
    return out


@pytest.mark.parametrize("name", list(GRAPHS))
def test_build_csr_bit_exact(graphs, ctx, name):
    n, s, t, g, (rp, col, deg) = graphs[name]
    grp, gcol, gdeg = g.export(ctx)
    assert np.array_equal(grp, rp) and np.array_equal(gcol, col) and np.array_equal(gdeg, deg)
    assert g.nnz == col.size


def test_build_csr_edge_cases(L, ctx):
    cases = [
        (1, [], []),                                # single vertex, no edges
        (5, [0, 0, 1, 1, 3], [0, 0, 1, 1, 3]),      # self loops only
        (4, [0, 1, 0, 2, 2, 3], [1, 0, 1, 3, 3, 2]),  # duplicates both directions
        (7, [6, 0], [0, 6]),                        # ragged: isolated vertices
    ]
    for n, s, t in cases:
        s = np.array(s, dtype=np.int32)
        t = np.array(t, dtype=np.int32)
        g = L.netmfp_build_csr(ctx, n, s, t)        # host buffers (e2e path)
        rp, col, deg = g.export(ctx)
        orp, ocol, odeg = O.build_csr(n, s, t)
        assert np.array_equal(rp, orp) and np.array_equal(col, ocol) and np.array_equal(deg, odeg)
    with pytest.raises(L.NetmfpError):
        L.netmfp_build_csr(ctx, 3, np.array([0, 5], np.int32), np.array([1, 1], np.int32))


def test_heavy_rows_present(graphs):
    assert graphs["star1500"][3].n_heavy == 1
    assert graphs["rmat_s13"][3].n_heavy > 0


# ---------------------------------------------------------------- SpMM
@pytest.mark.parametrize("name", list(GRAPHS))
@pytest.mark.parametrize("cols", [1, 3, 32, 37, 158])
@pytest.mark.parametrize("ab", [(0.45, 0.45), (0.5, 0.5), (1.0, 0.0), (0.0, 0.0)])
def test_spmm_parity(L, ctx, graphs, name, cols, ab):
    n, s, t, g, (rp, col, deg) = graphs[name]
    X = np.random.default_rng(cols).standard_normal((n, cols)).astype(np.float32)
    Xd = padded(n, cols)
    Xd.copy_(dev(X))
    Yd = padded(n, cols)
    L.netmfp_spmm(ctx, g, ab[0], ab[1], Xd, Yd)
    ref = O.spmm_scaled(rp, col, deg, X.astype(np.float64), ab[0], ab[1])
    assert relf(Yd.cpu().numpy(), ref) <= 1e-5


def test_spmm_host_buffers_and_unpadded_ld(L, ctx, graphs):
    n, s, t, g, (rp, col, deg) = graphs["rmat_s13"]
    X = np.random.default_rng(0).standard_normal((n, 5)).astype(np.float32)
    Y = np.zeros((n, 5), dtype=np.float32)
    L.netmfp_spmm(ctx, g, 0.5, 0.5, X, Y)            # host (e2e) path, ld = 5
    ref = O.normalized_spmm(rp, col, deg, X.astype(np.float64), 0.5)
    assert relf(Y, ref) <= 1e-5


# ---------------------------------------------------------------- Alg. 2
def recon(U, lam):
    return (U * lam[None, :]) @ U.T


@pytest.mark.parametrize("name,alpha,k,s1,q", [("er600", 0.45, 32, 10, 3), ("cfg0", 0.45, 128, 30, 2),
                                               ("rmat_s13", 0.4, 64, 20, 4)])
def test_eig_parity(L, ctx, graphs, name, alpha, k, s1, q):
    n, s, t, g, (rp, col, deg) = graphs[name]
    U = padded(n, k)
    lam = torch.zeros(k, dtype=torch.float64, device=DEV)
    L.netmfp_eig(ctx, g, alpha, k, s1, q, 7, U, lam)
    Ug = U.cpu().numpy().astype(np.float64)
    lg = lam.cpu().numpy()
    Uo, lo = O.freigs(lambda X: O.normalized_spmm(rp, col, deg, X, alpha), n, k, s1, q, 7)
    # leading eigenvalues (1e-3), all Ritz values (1e-3 of |lambda_1|)
    assert np.abs(lg[:8] - lo[:8]).max() <= 1e-3 * np.abs(lo[:8]).max()
    assert np.abs(lg - lo).max() <= 1e-3 * abs(lo[0])
    # orthonormal columns, same rank-k operator U Lambda U^T
    assert np.abs(Ug.T @ Ug - np.eye(k)).max() <= 1e-4
    assert relf(recon(Ug, lg), recon(Uo, lo)) <= 1e-3


def test_eig_alpha_half_top_pair(L, ctx, graphs):
    """North-star invariant on the GPU output: alpha = 1/2, connected graph:
    top eigenpair (1, D^1/2 1 / sqrt(vol))."""
    n, s, t, g, (rp, col, deg) = graphs["er600"]
    assert deg.min() > 0
    U = padded(n, 16)
    lam = torch.zeros(16, dtype=torch.float64, device=DEV)
    L.netmfp_eig(ctx, g, 0.5, 16, 10, 6, 3, U, lam)
    lg = lam.cpu().numpy()
    assert abs(lg[0] - 1.0) <= 1e-4 and np.all(np.abs(lg) <= 1 + 1e-4)
    v = np.sqrt(deg / deg.sum())
    assert abs(abs(U.cpu().numpy()[:, 0].astype(np.float64) @ v) - 1) <= 1e-4


# ---------------------------------------------------------------- Eq. 3
def test_factor_pair_parity(L, ctx, graphs):
    n, s, t, g, (rp, col, deg) = graphs["cfg0"]
    k, alpha, T = 48, 0.45, 10
    Uo, lo = O.freigs(lambda X: O.normalized_spmm(rp, col, deg, X, alpha), n, k, 10, 2, 1)
    U32 = Uo.astype(np.float32)
    Ud = padded(n, k)
    Ud.copy_(dev(U32))
    F = padded(n, k)
    Cm = torch.zeros(k, k, dtype=torch.float64, device=DEV)
    L.netmfp_factor_pair(ctx, g, alpha, T, Ud, dev(lo), F, Cm)
    K, Fo, Co = O.factor_pair(U32.astype(np.float64), lo, deg, alpha, T)
    assert relf(F.cpu().numpy(), Fo) <= 1e-6
    assert relf(Cm.cpu().numpy(), Co) <= 1e-5


# ---------------------------------------------------------------- Alg. 4
@pytest.mark.parametrize("logmode", [0, 1])
@pytest.mark.parametrize("name,k,d,s2,s3", [("er600", 32, 16, 16, 160), ("cfg0", 64, 32, 100, 1000)])
def test_sketch_svd_parity(L, ctx, graphs, name, k, d, s2, s3, logmode):
    n, s, t, g, (rp, col, deg) = graphs[name]
    alpha, T, b, z, seed = 0.45, 10, 1.0, 8, 11
    Uo, lo = O.freigs(lambda X: O.normalized_spmm(rp, col, deg, X, alpha), n, k, 10, 2, 1)
    K, Fo, Co = O.factor_pair(Uo, lo, deg, alpha, T)
    F32 = Fo.astype(np.float32)
    F64 = F32.astype(np.float64)
    scale = col.size / (b * T)
    Fd = padded(n, k)
    Fd.copy_(dev(F32))
    h2, h3 = d + s2, d + s3
    Ysk = padded(n, h2)
    Zsk = torch.zeros(h3, h3, dtype=torch.float64, device=DEV)
    sig = torch.zeros(d, dtype=torch.float64, device=DEV)
    E = padded(n, d)
    Ud = padded(n, d)
    L.netmfp_sketch_svd(ctx, Fd, dev(Co), scale, d, s2, s3, z, seed, logmode, U=Ud, sigma=sig, E=E,
                        Ysk=Ysk, Zsk=Zsk)
    r_psi, sg_psi, p_psi = O.gen_sparse_sign(n, h2, z, seed, O.TAG_PSI)
    Yo = O.sketch_y(F64, Co, scale, r_psi, sg_psi, p_psi, logmode)
    assert relf(Ysk.cpu().numpy(), Yo) <= 1e-4
    r_pi, sg_pi, p_pi = O.gen_sparse_sign(n, h3, z, seed, O.TAG_PI)
    Zo = O.sketch_z(F64, Co, scale, r_pi, sg_pi, p_pi, logmode)
    assert relf(Zsk.cpu().numpy(), Zo) <= 1e-4
    Uref, sref, Vref, Q = O.single_pass_svd(F64, Co, scale, d, s2, s3, z, seed, logmode)
    sg = sig.cpu().numpy()
    lead = sref >= 1e-2 * sref[0]          # "leading" singular values
    assert np.abs(sg - sref)[lead].max() <= 1e-3 * sref[0]
    assert np.abs(sg - sref).max() <= 1e-2 * sref[0]
    Ug = Ud.cpu().numpy().astype(np.float64)
    assert np.abs(Ug.T @ Ug - np.eye(d)).max() <= 1e-3
    # rank-d reconstruction U diag(sigma) U^T agrees (sign/rotation free)
    Eg = E.cpu().numpy().astype(np.float64)
    Eo = O.embedding_from_svd(Uref, sref)
    assert relf(Eg @ Eg.T, Eo @ Eo.T) <= 1e-3


# ---------------------------------------------------------------- propagation
@pytest.mark.parametrize("name", list(GRAPHS))
@pytest.mark.parametrize("order,d", [(0, 8), (1, 8), (2, 33), (3, 16), (10, 32)])
def test_propagate_parity(L, ctx, graphs, name, order, d):
    n, s, t, g, (rp, col, deg) = graphs[name]
    E0 = np.random.default_rng(order).standard_normal((n, d)).astype(np.float32)
    E = padded(n, d)
    E.copy_(dev(E0))
    L.netmfp_propagate(ctx, g, E, order, 0.2, 0.5)
    ref = O.spectral_propagate(rp, col, deg, E0.astype(np.float64), order, 0.2, 0.5)
    assert relf(E.cpu().numpy(), ref) <= 1e-4


# ---------------------------------------------------------------- Alg. 5
def test_embed_end_to_end(L, ctx, graphs):
    n, s, t, g, (rp, col, deg) = graphs["er600"]
    prm = dict(alpha=0.45, k=32, s1=10, q=3, T=10, b=1.0, d=16, s2=16, s3=160, z=8, prop_order=10,
               mu=0.2, theta=0.5, seed=5, logmode=0)
    E = padded(n, 16)
    sig = torch.zeros(16, dtype=torch.float64, device=DEV)
    lam = torch.zeros(32, dtype=torch.float64, device=DEV)
    L.netmfp_embed(ctx, g, L.make_params(**prm), E, sig, lam)
    ref = O.netmf_plus(n, s, t, **prm)
    assert np.abs(lam.cpu().numpy() - ref["lam"]).max() <= 1e-3 * abs(ref["lam"][0])
    sg = sig.cpu().numpy()
    assert np.abs(sg[:4] - ref["sigma"][:4]).max() <= 1e-3 * ref["sigma"][0]
    assert _match_cols_up_to_sign(E.cpu().numpy(), ref["E"], 4) <= 1e-3
    # host-buffer end-to-end path gives the same embedding
    Eh = np.zeros((n, 16), dtype=np.float32)
    L.netmfp_embed_edges(ctx, n, s, t, L.make_params(**prm), Eh)
    assert relf(Eh, E.cpu().numpy()) <= 1e-4


def _match_cols_up_to_sign(E, R, ncols):
    """max over the leading columns of min(|E_j - R_j|, |E_j + R_j|) / |R_j|"""
    worst = 0.0
    for j in range(ncols):
        r = np.linalg.norm(R[:, j])
        worst = max(worst, min(np.linalg.norm(E[:, j] - R[:, j]), np.linalg.norm(E[:, j] + R[:, j])) / r)
    return worst


def test_embed_isolated_vertices_compacted(L, ctx):
    """Isolated vertices interleaved with the graph (embed drops them on the
    GPU): same λ, σ and embedding as the oracle on the full
    vertex set, and exactly zero rows for the isolated vertices [R2]."""
    n0, s0, t0 = inputs.small_graph("er", 600, 3, avg_deg=10.0)
    n = 900
    perm = np.random.default_rng(11).permutation(n)[:n0].astype(np.int32)
    s, t = perm[s0], perm[t0]
    g = L.netmfp_build_csr(ctx, n, dev(s), dev(t))
    prm = dict(alpha=0.45, k=32, s1=10, q=3, T=10, b=1.0, d=16, s2=16, s3=160, z=8, prop_order=10,
               mu=0.2, theta=0.5, seed=5, logmode=0)
    E = padded(n, 16)
    sig = torch.zeros(16, dtype=torch.float64, device=DEV)
    lam = torch.zeros(32, dtype=torch.float64, device=DEV)
    L.netmfp_embed(ctx, g, L.make_params(**prm), E, sig, lam)
    ref = O.netmf_plus(n, s, t, **prm)
    assert np.abs(lam.cpu().numpy() - ref["lam"]).max() <= 1e-3 * abs(ref["lam"][0])
    assert np.abs(sig.cpu().numpy()[:4] - ref["sigma"][:4]).max() <= 1e-3 * ref["sigma"][0]
    Eh = E.cpu().numpy()
    iso = np.setdiff1d(np.arange(n), perm)
    assert np.all(Eh[iso] == 0.0)
    assert _match_cols_up_to_sign(Eh, ref["E"], 4) <= 1e-3
    # pinned host output (the GPU writes the n' rows straight into it, the
    # host zeroes it meanwhile): identical to the device result, whatever the
    # buffer held before; also with a padded leading dimension
    for ld in (16, 20):
        Ep = torch.full((n, ld), float("nan"), dtype=torch.float32).pin_memory()[:, :16]
        sg2 = np.zeros(16)
        L.netmfp_embed(ctx, g, L.make_params(**prm), Ep, sg2)
        assert np.array_equal(Ep.numpy(), Eh) and np.array_equal(sg2, sig.cpu().numpy())


def _separated(sig, j, rel=0.01):
    """singular value j is isolated from its neighbours by > rel (its vector is unique up to sign)"""
    lo = sig[j + 1] if j + 1 < len(sig) else -np.inf
    hi = sig[j - 1] if j > 0 else np.inf
    return (hi - sig[j]) > rel * sig[j] and (sig[j] - lo) > rel * sig[j]


@pytest.mark.parametrize("cfg", [0, 1])
def test_embed_full_config(L, ctx, cfg):
    """BASELINE configs[0] / configs[1] at full size and full parameters:
    lambda (all k), sigma (leading 8) and the embedding's well-separated
    leading columns (up to sign) vs the oracle's Alg. 5."""
    w = inputs.CONFIGS[cfg]
    n, s, t = inputs.make_graph(w.graph)
    prm = w.params()
    g = L.netmfp_build_csr(ctx, n, dev(s), dev(t))
    E = padded(n, w.d)
    sig = torch.zeros(w.d, dtype=torch.float64, device=DEV)
    lam = torch.zeros(w.k, dtype=torch.float64, device=DEV)
    L.netmfp_embed(ctx, g, L.make_params(**prm), E, sig, lam)
    ref = O.netmf_plus(n, s, t, **prm)
    lg, sg, Eg = lam.cpu().numpy(), sig.cpu().numpy(), E.cpu().numpy()
    assert np.abs(lg - ref["lam"]).max() <= 1e-3 * abs(ref["lam"][0])
    assert np.abs(sg[:8] - ref["sigma"][:8]).max() <= 1e-3 * ref["sigma"][0]
    cols = [j for j in range(8) if _separated(ref["sigma"], j)]
    assert cols, "no well-separated singular value among the leading 8"
    R = ref["E"][:, cols]
    assert _match_cols_up_to_sign(Eg[:, cols], R, len(cols)) <= 1e-3


def test_cfg2_full_size_properties(L, ctx):
    """BASELINE configs[2] at full size and full parameters (n = 2^20; the
    oracle's dense eigSVD / sketch do not finish in seconds there).  R-MAT at
    edge factor 3 has thousands of small components, so |lambda| = 1 and its
    neighbours are eigenvalues of huge multiplicity and single eigenvectors
    are not determined; what Alg. 2 guarantees at any size is checked
    instead (fp64 on the CPU): U has orthonormal columns and (U, Lambda) is a
    Ritz pair set, U^T X U = Lambda.  The embedding is finite with zero rows
    on isolated vertices, sigma sorted and non-negative."""
    import scipy.sparse as sp
    w = inputs.CONFIGS[2]
    n, s, t = inputs.make_graph(w.graph)
    g = L.netmfp_build_csr(ctx, n, dev(s), dev(t))
    rp, col, deg = g.export(ctx)
    U = padded(n, w.k)
    lam = torch.zeros(w.k, dtype=torch.float64, device=DEV)
    L.netmfp_eig(ctx, g, w.alpha, w.k, w.s1, w.q, w.seed, U, lam)
    lg = lam.cpu().numpy()
    Ug = U.cpu().numpy().astype(np.float64)
    dinv = np.zeros(n)
    dinv[deg > 0] = deg[deg > 0].astype(np.float64) ** -w.alpha
    A = sp.csr_matrix((np.ones(col.size), col, rp), shape=(n, n))
    XU = dinv[:, None] * (A @ (dinv[:, None] * Ug))
    assert np.abs(Ug.T @ Ug - np.eye(w.k)).max() <= 1e-4
    assert np.abs(Ug.T @ XU - np.diag(lg)).max() <= 1e-3 * abs(lg[0])
    assert np.all(np.diff(np.abs(lg)) <= 1e-12)          # ordered by |lambda| [R3]
    E = padded(n, w.d)
    sig = torch.zeros(w.d, dtype=torch.float64, device=DEV)
    L.netmfp_embed(ctx, g, L.make_params(**w.params()), E, sig)
    Eh, sg = E.cpu().numpy(), sig.cpu().numpy()
    assert np.isfinite(Eh).all() and np.all(Eh[deg == 0] == 0.0)
    assert np.all(sg >= 0) and np.all(np.diff(sg) <= 1e-9 * sg[0])
    assert np.linalg.norm(Eh[deg > 0], axis=0).min() > 0


def test_cfg2_full_size_sampled(L, ctx):
    """BASELINE configs[2] at full size: bit-exact CSR, sampled SpMM rows."""
    spec = inputs.CONFIGS[2]
    n, s, t = inputs.make_graph(spec.graph)
    g = L.netmfp_build_csr(ctx, n, dev(s), dev(t))
    rp, col, deg = O.build_csr(n, s, t)
    grp, gcol, gdeg = g.export(ctx)
    assert np.array_equal(grp, rp) and np.array_equal(gcol, col) and np.array_equal(gdeg, deg)
    l = spec.k + spec.s1
    X = torch.randn(n, 288, device=DEV)[:, :l].contiguous()
    Xp = padded(n, l)
    Xp.copy_(X)
    Y = padded(n, l)
    L.netmfp_spmm(ctx, g, spec.alpha, spec.alpha, Xp, Y)
    rng = np.random.default_rng(0)
    rows = np.concatenate([rng.integers(0, n, 200), np.argsort(deg)[-20:]])   # include hubs
    Xh = Xp.cpu().numpy()
    ref = O.spmm_scaled_rows(rp, col, deg, Xh, rows, spec.alpha, spec.alpha)
    assert relf(Y.cpu().numpy()[rows], ref) <= 1e-5


# ---------------------------------------------------------------- row partitions
@pytest.mark.parametrize("name", ["rmat_s13", "star1500", "cfg0"])
def test_build_csr_rows_is_a_slice(L, ctx, graphs, name):
    n, s, t, g, (rp, col, deg) = graphs[name]
    for b0, b1 in [(0, n // 3), (n // 3, n), (n // 2, n // 2 + 17)]:
        gp = L.netmfp_build_csr_rows(ctx, n, dev(s), dev(t), b0, b1)
        prp, pcol, pdeg = gp.export(ctx)
        assert np.array_equal(prp, rp[b0:b1 + 1] - rp[b0])
        assert np.array_equal(pcol, col[rp[b0]:rp[b1]])
        assert np.array_equal(pdeg, deg[b0:b1])
        assert L.netmfp_graph_rows(gp)[:2] == (b0, n)


@pytest.mark.parametrize("cols", [3, 128, 286])
def test_partition_spmm_rows(L, ctx, graphs, cols):
    n, s, t, g, (rp, col, deg) = graphs["rmat_s13"]
    X = np.random.default_rng(cols).standard_normal((n, cols)).astype(np.float32)
    Xd = padded(n, cols)
    Xd.copy_(dev(X))
    ref = O.spmm_scaled(rp, col, deg, X.astype(np.float64), 0.45, 0.0)
    bounds = L.netmfp_partition_rows(rp, 3)
    for r in range(3):
        b0, b1 = int(bounds[r]), int(bounds[r + 1])
        gp = L.netmfp_build_csr_rows(ctx, n, dev(s), dev(t), b0, b1)
        Yd = padded(b1 - b0, cols)
        L.netmfp_spmm(ctx, gp, 0.45, 0.0, Xd, Yd)       # full X in, this partition's rows out
        assert relf(Yd.cpu().numpy(), ref[b0:b1]) <= 1e-5


def test_dist_one_rank_is_the_single_gpu_path(L, ctx, graphs):
    n, s, t, g, _ = graphs["er600"]
    c1 = L.Context(0)
    L.netmfp_dist_init(c1, b"\0" * L.DIST_ID_BYTES, 1, 0)
    gd = L.netmfp_dist_build_csr(c1, n, dev(s), dev(t))
    assert L.netmfp_graph_rows(gd) == (0, n, g.nnz)
    prm = L.make_params(alpha=0.45, k=24, s1=8, q=2, T=10, b=1.0, d=12, s2=12, s3=100, z=8, prop_order=6,
                        mu=0.2, theta=0.5, seed=3, logmode=0)
    E1 = padded(n, 12)
    E2 = padded(n, 12)
    L.netmfp_embed(ctx, g, prm, E1)
    L.netmfp_embed(c1, gd, prm, E2)
    assert torch.equal(E1, E2)


@pytest.mark.parametrize("name", ["rmat_s13", "star1500"])
def test_repeatable_on_power_law_graphs(L, ctx, graphs, name):
    """Heavy rows (hubs split over many segments) are reduced in segment order,
    so SpMM and the whole embedding are bitwise repeatable."""
    n, s, t, g, (rp, col, deg) = graphs[name]
    assert deg.max() > 128                      # several heavy segments per hub
    X = padded(n, 286)
    X.copy_(torch.randn(n, 286, device=DEV))
    Y1, Y2 = padded(n, 286), padded(n, 286)
    L.netmfp_spmm(ctx, g, 0.45, 0.45, X, Y1)
    L.netmfp_spmm(ctx, g, 0.45, 0.45, X, Y2)
    assert torch.equal(Y1, Y2)
    L.netmfp_spmm(ctx, g, 0.45, 0.0, X, Y1)
    L.netmfp_spmm(ctx, g, 0.45, 0.0, X, Y2)
    assert torch.equal(Y1, Y2)
    prm = L.make_params(alpha=0.45, k=32, s1=10, q=3, T=10, b=1.0, d=16, s2=16, s3=160, z=8, prop_order=10,
                        mu=0.2, theta=0.5, seed=5, logmode=0)
    outs = []
    for _ in range(2):
        E = padded(n, 16)
        sig = torch.zeros(16, dtype=torch.float64, device=DEV)
        lam = torch.zeros(32, dtype=torch.float64, device=DEV)
        L.netmfp_embed(ctx, g, prm, E, sig, lam)
        outs.append((E, sig, lam))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_dist_nccl_path_with_one_rank(L, ctx, graphs):
    """The NCCL code path itself (per-slice all-gathers on the communicator's
    stream overlapping the SpMM passes, all-reduces, degree all-gather and
    compaction of the partition) executed with a one-rank communicator
    (NETMFP_DIST_FORCE_COMM=1): bitwise the single-GPU result."""
    import os
    n, s, t, g, (rp, col, deg) = graphs["rmat_s13"]
    os.environ["NETMFP_DIST_FORCE_COMM"] = "1"
    try:
        c1 = L.Context(0)
        L.netmfp_dist_init(c1, L.netmfp_dist_unique_id(), 1, 0)
    finally:
        del os.environ["NETMFP_DIST_FORCE_COMM"]
    gd = L.netmfp_dist_build_csr(c1, n, dev(s), dev(t))
    prm = L.make_params(alpha=0.45, k=40, s1=16, q=2, T=10, b=1.0, d=24, s2=24, s3=150, z=8, prop_order=6,
                        mu=0.2, theta=0.5, seed=3, logmode=0)
    E1, E2 = padded(n, 24), padded(n, 24)
    s1, s2 = torch.zeros(24, dtype=torch.float64, device=DEV), torch.zeros(24, dtype=torch.float64, device=DEV)
    L.netmfp_embed(ctx, g, prm, E1, s1)
    L.netmfp_dist_stats(c1)
    L.netmfp_embed(c1, gd, prm, E2, s2)
    nbytes, ncoll = L.netmfp_dist_stats(c1)
    assert ncoll > 0                      # the collectives were issued
    assert torch.equal(s1, s2) and torch.equal(E1, E2)
