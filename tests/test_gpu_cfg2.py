"""GPU parity on BASELINE.json configs[2] — the workload bench.py times —
at full size and full parameters, against the fp64 oracle's Alg. 5 stored by
scripts/oracle_cfg2.py (tests/golden/cfg2_oracle.npz; oracle-only, nothing
from the CUDA path).

Two GPU routes are checked: the ABI chain netmfp_eig -> netmfp_factor_pair ->
netmfp_sketch_svd (exposes the Alg. 4 sketches Y, Z) -> netmfp_propagate on the
uncompacted graph, and netmfp_embed (the bench's route: isolated vertices
compacted out).

Tolerances (north_star; "leading" = sigma_j >= 1e-2 sigma_1):
eigenvalues as a sorted multiset (Alg. 2 step 10, [R3]) 1e-3 |lambda_1|; Eq. 3's
M = F C F^T 1e-4; with identical inputs (the oracle's F, C) the sketches Y, Z
1e-4 relative Frobenius and the leading singular values 1e-3 sigma_1.  Through
the whole chain, sigma and E are held to the measured conditioning of Alg. 4 at
this input (see test_cfg2_leading_singular_values)."""
import os

import numpy as np
import pytest

from paper_2110_12782_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg2_oracle.npz")
DEV = "cuda:0"


def relf(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def padded(n, c, dtype=torch.float32):
    return torch.zeros(n, (c + 31) // 32 * 32, dtype=dtype, device=DEV)[:, :c]


def separated(sig, rel=0.01):
    out = []
    for j in range(len(sig)):
        hi = sig[j - 1] if j > 0 else np.inf
        lo = sig[j + 1] if j + 1 < len(sig) else -np.inf
        if hi - sig[j] > rel * sig[j] and sig[j] - lo > rel * sig[j]:
            out.append(j)
    return out


def cols_up_to_sign(E, R, cols):
    worst = 0.0
    for j in cols:
        r = np.linalg.norm(R[:, j])
        worst = max(worst, min(np.linalg.norm(E[:, j] - R[:, j]), np.linalg.norm(E[:, j] + R[:, j])) / r)
    return worst


@pytest.fixture(scope="module")
def gold():
    import oracle as O
    gd = dict(np.load(GOLD))
    w = inputs.CONFIGS[2]
    n, s, t = inputs.make_graph(w.graph)
    _, _, deg = O.build_csr(n, s, t)
    gd["iso_in_rows"] = np.flatnonzero(deg[gd["rows"]] == 0)
    return gd


@pytest.fixture(scope="module")
def run(gold):
    return run_cfg2(gold["rows"])


def run_cfg2(rows, extra=False):
    """Both GPU routes on configs[2]; outputs on the sampled rows."""
    import __graft_entry__ as ge
    ge.build()
    from paper_2110_12782_b200 import _lib as L
    w = inputs.CONFIGS[2]
    p = w.params()
    n, s, t = inputs.make_graph(w.graph)
    ctx = L.Context(0)
    g = L.netmfp_build_csr(ctx, n, torch.from_numpy(s).to(DEV), torch.from_numpy(t).to(DEV))
    out = {}
    # the bench's route
    E = padded(n, p["d"])
    sig = torch.zeros(p["d"], dtype=torch.float64, device=DEV)
    lam = torch.zeros(p["k"], dtype=torch.float64, device=DEV)
    L.netmfp_embed(ctx, g, L.make_params(**p), E, sig, lam)
    out["embed"] = dict(lam=lam.cpu().numpy(), sigma=sig.cpu().numpy(), E_rows=E.cpu().numpy()[rows])
    del E
    # the ABI chain (uncompacted graph), exposing the sketches
    k, d, h2, h3 = p["k"], p["d"], p["d"] + p["s2"], p["d"] + p["s3"]
    U = padded(n, k)
    lam2 = torch.zeros(k, dtype=torch.float64, device=DEV)
    L.netmfp_eig(ctx, g, p["alpha"], k, p["s1"], p["q"], p["seed"], U, lam2)
    F = padded(n, k)
    C = torch.zeros(k, k, dtype=torch.float64, device=DEV)
    L.netmfp_factor_pair(ctx, g, p["alpha"], p["T"], U, lam2, F, C)
    del U
    # basis-free Eq. 3 samples M = F C F^T on rows[:1024] x rows[:256]
    Fr = F.cpu().numpy()[rows[:1024]].astype(np.float64)
    out["M_rows"] = Fr @ C.cpu().numpy() @ Fr[:256].T
    scale = g.nnz / (p["b"] * p["T"])
    Ysk = padded(n, h2)
    Zsk = torch.zeros(h3, h3, dtype=torch.float64, device=DEV)
    sig2 = torch.zeros(d, dtype=torch.float64, device=DEV)
    E2 = padded(n, d)
    L.netmfp_sketch_svd(ctx, F, C, scale, d, p["s2"], p["s3"], p["z"], p["seed"], p["logmode"], sigma=sig2, E=E2,
                        Ysk=Ysk, Zsk=Zsk)
    del F
    Eraw = E2.cpu().numpy()[rows]
    L.netmfp_propagate(ctx, g, E2, p["prop_order"], p["mu"], p["theta"])
    Yg = Ysk.cpu().numpy()
    out["chain"] = dict(lam=lam2.cpu().numpy(), sigma=sig2.cpu().numpy(), Y_rows=Yg[rows],
                        Y_fro=np.linalg.norm(Yg.astype(np.float64)), Z=Zsk.cpu().numpy(), E_raw_rows=Eraw,
                        E_rows=E2.cpu().numpy()[rows])
    return out


@pytest.mark.parametrize("route", ["embed", "chain"])
def test_cfg2_eigenvalues(run, gold, route):
    """Alg. 2 (freigs) Ritz values, as a sorted multiset: 1e-3 |lambda_1|."""
    lg = np.sort(run[route]["lam"])
    lo = np.sort(gold["lam"])
    assert np.abs(lg - lo).max() <= 1e-3 * abs(gold["lam"][0])


def test_cfg2_eq3_product(run, gold):
    """Eq. 3 M = F C F^T (Alg. 5 steps 1-3) on sampled entries: basis-free,
    so it checks the whole rank-k factorisation, 1e-4 relative Frobenius."""
    assert relf(run["M_rows"], gold["M_rows"]) <= 1e-4


def test_cfg2_chain_sketches(run, gold):
    """Y and Z from the GPU's own F and C.  At this input Alg. 2 truncates at a
    Ritz gap of 4.4e-4 (|lambda_256| - |lambda_257|), so the fp32 eigenvectors
    next to the cut mix at ~1e-2 and the sketches inherit ~1e-4 from that
    (DESIGN.md §5); the sketch kernels themselves are held to 1e-4 on
    identical inputs by test_cfg2_sketch_same_inputs."""
    assert relf(run["chain"]["Y_rows"], gold["Y_rows"]) <= 1e-3
    assert abs(run["chain"]["Y_fro"] - float(gold["Y_fro"])) <= 1e-4 * float(gold["Y_fro"])
    zero = gold["zero_cols_Y"]          # Psi columns that drew only isolated vertices [R10]
    assert len(zero) > 0 and np.all(run["chain"]["Y_rows"][:, zero] == 0.0)
    Z = run["chain"]["Z"]
    assert relf(Z[gold["zrows"]], gold["Z_rows"]) <= 1e-3
    assert abs(np.linalg.norm(Z) - float(gold["Z_fro"])) <= 1e-4 * float(gold["Z_fro"])


@pytest.mark.parametrize("route", ["embed", "chain"])
def test_cfg2_leading_singular_values(run, gold, route):
    """Leading sigma (>= 1e-2 sigma_1) of the whole chain.  Alg. 4 is
    ill-conditioned at this input (Y has 3 zero columns and cond 6.8e4 on the
    rest): the oracle's own sigma moves by sens_sigma (1-3% of sigma_1) when its
    Y is perturbed by 1e-5 relative (scripts/oracle_cfg2.py), so the chain's
    sigma is held to that conditioning bound; with identical inputs the GPU's
    Alg. 4 meets 1e-3 (test_cfg2_sketch_same_inputs)."""
    so = gold["sigma"]
    lead = so >= 1e-2 * so[0]
    assert lead.sum() >= 8
    sg = run[route]["sigma"]
    assert np.abs(sg[lead] - so[lead]).max() <= float(gold["sens_sigma"]) * so[0]


@pytest.mark.parametrize("route,key", [("chain", "E_raw_rows"), ("chain", "E_rows"), ("embed", "E_rows")])
def test_cfg2_embedding(run, gold, route, key):
    """E = U sqrt(Sigma) (Alg. 5 step 5) and after propagation (step 6) on the
    sampled rows, basis-free (E E^T), within the conditioning bound; isolated
    vertices have exactly zero rows [R2]."""
    Eg = run[route][key].astype(np.float64)
    Eo = gold[key].astype(np.float64)
    print(route, key, "E E^T relF", relf(Eg @ Eg.T, Eo @ Eo.T))
    assert relf(Eg @ Eg.T, Eo @ Eo.T) <= 2.0 * float(gold["sens_sigma"])
    iso = gold["iso_in_rows"]
    assert len(iso) > 0 and np.all(run[route][key][iso] == 0.0)


@pytest.mark.slow
def test_cfg2_sketch_same_inputs(gold):
    """Alg. 4 on configs[2] with the ORACLE's F and C (fp64 Alg. 2 + Eq. 3 at
    full size, ~2-3 min of host CPU; F rounded to fp32 as the GPU block holds
    it): the sketches Y (sampled rows + norm) and Z at 1e-4 relative
    Frobenius, as north_star states for sketch outputs."""
    import oracle as O
    from paper_2110_12782_b200 import _lib as L
    w = inputs.CONFIGS[2]
    p = w.params()
    n, s, t = inputs.make_graph(w.graph)
    rp, col, deg = O.build_csr(n, s, t)
    U, lam = O.freigs(lambda M: O.normalized_spmm(rp, col, deg, M, p["alpha"]), n, p["k"], p["s1"], p["q"], p["seed"])
    _, F, C = O.factor_pair(U, lam, deg, p["alpha"], p["T"])
    del U
    F32 = F.astype(np.float32)
    F64 = F32.astype(np.float64)
    del F
    k, d, h2, h3, z, seed = p["k"], p["d"], p["d"] + p["s2"], p["d"] + p["s3"], p["z"], p["seed"]
    scale = col.size / (p["b"] * p["T"])
    ctx = L.Context(0)
    Fd = padded(n, k)
    Fd.copy_(torch.from_numpy(F32).to(DEV))
    Ysk = padded(n, h2)
    Zsk = torch.zeros(h3, h3, dtype=torch.float64, device=DEV)
    sig = torch.zeros(d, dtype=torch.float64, device=DEV)
    L.netmfp_sketch_svd(ctx, Fd, torch.from_numpy(C).to(DEV), scale, d, p["s2"], p["s3"], z, seed, p["logmode"],
                        sigma=sig, Ysk=Ysk, Zsk=Zsk)
    rows = gold["rows"]
    Yg = Ysk.cpu().numpy()
    r_psi, sg_psi, p_psi = O.gen_sparse_sign(n, h2, z, seed, O.TAG_PSI)
    Yo = O.sketch_y(F64, C, scale, r_psi, sg_psi, p_psi, p["logmode"])
    r_pi, sg_pi, p_pi = O.gen_sparse_sign(n, h3, z, seed, O.TAG_PI)
    Zo = O.sketch_z(F64, C, scale, r_pi, sg_pi, p_pi, p["logmode"])
    Q = O.orth_range(Yo)
    Sc = O.core_solve(O.sparse_sign_apply_T(r_pi, sg_pi, Q), Zo)
    so = np.linalg.svd(Sc, compute_uv=False)[:d]
    sg = sig.cpu().numpy()
    lead = so >= 1e-2 * so[0]
    print("cfg2 same-input sketch: Y relF", relf(Yg, Yo), "rows", relf(Yg[rows], Yo[rows]),
          "Z relF", relf(Zsk.cpu().numpy(), Zo), "sigma lead err/sigma1", np.abs(sg - so)[lead].max() / so[0],
          "sigma lead8", (np.abs(sg - so) / so[0])[:8])
    assert relf(Yg, Yo) <= 1e-4
    assert relf(Zsk.cpu().numpy(), Zo) <= 1e-4
    assert np.abs(sg - so)[lead].max() <= 1e-3 * so[0]
