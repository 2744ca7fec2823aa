"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the NetMF+ method (§4): it only
draws graphs (edge lists) and names the parameter sets of BASELINE.json's
configs.  Random numbers the *method* draws (the Gaussian test matrix of
Alg. 2 and the sparse-sign matrices of Alg. 3) are NOT generated here: the
CUDA library and ``oracle/`` each implement the same counter-based
generator (Philox4x32-10) independently; see DESIGN.md §3.

Graph recipes (DESIGN.md §4 "input recipe"):
  * ``er_graph``      Erdős–Rényi G(n, p), p = avg_deg/(n-1)      (configs[0])
  * ``chung_lu``      Chung–Lu expected-degree power law, exponent gamma,
                      max expected degree, exactly m unique edges   (configs[1];
                      BlogCatalog's n=10,312 / m=333,983, Table 2)
  * ``rmat``          R-MAT(a,b,c,d) recursive quadrant sampling, edge factor,
                      dedup + self-loop removal left to build_csr  (configs[2..4])

Every generator returns an *undirected, unprocessed* edge list (src, dst) as
int32 arrays; symmetrisation, deduplication and self-loop removal are the job
of ``netmfp_build_csr`` (and of ``oracle.build_csr``).
"""
from __future__ import annotations

from dataclasses import dataclass, field, asdict
import numpy as np


# --------------------------------------------------------------------------
# graph generators
# --------------------------------------------------------------------------

def er_graph(n: int, avg_deg: float, seed: int):
    """G(n, p) with p = avg_deg / (n - 1): every unordered pair independently.

    Exact Bernoulli sampling over the strict upper triangle (n <= ~20k)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    p = avg_deg / (n - 1)
    src_all, dst_all = [], []
    # row blocks of the upper triangle to bound memory
    blk = max(1, 4_000_000 // max(n, 1))
    for i0 in range(0, n, blk):
        i1 = min(n, i0 + blk)
        rows = np.arange(i0, i1)
        mask = rng.random((i1 - i0, n)) < p
        mask &= (np.arange(n)[None, :] > rows[:, None])
        r, c = np.nonzero(mask)
        src_all.append((r + i0).astype(np.int32))
        dst_all.append(c.astype(np.int32))
    return np.concatenate(src_all), np.concatenate(dst_all)


def _chung_lu_weights(n: int, m: int, gamma: float, max_deg: float):
    """Expected degrees w_i = c (i + i0)^(-1/(gamma-1)), i = 0..n-1, with
    w_0 = max_deg and sum_i w_i = 2m (i0 found by bisection)."""
    beta = 1.0 / (gamma - 1.0)
    idx = np.arange(n, dtype=np.float64)

    def total(i0):
        w = max_deg * ((idx + i0) / i0) ** (-beta)
        return w.sum()

    lo, hi = 1e-6, 1e9
    for _ in range(200):
        mid = np.sqrt(lo * hi)
        if total(mid) < 2 * m:
            lo = mid
        else:
            hi = mid
    i0 = np.sqrt(lo * hi)
    return max_deg * ((idx + i0) / i0) ** (-beta)


def chung_lu(n: int, m: int, gamma: float, max_deg: float, seed: int):
    """Chung–Lu graph with exactly m unique undirected edges (no self loops).

    Endpoints are drawn i.i.d. proportional to the expected degrees; candidate
    edges are canonicalised (min, max), self loops dropped, duplicates removed
    keeping first occurrence, until m unique edges exist (generation order)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    w = _chung_lu_weights(n, m, gamma, max_deg)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    keys = np.empty(0, dtype=np.int64)
    while keys.size < m:
        need = m - keys.size
        batch = int(need * 1.3) + 1024
        u = np.searchsorted(cdf, rng.random(batch), side="right")
        v = np.searchsorted(cdf, rng.random(batch), side="right")
        u = np.minimum(u, n - 1)
        v = np.minimum(v, n - 1)
        ok = u != v
        a = np.minimum(u, v)[ok].astype(np.int64)
        b = np.maximum(u, v)[ok].astype(np.int64)
        cand = np.concatenate([keys, a * n + b])
        _, first = np.unique(cand, return_index=True)
        first.sort()
        keys = cand[first]
    keys = keys[:m]
    return (keys // n).astype(np.int32), (keys % n).astype(np.int32)


def rmat(scale: int, edge_factor: int, a: float, b: float, c: float, seed: int,
         chunk: int = 1 << 22):
    """R-MAT: edge_factor * 2^scale directed draws, each choosing one of the
    four adjacency quadrants with probabilities (a, b, c, 1-a-b-c) at every
    one of `scale` bit levels (most significant first).  No noise, no vertex
    permutation (BASELINE.json states neither).  Duplicates and self loops are
    kept: build_csr removes them."""
    rng = np.random.Generator(np.random.PCG64(seed))
    total = edge_factor * (1 << scale)
    ab, abc = a + b, a + b + c
    srcs, dsts = [], []
    for s0 in range(0, total, chunk):
        cnt = min(chunk, total - s0)
        u = np.zeros(cnt, dtype=np.int64)
        v = np.zeros(cnt, dtype=np.int64)
        for lvl in range(scale):
            r = rng.random(cnt)
            bit = 1 << (scale - 1 - lvl)
            down = r >= ab                      # quadrants c, d: source bit set
            right = ((r >= a) & (r < ab)) | (r >= abc)   # quadrants b, d
            u |= np.where(down, bit, 0)
            v |= np.where(right, bit, 0)
        srcs.append(u.astype(np.int32))
        dsts.append(v.astype(np.int32))
    return np.concatenate(srcs), np.concatenate(dsts)


# --------------------------------------------------------------------------
# BASELINE.json configs (parameters the paper leaves open are filled from
# PAPER.md §5.2's classification preset; DESIGN.md §4 lists each choice)
# --------------------------------------------------------------------------

@dataclass
class Workload:
    name: str
    graph: dict                  # generator + args
    alpha: float = 0.45          # PAPER.md §5.4: alpha in [0.35, 0.5); OAG used 0.45
    k: int = 256                 # eigen rank (BASELINE.json calls it "h")
    s1: int = 30                 # §5.2 "s1=30"
    q: int = 4                   # power iterations
    T: int = 10                  # window
    b: float = 1.0               # negative samples
    d: int = 128                 # embedding dim
    s2: int = 100                # §5.2 "s2 = 100"
    s3: int = 1000               # §5.2 "s3 = 1000"
    z: int = 8                   # §4.2 "z = min(n, 8)"
    prop_order: int = 10         # §3 ProNE "the default setting is 10"
    mu: float = 0.2
    theta: float = 0.5
    seed: int = 0
    logmode: int = 0             # 0 = trunc_log (Eq. 1), 1 = log1p
    n_gpus: int = 1

    def params(self) -> dict:
        d = asdict(self)
        d.pop("graph")
        d.pop("name")
        d.pop("n_gpus")
        return d


CONFIGS = {
    0: Workload("er_n4096_deg16", dict(kind="er", n=4096, avg_deg=16, seed=0),
                k=128, q=2, d=32),
    1: Workload("chunglu_n10312_m333983", dict(kind="chung_lu", n=10312, m=333983,
                gamma=2.1, max_deg=3000, seed=1), k=256, q=4, d=128),
    2: Workload("rmat_s20_ef3", dict(kind="rmat", scale=20, edge_factor=3,
                a=0.57, b=0.19, c=0.19, seed=2), k=256, q=6, d=128),
    3: Workload("rmat_s26_ef28", dict(kind="rmat", scale=26, edge_factor=28,
                a=0.57, b=0.19, c=0.19, seed=3), k=256, q=6, d=128, n_gpus=8),
    4: Workload("rmat_s27_ef32", dict(kind="rmat", scale=27, edge_factor=32,
                a=0.57, b=0.19, c=0.19, seed=4), k=128, q=6, d=128, n_gpus=8),
}


def make_graph(spec: dict):
    """Return (n, src, dst) for a graph spec from CONFIGS."""
    kind = spec["kind"]
    if kind == "er":
        s, t = er_graph(spec["n"], spec["avg_deg"], spec["seed"])
        return spec["n"], s, t
    if kind == "chung_lu":
        s, t = chung_lu(spec["n"], spec["m"], spec["gamma"], spec["max_deg"], spec["seed"])
        return spec["n"], s, t
    if kind == "rmat":
        s, t = rmat(spec["scale"], spec["edge_factor"], spec["a"], spec["b"], spec["c"],
                    spec["seed"])
        return 1 << spec["scale"], s, t
    raise ValueError(kind)


def small_graph(kind: str, n: int, seed: int, **kw):
    """Tiny graphs for parity edge cases (ragged sizes, hubs, isolated vertices)."""
    if kind == "er":
        return (n,) + er_graph(n, kw.get("avg_deg", 6.0), seed)
    if kind == "star":                       # one hub of degree n-1
        s = np.zeros(n - 1, dtype=np.int32)
        t = np.arange(1, n, dtype=np.int32)
        return n, s, t
    if kind == "rmat":
        sc = int(np.ceil(np.log2(n)))
        s, t = rmat(sc, kw.get("edge_factor", 4), 0.57, 0.19, 0.19, seed)
        return 1 << sc, s, t
    raise ValueError(kind)


def rmat_device(scale: int, edge_factor: int, a: float, b: float, c: float, seed: int, device,
                chunk: int = 1 << 26):
    """The R-MAT recipe of `rmat` (same quadrant rule, most significant bit
    first, no noise, no permutation, duplicates and self loops kept) drawn on a
    GPU with torch's generator — for the billion-edge configs[3]/[4], where
    host numpy generation would take hours.  A different random stream than
    `rmat`: the same graph distribution, not the same graph.  Returns int32
    (src, dst) tensors on `device`; every rank calling it with the same seed
    gets the same edge list."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    total = edge_factor * (1 << scale)
    ab, abc = a + b, a + b + c
    src = torch.empty(total, dtype=torch.int32, device=device)
    dst = torch.empty(total, dtype=torch.int32, device=device)
    for s0 in range(0, total, chunk):
        cnt = min(chunk, total - s0)
        u = torch.zeros(cnt, dtype=torch.int32, device=device)
        v = torch.zeros(cnt, dtype=torch.int32, device=device)
        for lvl in range(scale):
            r = torch.rand(cnt, generator=g, device=device)
            bit = 1 << (scale - 1 - lvl)
            down = r >= ab
            right = ((r >= a) & (r < ab)) | (r >= abc)
            u |= down.to(torch.int32) * bit
            v |= right.to(torch.int32) * bit
        src[s0:s0 + cnt] = u
        dst[s0:s0 + cnt] = v
    return src, dst
