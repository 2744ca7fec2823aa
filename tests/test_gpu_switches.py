"""The A/B switches of the library must not change what is computed:
programmatic dependent launch (NETMFP_PDL) only changes when a kernel's launch
is processed, so an embedding is bitwise identical with and without it; the
fp16-split sketches (NETMFP_SKETCH_F16, default) and the 3xTF32 ones are two
~22-bit evaluations of the same Eq. 5 sums, within the sketch tolerance of
each other (1e-4 relative Frobenius, north_star); the tall GEMM's item order
(NETMFP_GEMM_TRI_ORDER: which CTA computes which output tile) cannot change
any tile's arithmetic, so CholeskyQR output is bitwise identical; running
Alg. 4's Z sketch on the side stream (NETMFP_SIDE_STREAM) only changes when
it runs, so the embedding is bitwise identical.  Each setting runs in its
own process (the switches are read once per process)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
import __graft_entry__ as ge
ge.build()
from paper_2110_12782_b200 import _lib as L, inputs
n, s, t = inputs.small_graph("rmat", 1 << 14, 3, edge_factor=6)
ctx = L.Context(0)
g = L.netmfp_build_csr(ctx, n, torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda())
prm = dict(alpha=0.45, k=96, s1=16, q=3, T=10, b=1.0, d=48, s2=40, s3=400, z=8, prop_order=10, mu=0.2, theta=0.5,
           seed=11, logmode=0)
E = torch.zeros(n, 64, dtype=torch.float32, device="cuda")[:, :48]
sig = torch.zeros(48, dtype=torch.float64, device="cuda")
lam = torch.zeros(96, dtype=torch.float64, device="cuda")
L.netmfp_embed(ctx, g, L.make_params(**prm), E, sig, lam)
# the Alg. 4 sketches on a fixed F, C (the embedding's own factor pair)
Ud = torch.zeros(n, 96, dtype=torch.float32, device="cuda")
lam2 = torch.zeros(96, dtype=torch.float64, device="cuda")
L.netmfp_eig(ctx, g, 0.45, 96, 16, 3, 11, Ud, lam2)
F = torch.zeros(n, 96, dtype=torch.float32, device="cuda")
C = torch.zeros(96, 96, dtype=torch.float64, device="cuda")
L.netmfp_factor_pair(ctx, g, 0.45, 10, Ud, lam2, F, C)
Y = torch.zeros(n, 96, dtype=torch.float32, device="cuda")[:, :88]
Z = torch.zeros(440, 440, dtype=torch.float64, device="cuda")
sg2 = torch.zeros(48, dtype=torch.float64, device="cuda")
L.netmfp_sketch_svd(ctx, F, C, float(g.nnz) / 10.0, 48, 40, 400, 8, 11, 0, sigma=sg2, Ysk=Y, Zsk=Z)
torch.cuda.synchronize()
np.savez(OUT, E=E.cpu().numpy(), sig=sig.cpu().numpy(), lam=lam.cpu().numpy(), Y=Y.cpu().numpy(),
         Z=Z.cpu().numpy())
'''


def run(tmp_path, tag, env):
    out = str(tmp_path / f"{tag}.npz")
    code = f"ROOT = {ROOT!r}\nOUT = {out!r}\n" + CHILD
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return dict(np.load(out))


def relf(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_pdl_is_bitwise_neutral(tmp_path):
    on = run(tmp_path, "pdl1", {"NETMFP_PDL": "1"})
    off = run(tmp_path, "pdl0", {"NETMFP_PDL": "0"})
    for key in on:
        assert np.array_equal(on[key], off[key]), key


def test_side_stream_is_bitwise_neutral(tmp_path):
    on = run(tmp_path, "side1", {"NETMFP_SIDE_STREAM": "1"})
    off = run(tmp_path, "side0", {"NETMFP_SIDE_STREAM": "0"})
    for key in on:
        assert np.array_equal(on[key], off[key]), key


def test_fp16_split_sketch_matches_3xtf32(tmp_path):
    h = run(tmp_path, "f16", {"NETMFP_SKETCH_F16": "1"})
    t = run(tmp_path, "tf32", {"NETMFP_SKETCH_F16": "0"})
    assert relf(h["Y"], t["Y"]) <= 1e-4, relf(h["Y"], t["Y"])
    assert relf(h["Z"], t["Z"]) <= 1e-4, relf(h["Z"], t["Z"])
    # the eigen side (Alg. 2) does not use the sketch: identical
    assert np.array_equal(h["lam"], t["lam"])


GEMM_CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
import __graft_entry__ as ge
ge.build()
from paper_2110_12782_b200 import _lib as L
ctx = L.Context(0)
n, c = 50001, 286  # two column parts of the triangular R^-1 GEMM, ragged last M tile
Yh = (np.random.default_rng(7).standard_normal((n, c)) * np.logspace(0, 2, c)[None, :]).astype(np.float32)
Y = torch.zeros(n, 288, dtype=torch.float32, device="cuda")[:, :c]
Y.copy_(torch.from_numpy(Yh))
outs = {}
for passes in (1, 2):
    Q = torch.zeros(n, 288, dtype=torch.float32, device="cuda")[:, :c]
    L.netmfp_orthonormalize(ctx, Y, Q, passes)
    outs[f"Q{passes}"] = Q.cpu().numpy()
torch.cuda.synchronize()
np.savez(OUT, **outs)
'''


def test_gemm_item_order_is_bitwise_neutral(tmp_path):
    res = {}
    for order in ("0", "1"):
        out = str(tmp_path / f"gemm{order}.npz")
        code = f"ROOT = {ROOT!r}\nOUT = {out!r}\n" + GEMM_CHILD
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, NETMFP_GEMM_TRI_ORDER=order),
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        res[order] = dict(np.load(out))
    for key in res["0"]:
        assert np.array_equal(res["0"][key], res["1"][key]), key
    q = res["0"]["Q2"].astype(np.float64)
    assert np.abs(q.T @ q - np.eye(q.shape[1])).max() <= 1e-4
