"""Diagnose tcgen05 3xTF32 Gram accuracy vs K (rows) — tuning aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2110_12782_b200 import _lib as L
ctx = L.Context(0)
for dist in ("normal", "positive"):
    for n in (128, 512, 2048, 8192, 32768, 131072):
        rng = np.random.default_rng(n)
        A = rng.standard_normal((n, 64)).astype(np.float32)
        if dist == "positive":
            A = np.abs(A)
        Ad = torch.zeros(n, 64, device="cuda"); Ad.copy_(torch.from_numpy(A))
        G = torch.zeros(64, 64, dtype=torch.float64, device="cuda")
        L.netmfp_gram(ctx, Ad, Ad, G)
        ref = A.astype(np.float64).T @ A.astype(np.float64)
        err = np.abs(G.cpu().numpy() - ref)
        rel_diag = (err.diagonal() / np.abs(ref.diagonal())).max()
        bias = ((G.cpu().numpy() - ref).diagonal() / ref.diagonal()).mean()
        print(f"{dist:8s} n={n:7d} max_rel_diag={rel_diag:.2e} mean_rel_bias={bias:+.2e} max_abs/max={err.max()/np.abs(ref).max():.2e}")
