"""3xTF32 Gram max relative error at the configs[2] block shape (n x 286) against an fp64 product."""
import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2110_12782_b200 import _lib as L
ctx = L.Context(0)
for n in (406727, 1048576):
    for dist in ("normal", "positive"):
        rng = np.random.default_rng(1)
        A = rng.standard_normal((n, 286)).astype(np.float32)
        if dist == "positive": A = np.abs(A)
        Ad = torch.zeros(n, 288, device="cuda")[:, :286]; Ad.copy_(torch.from_numpy(A))
        G = torch.zeros(286, 286, dtype=torch.float64, device="cuda")
        L.netmfp_gram(ctx, Ad, Ad, G)
        Ac = torch.from_numpy(A).double().cuda()
        ref = (Ac.T @ Ac).cpu().numpy()
        print(n, dist, "max rel err", float(np.abs(G.cpu().numpy() - ref).max() / np.abs(ref).max()))
