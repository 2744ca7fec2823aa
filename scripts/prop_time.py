"""Time netmfp_propagate (10 Clenshaw SpMMs on n' x 128) and a plain 286-column
SpMM on the compacted configs[2] graph (CUDA events, mean of 10 after warm-up)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2110_12782_b200 import _lib as L, inputs
n, s, t = inputs.make_graph(inputs.CONFIGS[2].graph)
keep = np.zeros(n, bool)
keep[s] = True
keep[t] = True
m = np.cumsum(keep) - 1
n, s, t = int(keep.sum()), m[s].astype(np.int32), m[t].astype(np.int32)
ctx = L.Context(0)
g = L.netmfp_build_csr(ctx, n, torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda())
E = torch.randn(n, 128, device="cuda")
for _ in range(3):
    L.netmfp_propagate(ctx, g, E, 10, 0.2, 0.5)
ctx.profile(True, "spmm")
for _ in range(10):
    L.netmfp_propagate(ctx, g, E, 10, 0.2, 0.5)
pr = ctx.profile_read()
ctx.profile(False)
out = {"propagate_spmm_ms": round(sum(v[1] for v in pr.values()) / 10, 4)}
X = torch.randn(n, 288, device="cuda")[:, :286]
Y = torch.zeros(n, 288, device="cuda")[:, :286]
for _ in range(3):
    L.netmfp_spmm(ctx, g, 0.45, 0.0, X, Y)
ctx.profile(True, "spmm")
for _ in range(10):
    L.netmfp_spmm(ctx, g, 0.45, 0.0, X, Y)
pr = ctx.profile_read()
ctx.profile(False)
out["spmm286_ms"] = round(sum(v[1] for v in pr.values()) / 10, 4)
print(json.dumps(out))
