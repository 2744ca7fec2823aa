"""One netmfp_spmm on configs[2] at n x cols (for ncu captures)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2110_12782_b200 import _lib as L, inputs
cols = int(sys.argv[1]) if len(sys.argv) > 1 else 286
w = inputs.CONFIGS[2]
n, s, t = inputs.make_graph(w.graph)
ctx = L.Context(0)
g = L.netmfp_build_csr(ctx, n, torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda())
ld = (cols + 31) // 32 * 32
X = torch.randn(n, ld, device="cuda")[:, :cols]
Y = torch.zeros(n, ld, device="cuda")[:, :cols]
for _ in range(3):
    L.netmfp_spmm(ctx, g, 0.45, 0.0, X, Y)
torch.cuda.synchronize()
print("ok", n, g.nnz, g.n_heavy)
