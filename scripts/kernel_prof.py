"""Per-kernel CUDA-event times of one configs[2] embedding (all launches profiled)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2110_12782_b200 import _lib as L, inputs
w = inputs.CONFIGS[int(os.environ.get("CFG", "2"))]
n, s, t = inputs.make_graph(w.graph)
src, dst = torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda()
ctx = L.Context(0)
prm = L.make_params(**w.params())
E = torch.zeros(n, (w.d + 31) // 32 * 32, device="cuda")[:, :w.d]
sig = torch.zeros(w.d, dtype=torch.float64, device="cuda")
for _ in range(3):
    L.netmfp_embed_edges(ctx, n, src, dst, prm, E, sig)
torch.cuda.synchronize()
reps = 3
ctx.profile(True, os.environ.get("FILTER", ""))
for _ in range(reps):
    L.netmfp_embed_edges(ctx, n, src, dst, prm, E, sig)
pr = ctx.profile_read()
ctx.profile(False)
for k, v in sorted(pr.items(), key=lambda x: -x[1][1]):
    print(f"{v[1] / reps:9.4f} ms  {v[0] // reps:4d}x  {k}")
