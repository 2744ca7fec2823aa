"""Where the stream is idle between kernels in one configs[2] embedding
(NETMFP_PROF_GAPS=1: gap before each kernel, attributed to that kernel)."""
import os, sys
os.environ["NETMFP_PROF_GAPS"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2110_12782_b200 import _lib as L, inputs
w = inputs.CONFIGS[2]
n, s, t = inputs.make_graph(w.graph)
src, dst = torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda()
ctx = L.Context(0)
prm = L.make_params(**w.params())
E = torch.zeros(n, 128, device="cuda")
for _ in range(3):
    L.netmfp_embed_edges(ctx, n, src, dst, prm, E)
ctx.profile(True, "")
L.netmfp_embed_edges(ctx, n, src, dst, prm, E)
pr = ctx.profile_read()
ctx.profile(False)
gaps = sorted(((k, v) for k, v in pr.items() if k.startswith("gap")), key=lambda x: -x[1][1])
kern = sum(v[1] for k, v in pr.items() if not k.startswith("gap") and not k.startswith("stage_"))
print(f"kernels total {kern:.3f} ms; stages: " + ", ".join(f"{k[6:]} {v[1]:.2f}" for k, v in pr.items() if k.startswith("stage_")))
for k, (cnt, ms) in gaps[:25]:
    print(f"{k:40s} {cnt:5d} {ms:8.3f} ms")
