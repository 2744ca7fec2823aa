"""Idle stream time before each kernel of one configs[2] embedding (NETMFP_PROF_GAPS=1)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["NETMFP_PROF_GAPS"] = "1"
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
ctx.profile(True, "")
reps = 3
for _ in range(reps):
    L.netmfp_embed_edges(ctx, n, src, dst, prm, E, sig)
pr = ctx.profile_read()
ctx.profile(False)
gaps = sorted(((v[1] / reps, v[0] // reps, k) for k, v in pr.items() if k.startswith("gap>")), reverse=True)
print("total gaps ms/embedding", round(pr.get("gaps", (0, 0))[1] / reps, 4))
for ms, cnt, k in gaps[:25]:
    print(f"{ms:8.4f} ms  {cnt:4d}x  {k}")
