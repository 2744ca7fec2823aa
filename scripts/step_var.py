"""Step-time variance probe: 15 embeddings of configs[2], per-step events and wall time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_12782_b200 import _lib as L, inputs
w = inputs.CONFIGS[2]
n, s, t = inputs.make_graph(w.graph)
ctx = L.Context(0)
src, dst = torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda()
prm = L.make_params(**w.params())
E = torch.zeros(n, 128, device="cuda")
sig = torch.zeros(128, device="cuda", dtype=torch.float64)
st = torch.cuda.current_stream()
for i in range(15):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record(st)
    if i == 8:
        ctx.profile(True, "stage_")
    L.netmfp_embed_edges(ctx, n, src, dst, prm, E, sig)
    e1.record(st)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - w0) * 1e3
    extra = ""
    if i == 8:
        extra = str({k: round(v[1], 2) for k, v in ctx.profile_read().items()})
        ctx.profile(False)
    print(f"step {i}: gpu {e0.elapsed_time(e1):.2f} ms wall {wall:.2f} ms {extra}", flush=True)
