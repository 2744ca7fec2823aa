"""Device time of netmfp_embed_edges on a BASELINE config (no per-kernel profiling), L2 flushed between calls."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2110_12782_b200 import _lib as L, inputs
w = inputs.CONFIGS[int(os.environ.get("CFG", "2"))]
n, s, t = inputs.make_graph(w.graph)
src, dst = torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda()
ctx = L.Context(0)
prm = L.make_params(**w.params())
E = torch.zeros(n, (w.d + 31) // 32 * 32, device="cuda")[:, :w.d]
sig = torch.zeros(w.d, dtype=torch.float64, device="cuda")
flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
for _ in range(3):
    L.netmfp_embed_edges(ctx, n, src, dst, prm, E, sig)
reps = int(os.environ.get("REPS", "10"))
st = torch.cuda.current_stream()
ms = []
for _ in range(reps):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    L.netmfp_embed_edges(ctx, n, src, dst, prm, E, sig)
    b.record(st)
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
print(f"{os.environ.get('TAG', '')} embed ms: median {np.median(ms):.3f}  min {min(ms):.3f}  all {[round(x, 3) for x in ms]}")
