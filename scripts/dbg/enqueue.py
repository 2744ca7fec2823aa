"""Host enqueue time vs device time of one configs[2] embedding (NETMFP_DEBUG_ENQUEUE)."""
import os, sys, time
os.environ["NETMFP_DEBUG_ENQUEUE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2110_12782_b200 import _lib as L, inputs
w = inputs.CONFIGS[2]
n, s, t = inputs.make_graph(w.graph)
src, dst = torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda()
ctx = L.Context(0)
prm = L.make_params(**w.params())
E = torch.zeros(n, 128, device="cuda")
for i in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L.netmfp_embed_edges(ctx, n, src, dst, prm, E)
    print(f"call {i}: {(time.perf_counter() - t0) * 1e3:.3f} ms wall", file=sys.stderr)
