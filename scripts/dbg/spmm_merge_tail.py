import os, sys
sys.path.insert(0, "/root/repo")
import torch, numpy as np
from paper_2110_12782_b200 import _lib as L, inputs
w = inputs.CONFIGS[2]
n, s, t = inputs.make_graph(w.graph)
keep = np.zeros(n, bool); keep[s] = True; keep[t] = True
m = np.cumsum(keep) - 1
n, s, t = int(keep.sum()), m[s].astype(np.int32), m[t].astype(np.int32)
ctx = L.Context(0)
g = L.netmfp_build_csr(ctx, n, torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda())
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
gen = torch.Generator(device="cuda").manual_seed(1)
X = torch.randn(n, 288, device="cuda", generator=gen)[:, :286]
Y = torch.zeros(n, 288, device="cuda")[:, :286]
for _ in range(3): L.netmfp_spmm(ctx, g, 0.45, 0.0, X, Y)
st = torch.cuda.current_stream()
ms = []
for _ in range(20):
    flush.fill_(1); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); L.netmfp_spmm(ctx, g, 0.45, 0.0, X, Y); b.record(st); torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
np.save(os.environ["OUT"], Y.cpu().numpy())
print(os.environ.get("NETMFP_SPMM_MERGE_TAIL", "1"), "median ms", np.median(ms), "min", min(ms))
