"""One-GPU embedding of a larger R-MAT graph (same recipe as configs[2..4],
drawn on the GPU) to check the path at scale: time per embedding and peak
device memory.  python scripts/scale_run.py SCALE EDGE_FACTOR [K]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2110_12782_b200 import _lib as L, inputs
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
ef = int(sys.argv[2]) if len(sys.argv) > 2 else 16
k = int(sys.argv[3]) if len(sys.argv) > 3 else 256
w = inputs.CONFIGS[2]
p = w.params()
p["k"] = k
dev = torch.device("cuda:0")
t0 = time.time()
src, dst = inputs.rmat_device(scale, ef, 0.57, 0.19, 0.19, 7, dev)
torch.cuda.synchronize()
gen_s = time.time() - t0
n = 1 << scale
os.environ.setdefault("NETMFP_POOL_RESERVE_GB", "0")
ctx = L.Context(0)
E = torch.zeros(n, 128, device=dev)
sig = torch.zeros(128, dtype=torch.float64, device=dev)
torch.cuda.reset_peak_memory_stats()
out = {"scale": scale, "edge_factor": ef, "n": n, "edges_in": int(src.numel()), "k": k, "gen_s": round(gen_s, 2)}
times = []
for i in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L.netmfp_embed_edges(ctx, n, src, dst, L.make_params(**p), E, sig)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
g = L.netmfp_build_csr(ctx, n, src, dst)
deg = g.export(ctx)[2]
free, total = torch.cuda.mem_get_info()
out.update(ms=[round(x, 1) for x in times], nnz=int(g.nnz), nonisolated=int((deg > 0).sum()),
           sigma0=float(sig[0]), finite=bool(torch.isfinite(E).all()), device_free_GB=round(free / 2**30, 1))
print(json.dumps(out))
