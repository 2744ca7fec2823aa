"""SpMM time on configs[2]'s compacted graph under vertex orderings (experiment)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, scipy.sparse as sp
from scipy.sparse import csgraph
import torch
from paper_2110_12782_b200 import _lib as L, inputs
w = inputs.CONFIGS[2]
n, s, t = inputs.make_graph(w.graph)
keep = np.zeros(n, bool); keep[s] = True; keep[t] = True
m = np.cumsum(keep) - 1
n, s, t = int(keep.sum()), m[s].astype(np.int64), m[t].astype(np.int64)
A = sp.csr_matrix((np.ones(2 * len(s)), (np.r_[s, t], np.r_[t, s])), shape=(n, n))
deg = np.asarray((A > 0).sum(1)).ravel()
orders = {"compact": np.arange(n),
          "degree": np.argsort(-deg, kind="stable"),
          "bfs": None, "rcm": csgraph.reverse_cuthill_mckee(A.tocsr(), symmetric_mode=True)}
bfs = []
seen = np.zeros(n, bool)
for root in np.argsort(-deg, kind="stable"):
    if seen[root]:
        continue
    o = csgraph.breadth_first_order(A, root, directed=False, return_predecessors=False)
    seen[o] = True
    bfs.append(o)
orders["bfs"] = np.concatenate(bfs)
ctx = L.Context(0)
for name, order in orders.items():
    inv = np.empty(n, np.int64); inv[order] = np.arange(n)
    ss, tt = inv[s].astype(np.int32), inv[t].astype(np.int32)
    g = L.netmfp_build_csr(ctx, n, torch.from_numpy(ss).cuda(), torch.from_numpy(tt).cuda())
    out = {}
    for cols in (286, 128):
        ld = (cols + 31) // 32 * 32
        X = torch.randn(n, ld, device="cuda")[:, :cols]
        Y = torch.zeros(n, ld, device="cuda")[:, :cols]
        for _ in range(3):
            L.netmfp_spmm(ctx, g, 0.45, 0.0, X, Y)
        ctx.profile(True, "spmm")
        for _ in range(10):
            L.netmfp_spmm(ctx, g, 0.45, 0.0, X, Y)
        pr = ctx.profile_read()
        ctx.profile(False)
        out[cols] = round(sum(v[1] for k, v in pr.items() if not k.startswith("gap")) / 10, 4)
    print(name, json.dumps(out), flush=True)
