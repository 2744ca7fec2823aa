"""Time netmfp_spmm variants on BASELINE configs shapes (tuning aid)."""
import os, sys, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch, numpy as np
    from paper_2110_12782_b200 import _lib as L, inputs
    w = inputs.CONFIGS[int(sys.argv[2])]
    n, s, t = inputs.make_graph(w.graph)
    if os.environ.get("COMPACT", "1") == "1":  # the rows embed works on (isolated vertices dropped)
        keep = np.zeros(n, bool)
        keep[s] = True
        keep[t] = True
        m = np.cumsum(keep) - 1
        n, s, t = int(keep.sum()), m[s].astype(np.int32), m[t].astype(np.int32)
    ctx = L.Context(0)
    g = L.netmfp_build_csr(ctx, n, torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda())
    out = {}
    for cols in [int(x) for x in os.environ.get("COLS", "286,128").split(",")]:
        ld = (cols + 31) // 32 * 32
        X = torch.randn(n, ld, device="cuda")[:, :cols]
        Y = torch.zeros(n, ld, device="cuda")[:, :cols]
        for _ in range(3):
            L.netmfp_spmm(ctx, g, 0.45, 0.0 if os.environ.get("SCOL", "0") == "0" else 0.45, X, Y)
        ctx.profile(True, "spmm")
        reps = 10
        for _ in range(reps):
            L.netmfp_spmm(ctx, g, 0.45, 0.0 if os.environ.get("SCOL", "0") == "0" else 0.45, X, Y)
        pr = ctx.profile_read()
        ctx.profile(False)
        ms = sum(v[1] for v in pr.values()) / reps
        byts = 8 * (n + 1) + 4 * g.nnz + 2 * 4 * n * cols
        out[cols] = dict(ms=round(ms, 4), gbs=round(byts / ms / 1e6, 1), k={k: round(v[1] / reps, 4) for k, v in pr.items()})
    print(json.dumps(out))
else:
    cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
    for v in [int(x) for x in os.environ.get("VARIANTS", "0,1,2,3,4,5,6,7").split(",")]:
        env = dict(os.environ, NETMFP_SPMM=str(v))
        r = subprocess.run([sys.executable, __file__, "child", cfg], env=env, capture_output=True, text=True)
        print("variant", v, r.stdout.strip() or r.stderr[-500:], flush=True)
