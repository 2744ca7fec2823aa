"""Heavy-row threshold x segment length sweep of netmfp_spmm on the compacted
configs[2] graph (NETMFP_LIGHT_CAP / NETMFP_HEAVY_SEG), ms per 286- and
128-column application (CUDA events, mean of 10 after 3 warm-ups)."""
import os, sys, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch, numpy as np
    from paper_2110_12782_b200 import _lib as L, inputs
    n, s, t = inputs.make_graph(inputs.CONFIGS[2].graph)
    keep = np.zeros(n, bool)
    keep[s] = True
    keep[t] = True
    m = np.cumsum(keep) - 1
    n, s, t = int(keep.sum()), m[s].astype(np.int32), m[t].astype(np.int32)
    ctx = L.Context(0)
    g = L.netmfp_build_csr(ctx, n, torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda())
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
        out[cols] = round(sum(v[1] for v in pr.values()) / 10, 4)
    print(json.dumps(out))
else:
    for cap in [int(x) for x in os.environ.get("CAPS", "16,24,32,48,64").split(",")]:
        for seg in [int(x) for x in os.environ.get("SEGS", "64,128").split(",")]:
            env = dict(os.environ, NETMFP_LIGHT_CAP=str(cap), NETMFP_HEAVY_SEG=str(seg))
            r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
            print(f"light_cap {cap:3d} heavy_seg {seg:3d}:", r.stdout.strip() or r.stderr[-300:], flush=True)
