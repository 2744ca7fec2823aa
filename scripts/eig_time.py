"""Time netmfp_sym_eig (tridiagonalisation and the rest) at the embed's l (286: Alg. 2 step 8, 228: Alg. 4 step 8)."""
import os, sys, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import numpy as np, torch
    from paper_2110_12782_b200 import _lib as L
    ctx = L.Context(0)
    out = {}
    for l in (286, 228):
        A = np.random.default_rng(l).standard_normal((l, l))
        S0 = (A + A.T) / 2
        S = torch.from_numpy(S0).cuda()
        lam = torch.zeros(l, dtype=torch.float64, device="cuda")
        V = torch.zeros(l, l, dtype=torch.float64, device="cuda")
        for _ in range(3):
            L.netmfp_sym_eig(ctx, S.clone(), lam, V, True)
        ctx.profile(True, "")
        reps = 20
        for _ in range(reps):
            L.netmfp_sym_eig(ctx, S, lam, V, True)
        pr = ctx.profile_read()
        ctx.profile(False)
        Vg, lg = V.cpu().numpy(), lam.cpu().numpy()
        err = np.abs(S0 @ Vg - Vg * lg[None, :]).max()
        out[l] = dict(err=float(err), **{k: round(v[1] / reps, 4) for k, v in pr.items()})
    print(json.dumps(out))
else:
    r = subprocess.run([sys.executable, __file__, "child"], capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-1500:], flush=True)
