"""Y/Z sketches on the same F, C with fp16-split vs 3xTF32 operands at a larger
R-MAT scale (each setting in its own process): relative Frobenius difference,
worst rows, and the operands' dynamic range.  python scripts/dbg/sketch_f16_check.py SCALE EF"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 3 and sys.argv[3] == "child":
    sys.path.insert(0, ROOT)
    import numpy as np, torch
    from paper_2110_12782_b200 import _lib as L, inputs
    scale, ef = int(sys.argv[1]), int(sys.argv[2])
    dev = torch.device("cuda:0")
    src, dst = inputs.rmat_device(scale, ef, 0.57, 0.19, 0.19, 7, dev)
    n = 1 << scale
    ctx = L.Context(0)
    g = L.netmfp_build_csr(ctx, n, src, dst)
    k, s1, q = 256, 30, 6
    U = torch.zeros(n, k, device=dev); lam = torch.zeros(k, dtype=torch.float64, device=dev)
    L.netmfp_eig(ctx, g, 0.45, k, s1, q, 0, U, lam)
    F = torch.zeros(n, k, device=dev); C = torch.zeros(k, k, dtype=torch.float64, device=dev)
    L.netmfp_factor_pair(ctx, g, 0.45, 10, U, lam, F, C)
    del U
    d, s2, s3 = 128, 100, 1000
    Y = torch.zeros(n, 256, device=dev)[:, :d + s2]
    Z = torch.zeros(d + s3, d + s3, dtype=torch.float64, device=dev)
    sig = torch.zeros(d, dtype=torch.float64, device=dev)
    L.netmfp_sketch_svd(ctx, F, C, float(g.nnz) / 10.0, d, s2, s3, 8, 0, 0, sigma=sig, Ysk=Y, Zsk=Z)
    torch.cuda.synchronize()
    rmax = F.abs().amax(1)
    nz = rmax[rmax > 0]
    np.save(sys.argv[4], Y.cpu().numpy())
    np.save(sys.argv[4] + ".z.npy", Z.cpu().numpy())
    print(json.dumps({"sigma0": float(sig[0]), "sigma4": sig[:4].tolist(), "F_rowmax_log2_range":
                      [float(torch.log2(nz.min())), float(torch.log2(nz.max()))], "C_absmax": float(C.abs().max())}))
else:
    scale, ef = sys.argv[1], sys.argv[2]
    import numpy as np
    res = {}
    for tag, v in (("f16", "1"), ("tf32", "0")):
        out = f"/tmp/skchk_{tag}.npy"
        r = subprocess.run([sys.executable, __file__, scale, ef, "child", out], env=dict(os.environ, NETMFP_SKETCH_F16=v),
                           capture_output=True, text=True)
        print(tag, r.stdout.strip() or r.stderr[-1500:], flush=True)
        res[tag] = (np.load(out), np.load(out + ".z.npy"))
    (Yh, Zh), (Yt, Zt) = res["f16"], res["tf32"]
    rel = np.linalg.norm(Yh - Yt) / np.linalg.norm(Yt)
    rz = np.linalg.norm(Zh - Zt) / np.linalg.norm(Zt)
    rowerr = np.linalg.norm(Yh - Yt, axis=1)
    worst = np.argsort(-rowerr)[:5]
    colerr = np.linalg.norm(Yh - Yt, axis=0) / np.maximum(np.linalg.norm(Yt, axis=0), 1e-300)
    print("Y relF", rel, "Z relF", rz, "worst rows", worst.tolist(), rowerr[worst].tolist(),
          "row norms there", np.linalg.norm(Yt[worst], axis=1).tolist(), "worst cols rel", np.sort(colerr)[-5:].tolist())
