import numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
from paper_2110_12782_b200 import _lib as L
ctx = L.Context(0)
bad = []
for l in list(range(3, 80)) + [96, 100, 128, 129, 130, 158, 200, 228, 286]:
    A = np.random.default_rng(l).standard_normal((l, l)); S0 = (A + A.T) / 2
    lam = torch.zeros(l, dtype=torch.float64, device="cuda"); V = torch.zeros(l, l, dtype=torch.float64, device="cuda")
    L.netmfp_sym_eig(ctx, torch.from_numpy(S0).cuda(), lam, V, True)
    err = np.abs(np.sort(lam.cpu().numpy()) - np.linalg.eigvalsh(S0)).max()
    if err > 1e-9: bad.append((l, float(err)))
print("bad", bad)
