"""One netmfp_sketch_svd at configs[2] shapes (n=2^20, k=256, d=128, s2=100, s3=1000, z=8): ncu target."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_12782_b200 import _lib as L
ctx = L.Context(0)
n, k, d = 1 << 20, 256, 128
g = torch.Generator(device="cuda").manual_seed(0)
F = (torch.randn(n, k, device="cuda", generator=g) * 1e-3)
Cm = torch.randn(k, k, device="cuda", dtype=torch.float64, generator=g) * 0.1
Cm = Cm @ Cm.T
E = torch.zeros(n, d, device="cuda")
sig = torch.zeros(d, device="cuda", dtype=torch.float64)
for _ in range(2):
    L.netmfp_sketch_svd(ctx, F, Cm, 6e6 / 10, d, 100, 1000, 8, 1, sigma=sig, E=E)
ctx.profile(True, "")
L.netmfp_sketch_svd(ctx, F, Cm, 6e6 / 10, d, 100, 1000, 8, 1, sigma=sig, E=E)
print(ctx.profile_read())
