"""One tc Gram + one CholeskyQR (tri GEMM) at configs[2] shapes (ncu target), timed with the ctx profiler."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_12782_b200 import _lib as L
ctx = L.Context(0)
n, c = 1 << 20, 286
Y = torch.randn(n, 288, device="cuda")[:, :c]
Q = torch.zeros(n, 288, device="cuda")[:, :c]
G = torch.zeros(c, c, dtype=torch.float64, device="cuda")
for _ in range(2):
    L.netmfp_gram(ctx, Y, Y, G)
    L.netmfp_orthonormalize(ctx, Y, Q, 1)
ctx.profile(True, "")
for _ in range(3):
    L.netmfp_gram(ctx, Y, Y, G)
    L.netmfp_orthonormalize(ctx, Y, Q, 1)
print(ctx.profile_read())
Yd = Y.double()
ref = (Yd.T @ Yd)
print("gram rel err", float((G - ref).abs().max() / ref.abs().max()))
Qd = Q.double()
print("orth err", float((Qd.T @ Qd - torch.eye(c, device="cuda", dtype=torch.float64)).abs().max()))
