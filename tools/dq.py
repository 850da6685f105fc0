import math, os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2110_04393_b200 as P
ctx = P.Context(0)
m, n, cond = 10240, 80, 1e9
g = torch.Generator(device="cuda").manual_seed(m + n)
U, _ = torch.linalg.qr(torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g))
V, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))
s = torch.logspace(0, -math.log10(cond), n, dtype=torch.float64, device="cuda")
A = ((U * s) @ V.T).t().contiguous().t()
G = A.T @ A
print("true gram norm", G.norm().item(), G[0,0].item(), "A[0,0]", A[0,0].item(), flush=True)
Q, R, fb = ctx.tt_qr(A, want_r=True)
print("res", ((Q @ R - A).norm() / A.norm()).item(), flush=True)
