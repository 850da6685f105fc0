"""Per-phase clock64 profile of chol_blk_kernel (library built with
TTR_EXTRA_FLAGS=-DTTR_CHOL_PROF): status words 32..37 accumulate cycles/64 of
C1 (diagonal blocks), C2 (panels), C3 (trailing), I0, I1-3 (inverse), load."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2110_04393_b200 as P

ctx = P.Context(0)
g = torch.Generator(device="cuda").manual_seed(3)
m, n = 36864, 144
U = torch.linalg.qr(torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g))[0]
s = torch.logspace(0, -10, n, dtype=torch.float64, device="cuda")
V = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))[0]
A = ((U * s) @ V.T).t().contiguous().t()
for _ in range(3):
    ctx.tt_qr(A, want_r=True)
torch.cuda.synchronize()
w = ctx.status_words(64)
names = (["C1-Xkk", "C2", "C3", "I0", "Iblk", "load", "C1-fact"] if os.environ.get("TTR_CHOL") == "blk"
         else ["wait-after-F", "(EMPTY waits in F)", "T(k)", "last-inverse", "outputs", "load", "F(warp0)"])
tot = sum(w[32:39]) - (0 if os.environ.get("TTR_CHOL") == "blk" else w[33])
calls = max(1, w[8] + 3 * w[10] + 4 * w[15])
print("status", w[:17])
ncall = 2 * w[8] + 3 * w[10] + 4 * w[15] + (2 if w[10] else 0)   # route 0 attempt + route 1
for i, nm in enumerate(names):
    print(f"{nm:8s} {w[32 + i] * 64 / max(ncall, 1):10.0f} cycles per Cholesky call  ({100 * w[32 + i] / max(tot, 1):.1f}%)")
print("cycles per Cholesky call:", tot * 64 / max(ncall, 1), "calls", ncall)
