import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_04393_b200 as P
ctx = P.Context(0)
for (m, n, cond) in [(10240, 80, 1e12), (10240, 80, 1e9), (36864, 144, 1e10), (2240, 35, 1e8)]:
    g = torch.Generator(device="cuda").manual_seed(m + n)
    U, _ = torch.linalg.qr(torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g))
    V, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))
    s = torch.logspace(0, -math.log10(cond), n, dtype=torch.float64, device="cuda")
    A = ((U * s) @ V.T).t().contiguous().t()
    Q, R, fb = ctx.tt_qr(A, want_r=True)
    st = ctx.status_words(16)
    Rt = torch.linalg.qr(A)[1]
    print(m, n, cond, "fb", fb, "status", st, "res", ((Q @ R - A).norm() / A.norm()).item(),
          "diagR", R.diagonal()[:3].tolist(), R.diagonal()[-3:].tolist(),
          "diagRt", Rt.diagonal()[:3].tolist(), Rt.diagonal()[-3:].tolist(), flush=True)
    _, R2, fb2 = ctx.tt_qr(A, want_r=True, want_q=False)
    print("   r-only", fb2, ctx.status_words(16), "sv diff",
          (torch.linalg.svdvals(R2) - torch.linalg.svdvals(A)).abs().max().item(), flush=True)
