"""Time tt_cholesky (factorisation + inverse) at n = 600 (the generic kernel)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2110_04393_b200 as P
ctx = P.Context(0)
for n in [161, 300, 600]:
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n)); G = A @ A.T + n * np.eye(n)
    Gd = torch.from_numpy(G).cuda().t().contiguous().t()
    for _ in range(2): ctx.tt_cholesky(Gd)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5): ctx.tt_cholesky(Gd)
    torch.cuda.synchronize()
    print(n, "ms per call", round((time.perf_counter() - t0) / 5 * 1e3, 3), flush=True)
