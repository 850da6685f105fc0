"""GPU diagnostic: QR fallback frequency and per-phase timing on reduced-depth configs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2110_04393_b200 as P
import ttsynth

ctx = P.Context(0)
ctx.set_timing(True)
for name, fn, kw in [("large d=6", ttsynth.config5_large, dict(d=6)),
                     ("gmres", ttsynth.config4_gmres, {}),
                     ("sum10 d=6", ttsynth.config3_sum10, dict(d=6))]:
    w = fn(device="cuda", **kw)
    if w.tol > 0:
        a = dict(mode="tol", tol=w.tol, oversample=w.ell, adaptive=w.adaptive)
    else:
        a = dict(mode="rank", rank=w.rank, oversample=w.ell - w.rank)
    for rep in range(2):
        r = ctx.tt_round_sum(w.terms, seed=1, **a)
        print(name, "flags", r.flags, "fallback", bool(r.flags & P.FLAG_QR_FALLBACK),
              "timing", [round(x, 3) for x in ctx.last_timing()], flush=True)

for m, n in [(36864, 144), (10240, 80), (7000, 70)]:
    for cond in [1.0, 1e6, 1e10]:
        g = torch.Generator(device="cuda")
        g.manual_seed(5)
        U, _ = torch.linalg.qr(torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g))
        V, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))
        s = torch.logspace(0, -torch.log10(torch.tensor(cond)).item(), n, dtype=torch.float64,
                           device="cuda")
        A = ((U * s) @ V.T).t().contiguous().t()
        Q, R, fb = ctx.tt_qr(A, want_r=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            Q, R, fb = ctx.tt_qr(A, want_r=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        orth = (Q.T @ Q - torch.eye(n, dtype=torch.float64, device="cuda")).norm().item()
        res = ((Q @ R - A).norm() / A.norm()).item()
        print(f"qr {m}x{n} cond {cond:.0e}: {dt * 1e3:.3f} ms fallback {fb} orth {orth:.2e} "
              f"res {res:.2e}", flush=True)
