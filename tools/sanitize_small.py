"""Small end-to-end calls for compute-sanitizer: one Alg. 7 rounding (config 5
shapes at d = 4: the cluster Jacobi, the blocked Cholesky, TMA GEMMs, the fused
projection-and-carry), one two-sided rounding, one deterministic rounding, one
TT-GMRES solve and one slab rounding."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2110_04393_b200 as P
import ttsynth

ctx = P.Context(0, stream=torch.cuda.current_stream())
w = ttsynth.config5_large(d=4, device="cuda")
r = ctx.tt_round_sum(w.terms, mode="rank", rank=w.rank, oversample=w.ell - w.rank, seed=1)
print("alg7", r.ranks)
r2 = ctx.tt_round_sum_two_sided(w.terms, w.rank, seed=1)
print("alg6", r2.ranks)
w3 = ttsynth.config3_sum10(d=5, I=20, S=3, device="cuda")
r3 = ctx.tt_round_deterministic(w3.terms, tol=1e-6)
print("det", r3.ranks)
op, f, dims = ttsynth.cookie_surrogate(grid=16, params=2, samples=4)
opd = [[None if A is None else torch.from_numpy(np.asarray(A)).cuda() for A in t] for t in op]
x, info = ctx.tt_gmres(opd, [torch.from_numpy(c).cuda() for c in f], tol=1e-8)
print("gmres", info["iters"], info["converged"])
r4 = ctx.tt_round_sum_slab(w3.terms, [20] * 5, [0] * 5, mode="rank", rank=20, oversample=5)
print("slab", r4.ranks)
torch.cuda.synchronize()
print("done")
