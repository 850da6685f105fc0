"""Time the fused CholeskyQR pass (tt_cholqr_pass) on a C5-sized 36864 x 144
matrix against the two-GEMM form (tt_dgemm Q = A Rinv, G = Q^T Q).
python tools/cqr_bench.py [m] [n] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2110_04393_b200 as P

m = int(sys.argv[1]) if len(sys.argv) > 1 else 36864
n = int(sys.argv[2]) if len(sys.argv) > 2 else 144
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
ctx = P.Context(0, stream=torch.cuda.current_stream())
g = torch.Generator(device="cuda").manual_seed(3)
A = torch.randn((n, m), dtype=torch.float64, device="cuda", generator=g).t()
At = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g).t()   # n x m col-major
R = (torch.triu(torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g))
     + 4 * torch.eye(n, dtype=torch.float64, device="cuda")).t().contiguous().t()
Q = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
G = torch.empty((n, n), dtype=torch.float64, device="cuda").t()


def timeit(f):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


flop_tr = 2.0 * m * n * (n + 1) / 2 + 0.0   # triangular product
flop_g = 2.0 * m * n * (n + 1) / 2
for name, f, fl in [
    ("fused Q=A Rinv + G", lambda: ctx.tt_cholqr_pass(A, R), flop_tr + flop_g),
    ("fused trans", lambda: ctx.tt_cholqr_pass(At, R, trans=True), flop_tr + flop_g),
    ("gram only", lambda: ctx.tt_cholqr_pass(A, None, want_q=False), flop_g),
    ("Q only", lambda: ctx.tt_cholqr_pass(A, R, want_g=False), flop_tr),
    ("2 GEMMs (full)", lambda: (ctx.tt_dgemm(A, R, C_out=Q), ctx.tt_dgemm(Q, Q, trans_a=True, C_out=G)), 2 * m * n * n * 2.0),
]:
    try:
        us = timeit(f)
        print(f"{name:22s} {us:9.1f} us  {fl / us / 1e6:7.2f} TF/s (useful flop)", flush=True)
    except Exception as e:
        print(name, "failed", e)
