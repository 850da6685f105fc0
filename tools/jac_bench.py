"""Time the truncation's V-free Jacobi SVD (tt_svd_nov) on C5-like R^T factors:
R of the QR of a 36864 x 144 matrix with 96 O(1) and 48 O(1e-6) singular values.
Set TTR_JACOBI=cta to force the single-CTA kernel."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2110_04393_b200 as P

ctx = P.Context(0, stream=torch.cuda.current_stream())
g = torch.Generator(device="cuda").manual_seed(7)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 144
m = 256 * 128
s = torch.cat([torch.linspace(1, 0.3, 96, dtype=torch.float64, device="cuda"),
               1e-6 * torch.linspace(1, 0.2, n - 96, dtype=torch.float64, device="cuda")])
U = torch.linalg.qr(torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g))[0]
V = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))[0]
A = (U * s) @ V.T
R = torch.linalg.qr(A, mode="r")[1]
Rt = R.t().contiguous().t()          # column-major storage of R^T ... (n x n)
Rt = R.t().clone().t().t()           # R^T as a column-major matrix
Rt = R.t().contiguous()              # row-major R^T == column-major R: transpose once more
RtT = Rt.t().contiguous().t()        # column-major R^T
for _ in range(2):
    AV, sig = ctx.tt_svd_nov(RtT)
torch.cuda.synchronize()
w0 = ctx.status_words(16)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
e0.record()
for _ in range(reps):
    AV, sig = ctx.tt_svd_nov(RtT)
e1.record()
torch.cuda.synchronize()
w1 = ctx.status_words(16)
ref = torch.linalg.svdvals(R)
err = ((sig - ref).abs().max() / ref[0]).item()
print(f"variant={os.environ.get('TTR_JACOBI', 'default')} n={n}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us per SVD, "
      f"sweeps/call {(w1[12] - w0[12]) / max(1, w1[13] - w0[13]):.2f}, max |sigma - ref| / sigma_1 = {err:.2e}")
