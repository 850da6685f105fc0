"""Diagnostic (not product code): spectra of the sketches Y_n and of the truncation
bond matrices for a BASELINE config, computed with plain torch fp64 on the GPU
(torch.linalg.svd), to see how ill-conditioned the QRs of the sweep are.

python tools/diag_spectra.py <workload> [d]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import ttsynth

name = sys.argv[1]
d = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = ttsynth.CONFIGS[name](device=os.environ.get("DEV", "cuda"), **({"d": d} if d else {}))
terms = w.terms
S, D = len(terms), len(terms[0])
dims = [c.shape[1] for c in terms[0]]
dev = os.environ.get("DEV", "cuda")
g = torch.Generator(device=dev).manual_seed(1)
sumR = [1] + [sum(t[n].shape[2] for t in terms) for n in range(D - 1)] + [1]
ell = w.ell
l = [1]
for n in range(1, D):
    tail = 1
    for k in range(n, D):
        tail = min(tail * dims[k], 10 ** 18)
    l.append(max(1, min(ell, l[-1] * dims[n - 1], tail, sumR[n])))
l.append(1)
G = [None] + [torch.randn(l[n - 1], dims[n - 1], l[n], dtype=torch.float64, device=dev,
                          generator=g) / (l[n - 1] * dims[n - 1] * l[n]) ** 0.5
              for n in range(2, D + 1)]


def Hm(c):   # R0 x (I R1), column (i, b) in any consistent order
    return c.reshape(c.shape[0], -1)


def Vm(c):
    return c.reshape(-1, c.shape[2])


# phase 1: W^(j)_n
W = [[None] * (D + 1) for _ in range(S)]
for j, t in enumerate(terms):
    W[j][D - 1] = Hm(t[D - 1]) @ Hm(G[D - 1]).T
    for n in range(D - 1, 1, -1):
        Z = (Vm(t[n - 1]) @ W[j][n]).reshape(t[n - 1].shape[0], dims[n - 1], l[n])
        W[j][n - 1] = Hm(Z) @ Hm(G[n - 1]).T

X = torch.cat([t[0] for t in terms], dim=2)
out = []
for n in range(1, D):
    Wst = torch.cat([W[j][n] for j in range(S)], dim=0)
    Yn = Vm(X) @ Wst
    s = torch.linalg.svdvals(Yn)
    print(f"sweep n={n:2d} Y {tuple(Yn.shape)} |W|={Wst.norm():.2e} smax={s[0]:.3e} "
          f"smin={s[-1]:.3e} kappa={s[0] / s[-1]:.2e}", flush=True)
    Q, _ = torch.linalg.qr(Yn)
    out.append(Q.reshape(X.shape[0], dims[n - 1], -1))
    M = Q.T @ Vm(X)
    offs = [0]
    for t in terms:
        offs.append(offs[-1] + t[n - 1].shape[2])
    if n < D - 1:
        blocks = [(M[:, offs[j]:offs[j + 1]] @ Hm(terms[j][n])).reshape(-1, dims[n],
                                                                     terms[j][n].shape[2])
                  for j in range(S)]
        X = torch.cat(blocks, dim=2)
    else:
        last = sum(M[:, offs[j]:offs[j + 1]] @ Hm(terms[j][D - 1]) for j in range(S))
        out.append(last.reshape(-1, dims[D - 1], 1))

# truncation sweep (mirrored Alg. 2)
r = w.rank
for n in range(D, 1, -1):
    Xn = out[n - 1]
    A = Hm(Xn).T
    Q, R = torch.linalg.qr(A)
    U, s, Vt = torch.linalg.svd(R.T)
    k = min(r, s.numel()) if r else s.numel()
    print(f"trunc n={n:2d} H^T {tuple(A.shape)} smax={s[0]:.3e} s[k-1]={s[k - 1]:.3e} "
          f"smin={s[-1]:.3e} kappa={s[0] / s[-1]:.2e}", flush=True)
    out[n - 1] = (Vt[:k] @ Q.T).reshape(k, dims[n - 1], -1)
    Xp = out[n - 2]
    out[n - 2] = (Vm(Xp) @ (U[:, :k] * s[:k])).reshape(Xp.shape[0], dims[n - 2], k)
