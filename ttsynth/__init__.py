"""Seeded synthetic inputs shared by the tests, ``bench.py`` and ``smoke()``.

This module is deliberately neither the oracle nor the product: it holds NO
arithmetic of the rounding method (no sketching, no contraction, no QR of a
sketch, no truncation).  It only draws random TT-tensors with the shapes and
value distributions of the paper's workloads (§4.1, P:1010-1016:
"𝒳₁ + ε𝒳₂"; §4.2: sums arising in TT-GMRES) restated as the five
BASELINE.json configs (recipes in DESIGN.md §"Input recipe", following
SURVEY.md §8d).  Both the oracle (CPU) and the CUDA path consume the same bits.

Cores are torch tensors of logical shape (R_{n-1}, I_n, R_n) stored
"a-fastest" (element (a,i,b) at a + R_{n-1}(i + I_n b)), which is the layout
include/ttround.h documents; ``.numpy()`` of such a tensor is a Fortran-ordered
numpy array with the same logical shape, which is what the oracle indexes.

Random numbers come from a ``torch.Generator`` (CPU for parity-sized inputs,
CUDA for bench-sized inputs); the recipe is the same on both, the bit streams
are not, and nothing requires them to be (inputs are generated once and handed
to both sides).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence

import torch

Core = torch.Tensor
TT = List[Core]


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def empty_core(r0: int, n: int, r1: int, device="cpu", dtype=torch.float64) -> Core:
    """Uninitialised core with logical shape (r0, n, r1) in the a-fastest layout."""
    return torch.empty((r1, n, r0), dtype=dtype, device=device).permute(2, 1, 0)


def gaussian_tt(dims: Sequence[int], ranks: Sequence[int], std, g: torch.Generator,
                device="cpu") -> TT:
    """TT-tensor with i.i.d. N(0, std_n^2) core entries; ranks has length d+1.

    ``std`` is a float or a callable (r0, I, r1) -> float."""
    d = len(dims)
    assert len(ranks) == d + 1 and ranks[0] == 1 and ranks[d] == 1
    cores = []
    for n in range(d):
        r0, I, r1 = int(ranks[n]), int(dims[n]), int(ranks[n + 1])
        s = std(r0, I, r1) if callable(std) else float(std)
        c = torch.randn((r1, I, r0), generator=g, dtype=torch.float64, device=device)
        c.mul_(s)
        cores.append(c.permute(2, 1, 0))
    return cores


def block_sum(parts: Sequence[TT], weights: Sequence[float]) -> TT:
    """Cores of c_1·A_1 ⊕ c_2·A_2 ⊕ … (block structure of PAPER.md P:388-391).

    Input construction only (e.g. the summand c_j·Y ⊕ 1e-6·Z_j of config 3);
    the weights are folded into the first core of each block."""
    d = len(parts[0])
    dev = parts[0][0].device
    out = []
    for n in range(d):
        r0 = 1 if n == 0 else sum(p[n].shape[0] for p in parts)
        r1 = 1 if n == d - 1 else sum(p[n].shape[2] for p in parts)
        I = parts[0][n].shape[1]
        c = empty_core(r0, I, r1, device=dev)
        c.zero_()
        a = b = 0
        for p, w in zip(parts, weights):
            x = p[n] * (w if n == 0 else 1.0)
            ra, rb = x.shape[0], x.shape[2]
            if n == 0:
                c[:, :, b:b + rb] = x
            elif n == d - 1:
                c[a:a + ra, :, :] = x
            else:
                c[a:a + ra, :, b:b + rb] = x
            a += ra
            b += rb
        out.append(c)
    return out


@dataclasses.dataclass
class Workload:
    """One rounding problem: the summands plus the options of the call."""
    name: str
    terms: List[TT]
    ell: int                      # sketch rank ℓ (oversampling included)
    rank: int = 0                 # target rank r after truncation (0: none)
    tol: float = 0.0              # relative tolerance ε0 (0: none)
    adaptive: bool = False
    max_rank: int = 0
    note: str = ""

    @property
    def d(self) -> int:
        return len(self.terms[0])

    @property
    def dims(self) -> List[int]:
        return [int(c.shape[1]) for c in self.terms[0]]

    def to(self, device) -> "Workload":
        return dataclasses.replace(self, terms=[[_move(c, device) for c in t]
                                                for t in self.terms])


def _move(c: Core, device) -> Core:
    """Copy preserving the a-fastest layout."""
    return c.permute(2, 1, 0).contiguous().to(device).permute(2, 1, 0)


# --------------------------------------------------------------------------
# the five BASELINE.json configs (SURVEY.md §8d "Configs restated")
# --------------------------------------------------------------------------

def _std_ri(r0, I, r1):
    # "fp64 N(0,1/sqrt(R·I)) cores" read as std 1/sqrt(R·I) with R
    # the TT rank of the tensor the core belongs to (max of its two bonds).
    return 1.0 / math.sqrt(max(r0, r1) * I)


def config1_tiny(seed: int = 1001, device="cpu", d=4, I=4, R=3, S=2) -> Workload:
    g = _gen(seed, device)
    ranks = [1] + [R] * (d - 1) + [1]
    terms = [gaussian_tt([I] * d, ranks, 1.0, g, device) for _ in range(S)]
    return Workload("tiny", terms, ell=6, rank=4,
                    note="S=2 d=4 I=4 R=3, N(0,1) cores, rank 4 + oversampling 2")


def perturbed(seed, device, S, d, I, Ry, Rz, eps, shared=1, cj=True) -> List[TT]:
    """Summand j = c_j·Y_{j mod shared} ⊕ eps·Z_j (§4.1's 𝒳₁+ε𝒳₂)."""
    g = _gen(seed, device)
    Ys = [gaussian_tt([I] * d, [1] + [Ry] * (d - 1) + [1], _std_ri, g, device)
          for _ in range(shared)]
    terms = []
    for j in range(S):
        Z = gaussian_tt([I] * d, [1] + [Rz] * (d - 1) + [1], _std_ri, g, device)
        c = float(0.5 + torch.rand((), generator=g, device=device, dtype=torch.float64)) if cj else 1.0
        terms.append(block_sum([Ys[j % shared], Z], [c, eps]))
    return terms


def config2_single(seed: int = 1002, device="cpu", d=16, I=64) -> Workload:
    terms = perturbed(seed, device, S=1, d=d, I=I, Ry=25, Rz=25, eps=1e-8, cj=False)
    return Workload("single", terms, ell=35, rank=25,
                    note="X = Y + 1e-8 Z, rank 25+25, round to 25 with sketch 35")


def config3_sum10(seed: int = 1003, device="cpu", d=20, I=100, S=10) -> Workload:
    terms = perturbed(seed, device, S=S, d=d, I=I, Ry=50, Rz=10, eps=1e-6)
    return Workload("sum10", terms, ell=70, rank=60,
                    note="X_j = c_j Y + 1e-6 Z_j, rank 50+10, round to 60 with sketch 70")


def config5_large(seed: int = 1005, device="cpu", d=50, I=256, S=32) -> Workload:
    terms = perturbed(seed, device, S=S, d=d, I=I, Ry=48, Rz=16, eps=1e-6, shared=2)
    return Workload("large", terms, ell=144, rank=128,
                    note="reading C: X_j = c_j Y_{A|B} + 1e-6 Z_j, per-summand rank 64, "
                         "signal rank 96, round to 128 with sketch 144")


def _decay_tt(d, I, R, g, device, decay=8.0) -> TT:
    """T with V(T_n) = Q_n·diag(10^{-k/decay}) (n < d), Q_n orthonormal; last core
    N(0, 1/(R·I)).  Q_n is the Q of a Householder QR of a Gaussian block with
    diag(R) > 0 (input construction only)."""
    ranks = [1] + [R] * (d - 1) + [1]
    s = torch.pow(10.0, -torch.arange(R, dtype=torch.float64, device=device) / decay)
    cores = []
    for n in range(d):
        r0, r1 = ranks[n], ranks[n + 1]
        if n < d - 1:
            A = torch.randn((r0 * I, r1), generator=g, dtype=torch.float64, device=device)
            Q, Rf = torch.linalg.qr(A)
            Q = Q * torch.sign(torch.diagonal(Rf))[None, :]
            V = Q * s[None, :r1]
            # V rows are (a, i) with a fastest  -> a-fastest core (r0, I, r1)
            c = empty_core(r0, I, r1, device=device)
            c.copy_(V.reshape(I, r0, r1).permute(1, 0, 2))
        else:
            c = torch.randn((r1, I, r0), generator=g, dtype=torch.float64,
                            device=device).permute(2, 1, 0) / math.sqrt(R * I)
        cores.append(c)
    return cores


def _norm_by_gram(cores: TT) -> float:
    """‖T‖ by the plain Gram recursion G ← Σ_i T_iᵀ G T_i (input normalisation only)."""
    G = torch.ones((1, 1), dtype=torch.float64, device=cores[0].device)
    for c in cores:
        G = torch.einsum("ab,aic,bid->cd", G, c, c)
    return float(G.reshape(()).clamp_min(0).sqrt())


def config4_gmres(seed: int = 1004, device="cpu", d=12, I=128, R=40, S=20,
                  stress: bool = False) -> Workload:
    g = _gen(seed, device)
    terms = []
    for j in range(S):
        T = _decay_tt(d, I, R, g, device)
        nrm = _norm_by_gram(T)
        c = (1.0 if stress else 10.0 ** (-5.0 * j)) / nrm
        T[0] = T[0] * c
        terms.append(T)
    return Workload("gmres" + ("_stress" if stress else ""), terms, ell=80, rank=0,
                    tol=1e-8, adaptive=True, max_rank=0,
                    note="GMRES-like: S=20 rank-40 summands with core spectra 10^(-k/8), "
                         + ("equal weights (stress)" if stress else "weights 10^(-5(j-1))"))


CONFIGS = {
    "tiny": config1_tiny,
    "single": config2_single,
    "sum10": config3_sum10,
    "gmres": config4_gmres,
    "large": config5_large,
}


def hilbert_tt(dims: Sequence[int], ranks: Sequence[int], device="cpu") -> TT:
    """Hilbert-type TT of PAPER.md App. C: X_n(i1,i2,i3) = 1/(i1+i2+i3-1)."""
    cores = []
    for n in range(len(dims)):
        r0, I, r1 = ranks[n], dims[n], ranks[n + 1]
        a = torch.arange(1, r0 + 1, dtype=torch.float64, device=device)[:, None, None]
        i = torch.arange(1, I + 1, dtype=torch.float64, device=device)[None, :, None]
        b = torch.arange(1, r1 + 1, dtype=torch.float64, device=device)[None, None, :]
        c = empty_core(r0, I, r1, device=device)
        c.copy_(1.0 / (a + i + b - 1.0))
        cores.append(c)
    return cores


def random_terms(seed: int, dims: Sequence[int], term_ranks: Sequence[Sequence[int]],
                 std=1.0, device="cpu") -> List[TT]:
    """Generic ragged summands (per-summand rank profiles, per-mode dims)."""
    g = _gen(seed, device)
    return [gaussian_tt(dims, r, std, g, device) for r in term_ranks]


def to_numpy(tt: TT):
    return [c.detach().cpu().numpy() for c in tt]


# ---------------------------------------------------------------- TT-GMRES surrogate (NEXT-4)
def cookie_surrogate(grid: int = 16, params: int = 2, samples: int = 4,
                     rho=(1.0, 10.0)):
    """Kronecker-sum stand-in for the paper's cookie problem (its FEM
    operator and mesh are not available): N = 1 + params modes.
      A_{1,1} = 1-D finite-difference Dirichlet Laplacian on `grid` interior points
                (the operator with constant coefficient),
      A_{p+1,1} = the same stiffness restricted to the edges of a disjoint index block
                (the characteristic function of "subdomain" p),
      A_{p+1,p+1} = diag(ρ samples linearly spaced in [1, 10]),
      every other factor the identity;  f = the rank-1 all-ones TT.
    Returns (op, f, dims) with op in oracle.gmres's format (None = identity,
    1-D = diagonal, 2-D = dense), numpy fp64.  Input synthesis only."""
    import numpy as np
    h2 = float((grid + 1) ** 2)
    edges = [(k, k + 1) for k in range(grid - 1)]

    def stiffness(edge_list, dirichlet):
        A = np.zeros((grid, grid))
        for a, b in edge_list:
            A[a, a] += h2
            A[b, b] += h2
            A[a, b] -= h2
            A[b, a] -= h2
        if dirichlet:
            A[0, 0] += h2
            A[grid - 1, grid - 1] += h2
        return A

    L0 = stiffness(edges, True)
    N = 1 + params
    op = [[L0] + [None] * params]
    width = max(1, grid // (2 * params + 1))
    for p in range(params):
        lo = (2 * p + 1) * width
        blk = [(a, b) for (a, b) in edges if lo <= a and b < min(grid, lo + width + 1)]
        term = [stiffness(blk, False)] + [None] * params
        term[1 + p] = np.linspace(rho[0], rho[1], samples)
        op.append(term)
    dims = [grid] + [samples] * params
    f = [np.ones((1, dims[n], 1)) for n in range(N)]
    return op, f, dims
