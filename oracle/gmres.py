"""Oracle: preconditioned TT-GMRES on a Kronecker-sum operator (§4.2,
P:1020-1045), with every TT linear combination followed by a rounding.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's application of the rounding:
  * the global system  (Σ_i A_{i,1} ⊗ … ⊗ A_{i,N}) x = f
  * right preconditioning  Y = ((Σ_i A_{i,1})^{-1} ⊗ I ⊗ … ⊗ I) V_k
  * W = Σ_i (A_{i,1} ⊗ … ⊗ A_{i,N}) Y, a sum of N TT-tensors, rounded
  * h_jk = ⟨V_j, W⟩ (j = 1..k), Z = W − Σ_j h_jk V_j, a sum of k+1 TT-tensors,
    rounded; h_{k+1,k} = ‖Z‖_F, V_{k+1} = Z / h_{k+1,k}
  * "the addition of TT-tensors is followed by a TT-rounding operation",
    either deterministic (Alg. 2 on the assembled sum, ``tt_round``) or randomized
    (Alg. 7 + truncation, ``round_sum``), the comparison the paper makes.
The paper cites TT-GMRES [Dol13] without listing it; the Arnoldi loop, the
least-squares solve on the (k+1) x k Hessenberg matrix and the solution update
x = M^{-1} Σ_j y_j V_j are textbook GMRES (readings G1-G4 in DESIGN.md).

Operator format: a list of terms; term i is a list of N per-mode factors, each
None (identity), a 1-D array (diagonal matrix) or a 2-D I_n x I_n array.
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence

import numpy as np

from .tt import inner, norm, ranks_of, round_sum, tt_add, tt_round

__all__ = ["kron_apply", "kron_dense", "precond_matrix", "apply_precond", "gmres_rounding",
           "tt_gmres", "GmresResult"]


def _mode_mult(A, c: np.ndarray) -> np.ndarray:
    """Mode-2 product core(a, i, b) <- Σ_j A(i, j) core(a, j, b) (one Kronecker factor)."""
    if A is None:
        return c
    A = np.asarray(A, dtype=np.float64)
    if A.ndim == 1:
        return c * A[None, :, None]
    return np.einsum("ij,ajb->aib", A, c)


def kron_apply(op: Sequence[Sequence], X: List[np.ndarray]) -> List[List[np.ndarray]]:
    """(Σ_i A_{i,1} ⊗ … ⊗ A_{i,N}) X as the UNROUNDED list of its N summands: term i
    is X with core n multiplied by A_{i,n} in mode 2."""
    return [[_mode_mult(A, c) for A, c in zip(term, X)] for term in op]


def _dense(A, n: int) -> np.ndarray:
    if A is None:
        return np.eye(n)
    A = np.asarray(A, dtype=np.float64)
    return np.diag(A) if A.ndim == 1 else A


def kron_dense(op: Sequence[Sequence], dims: Sequence[int]) -> np.ndarray:
    """The assembled Kronecker-sum matrix (tiny problems only).  Row/column order
    follows oracle.full(): mode 1 slowest (numpy C order of the full tensor)."""
    tot = None
    for term in op:
        K = np.ones((1, 1))
        for A, n in zip(term, dims):
            K = np.kron(K, _dense(A, n))
        tot = K if tot is None else tot + K
    return tot


def precond_matrix(op: Sequence[Sequence], I1: int) -> np.ndarray:
    """M^{-1} = (Σ_i A_{i,1})^{-1}, the mode-1 factor of the preconditioner."""
    M = sum(_dense(term[0], I1) for term in op)
    return np.linalg.inv(M)


def apply_precond(P: np.ndarray, X: List[np.ndarray]) -> List[np.ndarray]:
    """(P ⊗ I ⊗ … ⊗ I) X: mode-2 product of the first core with P (ranks unchanged)."""
    return [_mode_mult(P, X[0])] + [np.asarray(c) for c in X[1:]]


def _scale(X: List[np.ndarray], a: float) -> List[np.ndarray]:
    return [X[0] * a] + [np.asarray(c) for c in X[1:]]


def gmres_rounding(terms: Sequence[List[np.ndarray]], round_tol: float, randomized: bool,
                   seed: int, oversample: int = 10, max_rank: int = 0) -> List[np.ndarray]:
    """Round the sum of ``terms`` to relative accuracy round_tol.
    deterministic: Alg. 2 on the assembled sum;
    randomized: Alg. 7 + truncation with adaptive sketch rank (R8), initial
    sketch rank ℓ0 = (largest bond rank of a summand) + oversample (reading G3)."""
    if not randomized:
        X = tt_round(tt_add(terms), round_tol, max_rank)
        return X
    ell0 = max(max(ranks_of(t)) for t in terms) + oversample
    if max_rank > 0:
        ell0 = min(ell0, max_rank)
    r = round_sum(terms, ell=ell0, seed=seed, tol=round_tol, adaptive=True, max_rank=max_rank)
    return r.X


class GmresResult:
    def __init__(self, x, iters, residuals, ranks, converged):
        self.x = x
        self.iters = iters
        self.residuals = residuals      # relative residual estimates |beta e1 - H y| / beta
        self.ranks = ranks              # internal ranks of each basis vector V_k
        self.converged = converged


def _lstsq(Hb: np.ndarray, beta: float):
    """min_y ‖β e1 − H̄ y‖ for the (k+1) x k Hessenberg H̄ (textbook GMRES, G2)."""
    rhs = np.zeros(Hb.shape[0])
    rhs[0] = beta
    y, *_ = np.linalg.lstsq(Hb, rhs, rcond=None)
    return y, float(np.linalg.norm(rhs - Hb @ y))


def tt_gmres(op: Sequence[Sequence], f: List[np.ndarray], tol: float = 1e-8,
             max_iter: int = 50, round_tol: Optional[float] = None, randomized: bool = True,
             seed: int = 1, oversample: int = 10, max_rank: int = 0,
             precond: bool = True) -> GmresResult:
    """Right-preconditioned TT-GMRES.  Rounding calls are numbered
    c = 0, 1, 2, … in the order they happen; call c uses sketch seed ``seed + c``
    (reading G4).  round_tol defaults to tol / 10 (reading G1)."""
    f = [np.asarray(c, dtype=np.float64) for c in f]
    rt = tol / 10.0 if round_tol is None else float(round_tol)
    I1 = f[0].shape[1]
    P = precond_matrix(op, I1) if precond else np.eye(I1)
    calls = [0]

    def rnd(terms):
        X = gmres_rounding(terms, rt, randomized, seed + calls[0], oversample, max_rank)
        calls[0] += 1
        return X

    beta = norm(f)
    V = [_scale(f, 1.0 / beta)]
    Hb = np.zeros((max_iter + 1, max_iter))
    res, ranks = [1.0], [ranks_of(V[0])]
    y = np.zeros(0)
    k = 0
    converged = False
    while k < max_iter:
        Y = apply_precond(P, V[k])
        W = rnd(kron_apply(op, Y))
        h = np.array([inner(V[j], W) for j in range(k + 1)])
        Z = rnd([W] + [_scale(V[j], -h[j]) for j in range(k + 1)])
        hk1 = norm(Z)
        Hb[:k + 1, k] = h
        Hb[k + 1, k] = hk1
        y, r = _lstsq(Hb[:k + 2, :k + 1], beta)
        res.append(r / beta)
        k += 1
        if res[-1] <= tol or hk1 == 0.0:
            converged = res[-1] <= tol
            break
        V.append(_scale(Z, 1.0 / hk1))
        ranks.append(ranks_of(V[-1]))
    # x = M^{-1} Σ_j y_j V_j (right preconditioning)
    x = apply_precond(P, rnd([_scale(V[j], y[j]) for j in range(len(y))]))
    return GmresResult(x, k, res, ranks, converged)
