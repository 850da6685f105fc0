"""Oracle: TT arithmetic and the rounding algorithms of PAPER.md, in fp64 NumPy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Conventions follow the paper: a TT-tensor is a list of
cores X_n of shape (R_{n-1}, I_n, R_n) with R_0 = R_N = 1.  The unfoldings are
exactly the paper's (Fig. 1):
  * H(X_n) = [X_n(:,1,:) X_n(:,2,:) … ]   (R_{n-1} × I_n R_n, slices side by side)
  * V(X_n) = [X_n(:,1,:); X_n(:,2,:); …]  (R_{n-1} I_n × R_n, slices stacked)
Modes are numbered 1..N in docstrings (the paper's) and 0..N-1 in Python lists.
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional, Sequence, Tuple, Union

import numpy as np

from .philox import sketch_core

__all__ = [
    "H", "V", "fold_H", "fold_V", "ranks_of", "dims_of", "full", "tt_add", "tt_scale",
    "inner", "norm", "diff_norm", "rel_diff", "orthogonalize_rl", "orthogonalize_lr",
    "partial_contractions_rl", "tt_round", "thin_qr", "eps_rank", "rank_caps",
    "structural_caps", "gaussian_sketch", "round_rand_orth", "round_sum_rand_orth",
    "truncate_left_orthogonal", "round_sum", "RoundResult", "left_orth_residual",
    "right_orth_residual", "partial_contractions_lr", "gaussian_sketch_left", "pinv_rtol",
    "round_two_sided", "round_sum_two_sided", "round_sum_2s", "two_sided_ranks",
    "TAG_2S_L", "TAG_2S_R",
]

Core = np.ndarray
TT = List[Core]


# ---------------------------------------------------------------- unfoldings
def H(c: Core) -> np.ndarray:
    """Horizontal unfolding: R_{n-1} × I_n R_n, column index i·R_n + b."""
    r0, I, r1 = c.shape
    return np.ascontiguousarray(c).reshape(r0, I * r1)


def V(c: Core) -> np.ndarray:
    """Vertical unfolding: R_{n-1} I_n × R_n, row index i·R_{n-1} + a."""
    r0, I, r1 = c.shape
    return np.ascontiguousarray(c.transpose(1, 0, 2)).reshape(I * r0, r1)


def fold_H(m: np.ndarray, I: int) -> Core:
    r0 = m.shape[0]
    return m.reshape(r0, I, m.shape[1] // I)


def fold_V(m: np.ndarray, I: int) -> Core:
    r1 = m.shape[1]
    return m.reshape(I, m.shape[0] // I, r1).transpose(1, 0, 2)


def ranks_of(tt: TT) -> List[int]:
    return [tt[0].shape[0]] + [c.shape[2] for c in tt]


def dims_of(tt: TT) -> List[int]:
    return [c.shape[1] for c in tt]


# ---------------------------------------------------------------- basics
def full(tt: TT) -> np.ndarray:
    """Dense tensor: entry = X_1(i_1)·X_2(i_2)···X_N(i_N).  Tiny inputs only."""
    t = np.asarray(tt[0])[0]                      # I_1 × R_1
    for c in tt[1:]:
        t = np.tensordot(t, c, axes=([t.ndim - 1], [0]))
    return t[..., 0]


def tt_add(terms: Sequence[TT], weights: Optional[Sequence[float]] = None) -> TT:
    """Assembled sum Σ_j w_j·Y^(j) with the block structure of P:388-391:
    block-diagonal middle cores, concatenated first and last cores."""
    s = len(terms)
    w = [1.0] * s if weights is None else list(weights)
    N = len(terms[0])
    out = []
    for n in range(N):
        blocks = [np.asarray(t[n]) for t in terms]
        I = blocks[0].shape[1]
        if N == 1:
            out.append(sum(wj * b for wj, b in zip(w, blocks)))
            continue
        if n == 0:
            out.append(np.concatenate([wj * b for wj, b in zip(w, blocks)], axis=2))
        elif n == N - 1:
            out.append(np.concatenate(blocks, axis=0))
        else:
            r0 = sum(b.shape[0] for b in blocks)
            r1 = sum(b.shape[2] for b in blocks)
            c = np.zeros((r0, I, r1))
            a = b_ = 0
            for blk in blocks:
                c[a:a + blk.shape[0], :, b_:b_ + blk.shape[2]] = blk
                a += blk.shape[0]
                b_ += blk.shape[2]
            out.append(c)
    return out


def tt_scale(tt: TT, alpha: float) -> TT:
    return [tt[0] * alpha] + [np.asarray(c) for c in tt[1:]]


def thin_qr(A: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Thin Householder QR with explicit Q; economy size when m < n."""
    return np.linalg.qr(A, mode="reduced")


# ---------------------------------------------------------------- Alg. 3
def partial_contractions_rl(X: TT, Y: TT) -> Dict[int, np.ndarray]:
    """Alg. 3 PartialContractionsRL, eq. (2.5).

    Returns {n: W_n} for n = 1..N-1 with W_n = H(X^{n+1:N}) H(Y^{n+1:N})ᵀ,
    W_n of shape R^X_n × R^Y_n."""
    N = len(X)
    W: Dict[int, np.ndarray] = {}
    if N < 2:
        return W
    W[N - 1] = H(X[N - 1]) @ H(Y[N - 1]).T                  # line 2
    for n in range(N - 1, 1, -1):                           # line 3: n = N-1 down to 2
        Xn, Yn = X[n - 1], Y[n - 1]
        Z = fold_V(V(Xn) @ W[n], Xn.shape[1])               # line 4: V(Z_n) = V(X_n) W_n
        W[n - 1] = H(Z) @ H(Yn).T                           # line 5: W_{n-1} = H(Z_n) H(Y_n)ᵀ
    return W


def inner(X: TT, Y: TT) -> float:
    """⟨X, Y⟩ = full right-to-left contraction (App. A: "ℓ = R ... inner product")."""
    N = len(X)
    if N == 1:
        return float(np.sum(X[0] * Y[0]))
    W = partial_contractions_rl(X, Y)
    Z = fold_V(V(X[0]) @ W[1], X[0].shape[1])
    return float((H(Z) @ H(Y[0]).T)[0, 0])


# ---------------------------------------------------------------- Alg. 1 / norms
def orthogonalize_rl(Y: TT) -> TT:
    """Alg. 1 OrthogonalizeRL.  Economy QR when H(X_n)ᵀ is wide, in
    which case the bond shrinks to I_n R_n (SPEC S:328 reading, R14)."""
    X = [np.array(c, dtype=np.float64, copy=True) for c in Y]
    N = len(X)
    for n in range(N, 1, -1):                               # line 3: n = N down to 2
        Xn = X[n - 1]
        I = Xn.shape[1]
        Q, R = thin_qr(H(Xn).T)                             # line 4
        X[n - 1] = fold_H(Q.T, I)                           # H(X_n) = Qᵀ
        Xp = X[n - 2]
        X[n - 2] = fold_V(V(Xp) @ R.T, Xp.shape[1])         # line 5: V(X_{n-1}) Rᵀ
    return X


def orthogonalize_lr(Y: TT) -> TT:
    """Left-to-right mirror of Alg. 1 ("similarly ... starting from mode-1")."""
    X = [np.array(c, dtype=np.float64, copy=True) for c in Y]
    N = len(X)
    for n in range(1, N):
        Xn = X[n - 1]
        Q, R = thin_qr(V(Xn))
        X[n - 1] = fold_V(Q, Xn.shape[1])
        Xq = X[n]
        X[n] = fold_H(R @ H(Xq), Xq.shape[1])
    return X


def norm(X: TT) -> float:
    """‖X‖ = ‖X_1‖_F after right-to-left orthogonalisation (Alg. 2 line 3)."""
    return float(np.linalg.norm(orthogonalize_rl(X)[0]))


def diff_norm(A: TT, B: TT) -> float:
    """‖A − B‖ computed in TT arithmetic: orthogonalise the assembled TT [A, −B]
     and take ‖first core‖ (R12; not the Gram identity)."""
    return norm(tt_add([A, B], [1.0, -1.0]))


def rel_diff(A: TT, B: TT) -> float:
    nb = norm(B)
    return diff_norm(A, B) / nb if nb > 0 else diff_norm(A, B)


def left_orth_residual(X: TT) -> float:
    """max_n ‖V(X_n)ᵀV(X_n) − I‖_F over n = 1..N-1 (left-orthogonality)."""
    r = 0.0
    for c in X[:-1]:
        v = V(c)
        r = max(r, float(np.linalg.norm(v.T @ v - np.eye(v.shape[1]))))
    return r


def right_orth_residual(X: TT) -> float:
    """max_n ‖H(X_n)H(X_n)ᵀ − I‖_F over n = 2..N (right-orthogonality)."""
    r = 0.0
    for c in X[1:]:
        h = H(c)
        r = max(r, float(np.linalg.norm(h @ h.T - np.eye(h.shape[0]))))
    return r


# ---------------------------------------------------------------- truncation rule
def eps_rank(s: np.ndarray, eps: float, rmax: int = 0) -> int:
    """ε-truncated SVD rank (Alg. 2 line 7): smallest k ≥ 1 with
    √(Σ_{i>k} σ_i²) ≤ ε (ties kept inclusive, R5); capped by rmax > 0."""
    s = np.asarray(s, dtype=np.float64)
    n = len(s)
    k = n
    if eps > 0:
        tail = 0.0
        k = n
        # walk from the smallest singular value up while the dropped tail stays ≤ ε
        for i in range(n - 1, 0, -1):
            t2 = tail + s[i] * s[i]
            if math.sqrt(t2) <= eps:
                tail = t2
                k = i
            else:
                break
    if rmax > 0:
        k = min(k, rmax)
    return max(1, min(k, n))


# ---------------------------------------------------------------- Alg. 2
def tt_round(Y: TT, eps0: float, rmax: Union[int, Sequence[int]] = 0) -> TT:
    """Alg. 2 TT-Rounding: OrthogonalizeRL, then a left-to-right
    ε-truncated QR+SVD sweep.  Line 8 reads V(X_n) ← Q·Û (R13)."""
    N = len(Y)
    X = orthogonalize_rl(Y)                                 # line 2
    nrm = float(np.linalg.norm(X[0]))                       # line 3: ‖Y‖ = ‖X_1‖_F
    eps = nrm * eps0 / math.sqrt(N - 1) if N > 1 else 0.0
    for n in range(1, N):                                   # line 5
        Xn = X[n - 1]
        I = Xn.shape[1]
        Q, R = thin_qr(V(Xn))                               # line 6
        U, s, Vt = np.linalg.svd(R, full_matrices=False)    # line 7
        r = rmax if isinstance(rmax, int) else int(rmax[n - 1])
        k = eps_rank(s, eps, r)
        X[n - 1] = fold_V(Q @ U[:, :k], I)                  # line 8
        Xq = X[n]
        X[n] = fold_H((s[:k, None] * Vt[:k]) @ H(Xq), Xq.shape[1])   # line 9
    return X


# ---------------------------------------------------------------- sketch + caps
def structural_caps(dims: Sequence[int], sumR: Sequence[int]) -> List[int]:
    """Largest useful sketch rank per bond n = 1..N-1 ignoring the request."""
    return rank_caps(dims, sumR, [10 ** 18] * (len(dims) - 1))


def rank_caps(dims: Sequence[int], sumR: Sequence[int],
              ell: Union[int, Sequence[int]]) -> List[int]:
    """Capped target ranks ℓ_n, n = 1..N-1 (R7; the paper is silent):
    ℓ_n = min(ℓ, ℓ_{n-1}·I_n, Π_{k>n} I_k, ΣR_n), ℓ_0 = 1.  ``sumR[n]`` is the
    bond-n rank of the (assembled) input, n = 0..N."""
    N = len(dims)
    req = [int(ell)] * (N - 1) if np.isscalar(ell) else [int(x) for x in ell]
    caps = []
    prev = 1
    for n in range(1, N):
        tail = 1
        for k in range(n, N):
            tail *= int(dims[k])
            if tail > 10 ** 18:
                break
        c = min(req[n - 1], prev * int(dims[n - 1]), tail, int(sumR[n]))
        caps.append(max(1, c))
        prev = caps[-1]
    return caps


def gaussian_sketch(dims: Sequence[int], ell_caps: Sequence[int], seed: int,
                    tag: int = 0) -> List[Optional[Core]]:
    """Random Gaussian TT 𝓡 of Def. 3.1 with ranks (1, ℓ_1..ℓ_{N-1}, 1).
    Core 1 is never used by Alg. 3/5/7 (only 𝓡^{n+1:N} enter W_n) and is None."""
    N = len(dims)
    l = [1] + list(ell_caps) + [1]
    G: List[Optional[Core]] = [None]
    for n in range(2, N + 1):
        G.append(sketch_core(seed, n, l[n - 1], dims[n - 1], l[n], tag))
    return G


# ---------------------------------------------------------------- Alg. 5 / Alg. 7
def round_rand_orth(Y: TT, G: List[Optional[Core]]) -> TT:
    """Alg. 5 TT-Rounding-RandOrth on a single (possibly assembled) TT."""
    N = len(Y)
    Gc = [g if g is not None else np.zeros((1, 1, 1)) for g in G]
    W = partial_contractions_rl(Y, Gc)                      # line 3
    X = [None] * N
    Xn = np.asarray(Y[0])                                   # line 4
    for n in range(1, N):                                   # line 5
        I = Xn.shape[1]
        Zn = V(Xn)                                          # line 6
        Yn = Zn @ W[n]                                      # line 7
        Q, _ = thin_qr(Yn)                                  # line 8
        X[n - 1] = fold_V(Q, I)
        Mn = Q.T @ Zn                                       # line 9
        Yq = np.asarray(Y[n])
        Xn = fold_H(Mn @ H(Yq), Yq.shape[1])                # line 10
    X[N - 1] = Xn
    return X


def round_sum_rand_orth(terms: Sequence[TT], G: List[Optional[Core]],
                        return_sketches: bool = False):
    """Alg. 7 TT-Rounding-sum-RandOrth, never forming the block cores.

    Q2 reading (R2): the carried core X_{n+1} concatenates the blocks
    M^(j) ×₁ T^(j)_{n+1} along its right-rank (third) mode.  Q1 reading: the last
    core is X_N = Σ_j M^(j)_{N-1} H(T^(j)_N) (line 14 prints M_{n-1})."""
    s = len(terms)
    N = len(terms[0])
    Gc = [g if g is not None else np.zeros((1, 1, 1)) for g in G]
    Wj = [partial_contractions_rl(t, Gc) for t in terms]   # lines 3-5
    X: List[Optional[Core]] = [None] * N
    Xn = np.concatenate([np.asarray(t[0]) for t in terms], axis=2)   # line 6
    Ys = {}
    if N < 2:
        raise ValueError("a TT-tensor to round needs N >= 2 modes")
    for n in range(1, N):                                   # line 7
        I = Xn.shape[1]
        Zn = V(Xn)                                          # line 8
        Wstack = np.concatenate([Wj[j][n] for j in range(s)], axis=0)
        Yn = Zn @ Wstack                                    # line 9
        Ys[n] = Yn
        if not np.any(Yn):
            # zero sum (R16): zero TT with all ranks 1
            z = [np.zeros((1, d, 1)) for d in dims_of(terms[0])]
            return (z, Wj, Ys) if return_sketches else z
        Q, _ = thin_qr(Yn)                                  # line 10
        X[n - 1] = fold_V(Q, I)
        M = Q.T @ Zn                                        # line 11
        offs = np.cumsum([0] + [t[n - 1].shape[2] for t in terms])
        Mj = [M[:, offs[j]:offs[j + 1]] for j in range(s)]
        if n < N - 1:                                       # line 12
            blocks = [fold_H(Mj[j] @ H(np.asarray(terms[j][n])), terms[j][n].shape[1])
                      for j in range(s)]
            Xn = np.concatenate(blocks, axis=2)             # line 13
        else:                                               # line 15
            last = sum(Mj[j] @ H(np.asarray(terms[j][N - 1])) for j in range(s))
            X[N - 1] = fold_H(last, terms[0][N - 1].shape[1])
    return (X, Wj, Ys) if return_sketches else X


# ---------------------------------------------------------------- truncation
def truncate_left_orthogonal(X: TT, eps0: float = 0.0,
                             rmax: Union[int, Sequence[int]] = 0) -> Tuple[TT, List[int]]:
    """Truncate a LEFT-orthogonal TT (output of Alg. 5/7) without re-orthogonalising.

    P:667-670: "skip the orthogonalization phase (line 2 of Alg. 2) and execute
    lines 3-10".  Alg. 2's sweep needs a right-orthogonal input, so on a
    left-orthogonal one it runs mirrored, right to left (R3):
      ‖X‖ = ‖X_N‖_F;  ε = ‖X‖ ε0 / √(N-1)
      for n = N..2:  [Q,R] = qr(H(X_n)ᵀ);  [U,Σ,V] = svd(Rᵀ, ε);
                     H(X_n) ← V_kᵀQᵀ;  V(X_{n-1}) ← V(X_{n-1}) U_k Σ_k
    Returns the truncated TT (right-orthogonal) and the kept ranks k_1..k_{N-1}."""
    N = len(X)
    X = [np.array(c, dtype=np.float64, copy=True) for c in X]
    nrm = float(np.linalg.norm(X[N - 1]))
    eps = nrm * eps0 / math.sqrt(N - 1) if (N > 1 and eps0 > 0) else 0.0
    ks = [0] * (N - 1)
    for n in range(N, 1, -1):
        Xn = X[n - 1]
        I = Xn.shape[1]
        Q, R = thin_qr(H(Xn).T)
        U, s, Vt = np.linalg.svd(R.T, full_matrices=False)
        r = rmax if isinstance(rmax, int) else int(rmax[n - 2])
        k = eps_rank(s, eps, r)
        ks[n - 2] = k
        X[n - 1] = fold_H(Vt[:k] @ Q.T, I)
        Xp = X[n - 2]
        X[n - 2] = fold_V(V(Xp) @ (U[:, :k] * s[None, :k]), Xp.shape[1])
    return X, ks


# ---------------------------------------------------------------- user-level call
class RoundResult:
    def __init__(self, X, ranks, sketch_ranks, passes, capped):
        self.X = X
        self.ranks = ranks
        self.sketch_ranks = sketch_ranks
        self.passes = passes
        self.capped = capped


P_MIN = 5  # adaptive saturation margin (R8)


def round_sum(terms: Sequence[TT], ell: Union[int, Sequence[int]], seed: int = 1,
              rank: Union[int, Sequence[int]] = 0,
              tol: float = 0.0, adaptive: bool = False, max_rank: int = 0,
              sketch_only: bool = False) -> RoundResult:
    """The operation behind ``tt_round_sum``: caps → sketch → Alg. 7 → truncation
    (→ adaptive growth of ℓ, tolerance mode only).  See DESIGN.md R3-R8.
    ``ell`` and ``rank`` may be sequences of N-1 per-bond values, the paper's
    "target TT-ranks {ℓ_n}" (R22): one pass, bond n
    sketched with ℓ_n (capped, R7) and truncated to rank_n."""
    if not np.isscalar(ell) or not np.isscalar(rank):
        return _round_sum_per_bond(terms, ell, seed, rank, tol, sketch_only)
    terms = [[np.asarray(c, dtype=np.float64) for c in t] for t in terms]
    dims = dims_of(terms[0])
    N = len(dims)
    if N < 2:
        raise ValueError("a TT-tensor to round needs N >= 2 modes")
    sumR = [1] + [sum(t[n].shape[2] for t in terms) for n in range(N - 1)] + [1]
    scap = structural_caps(dims, sumR)
    cur = int(ell)
    passes = 0
    while True:
        caps = rank_caps(dims, sumR, cur)
        G = gaussian_sketch(dims, caps, seed, tag=passes)
        X = round_sum_rand_orth(terms, G)
        passes += 1
        capped = any(c < cur for c in caps)
        lr = ranks_of(X)[1:-1]
        is_zero = all(r == 1 for r in lr) and not any(np.any(c) for c in X)
        if sketch_only or is_zero:
            return RoundResult(X, lr, caps, passes, capped)
        need = tol > 0 or (rank > 0 and any(c > rank for c in caps))
        if not need:
            return RoundResult(X, lr, caps, passes, capped)
        Xt, ks = truncate_left_orthogonal(X, tol, rank)
        if not (adaptive and tol > 0):
            return RoundResult(Xt, ks, caps, passes, capped)
        sat = [k > c - P_MIN and c < sc for k, c, sc in zip(ks, caps, scap)]
        if not any(sat) or (max_rank > 0 and cur >= max_rank):
            return RoundResult(Xt, ks, caps, passes, capped)
        nxt = 2 * cur
        if max_rank > 0:
            nxt = min(nxt, max_rank)
        if nxt >= max(scap):
            nxt = max(scap)
        if nxt <= cur:
            return RoundResult(Xt, ks, caps, passes, capped)
        cur = nxt


def _round_sum_per_bond(terms, ell, seed, rank, tol, sketch_only) -> RoundResult:
    """round_sum with per-bond sketch ranks ℓ_1..ℓ_{N-1} and target ranks
    r_1..r_{N-1} (scalars are broadcast; r_n = 0 means no cap on bond n)."""
    terms = [[np.asarray(c, dtype=np.float64) for c in t] for t in terms]
    dims = dims_of(terms[0])
    N = len(dims)
    if N < 2:
        raise ValueError("a TT-tensor to round needs N >= 2 modes")
    req = [int(ell)] * (N - 1) if np.isscalar(ell) else [int(x) for x in ell]
    rk = [int(rank)] * (N - 1) if np.isscalar(rank) else [int(x) for x in rank]
    if len(req) != N - 1 or len(rk) != N - 1:
        raise ValueError("per-bond ranks need N-1 entries")
    sumR = [1] + [sum(t[n].shape[2] for t in terms) for n in range(N - 1)] + [1]
    caps = rank_caps(dims, sumR, req)
    G = gaussian_sketch(dims, caps, seed, tag=0)
    X = round_sum_rand_orth(terms, G)
    capped = any(c < q for c, q in zip(caps, req))
    lr = ranks_of(X)[1:-1]
    is_zero = all(r == 1 for r in lr) and not any(np.any(c) for c in X)
    need = tol > 0 or any(r > 0 and c > r for c, r in zip(caps, rk))
    if sketch_only or is_zero or not need:
        return RoundResult(X, lr, caps, 1, capped)
    Xt, ks = truncate_left_orthogonal(X, tol, rk)
    return RoundResult(Xt, ks, caps, 1, capped)


# ---------------------------------------------------------------- Alg. 6
# Two-Sided-Randomization (generalized Nyström), P:755-783 and its derivation
# P:786-830.  Readings (R18-R21): PartialContractionsLR is the
# left-to-right mirror of Alg. 3 (the paper names it, line 4, without a listing);
# ρ = ⌈1.5ℓ⌉ by default; Σ† is the pseudo-inverse with numpy's
# cutoff σ_i > max(ℓ_n, ρ_n)·ε·σ_1; on a sum the block structure of P:388-391
# makes W^L_n = [W^L_n(Y^(1)) ⋯ W^L_n(Y^(s))] and W^R_n = [W^R_n(Y^(1)); ⋯], the
# stacking identity of P:884-890 applied to Alg. 6.

TAG_2S_L = 0x10001   # Philox tag of the left sketch 𝓛 (R21)
TAG_2S_R = 0x10002   # Philox tag of the right sketch 𝓡


def partial_contractions_lr(X: TT, Y: TT) -> Dict[int, np.ndarray]:
    """PartialContractionsLR (Alg. 6 line 4), the mirror of Alg. 3:
    {n: W_n}, n = 1..N-1, W_n = V(X^{1:n})ᵀ V(Y^{1:n}) (R^X_n × R^Y_n), so that
    with X = 𝓛, W_n = Ψ_n V(Y^{1:n}).
      W_1 = V(X_1)ᵀ V(Y_1);  n = 2..N-1: Z_n = Y_n ×₁ W_{n-1}, W_n = V(X_n)ᵀ V(Z_n)."""
    N = len(X)
    W: Dict[int, np.ndarray] = {}
    if N < 2:
        return W
    W[1] = V(np.asarray(X[0])).T @ V(np.asarray(Y[0]))
    for n in range(2, N):
        Yn = np.asarray(Y[n - 1])
        Z = fold_H(W[n - 1] @ H(Yn), Yn.shape[1])           # H(Z_n) = W_{n-1} H(Y_n)
        W[n] = V(np.asarray(X[n - 1])).T @ V(Z)
    return W


def gaussian_sketch_left(dims: Sequence[int], ell_caps: Sequence[int], seed: int,
                         tag: int = TAG_2S_L) -> List[Optional[Core]]:
    """Random Gaussian TT 𝓛 of Def. 3.1 with ranks (1, ℓ_1..ℓ_{N-1}, 1)
    for the left side of Alg. 6.  Only 𝓛^{1:N-1} enter Ψ_n: core N is None."""
    N = len(dims)
    l = [1] + list(ell_caps) + [1]
    L: List[Optional[Core]] = []
    for n in range(1, N):
        L.append(sketch_core(seed, n, l[n - 1], dims[n - 1], l[n], tag))
    L.append(None)
    return L


def pinv_rtol(shape: Tuple[int, int]) -> float:
    """Relative cutoff of Σ† (R20): numpy.linalg.pinv's default max(M, N)·ε."""
    return max(shape) * float(np.finfo(np.float64).eps)


def _two_sided_factors(WL: np.ndarray, WR: np.ndarray):
    """Alg. 6 lines 7-10 for one bond: SVD of W^L W^R, then
    L_n = W^R V (Σ†)^{1/2} and R_n = (Σ†)^{1/2} Uᵀ W^L (eq. (3.3)).
    Returns (L_n, R_n, σ)."""
    P = WL @ WR                                             # ℓ_n × ρ_n
    U, s, Vt = np.linalg.svd(P, full_matrices=False)        # line 8
    keep = s > pinv_rtol(P.shape) * (s[0] if s.size else 0.0)
    sih = np.zeros_like(s)
    sih[keep] = 1.0 / np.sqrt(s[keep])                      # (Σ†)^{1/2}
    Ln = (WR @ Vt.T) * sih[None, :]                         # line 9
    Rn = sih[:, None] * (U.T @ WL)                          # line 10
    return Ln, Rn, s


def round_two_sided(Y: TT, L: List[Optional[Core]], R: List[Optional[Core]]) -> TT:
    """Alg. 6 TT-Rounding two-sided on one (possibly assembled) TT,
    line by line.  L has ranks ℓ, R ranks ρ (cores 1 of R / N of L unused)."""
    N = len(Y)
    Y = [np.asarray(c, dtype=np.float64) for c in Y]
    Lc = [g if g is not None else np.zeros((1, 1, 1)) for g in L]
    Rc = [g if g is not None else np.zeros((1, 1, 1)) for g in R]
    WLd = partial_contractions_lr(Lc, Y)                    # line 4
    WRd = partial_contractions_rl(Y, Rc)                    # line 5
    Lf, Rf = {}, {}
    for n in range(1, N):                                   # lines 6-11
        Lf[n], Rf[n], s = _two_sided_factors(WLd[n], WRd[n])
        if not s.size or s[0] == 0.0:
            return [np.zeros((1, d, 1)) for d in dims_of(Y)]   # zero tensor (R16)
    X: TT = [None] * N
    X[0] = fold_V(V(Y[0]) @ Lf[1], Y[0].shape[1])           # line 12
    for n in range(2, N):                                   # lines 13-15
        I = Y[n - 1].shape[1]
        T = fold_V(V(Y[n - 1]) @ Lf[n], I)
        X[n - 1] = fold_H(Rf[n - 1] @ H(T), I)
    X[N - 1] = fold_H(Rf[N - 1] @ H(Y[N - 1]), Y[N - 1].shape[1])   # line 16
    return X


def round_sum_two_sided(terms: Sequence[TT], L: List[Optional[Core]],
                        R: List[Optional[Core]]) -> TT:
    """Alg. 6 on Σ_j Y^(j) without forming the block cores (R19): per-summand
    partial contractions, W^L_n = [W^L_n(Y^(j))]_j (ℓ_n × ΣR_n), W^R_n stacked
    (ΣR_n × ρ_n); L_n / R_n split into the summands' row / column blocks and
    X_n = Σ_j Y^(j)_n ×₁ R^(j)_{n-1} ×₃ L^(j)_n."""
    s = len(terms)
    N = len(terms[0])
    if N < 2:
        raise ValueError("a TT-tensor to round needs N >= 2 modes")
    terms = [[np.asarray(c, dtype=np.float64) for c in t] for t in terms]
    Lc = [g if g is not None else np.zeros((1, 1, 1)) for g in L]
    Rc = [g if g is not None else np.zeros((1, 1, 1)) for g in R]
    WLj = [partial_contractions_lr(Lc, t) for t in terms]   # line 4, per summand
    WRj = [partial_contractions_rl(t, Rc) for t in terms]   # line 5, per summand
    Lb, Rb = {}, {}
    for n in range(1, N):
        offs = np.cumsum([0] + [t[n - 1].shape[2] for t in terms])
        WL = np.concatenate([WLj[j][n] for j in range(s)], axis=1)
        WR = np.concatenate([WRj[j][n] for j in range(s)], axis=0)
        Ln, Rn, sv = _two_sided_factors(WL, WR)
        if not sv.size or sv[0] == 0.0:
            return [np.zeros((1, d, 1)) for d in dims_of(terms[0])]
        Lb[n] = [Ln[offs[j]:offs[j + 1], :] for j in range(s)]
        Rb[n] = [Rn[:, offs[j]:offs[j + 1]] for j in range(s)]
    X: TT = [None] * N
    I1 = terms[0][0].shape[1]
    X[0] = fold_V(sum(V(t[0]) @ Lb[1][j] for j, t in enumerate(terms)), I1)
    for n in range(2, N):
        I = terms[0][n - 1].shape[1]
        X[n - 1] = sum(fold_H(Rb[n - 1][j] @ H(fold_V(V(t[n - 1]) @ Lb[n][j], I)), I)
                       for j, t in enumerate(terms))
    IN = terms[0][N - 1].shape[1]
    X[N - 1] = fold_H(sum(Rb[N - 1][j] @ H(t[N - 1]) for j, t in enumerate(terms)), IN)
    return X


def two_sided_ranks(dims: Sequence[int], sumR: Sequence[int], ell: int,
                    rho: int = 0) -> Tuple[List[int], List[int]]:
    """Capped (ℓ_n, ρ_n), n = 1..N-1: R7's caps applied to ℓ and to
    ρ = ⌈1.5ℓ⌉ when rho = 0; ℓ_n ≤ ρ_n follows."""
    rho = int(rho) if rho > 0 else int(math.ceil(1.5 * int(ell)))
    if rho < ell:
        raise ValueError("Alg. 6 needs rho >= ell (P:763)")
    return rank_caps(dims, sumR, ell), rank_caps(dims, sumR, rho)


def round_sum_2s(terms: Sequence[TT], ell: int, rho: int = 0, seed: int = 1):
    """The operation behind ``tt_round_sum_two_sided``: caps → 𝓛 (tag TAG_2S_L)
    and 𝓡 (tag TAG_2S_R) from the seed → Alg. 6 on the sum.  Returns
    (X, ℓ caps, ρ caps)."""
    terms = [[np.asarray(c, dtype=np.float64) for c in t] for t in terms]
    dims = dims_of(terms[0])
    N = len(dims)
    sumR = [1] + [sum(t[n].shape[2] for t in terms) for n in range(N - 1)] + [1]
    lc, rc = two_sided_ranks(dims, sumR, ell, rho)
    L = gaussian_sketch_left(dims, lc, seed)
    R = gaussian_sketch(dims, rc, seed, tag=TAG_2S_R)
    return round_sum_two_sided(terms, L, R), lc, rc
