"""Algorithmic flop counts of one rounding (metric accounting).

These count what the method must compute (Alg. 3 per summand, Alg. 7's sweep,
the truncation QR + products), not the extra work an implementation chooses
(CholeskyQR3's repeated Gram products are not credited: QR is credited at the
Householder count 4mn² − 4n³/3 of P:397).  Pinned in tests/test_cost_model.py
against the paper's leading-order formulas (Table 1)."""
from __future__ import annotations

from typing import Dict, List, Sequence


def caps(dims: Sequence[int], sumR: Sequence[int], ell: int) -> List[int]:
    """l_0..l_N with the R7 caps (same rule as the library and the oracle)."""
    N = len(dims)
    l = [1] * (N + 1)
    for n in range(1, N):
        tail = 1
        for k in range(n, N):
            tail *= dims[k]
            if tail > 1 << 40:
                break
        l[n] = max(1, min(ell, l[n - 1] * dims[n - 1], tail, sumR[n]))
    return l


def rounding_flops(dims: Sequence[int], term_ranks: Sequence[Sequence[int]], l: Sequence[int],
                   kept: Sequence[int] | None = None) -> Dict[str, float]:
    """Exact per-step counts.  term_ranks[j] = (R_0..R_N) of summand j; l = (l_0..l_N);
    kept = ranks after truncation (None: no truncation)."""
    N = len(dims)
    I = list(dims)
    sumR = [sum(r[n] for r in term_ranks) for n in range(N + 1)]
    p1 = 0.0
    for R in term_ranks:
        p1 += 2.0 * R[N - 1] * I[N - 1] * l[N - 1]                      # Alg. 3 line 2
        for n in range(2, N):                                             # lines 4-5
            p1 += 2.0 * R[n - 1] * I[n - 1] * R[n] * l[n]
            p1 += 2.0 * R[n - 1] * I[n - 1] * l[n] * l[n - 1]
    sk = qr = pr = ca = 0.0
    for n in range(1, N):
        m = l[n - 1] * I[n - 1]
        sk += 2.0 * sumR[n] * m * l[n]                                    # Alg. 7 line 9
        qr += 4.0 * m * l[n] ** 2 - 4.0 * l[n] ** 3 / 3.0                 # line 10
        pr += 2.0 * sumR[n] * m * l[n]                                    # line 11
        if n < N - 1:
            ca += sum(2.0 * l[n] * R[n] * I[n] * R[n + 1] for R in term_ranks)   # line 13
        else:
            ca += 2.0 * l[n] * sumR[n] * I[n]                             # line 15
    tr = 0.0
    if kept is not None:
        r = list(l)
        for n in range(N, 1, -1):
            mrow = I[n - 1] * r[n]
            c = min(mrow, r[n - 1])
            tr += 4.0 * mrow * c * c - 4.0 * c ** 3 / 3.0
            tr += 2.0 * kept[n - 1] * r[n - 1] * mrow
            r[n - 1] = kept[n - 1]
    total = p1 + sk + qr + pr + ca + tr
    return {"phase1": p1, "sketch": sk, "qr": qr, "project": pr, "carry": ca, "truncate": tr,
            "total": total}


def two_sided_flops(dims: Sequence[int], term_ranks: Sequence[Sequence[int]],
                    l: Sequence[int], rho: Sequence[int]) -> Dict[str, float]:
    """Exact per-step counts of Alg. 6 on a sum (R18-R20): l = (l_0..l_N) left /
    output ranks, rho = (rho_0..rho_N) right sketch ranks.  The bond SVD of the
    l x rho matrix W^L W^R is credited at the Householder QR count of its
    transpose, the SVD of the l x l factor is not credited."""
    N = len(dims)
    I = list(dims)
    sumR = [sum(r[n] for r in term_ranks) for n in range(N + 1)]
    right = rounding_flops(dims, term_ranks, rho)["phase1"]              # line 5 (Alg. 3)
    left = 0.0
    for R in term_ranks:                                                  # line 4 (R18)
        left += 2.0 * I[0] * l[1] * R[1]
        for n in range(2, N):
            left += 2.0 * l[n - 1] * R[n - 1] * I[n - 1] * R[n]
            left += 2.0 * l[n] * l[n - 1] * I[n - 1] * R[n]
    bond = 0.0
    for n in range(1, N):                                                 # lines 7-10
        bond += 2.0 * l[n] * sumR[n] * rho[n]                             # W^L W^R
        bond += 4.0 * rho[n] * l[n] ** 2 - 4.0 * l[n] ** 3 / 3.0          # QR of its transpose
        bond += 2.0 * sumR[n] * rho[n] * l[n] + 2.0 * l[n] * l[n] * sumR[n]   # L_n, R_n
    asm = 2.0 * I[0] * sumR[1] * l[1]                                     # lines 12-16
    for n in range(2, N):
        asm += sum(2.0 * l[n - 1] * R[n - 1] * I[n - 1] * R[n] for R in term_ranks)
        asm += 2.0 * l[n - 1] * I[n - 1] * sumR[n] * l[n]
    asm += 2.0 * l[N - 1] * sumR[N - 1] * I[N - 1]
    total = right + left + bond + asm
    return {"phase1": right, "left": left, "bond": bond, "assembly": asm, "total": total}


def paper_two_sided(N: int, I: int, R: int, ell: int, rho: int) -> float:
    """Leading-order cost of Alg. 6 on one TT: (N-2)I(2R²ρ + 2Rρ²)
    for the right contraction + (N-2)I(2R²l + 2Rl²) left + (N-2)I(2R²l + 2Rl²)
    assembly; with rho = 1.5 l this is P:944's I(N-2)(7R²l + 8.5Rl²)."""
    return I * (N - 2) * (2.0 * R * R * rho + 2.0 * R * rho * rho
                          + 4.0 * R * R * ell + 4.0 * R * ell * ell)


def paper_rto_sum(N: int, I: int, R: int, ell: int, s: int) -> float:
    """Leading-order cost of Alg. 7 printed at P:985-987 (last term read 4l³, R14)."""
    return I * (N - 2) * (4.0 * s * R * R * ell + 6.0 * s * R * ell * ell + 4.0 * ell ** 3)


def table1_simplified(beta: float) -> Dict[str, float]:
    """Table 1 simplified coefficients of (N-2) I R³."""
    return {"tt_rounding": 5 + 6 * beta + 2 * beta ** 2,
            "orth_then_rand": 5 + 2 * beta + 4 * beta ** 2 + 4 * beta ** 3,
            "rand_then_orth": 4 * beta + 6 * beta ** 2 + 4 * beta ** 3,
            "two_sided": 6 * beta + 6 * beta ** 2}
