"""Oracle: counter-based Philox4x32-10 and the Gaussian sketch of Def. 3.1.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md Def. 3.1: a random Gaussian TT-tensor has cores
R^(n) ∈ R^{ℓ_{n-1}×I_n×ℓ_n} "filled with random, independent, normally
distributed entries with mean 0 and variance 1/(ℓ_{n-1} I_n ℓ_n)".  The paper's
Matlab code draws them with ``randn``; the paper fixes no generator, so the
reading (R9) is:

  * Philox4x32 with 10 rounds (Salmon et al., SC'11 "Random123"): round
    function (c0,c1,c2,c3) -> (hi(M1·c2)^c1^k0, lo(M1·c2), hi(M0·c0)^c3^k1,
    lo(M0·c0)), key bumped by the Weyl constants (W0, W1) between rounds.
  * key = (seed mod 2^32, seed >> 32); counter = (k mod 2^32, k >> 32, n, tag)
    for element pair k = e // 2 of core n (1-based mode index), where e is the
    element's index in the layout order e = a + ℓ_{n-1}(i + I_n b).
  * u1 from words (x0, x1), u2 from (x2, x3):  u = ((x_hi·2^32 + x_lo) >> 11
    + 0.5)·2^-53 ∈ (0, 1);  Box–Muller: z_{2k} = √(-2 ln u1)·cos(2π u2),
    z_{2k+1} = √(-2 ln u1)·sin(2π u2);  entry = z_e · (ℓ_{n-1} I_n ℓ_n)^{-1/2}.

Pinned by tests/test_oracle_philox.py against cuRAND's own
``curand_Philox4x32_10`` (golden vectors written by tests/golden/philox_kat.cu)
and by the moments of Def. 3.1 (E‖R^(n)‖_F² = 1).
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint32(0x9E3779B9)
W1 = np.uint32(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Ten Philox4x32 rounds on uint32 arrays (broadcast); returns 4 uint32 arrays."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint32) for x in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint32).copy()
    k1 = np.asarray(k1, dtype=np.uint32).copy()
    with np.errstate(over="ignore"):
        for r in range(10):
            p0 = M0 * c0.astype(np.uint64)
            p1 = M1 * c2.astype(np.uint64)
            hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
            lo0 = (p0 & _MASK).astype(np.uint32)
            hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
            lo1 = (p1 & _MASK).astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            k0 = k0 + W0
            k1 = k1 + W1
    return c0, c1, c2, c3


def _unit(lo, hi):
    """53-bit uniform in (0,1] from two 32-bit words (fp64, round-to-nearest)."""
    v = (hi.astype(np.uint64) << np.uint64(32)) | lo.astype(np.uint64)
    return ((v >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def philox_normal(count: int, seed: int, n: int, tag: int = 0) -> np.ndarray:
    """The first ``count`` standard normals of stream (seed, n, tag), element order e."""
    npair = (count + 1) // 2
    k = np.arange(npair, dtype=np.uint64)
    c0 = (k & _MASK).astype(np.uint32)
    c1 = (k >> np.uint64(32)).astype(np.uint32)
    c2 = np.full(npair, n, dtype=np.uint32)
    c3 = np.full(npair, tag, dtype=np.uint32)
    seed = int(seed)
    x0, x1, x2, x3 = philox4x32_10(c0, c1, c2, c3, np.uint32(seed & 0xFFFFFFFF),
                                   np.uint32((seed >> 32) & 0xFFFFFFFF))
    u1 = _unit(x0, x1)
    u2 = _unit(x2, x3)
    r = np.sqrt(-2.0 * np.log(u1))
    z = np.empty(2 * npair, dtype=np.float64)
    z[0::2] = r * np.cos(2.0 * np.pi * u2)
    z[1::2] = r * np.sin(2.0 * np.pi * u2)
    return z[:count]


def sketch_core(seed: int, n: int, l0: int, I: int, l1: int, tag: int = 0) -> np.ndarray:
    """Core n (1-based) of the random Gaussian TT of Def. 3.1, shape (l0, I, l1)."""
    cnt = l0 * I * l1
    z = philox_normal(cnt, seed, n, tag) * (1.0 / np.sqrt(float(cnt)))
    return z.reshape((l0, I, l1), order="F")
