"""Pins for oracle/philox.py (CPU only).

* cuRAND's own curand_Philox4x32_10 (golden words written on the host by
  tests/golden/philox_kat.cu from /usr/local/cuda/include/curand_philox4x32_x.h).
* The three published Random123 known-answer vectors for philox4x32-10
  (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers: as easy as 1, 2, 3";
  kat_vectors of the Random123 distribution).
* Def. 3.1: entries N(0, 1/(ℓ_{n-1} I_n ℓ_n)) so that
  E‖R^(n)‖_F² = 1 ("This normalization is chosen such that E‖R^(n)‖²_F = 1").
"""
import math
import os

import numpy as np
import pytest
from scipy import stats

import oracle


GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")


def test_philox_matches_curand_golden():
    rows = [l.split() for l in open(GOLD) if l.strip() and not l.startswith("#")]
    assert len(rows) > 100
    for r in rows:
        s, k, n, t, *x = map(int, r)
        got = oracle.philox4x32_10(k & 0xFFFFFFFF, k >> 32, n, t, s & 0xFFFFFFFF, s >> 32)
        assert [int(v) for v in got] == x, r


@pytest.mark.parametrize("ctr,key,want", [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
])
def test_philox_random123_kat(ctr, key, want):
    got = oracle.philox4x32_10(*ctr, *key)
    assert tuple(int(v) for v in got) == want


def test_uniform_mapping_in_open_interval():
    # word pair (0,0) -> 0.5·2^-53 > 0, so ln(u1) is finite; (max,max) rounds
    # (ties-to-even, 2^53 - 0.5 -> 2^53) to exactly 1.0, where Box–Muller gives r = 0
    from oracle.philox import _unit
    lo = _unit(np.array([0], np.uint32), np.array([0], np.uint32))[0]
    hi = _unit(np.array([0xFFFFFFFF], np.uint32), np.array([0xFFFFFFFF], np.uint32))[0]
    assert lo == 0.5 * 2.0 ** -53 and 0 < lo
    assert hi == 1.0


def test_box_muller_pairs_share_radius():
    z = oracle.philox_normal(2000, seed=7, n=3)
    # (z_2k, z_2k+1) = r(cos θ, sin θ) with r² = -2 ln u1: each pair's radius is
    # recomputed independently from the same Philox words
    x0, x1, x2, x3 = oracle.philox4x32_10(np.arange(1000, dtype=np.uint32), 0, 3, 0, 7, 0)
    from oracle.philox import _unit
    r2 = -2.0 * np.log(_unit(x0, x1))
    th = 2 * np.pi * _unit(x2, x3)
    np.testing.assert_allclose(z[0::2] ** 2 + z[1::2] ** 2, r2, rtol=1e-13)
    np.testing.assert_allclose(np.arctan2(z[1::2], z[0::2]) % (2 * np.pi), th, rtol=0, atol=1e-12)


def test_standard_normal_distribution():
    z = oracle.philox_normal(200_000, seed=12345, n=2)
    assert abs(z.mean()) < 4 / math.sqrt(len(z))
    assert abs(z.var() - 1) < 4 * math.sqrt(2 / len(z))
    assert stats.kstest(z, "norm").pvalue > 1e-3
    # the two halves of a Box–Muller pair are independent
    assert abs(np.corrcoef(z[0::2], z[1::2])[0, 1]) < 4 / math.sqrt(len(z) / 2)


def test_def31_expected_core_norm_is_one():
    # sample mean of 1000 draws of a (4,8,4) core's squared norm is
    # within 3 standard errors of 1 (E‖R^(n)‖² = 1)
    v = np.array([np.sum(oracle.sketch_core(seed, 2, 4, 8, 4) ** 2) for seed in range(1000)])
    se = v.std(ddof=1) / math.sqrt(len(v))
    assert abs(v.mean() - 1.0) < 3 * se
    # variance of each entry is 1/(ℓ_{n-1} I_n ℓ_n)
    c = oracle.sketch_core(99, 5, 30, 40, 50)
    assert abs(c.var() * 30 * 40 * 50 - 1) < 4 * math.sqrt(2 / c.size)


def test_sketch_layout_order_and_independence_of_modes():
    c = oracle.sketch_core(3, 4, 5, 6, 7)
    z = oracle.philox_normal(5 * 6 * 7, 3, 4) * (1.0 / math.sqrt(5 * 6 * 7))
    # element (a,i,b) is stream element e = a + ℓ0(i + I b)
    for (a, i, b) in [(0, 0, 0), (4, 0, 0), (0, 5, 0), (2, 3, 6), (4, 5, 6)]:
        assert c[a, i, b] == z[a + 5 * (i + 6 * b)]
    other = oracle.sketch_core(3, 5, 5, 6, 7)
    assert not np.allclose(c, other)
    same = oracle.sketch_core(3, 4, 5, 6, 7)
    assert np.array_equal(c, same)
