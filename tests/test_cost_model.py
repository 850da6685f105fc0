"""Pins of the metric's flop accounting against the paper's cost formulas (CPU)."""
import pytest

from paper_2110_04393_b200 import cost


def test_exact_count_reproduces_paper_leading_order():
    # uniform ranks, large I: the exact count approaches I(N-2)(4sR²l + 6sRl² + 4l³)
    N, I, R, ell, s = 50, 256, 64, 144, 32
    dims = [I] * N
    tr = [[1] + [R] * (N - 1) + [1]] * s
    l = cost.caps(dims, [1] + [s * R] * (N - 1) + [1], ell)
    f = cost.rounding_flops(dims, tr, l)
    ref = cost.paper_rto_sum(N, I, R, ell, s)
    assert abs(f["total"] / ref - 1) < 0.03       # boundary cores + QR -4n³/3 terms
    # C5 canonical total 4.21e12, phase 1 1.51e12
    assert abs(f["total"] - 4.21e12) / 4.21e12 < 0.01
    assert abs(f["phase1"] - 1.51e12) / 1.51e12 < 0.01


def test_phase1_is_s_times_contraction_cost():
    # App. A: C_Contr = I(N-2)(2Rl² + 2R²l) per summand
    N, I, R, ell, s = 20, 100, 60, 70, 10
    dims = [I] * N
    tr = [[1] + [R] * (N - 1) + [1]] * s
    l = [1] + [ell] * (N - 1) + [1]
    f = cost.rounding_flops(dims, tr, l)
    lead = s * I * (N - 2) * (2 * R * ell ** 2 + 2 * R ** 2 * ell)
    exact_extra = s * 2 * R * I * ell                      # line 2 (order IRl)
    assert f["phase1"] == pytest.approx(lead + exact_extra, rel=1e-12)


def test_table1_ratio_at_half():
    # SPEC S:604 / Table 1: TT-Rounding / Rand-then-Orth = 2.125 at beta = 0.5
    t = cost.table1_simplified(0.5)
    assert t["tt_rounding"] / t["rand_then_orth"] == pytest.approx(2.125)


def test_caps_match_oracle_rule():
    import oracle
    dims = [4, 4, 4, 4]
    assert cost.caps(dims, [1, 6, 6, 6, 1], 6) == [1] + oracle.rank_caps(dims, [1, 6, 6, 6, 1], 6) + [1]


@pytest.mark.parametrize("rho_factor", [1.0, 1.5])
def test_two_sided_count_matches_paper(rho_factor):
    """Alg. 6 on one TT: Table 1's (6β + 6β²)(N-2)IR³ for ρ = ℓ and
    P:944's I(N-2)(7R²ℓ + 8.5Rℓ²) for ρ = 1.5ℓ, to leading order."""
    N, I, R, ell = 60, 300, 80, 40
    rho = int(rho_factor * ell)
    dims = [I] * N
    tr = [[1] + [R] * (N - 1) + [1]]
    sumR = [1] + [R] * (N - 1) + [1]
    f = cost.two_sided_flops(dims, tr, cost.caps(dims, sumR, ell), cost.caps(dims, sumR, rho))
    if rho_factor == 1.0:
        beta = ell / R
        lead = cost.table1_simplified(beta)["two_sided"] * (N - 2) * I * R ** 3
    else:
        lead = I * (N - 2) * (7.0 * R * R * ell + 8.5 * R * ell * ell)
    assert f["total"] / lead == pytest.approx(1.0, abs=0.03)
    assert cost.paper_two_sided(N, I, R, ell, rho) == pytest.approx(lead, rel=1e-12)
