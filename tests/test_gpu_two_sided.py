"""Parity of tt_round_sum_two_sided (Alg. 6 on a sum, CUDA through the C-ABI)
with the oracle's round_sum_2s on identical inputs and the same Philox seeds.
Metric as for Alg. 7: ‖X_gpu − X_oracle‖ / ‖X_oracle‖ in TT arithmetic (R12),
bar 1e-10 (BASELINE.json).  Run with -m gpu."""
import math

import numpy as np
import pytest
import torch

import oracle
import ttsynth

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def ctx():
    import paper_2110_04393_b200 as P
    return P.Context(0)


def gpu_terms(terms):
    return [[ttsynth._move(c, "cuda") for c in t] for t in terms]


def run_2s(ctx, terms, ell, rho=0, seed=1, host=False, tol=TOL):
    ref, lc, rc = oracle.round_sum_2s([ttsynth.to_numpy(t) for t in terms], ell, rho, seed)
    res = ctx.tt_round_sum_two_sided(terms if host else gpu_terms(terms), ell, rho, seed)
    X = res.numpy()
    assert res.ranks == oracle.ranks_of(ref), (res.ranks, oracle.ranks_of(ref))
    r = oracle.rel_diff(X, ref)
    assert r <= tol, r
    return res, X, ref, lc, rc


def test_config1_tiny(ctx):
    w = ttsynth.config1_tiny()
    res, X, ref, lc, rc = run_2s(ctx, w.terms, 4)
    assert lc == [4, 4, 4] and rc == [4, 6, 4]


def test_config2_single(ctx):
    w = ttsynth.config2_single()
    res, X, ref, lc, rc = run_2s(ctx, w.terms, w.rank)
    assert rc[5] == math.ceil(1.5 * w.rank)


def test_config3_sum10(ctx):
    w = ttsynth.config3_sum10()
    run_2s(ctx, w.terms, w.rank)


def test_config4_gmres(ctx):
    w = ttsynth.config4_gmres()
    run_2s(ctx, w.terms, 80)


def test_config5_shapes_reduced_depth(ctx):
    # config 5 per-core shapes (S=32, I=256, summand rank 64, l=128, rho=192) at d=5
    w = ttsynth.config5_large(d=5)
    res, X, ref, lc, rc = run_2s(ctx, w.terms, w.rank)
    assert lc == [128] * 4 and rc == [192] * 4


@pytest.mark.parametrize("seed", [11, 12])
def test_ragged_summand_ranks_and_dims(ctx, seed):
    dims = [3, 11, 5, 7, 2, 13]
    rng = np.random.default_rng(seed)
    tr = [[1] + [int(x) for x in rng.integers(1, 9, size=len(dims) - 1)] + [1] for _ in range(5)]
    terms = ttsynth.random_terms(seed, dims, tr)
    run_2s(ctx, terms, 6)
    run_2s(ctx, terms, 5, rho=11, seed=3)


def test_general_svd_path_above_160(ctx):
    # bond 2 has l = 175 > 160 (rho capped at sum R = 180): the Jacobi that
    # accumulates its rotations factors W^L W^R instead of QR + V-free Jacobi
    terms = ttsynth.random_terms(41, [14, 14, 14, 14], [[1, 14, 30, 14, 1]] * 6)
    res, X, ref, lc, rc = run_2s(ctx, terms, 175)
    assert lc[1] == 175 and rc[1] == 180


def test_exact_recovery_of_rank_deficient_sum(ctx):
    a = ttsynth.random_terms(51, [6, 5, 6, 5], [[1, 2, 3, 2, 1]])[0]
    b = ttsynth.random_terms(52, [6, 5, 6, 5], [[1, 3, 2, 2, 1]])[0]
    terms = [a, a, b]
    res, X, ref, lc, rc = run_2s(ctx, terms, 6)
    S = oracle.tt_add([ttsynth.to_numpy(t) for t in terms])
    assert oracle.rel_diff(X, S) < 1e-12


def test_zero_sum(ctx):
    import paper_2110_04393_b200 as P
    Z = [torch.zeros((1, 4, 2), dtype=torch.float64), torch.zeros((2, 4, 2), dtype=torch.float64),
         torch.zeros((2, 4, 1), dtype=torch.float64)]
    res = ctx.tt_round_sum_two_sided(gpu_terms([Z, Z]), 2)
    assert res.ranks == [1, 1, 1, 1] and res.flags & P.FLAG_ZERO
    assert all(not np.any(c) for c in res.numpy())


def test_two_modes_single_summand_and_unit_ranks(ctx):
    run_2s(ctx, ttsynth.random_terms(3, [17, 9], [[1, 5, 1]]), 3)
    run_2s(ctx, ttsynth.random_terms(4, [5, 6, 7], [[1, 1, 1, 1]] * 3), 2)


def test_host_inputs_are_staged(ctx):
    w = ttsynth.config3_sum10(d=6, I=40, S=3)
    pinned = [[c.permute(2, 1, 0).contiguous().pin_memory().permute(2, 1, 0) for c in t]
              for t in w.terms]
    run_2s(ctx, pinned, 30, host=True)


def test_more_summands_than_one_gemm_batch(ctx):
    terms = ttsynth.random_terms(61, [4, 5, 4, 5], [[1, 2, 2, 2, 1]] * 70)
    run_2s(ctx, terms, 12)


def test_determinism_bitwise(ctx):
    w = ttsynth.config3_sum10(d=5, I=30, S=4)
    t = gpu_terms(w.terms)
    a = ctx.tt_round_sum_two_sided(t, 20, seed=4).numpy()
    b = ctx.tt_round_sum_two_sided(t, 20, seed=4).numpy()
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_errors_are_reported(ctx):
    import paper_2110_04393_b200 as P
    terms = ttsynth.random_terms(1, [4, 4, 4], [[1, 2, 2, 1], [1, 2, 2, 1]])
    with pytest.raises(P.TTError) as e:
        ctx.tt_round_sum_two_sided(gpu_terms(terms), 4, rho=3)
    assert e.value.code == -1
    with pytest.raises(P.TTError):
        ctx.tt_round_sum_two_sided(gpu_terms(terms), 0)


def test_config5_full_size_in_bench_launch_configuration():
    """Config 5 at full size (S=32, d=50, I=256, summand rank 64; l = 128,
    rho = 192) in bench.py's launch configuration (library on torch's current
    stream), against the oracle's Alg. 6 on the host (round_sum_2s, minutes) in
    TT arithmetic at the 1e-10 bar -- the depth at which the bond scaling and the
    output gauge rebalancing matter (DESIGN.md §6 "Two-sided design")."""
    import paper_2110_04393_b200 as P
    w = ttsynth.config5_large()
    c = P.Context(0, stream=torch.cuda.current_stream())
    res = c.tt_round_sum_two_sided(gpu_terms(w.terms), w.rank, seed=1)
    X = res.numpy()
    assert res.ranks == [1] + [w.rank] * (w.d - 1) + [1]
    del res
    ref, _, _ = oracle.round_sum_2s([ttsynth.to_numpy(t) for t in w.terms], w.rank, 0, 1)
    assert oracle.ranks_of(ref) == [1] + [w.rank] * (w.d - 1) + [1]
    r = oracle.rel_diff(X, ref)
    assert r <= TOL, r
