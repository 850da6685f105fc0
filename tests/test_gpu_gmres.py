"""TT-GMRES (§4.2) through the C-ABI
against the oracle's tt_gmres (oracle/gmres.py) on the cookie surrogate:
the same rounding calls with the same Philox seeds, so both solvers take the
same Arnoldi steps.  Run with -m gpu."""
import numpy as np
import pytest
import torch

import oracle
import ttsynth
from oracle import gmres as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2110_04393_b200 as P
    return P.Context(0)


def to_dev(op):
    return [[None if A is None else torch.from_numpy(np.asarray(A)).cuda() for A in t] for t in op]


def gpu_tt(tt):
    return [torch.from_numpy(np.ascontiguousarray(c)).cuda() for c in tt]


def test_kron_apply_matches_oracle(ctx):
    rng = np.random.default_rng(0)
    dims = [6, 5, 7]
    op = [[rng.standard_normal((6, 6)), None, rng.standard_normal(7)],
          [None, rng.standard_normal((5, 5)), None],
          [rng.standard_normal(6), rng.standard_normal(5), rng.standard_normal((7, 7))]]
    X = [rng.standard_normal((r0, n, r1)) for r0, n, r1 in [(1, 6, 3), (3, 5, 4), (4, 7, 1)]]
    got = ctx.tt_kron_apply(to_dev(op), gpu_tt(X))
    want = G.kron_apply(op, X)
    for g, w in zip(got, want):
        for a, b in zip(g.numpy(), w):
            assert np.abs(a - b).max() <= 1e-13 * max(1.0, np.abs(b).max())


@pytest.mark.parametrize("cfg,randomized", [((16, 2, 4), True), ((16, 2, 4), False),
                                            ((32, 3, 8), True), ((32, 3, 8), False)])
def test_gmres_matches_oracle(ctx, cfg, randomized):
    g, p, s = cfg
    op, f, dims = ttsynth.cookie_surrogate(grid=g, params=p, samples=s)
    ref = G.tt_gmres(op, f, tol=1e-8, max_iter=60, randomized=randomized, seed=7)
    x, info = ctx.tt_gmres(to_dev(op), gpu_tt(f), tol=1e-8, max_iter=60, randomized=randomized,
                           seed=7)
    assert info["converged"] and ref.converged
    assert info["iters"] == ref.iters, (info["iters"], ref.iters)
    assert info["roundings"] == 2 * ref.iters + 1
    np.testing.assert_allclose(info["residuals"], ref.residuals, rtol=1e-5, atol=1e-12)
    X = x.numpy()
    assert oracle.rel_diff(X, ref.x) <= 1e-8
    if g == 16:   # and the dense direct solve of the assembled system
        K = G.kron_dense(op, dims)
        xd = np.linalg.solve(K, oracle.full(f).reshape(-1))
        assert np.linalg.norm(oracle.full(X).reshape(-1) - xd) <= 1e-6 * np.linalg.norm(xd)


def test_gmres_rejects_bad_operator(ctx):
    import paper_2110_04393_b200 as P
    op, f, dims = ttsynth.cookie_surrogate(grid=8, params=2, samples=3)
    bad = [t[:2] for t in op]
    with pytest.raises((P.TTError, ValueError)):
        ctx.tt_gmres(to_dev(bad), gpu_tt(f))
