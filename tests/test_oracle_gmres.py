"""Pins for oracle/gmres.py (TT-GMRES, §4.2) against dense
linear algebra: the assembled Kronecker-sum matrix, a dense direct solve, and the
textbook GMRES special cases.  CPU only."""
import numpy as np
import pytest

import oracle
import ttsynth
from oracle import gmres as G


def rnd_tt(rng, dims, ranks):
    return [rng.standard_normal((ranks[n], dims[n], ranks[n + 1])) for n in range(len(dims))]


def test_kron_apply_matches_assembled_matrix():
    rng = np.random.default_rng(0)
    dims = [4, 3, 5]
    op = [[rng.standard_normal((4, 4)), None, rng.standard_normal(5)],
          [None, rng.standard_normal((3, 3)), None],
          [rng.standard_normal(4), rng.standard_normal(3), rng.standard_normal((5, 5))]]
    X = rnd_tt(rng, dims, [1, 2, 3, 1])
    terms = G.kron_apply(op, X)
    assert len(terms) == 3
    got = sum(oracle.full(t) for t in terms).reshape(-1)
    want = G.kron_dense(op, dims) @ oracle.full(X).reshape(-1)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
    # each term keeps the ranks of X (rank-preserving factors)
    assert all(oracle.ranks_of(t) == oracle.ranks_of(X) for t in terms)


def test_preconditioner_is_the_inverse_mode1_mean_operator():
    op, f, dims = ttsynth.cookie_surrogate(grid=8, params=2, samples=3)
    P = G.precond_matrix(op, dims[0])
    M = sum(t[0] for t in op)
    assert np.allclose(P @ M, np.eye(dims[0]), atol=1e-12)
    rng = np.random.default_rng(1)
    X = rnd_tt(rng, dims, [1, 2, 2, 1])
    got = oracle.full(G.apply_precond(P, X)).reshape(-1)
    K = np.kron(np.kron(P, np.eye(dims[1])), np.eye(dims[2]))
    want = K @ oracle.full(X).reshape(-1)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def test_surrogate_is_symmetric_positive_definite():
    op, f, dims = ttsynth.cookie_surrogate(grid=16, params=2, samples=4)
    K = G.kron_dense(op, dims)
    assert np.allclose(K, K.T)
    assert np.linalg.eigvalsh(K).min() > 0


def test_identity_operator_converges_in_one_iteration():
    rng = np.random.default_rng(2)
    dims = [5, 4, 3]
    f = rnd_tt(rng, dims, [1, 2, 2, 1])
    op = [[None, None, None]]
    r = G.tt_gmres(op, f, tol=1e-10, precond=False, randomized=False)
    assert r.iters == 1 and r.converged
    assert oracle.diff_norm(r.x, f) <= 1e-9 * oracle.norm(f)


@pytest.mark.parametrize("randomized", [False, True])
def test_gmres_matches_dense_direct_solve(randomized):
    """Surrogate with N = 3 modes, 16 x 4 x 4 unknowns: the TT-GMRES solution equals
    the dense direct solve of the assembled Kronecker-sum system."""
    op, f, dims = ttsynth.cookie_surrogate(grid=16, params=2, samples=4)
    r = G.tt_gmres(op, f, tol=1e-8, max_iter=40, randomized=randomized, seed=3)
    assert r.converged, r.residuals[-3:]
    K = G.kron_dense(op, dims)
    xd = np.linalg.solve(K, oracle.full(f).reshape(-1))
    xt = oracle.full(r.x).reshape(-1)
    assert np.linalg.norm(xt - xd) <= 1e-6 * np.linalg.norm(xd)
    # residual estimates are nonincreasing (least squares over a growing space)
    assert all(b <= a * (1 + 1e-6) for a, b in zip(r.residuals, r.residuals[1:]))


def test_randomized_and_deterministic_take_the_same_iterations():
    """"the ranks of the basis vectors and number of iterations are the
    same using both implementations" (here within one iteration)."""
    op, f, dims = ttsynth.cookie_surrogate(grid=16, params=2, samples=4)
    a = G.tt_gmres(op, f, tol=1e-8, max_iter=40, randomized=False)
    b = G.tt_gmres(op, f, tol=1e-8, max_iter=40, randomized=True, seed=5)
    assert abs(a.iters - b.iters) <= 1
