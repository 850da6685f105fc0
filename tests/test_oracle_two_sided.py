"""Pins for the oracle's Alg. 6 (Two-Sided-Randomization; SURVEY §8f
NEXT-3) against things other than itself: dense brute force of the partial
contractions Ψ_n V(Y^{1:n}) and H(Y^{n+1:N}) Ω_n, the textbook
generalized Nyström formula for matrices, the dense bond-projector
form of the result, exact recovery when ℓ reaches the true TT rank,
and the stacking identity of a sum.  CPU only."""
import math

import numpy as np
import pytest

import oracle


def rnd_tt(rng, dims, ranks, scale=1.0):
    return [rng.standard_normal((ranks[n], dims[n], ranks[n + 1])) * scale
            for n in range(len(dims))]


def dense_left(tt, n):
    """Dense V(X^{1:n}) ((Π_{k≤n} I_k) × R_n), n 1-based, by brute-force contraction."""
    t = np.asarray(tt[0])[0]
    for c in tt[1:n]:
        t = np.tensordot(t, c, axes=([t.ndim - 1], [0]))
    return t.reshape(-1, t.shape[-1])


def dense_right(tt, n):
    """Dense H(X^{n+1:N}) (R_n × Π_{k>n} I_k), n 1-based."""
    t = tt[n]
    for c in tt[n + 1:]:
        t = np.tensordot(t, c, axes=([t.ndim - 1], [0]))
    return t[..., 0].reshape(t.shape[0], -1)


def sketches(dims, sumR, ell, rho=0, seed=3):
    lc, rc = oracle.two_sided_ranks(dims, sumR, ell, rho)
    return (oracle.gaussian_sketch_left(dims, lc, seed),
            oracle.gaussian_sketch(dims, rc, seed, tag=oracle.TAG_2S_R), lc, rc)


def sum_ranks(terms):
    N = len(terms[0])
    return [1] + [sum(t[n].shape[2] for t in terms) for n in range(N - 1)] + [1]


def test_partial_contractions_lr_against_dense():
    rng = np.random.default_rng(1)
    dims = [3, 4, 2, 5]
    X = rnd_tt(rng, dims, [1, 2, 3, 4, 1])
    Y = rnd_tt(rng, dims, [1, 3, 2, 3, 1])
    W = oracle.partial_contractions_lr(X, Y)
    assert sorted(W) == [1, 2, 3]
    for n in (1, 2, 3):
        ref = dense_left(X, n).T @ dense_left(Y, n)
        assert W[n].shape == (X[n - 1].shape[2], Y[n - 1].shape[2])
        assert np.allclose(W[n], ref, rtol=1e-13, atol=1e-12)


def test_matrix_case_is_generalized_nystrom():
    """N = 2: X = AΩ(ΨAΩ)†ΨA with Ψ = V(𝓛_1)ᵀ, Ω = H(𝓡_2)ᵀ."""
    rng = np.random.default_rng(2)
    dims = [9, 11]
    Y = rnd_tt(rng, dims, [1, 7, 1])
    L, R, lc, rc = sketches(dims, [1, 7, 1], 4)
    assert lc == [4] and rc == [6]
    A = oracle.full(Y)
    Psi = np.asarray(L[0])[0].T               # ℓ × I_1
    Om = np.asarray(R[1])[:, :, 0].T          # I_2 × ρ
    ref = A @ Om @ np.linalg.pinv(Psi @ A @ Om) @ Psi @ A
    X = oracle.round_two_sided(Y, L, R)
    assert [c.shape[2] for c in X[:-1]] == [4]
    assert np.linalg.norm(oracle.full(X) - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("ell", [3, 4])
def test_sum_matches_dense_bond_projectors(ell):
    """Σ_j Y^(j) with P_n = W^R_n (W^L_n W^R_n)† W^L_n inserted at every bond
    (P:812-818), every W formed densely from the full unfoldings."""
    rng = np.random.default_rng(3 + ell)
    dims = [3, 4, 3, 4]
    terms = [rnd_tt(rng, dims, [1, 3, 3, 3, 1]) for _ in range(2)]
    Ysum = oracle.tt_add(terms)
    sr = sum_ranks(terms)
    L, R, lc, rc = sketches(dims, sr, ell)
    X = oracle.round_sum_two_sided(terms, L, R)
    cores = []
    for n in range(1, len(dims) + 1):
        c = np.asarray(Ysum[n - 1])
        if n < len(dims):
            WL = dense_left(L, n).T @ dense_left(Ysum, n)
            WR = dense_right(Ysum, n) @ dense_right(R, n).T
            P = WR @ np.linalg.pinv(WL @ WR) @ WL
            c = np.tensordot(c, P, axes=([2], [0]))
        cores.append(c)
    ref = oracle.full(cores)
    assert [c.shape[2] for c in X[:-1]] == lc
    assert np.linalg.norm(oracle.full(X) - ref) <= 1e-11 * np.linalg.norm(ref)


def test_exact_recovery_at_true_rank_with_rank_deficient_core():
    """ΣR = 6 but the sum A + A + B has TT rank 4: W^L W^R is rank deficient and
    the pseudo-inverse cutoff (R20) must drop its null direction; generalized
    Nyström is then exact."""
    rng = np.random.default_rng(5)
    dims = [4, 4, 4, 4]
    A = rnd_tt(rng, dims, [1, 2, 2, 2, 1])
    B = rnd_tt(rng, dims, [1, 2, 2, 2, 1])
    X, lc, rc = oracle.round_sum_2s([A, A, B], ell=5, seed=7)
    assert lc == [4, 5, 4] and rc == [4, 6, 4]
    ref = oracle.tt_add([A, A, B])
    assert oracle.rel_diff(X, ref) <= 1e-12


def test_sum_equals_alg6_on_assembled_sum():
    rng = np.random.default_rng(6)
    dims = [5, 3, 4, 3, 5]
    terms = [rnd_tt(rng, dims, [1, 2, 3, 3, 2, 1]) for _ in range(3)]
    sr = sum_ranks(terms)
    L, R, lc, rc = sketches(dims, sr, 4)
    X1 = oracle.round_sum_two_sided(terms, L, R)
    X2 = oracle.round_two_sided(oracle.tt_add(terms), L, R)
    assert oracle.rel_diff(X1, X2) <= 1e-12
    assert oracle.ranks_of(X1) == [1] + lc + [1]


def test_error_tracks_perturbation():
    """X = Y + δZ with TT rank(Y) = ℓ: the two-sided result's error is O(δ)
    (generalized Nyström is exact on Y)."""
    rng = np.random.default_rng(8)
    dims = [6, 6, 6, 6]
    Y = rnd_tt(rng, dims, [1, 3, 3, 3, 1])
    Z = rnd_tt(rng, dims, [1, 2, 2, 2, 1])
    ny = oracle.norm(Y)
    errs = []
    for delta in (1e-4, 1e-8):
        Xs, lc, rc = oracle.round_sum_2s([Y, oracle.tt_scale(Z, delta)], ell=3, seed=9)
        errs.append(oracle.diff_norm(Xs, Y) / ny)
    assert errs[0] < 1e-2 and errs[1] < 1e-6
    assert 1e2 < errs[0] / errs[1] < 1e6   # scales like δ


def test_ranks_default_rho_and_order():
    lc, rc = oracle.two_sided_ranks([8] * 6, [1, 50, 50, 50, 50, 50, 1], 20)
    assert rc[2] == math.ceil(1.5 * 20) == 30
    assert all(a <= b for a, b in zip(lc, rc))
    assert lc == [8, 20, 20, 20, 8] and rc == [8, 30, 30, 30, 8]
    with pytest.raises(ValueError):
        oracle.two_sided_ranks([8] * 4, [1, 9, 9, 9, 1], 10, rho=5)


def test_zero_sum_gives_zero_tensor():
    rng = np.random.default_rng(10)
    dims = [3, 3, 3]
    A = rnd_tt(rng, dims, [1, 2, 2, 1])
    A[1][:] = 0.0
    X, lc, rc = oracle.round_sum_2s([A, A], ell=2)
    assert oracle.ranks_of(X) == [1, 1, 1, 1]
    assert not any(np.any(c) for c in X)


def test_sketch_streams_are_distinct():
    dims = [4, 5, 6]
    L = oracle.gaussian_sketch_left(dims, [3, 3], seed=1)
    R = oracle.gaussian_sketch(dims, [3, 3], seed=1, tag=oracle.TAG_2S_R)
    G = oracle.gaussian_sketch(dims, [3, 3], seed=1)
    assert L[2] is None and R[0] is None
    assert L[0].shape == (1, 4, 3) and L[1].shape == (3, 5, 3)
    assert not np.allclose(R[1], G[1]) and not np.allclose(L[1], R[1])
    # Def. 3.1 scaling: entries N(0, 1/(ℓ_{n-1} I_n ℓ_n))
    big = oracle.gaussian_sketch_left([50, 40, 2], [30, 2], seed=4)
    assert abs(np.var(big[1]) * 30 * 40 * 2 - 1.0) < 0.1
