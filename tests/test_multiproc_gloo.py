"""World-size-2 check of the summand-sharded sweep on CPU with gloo.

The CUDA path shards summands over ranks: phase 1 (Alg. 3) and the carries stay
local, every sweep step all-reduces the partial sketched core Y_n and
the last core, and the QR of Y_n is replicated.  This test runs that
exact decomposition with the oracle's primitives on two gloo processes and
checks it against the unsharded oracle Alg. 7 (oracle.round_sum_rand_orth),
plus the contiguous shard bounds that bench.py uses."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import ttsynth
from paper_2110_04393_b200.shard import shard_bounds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def sharded_alg7(local_terms, G, allreduce):
    """Alg. 7 with the summands split over ranks: Y_n and the last
    core are sums over summands, so each rank forms its partial
    sum and one all-reduce completes it; Q_n is then identical on every rank."""
    N = len(local_terms[0])
    Gc = [g if g is not None else np.zeros((1, 1, 1)) for g in G]
    Wj = [oracle.partial_contractions_rl(t, Gc) for t in local_terms]
    Xn = np.concatenate([t[0] for t in local_terms], axis=2)
    X = [None] * N
    for n in range(1, N):
        I = Xn.shape[1]
        Zn = oracle.V(Xn)
        Yn = allreduce(Zn @ np.concatenate([w[n] for w in Wj], axis=0))
        Q, _ = oracle.thin_qr(Yn)
        X[n - 1] = oracle.fold_V(Q, I)
        M = Q.T @ Zn
        offs = np.cumsum([0] + [t[n - 1].shape[2] for t in local_terms])
        Mj = [M[:, offs[j]:offs[j + 1]] for j in range(len(local_terms))]
        if n < N - 1:
            Xn = np.concatenate([oracle.fold_H(Mj[j] @ oracle.H(t[n]), t[n].shape[1])
                                 for j, t in enumerate(local_terms)], axis=2)
        else:
            last = sum(Mj[j] @ oracle.H(t[N - 1]) for j, t in enumerate(local_terms))
            X[N - 1] = oracle.fold_H(allreduce(last), local_terms[0][N - 1].shape[1])
    return X


def sharded_alg6(local_terms, L, R, allreduce):
    """Alg. 6 on the sum (R19) with the summands split over ranks, as
    tt_round_sum_two_sided does: W^L / W^R stay local, P_n = Σ_j W^L_j W^R_j is
    all-reduced, its SVD is replicated, and every output core X_n = Σ_j (…) is a
    sum over summands (one all-reduce each)."""
    N = len(local_terms[0])
    Lc = [g if g is not None else np.zeros((1, 1, 1)) for g in L]
    Rc = [g if g is not None else np.zeros((1, 1, 1)) for g in R]
    WL = [oracle.partial_contractions_lr(Lc, t) for t in local_terms]
    WR = [oracle.partial_contractions_rl(t, Rc) for t in local_terms]
    Lb, Rb = {}, {}
    for n in range(1, N):
        P = allreduce(sum(WL[j][n] @ WR[j][n] for j in range(len(local_terms))))
        U, s, Vt = np.linalg.svd(P, full_matrices=False)
        keep = s > oracle.pinv_rtol(P.shape) * s[0]
        sih = np.where(keep, 1.0 / np.sqrt(np.where(keep, s, 1.0)), 0.0)
        Lb[n] = [(WR[j][n] @ Vt.T) * sih[None, :] for j in range(len(local_terms))]
        Rb[n] = [sih[:, None] * (U.T @ WL[j][n]) for j in range(len(local_terms))]
    X = [None] * N
    I1 = local_terms[0][0].shape[1]
    X[0] = oracle.fold_V(allreduce(sum(oracle.V(t[0]) @ Lb[1][j]
                                       for j, t in enumerate(local_terms))), I1)
    for n in range(2, N):
        I = local_terms[0][n - 1].shape[1]
        X[n - 1] = allreduce(sum(
            oracle.fold_H(Rb[n - 1][j] @ oracle.H(oracle.fold_V(oracle.V(t[n - 1]) @ Lb[n][j], I)), I)
            for j, t in enumerate(local_terms)))
    IN = local_terms[0][N - 1].shape[1]
    X[N - 1] = oracle.fold_H(allreduce(sum(Rb[N - 1][j] @ oracle.H(t[N - 1])
                                           for j, t in enumerate(local_terms))), IN)
    return X


def _sketches_2s(terms, ell):
    dims = oracle.dims_of(terms[0])
    sumR = [1] + [sum(t[n].shape[2] for t in terms) for n in range(len(dims) - 1)] + [1]
    lc, rc = oracle.two_sided_ranks(dims, sumR, ell)
    return (oracle.gaussian_sketch_left(dims, lc, 2),
            oracle.gaussian_sketch(dims, rc, 2, tag=oracle.TAG_2S_R))


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = ttsynth.config3_sum10(d=5, I=12, S=5)
        terms = [ttsynth.to_numpy(t) for t in w.terms]
        lo, hi = shard_bounds(len(terms), world, rank)
        dims = oracle.dims_of(terms[0])
        sumR = [1] + [sum(t[n].shape[2] for t in terms) for n in range(len(dims) - 1)] + [1]
        G = oracle.gaussian_sketch(dims, oracle.rank_caps(dims, sumR, 9), seed=1)

        def allreduce(a):
            t = torch.from_numpy(np.ascontiguousarray(a))
            dist.all_reduce(t)          # fp64 sum, as ncclAllReduce in the CUDA path
            return t.numpy()

        X = sharded_alg7(terms[lo:hi], G, allreduce)
        L, R = _sketches_2s(terms, 7)
        X2 = sharded_alg6(terms[lo:hi], L, R, allreduce)
        out_q.put((rank, ([c.copy() for c in X], [c.copy() for c in X2])))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_cover_contiguously():
    for S in (1, 5, 10, 32):
        for world in (1, 2, 3, 8):
            b = [shard_bounds(S, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == S
            assert all(b[r][1] == b[r + 1][0] for r in range(world - 1))
            assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1


def test_sharded_alg7_and_alg6_world2_match_unsharded_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = ttsynth.config3_sum10(d=5, I=12, S=5)
    terms = [ttsynth.to_numpy(t) for t in w.terms]
    dims = oracle.dims_of(terms[0])
    sumR = [1] + [sum(t[n].shape[2] for t in terms) for n in range(len(dims) - 1)] + [1]
    G = oracle.gaussian_sketch(dims, oracle.rank_caps(dims, sumR, 9), seed=1)
    ref = oracle.round_sum_rand_orth(terms, G)
    for r in (0, 1):
        assert oracle.rel_diff(res[r][0], ref) <= 1e-12
    # replicated QR on identical all-reduced inputs: ranks agree bit for bit
    for a, b in zip(res[0][0], res[1][0]):
        assert np.array_equal(a, b)
    assert oracle.left_orth_residual(res[0][0]) < 1e-12
    # Alg. 6 (NEXT-3): sharded == unsharded oracle, identical on both ranks
    L, R = _sketches_2s(terms, 7)
    ref2 = oracle.round_sum_two_sided(terms, L, R)
    for r in (0, 1):
        assert oracle.rel_diff(res[r][1], ref2) <= 1e-12
    for a, b in zip(res[0][1], res[1][1]):
        assert np.array_equal(a, b)


# ---------------------------------------------------------------- mode-slab sharding (NEXT-2)
def _cholqr2_dist(Y, allreduce):
    """Thin Q of the row-distributed Y by CholeskyQR2 with all-reduced Grams (the
    distributed QR of tt_round_sum_slab): G = Σ_ranks Y_rᵀY_r, R = chol(G)ᵀ,
    Q_r = Y_r R⁻¹, twice."""
    for _ in range(2):
        G = allreduce(Y.T @ Y)
        R = np.linalg.cholesky(G).T
        Y = np.linalg.solve(R.T, Y.T).T
    return Y


def slab_alg7(terms, Gs, allreduce):
    """Alg. 7 with every core split into mode-index slabs over the ranks
    (all summands on every rank): Alg. 3's W_{n-1} = H(Z_n)H(G_n)ᵀ and line 11's
    M = QᵀV(X_n) contract the mode index -> partial sums + one all-reduce each; the
    QR of the row-distributed Y_n takes all-reduced Grams; carries stay local."""
    N = len(terms[0])
    Wj = []
    for t in terms:
        W = {N - 1: allreduce(oracle.H(t[N - 1]) @ oracle.H(Gs[N - 1]).T)}
        for n in range(N - 1, 1, -1):
            Z = oracle.fold_V(oracle.V(t[n - 1]) @ W[n], t[n - 1].shape[1])
            W[n - 1] = allreduce(oracle.H(Z) @ oracle.H(Gs[n - 1]).T)
        Wj.append(W)
    Xn = np.concatenate([t[0] for t in terms], axis=2)
    X = [None] * N
    for n in range(1, N):
        I = Xn.shape[1]
        Zn = oracle.V(Xn)
        Q = _cholqr2_dist(Zn @ np.concatenate([w[n] for w in Wj], axis=0), allreduce)
        X[n - 1] = oracle.fold_V(Q, I)
        M = allreduce(Q.T @ Zn)
        offs = np.cumsum([0] + [t[n - 1].shape[2] for t in terms])
        Mj = [M[:, offs[j]:offs[j + 1]] for j in range(len(terms))]
        if n < N - 1:
            Xn = np.concatenate([oracle.fold_H(Mj[j] @ oracle.H(t[n]), t[n].shape[1])
                                 for j, t in enumerate(terms)], axis=2)
        else:
            X[N - 1] = oracle.fold_H(sum(Mj[j] @ oracle.H(t[N - 1]) for j, t in enumerate(terms)),
                                     terms[0][N - 1].shape[1])
    return X


def _slab_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = ttsynth.config3_sum10(d=5, I=12, S=5)
        terms = [ttsynth.to_numpy(t) for t in w.terms]
        dims = oracle.dims_of(terms[0])
        sumR = [1] + [sum(t[n].shape[2] for t in terms) for n in range(len(dims) - 1)] + [1]
        G = oracle.gaussian_sketch(dims, oracle.rank_caps(dims, sumR, 9), seed=1)
        sl = [((rank * I) // world, ((rank + 1) * I) // world) for I in dims]
        loc = [[c[:, a:b, :] for c, (a, b) in zip(t, sl)] for t in terms]
        Gs = [None] + [g[:, a:b, :] for g, (a, b) in zip(G[1:], sl[1:])]

        def allreduce(a):
            t = torch.from_numpy(np.ascontiguousarray(a))
            dist.all_reduce(t)
            return t.numpy()

        X = slab_alg7(loc, Gs, allreduce)
        out_q.put((rank, [c.copy() for c in X]))
    finally:
        dist.destroy_process_group()


def test_slab_sharded_alg7_world2_matches_unsharded_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = ttsynth.config3_sum10(d=5, I=12, S=5)
    terms = [ttsynth.to_numpy(t) for t in w.terms]
    dims = oracle.dims_of(terms[0])
    sumR = [1] + [sum(t[n].shape[2] for t in terms) for n in range(len(dims) - 1)] + [1]
    G = oracle.gaussian_sketch(dims, oracle.rank_caps(dims, sumR, 9), seed=1)
    ref = oracle.round_sum_rand_orth(terms, G)
    X = [np.concatenate([res[0][n], res[1][n]], axis=1) for n in range(len(dims))]
    assert oracle.rel_diff(X, ref) <= 1e-12
    assert oracle.left_orth_residual(X) < 1e-12
