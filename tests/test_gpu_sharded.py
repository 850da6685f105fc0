"""The sharded (multi-rank) code path of libttround on one GPU.

Ranks are contexts of a loopback communicator (include/ttround.h
tt_loopback_create), one host thread each: every rank holds a contiguous shard
of the summands (paper_2110_04393_b200/shard.py), runs Alg. 3 on its own
summands, exchanges the partial sketched cores Y_n (Alg. 7 line 9) and
the last core (line 15) through the communicator, and must end with the
same tensor as the oracle's unsharded rounding (<= 1e-10 in TT arithmetic) and
identical bits on every rank.  A rank with no summands and a bad argument on one
rank are covered (every rank must return, never hang)."""
import concurrent.futures as cf

import numpy as np
import pytest
import torch

import oracle
import ttsynth

pytestmark = pytest.mark.gpu
TOL = 1e-10


def gpu_terms(terms):
    return [[ttsynth._move(c, "cuda") for c in t] for t in terms]


def run_ranks(world, fn, timeout=600):
    """fn(ctx, rank) on `world` loopback ranks, one thread + stream each."""
    import paper_2110_04393_b200 as P
    g = P.LoopbackGroup(world)
    torch.cuda.synchronize()

    def lane(r):
        st = torch.cuda.Stream()
        ctx = P.Context(0, stream=st, loopback=g, rank=r)
        try:
            return fn(ctx, r)
        finally:
            torch.cuda.synchronize()
            ctx.close()

    with cf.ThreadPoolExecutor(world) as ex:
        futs = [ex.submit(lane, r) for r in range(world)]
        out = [f.result(timeout=timeout) for f in futs]
    del g
    return out


def shards(S, world):
    from paper_2110_04393_b200.shard import shard_bounds
    return [shard_bounds(S, world, r) for r in range(world)]


def check_same_bits(results):
    X0 = results[0]
    for X in results[1:]:
        assert len(X) == len(X0)
        for a, b in zip(X, X0):
            assert a.shape == b.shape and np.array_equal(a, b)


@pytest.mark.parametrize("cfg,world", [("config3_sum10", 2), ("config3_sum10", 3),
                                       ("config4_gmres", 2)])
def test_sharded_round_sum_matches_oracle(cfg, world):
    w = getattr(ttsynth, cfg)()
    np_terms = [ttsynth.to_numpy(t) for t in w.terms]
    if w.tol > 0:
        kw = dict(mode="tol", tol=w.tol, oversample=w.ell, adaptive=w.adaptive)
        ref = oracle.round_sum(np_terms, ell=w.ell, seed=1, tol=w.tol, adaptive=w.adaptive)
    else:
        kw = dict(mode="rank", rank=w.rank, oversample=w.ell - w.rank)
        ref = oracle.round_sum(np_terms, ell=w.ell, seed=1, rank=w.rank)
    g = gpu_terms(w.terms)
    bounds = shards(len(g), world)

    def fn(ctx, r):
        lo, hi = bounds[r]
        res = ctx.tt_round_sum(g[lo:hi], seed=1, **kw)
        return res.ranks, res.numpy()

    out = run_ranks(world, fn)
    for ranks, X in out:
        assert ranks[1:-1] == list(ref.ranks)
        assert oracle.rel_diff(X, ref.X) <= TOL
    check_same_bits([X for _, X in out])


def test_rank_without_summands_contributes_zeros():
    """S = 2 summands on 3 ranks: rank 2 holds none (S_local = 0)."""
    w = ttsynth.config1_tiny()
    ref = oracle.round_sum([ttsynth.to_numpy(t) for t in w.terms], ell=w.ell, seed=1,
                           rank=w.rank)
    g = gpu_terms(w.terms)
    bounds = shards(len(g), 3)
    assert bounds[0][1] - bounds[0][0] == 0 or any(hi == lo for lo, hi in bounds)

    def fn(ctx, r):
        lo, hi = bounds[r]
        res = ctx.tt_round_sum(g[lo:hi], mode="rank", rank=w.rank,
                               oversample=w.ell - w.rank, seed=1)
        return res.numpy()

    out = run_ranks(3, fn)
    for X in out:
        assert oracle.rel_diff(X, ref.X) <= TOL
    check_same_bits(out)


def test_sharded_two_sided_matches_oracle():
    w = ttsynth.config3_sum10(d=8, I=30, S=6)
    ell = w.rank
    X2, _, _ = oracle.round_sum_2s([ttsynth.to_numpy(t) for t in w.terms], ell=ell, seed=1)
    g = gpu_terms(w.terms)
    bounds = shards(len(g), 2)

    def fn(ctx, r):
        lo, hi = bounds[r]
        return ctx.tt_round_sum_two_sided(g[lo:hi], ell=ell, seed=1).numpy()

    out = run_ranks(2, fn)
    for X in out:
        assert oracle.rel_diff(X, X2) <= TOL
    check_same_bits(out)


def test_bad_argument_on_one_rank_fails_every_rank():
    import paper_2110_04393_b200 as P
    w = ttsynth.config3_sum10(d=6, I=12, S=4)
    g = gpu_terms(w.terms)
    bad = gpu_terms(ttsynth.config3_sum10(d=6, I=13, S=2).terms)   # other mode size

    def fn(ctx, r):
        try:
            ctx.tt_round_sum(g[:2] if r == 0 else bad, mode="rank", rank=8, oversample=4)
            return None
        except P.TTError as e:
            return e.code

    codes = run_ranks(2, fn, timeout=120)
    assert all(c is not None and c < 0 for c in codes), codes

    def fn2(ctx, r):   # ranks disagree on the options
        try:
            ctx.tt_round_sum(g[2 * r:2 * r + 2], mode="rank", rank=8 + r, oversample=4)
            return None
        except P.TTError as e:
            return e.code

    codes = run_ranks(2, fn2, timeout=120)
    assert all(c is not None and c < 0 for c in codes), codes


def test_nccl_plumbing_one_rank():
    """The NCCL communicator of the world > 1 path (dlopen'd libnccl,
    ncclCommInitRank, the fp64-sum and int64 allreduce on the context's stream)
    with ONE rank, where a sum allreduce returns its input exactly."""
    import paper_2110_04393_b200 as P
    ctx = P.Context(0)
    for n in (0, 1, 144 * 64 + 3, 1 << 20):
        assert ctx.nccl_selftest(n) == 0.0
    with pytest.raises(P.TTError):
        ctx.nccl_selftest(-1)


@pytest.mark.parametrize("cfg", ["config3_sum10", "config4_gmres"])
def test_one_rank_nccl_context_runs_the_sharded_path(cfg):
    """tt_ctx_create with world == 1 AND an NCCL id: the sharded code path (agreed
    validation, ncclAllReduce of Y_n per sweep step; the last core)
    runs through a real one-rank NCCL communicator.  Same result as the oracle,
    and the same bits as the plain single-GPU context (a one-rank sum is exact)."""
    import paper_2110_04393_b200 as P
    w = getattr(ttsynth, cfg)()
    np_terms = [ttsynth.to_numpy(t) for t in w.terms]
    if w.tol > 0:
        kw = dict(mode="tol", tol=w.tol, oversample=w.ell, adaptive=w.adaptive)
        ref = oracle.round_sum(np_terms, ell=w.ell, seed=1, tol=w.tol, adaptive=w.adaptive)
    else:
        kw = dict(mode="rank", rank=w.rank, oversample=w.ell - w.rank)
        ref = oracle.round_sum(np_terms, ell=w.ell, seed=1, rank=w.rank)
    g = gpu_terms(w.terms)
    nc = P.Context(0, nccl_id=P.tt_get_nccl_unique_id(), rank=0, world=1)
    res = nc.tt_round_sum(g, seed=1, **kw)
    assert res.ranks[1:-1] == list(ref.ranks)
    X = res.numpy()
    assert oracle.rel_diff(X, ref.X) <= TOL
    plain = P.Context(0).tt_round_sum(g, seed=1, **kw).numpy()
    check_same_bits([X, plain])
    # two-sided (Alg. 6) and the mode-slab partition through the same communicator
    if w.tol == 0:
        r2 = nc.tt_round_sum_two_sided(g, ell=w.rank, seed=1)
        p2 = P.Context(0).tt_round_sum_two_sided(g, ell=w.rank, seed=1)
        assert oracle.rel_diff(r2.numpy(), p2.numpy()) <= TOL
    dims = [c.shape[1] for c in g[0]]
    rs = nc.tt_round_sum_slab(g, dims, [0] * len(dims), seed=1, **kw)
    assert rs.ranks[1:-1] == list(ref.ranks)
    assert oracle.rel_diff(rs.numpy(), ref.X) <= TOL
    nc.close()


def test_one_rank_nccl_context_bad_argument_returns():
    import paper_2110_04393_b200 as P
    nc = P.Context(0, nccl_id=P.tt_get_nccl_unique_id(), rank=0, world=1)
    with pytest.raises(P.TTError):
        nc.tt_round_sum([], mode="rank", rank=2, oversample=1, seed=1)
    nc.close()


def test_sharded_per_bond_target_ranks():
    """Per-bond target ranks (tt_round_opts.ranks, R24) with the summands sharded
    over 2 loopback ranks: same tensor as the unsharded oracle, same bits on both
    ranks; ranks that disagree on one entry (or on passing the array at all) all
    return an error."""
    import paper_2110_04393_b200 as P
    w = ttsynth.config3_sum10(d=6, I=20, S=4)
    ranks, p = [9, 25, 31, 17, 6], 6
    ref = oracle.round_sum([ttsynth.to_numpy(t) for t in w.terms],
                           ell=[r + p for r in ranks], seed=3, rank=ranks)
    g = gpu_terms(w.terms)

    def fn(ctx, r):
        res = ctx.tt_round_sum(g[2 * r:2 * r + 2], mode="rank", rank=ranks, oversample=p, seed=3)
        return res.ranks, res.numpy()

    out = run_ranks(2, fn)
    for rk, X in out:
        assert rk[1:-1] == list(ref.ranks) == ranks
        assert oracle.rel_diff(X, ref.X) <= TOL
    check_same_bits([X for _, X in out])

    def bad(ctx, r):
        rr = list(ranks)
        rr[2] += r
        try:
            ctx.tt_round_sum(g[2 * r:2 * r + 2], mode="rank", rank=rr, oversample=p, seed=3)
            return None
        except P.TTError as e:
            return e.code

    codes = run_ranks(2, bad, timeout=120)
    assert all(c is not None and c < 0 for c in codes), codes

    def bad2(ctx, r):
        try:
            ctx.tt_round_sum(g[2 * r:2 * r + 2], mode="rank", rank=ranks if r else 31,
                             oversample=p, seed=3)
            return None
        except P.TTError as e:
            return e.code

    codes = run_ranks(2, bad2, timeout=120)
    assert all(c is not None and c < 0 for c in codes), codes
