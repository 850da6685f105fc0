"""Mode-slab sharding (SURVEY §8e alternative, §8f NEXT-2) of the Alg. 7 rounding
through the C-ABI (tt_round_sum_slab) on loopback ranks (one thread each, one GPU):
every rank holds all summands but a slab of every mode index; the slabs of the
result, concatenated along the mode axis, must equal the oracle's unsharded
rounding (<= 1e-10 in TT arithmetic) whatever the number of ranks."""
import numpy as np
import pytest
import torch

import oracle
import ttsynth
from test_gpu_sharded import run_ranks

pytestmark = pytest.mark.gpu
TOL = 1e-10


def split(I, world):
    """Contiguous, possibly uneven slabs of 0..I-1 (rank r gets [lo, hi))."""
    cuts = [(r * I) // world for r in range(world + 1)]
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def slab_run(terms, world, **kw):
    dims = [int(c.shape[1]) for c in terms[0]]
    g = [[ttsynth._move(c, "cuda") for c in t] for t in terms]
    parts = [split(I, world) for I in dims]

    def fn(ctx, r):
        lo = [parts[n][r][0] for n in range(len(dims))]
        loc = [[c[:, parts[n][r][0]:parts[n][r][1], :] for n, c in enumerate(t)] for t in g]
        res = ctx.tt_round_sum_slab(loc, dims, lo, seed=1, **kw)
        return res.ranks, res.numpy()

    out = run_ranks(world, fn)
    ranks = out[0][0]
    assert all(o[0] == ranks for o in out)
    X = [np.concatenate([o[1][n] for o in out], axis=1) for n in range(len(dims))]
    return ranks, X


@pytest.mark.parametrize("world", [1, 2, 3])
def test_slab_rounding_matches_oracle_rank_mode(world):
    w = ttsynth.config3_sum10(d=8, I=40, S=6)
    ref = oracle.round_sum([ttsynth.to_numpy(t) for t in w.terms], ell=w.ell, seed=1,
                           rank=w.rank)
    ranks, X = slab_run(w.terms, world, mode="rank", rank=w.rank, oversample=w.ell - w.rank)
    assert ranks[1:-1] == list(ref.ranks)
    assert oracle.rel_diff(X, ref.X) <= TOL


def test_slab_rounding_tolerance_mode_adaptive():
    w = ttsynth.config4_gmres(d=6, I=64, S=6)
    ref = oracle.round_sum([ttsynth.to_numpy(t) for t in w.terms], ell=w.ell, seed=1,
                           tol=w.tol, adaptive=True)
    ranks, X = slab_run(w.terms, 2, mode="tol", tol=w.tol, oversample=w.ell, adaptive=True)
    assert ranks[1:-1] == list(ref.ranks)
    assert oracle.rel_diff(X, ref.X) <= TOL


def test_slab_rounding_config5_shapes():
    """Config 5 shapes (S=32, I=256, summand rank 64, l=144 -> r=128) at d = 5 on
    4 ranks (64 mode indices each)."""
    w = ttsynth.config5_large(d=5)
    ref = oracle.round_sum([ttsynth.to_numpy(t) for t in w.terms], ell=w.ell, seed=1,
                           rank=w.rank)
    ranks, X = slab_run(w.terms, 4, mode="rank", rank=w.rank, oversample=w.ell - w.rank)
    assert ranks[1:-1] == list(ref.ranks)
    assert oracle.rel_diff(X, ref.X) <= TOL


def test_slabs_that_do_not_tile_fail_on_every_rank():
    import paper_2110_04393_b200 as P
    w = ttsynth.config3_sum10(d=4, I=10, S=2)
    g = [[ttsynth._move(c, "cuda") for c in t] for t in w.terms]

    def fn(ctx, r):
        loc = [[c[:, 0:5, :] for c in t] for t in g]    # both ranks claim slab 0..4
        try:
            ctx.tt_round_sum_slab(loc, [10] * 4, [0] * 4, mode="rank", rank=4, oversample=2)
            return None
        except P.TTError as e:
            return e.code

    codes = run_ranks(2, fn, timeout=120)
    assert all(c is not None and c < 0 for c in codes), codes
