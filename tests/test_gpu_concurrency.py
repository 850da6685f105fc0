"""Several roundings in flight on one GPU (tt_ctx_set_concurrency).  The QR /
truncation chain (Alg. 7 line 10; truncation P:667-670) on a
highest-priority stream changes when kernels run, not what they compute: results
are bit-identical to the default context.  Persistent grids sized to fewer SMs
change summation orders (split-K slices, partial Grams): results equal to
rounding, and bit-identical between two contexts with the same setting driven
concurrently from two host threads and one after the other.  Run with -m gpu."""
import concurrent.futures as cf

import numpy as np
import pytest
import torch

import oracle
import ttsynth

pytestmark = pytest.mark.gpu


def _kw(w):
    if w.tol > 0:
        return dict(mode="tol", tol=w.tol, oversample=w.ell, adaptive=w.adaptive, rank=w.rank)
    return dict(mode="rank", rank=w.rank, oversample=w.ell - w.rank)


def _same(a, b):
    return len(a) == len(b) and all(x.shape == y.shape and np.array_equal(x, y)
                                    for x, y in zip(a, b))


@pytest.mark.parametrize("cfg", ["config2_single", "config3_sum10", "config4_gmres"])
def test_concurrency_mode_results(cfg):
    import paper_2110_04393_b200 as P
    w = getattr(ttsynth, cfg)(device="cuda")
    torch.cuda.synchronize()
    ref = P.Context(0, stream=torch.cuda.Stream()).tt_round_sum(w.terms, seed=7, **_kw(w))
    cx = P.Context(0, stream=torch.cuda.Stream())
    cx.set_concurrency(0, True)          # chain stream only: same bits
    got = cx.tt_round_sum(w.terms, seed=7, **_kw(w))
    assert got.ranks == ref.ranks
    assert _same(got.numpy(), ref.numpy())
    cx.set_concurrency(16, True)         # smaller persistent grids: other summation order
    got = cx.tt_round_sum(w.terms, seed=7, **_kw(w))
    assert got.ranks == ref.ranks
    assert oracle.rel_diff(got.numpy(), ref.numpy()) <= 1e-10
    if cfg != "config4_gmres":
        ora = oracle.round_sum([ttsynth.to_numpy(t) for t in w.terms], ell=w.ell, seed=7,
                               rank=w.rank)
        assert oracle.rel_diff(got.numpy(), ora.X) <= 1e-10


def test_two_concurrent_contexts_equal_sequential():
    import paper_2110_04393_b200 as P
    w = ttsynth.config3_sum10(device="cuda")
    torch.cuda.synchronize()
    seeds = [11, 12, 13, 14]
    base = P.Context(0, stream=torch.cuda.Stream())
    base.set_concurrency(12, True)
    ref = [base.tt_round_sum(w.terms, seed=s, **_kw(w)).numpy() for s in seeds]
    ctxs = [P.Context(0, stream=torch.cuda.Stream()) for _ in range(2)]
    for cx in ctxs:
        cx.set_concurrency(12, True)

    def lane(t):
        return [ctxs[t].tt_round_sum(w.terms, seed=seeds[b], **_kw(w)).numpy()
                for b in range(t, len(seeds), 2)]

    with cf.ThreadPoolExecutor(2) as ex:
        outs = list(ex.map(lane, range(2)))
    for t in range(2):
        for i, b in enumerate(range(t, len(seeds), 2)):
            assert _same(outs[t][i], ref[b])


def test_concurrency_arguments_checked():
    import paper_2110_04393_b200 as P
    cx = P.Context(0, stream=torch.cuda.Stream())
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    with pytest.raises(P.TTError):
        cx.set_concurrency(-1, True)
    with pytest.raises(P.TTError):
        cx.set_concurrency(sms, True)
    cx.set_concurrency(8, True)
    cx.set_concurrency(0, False)   # back to the default
    w = ttsynth.config1_tiny(device="cuda")
    r = cx.tt_round_sum(w.terms, seed=1, **_kw(w))
    ora = oracle.round_sum([ttsynth.to_numpy(t) for t in w.terms], ell=w.ell, seed=1,
                           rank=w.rank)
    assert oracle.rel_diff(r.numpy(), ora.X) <= 1e-10


def test_bench_concurrent_batched_line():
    """bench.py --batch B --streams k --reserve-sms R prints one contract line timed
    with CUDA events."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--workload", "sum10",
                          "--batch", "4", "--streams", "2", "--reserve-sms", "12", "--steps", "2",
                          "--warmup", "3", "--no-cpu"], capture_output=True, text=True,
                         timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["value"] > 0 and d["config"]["concurrency"]["reserve_sms"] == 12
