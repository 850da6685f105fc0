"""CUDA-graph plans (tt_plan_create / tt_plan_launch): B rank-mode roundings of the
small configs captured in one graph and replayed give exactly the results of the
eager tt_round_sum calls with the same sketch seeds.  Run with -m gpu."""
import numpy as np
import pytest
import torch

import oracle
import ttsynth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,branches", [("config1_tiny", 1), ("config1_tiny", 3),
                                          ("config2_single", 2)])
def test_plan_replays_equal_eager_roundings(cfg, branches):
    import paper_2110_04393_b200 as P
    st = torch.cuda.Stream()
    ctx = P.Context(0, stream=st)
    w = getattr(ttsynth, cfg)(device="cuda")
    torch.cuda.synchronize()
    seeds = [3, 4, 5, 6]
    kw = dict(mode="rank", rank=w.rank, oversample=w.ell - w.rank)
    plan = P.Plan(ctx, w.terms, seeds, branches=branches, **kw)
    for _ in range(2):
        plan.launch()
    for b, sd in enumerate(seeds):
        got = plan.result(b).numpy()
        ref = ctx.tt_round_sum(w.terms, seed=sd, **kw).numpy()
        assert oracle.rel_diff(got, ref) <= 1e-13
        ora = oracle.round_sum([ttsynth.to_numpy(t) for t in w.terms], ell=w.ell, seed=sd,
                               rank=w.rank)
        assert oracle.rel_diff(got, ora.X) <= 1e-10


def test_plan_rejects_tolerance_mode_and_default_stream():
    import paper_2110_04393_b200 as P
    w = ttsynth.config1_tiny(device="cuda")
    ctx = P.Context(0, stream=torch.cuda.Stream())
    with pytest.raises(P.TTError):
        P.Plan(ctx, w.terms, [1], mode="tol")
    ctx2 = P.Context(0, stream=torch.cuda.default_stream())
    with pytest.raises(P.TTError):
        P.Plan(ctx2, w.terms, [1], mode="rank", rank=w.rank, oversample=2)


def test_bench_batched_graph_line():
    """bench.py --batch B --graph --streams k prints one contract line."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--workload", "tiny",
                          "--batch", "16", "--graph", "--streams", "4", "--steps", "2",
                          "--warmup", "3", "--no-cpu"], capture_output=True, text=True,
                         timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["value"] > 0 and d["config"]["cuda_graph"] and d["config"]["graph_branches"] == 4
