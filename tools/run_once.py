"""One tt_round_sum call on a (possibly reduced) BASELINE config, for ncu launch lists.

python tools/run_once.py <workload> [d] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2110_04393_b200 as P
import ttsynth

name = sys.argv[1]
d = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
fn = ttsynth.CONFIGS[name]
w = fn(device="cuda", **({"d": d} if d else {}))
ctx = P.Context(0, stream=torch.cuda.current_stream())
ctx.set_timing(True)
if w.tol > 0:
    kw = dict(mode="tol", tol=w.tol, oversample=w.ell, adaptive=w.adaptive)
else:
    kw = dict(mode="rank", rank=w.rank, oversample=w.ell - w.rank)
for _ in range(reps):
    r = ctx.tt_round_sum(w.terms, seed=1, **kw)
    print(name, d, "ranks", r.ranks[:4], "passes", r.passes, "flags", r.flags, "timing",
          [round(x, 3) for x in ctx.last_timing()], "status", ctx.status_words(64), flush=True)
