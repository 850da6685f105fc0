"""One tt_round_deterministic call on a BASELINE config: phase timings and the
device status words (route counters: 8 CholQR2, 10 sCholQR3, 15 sCholQR4,
11 Householder, 14 TSQR; 12/13 Jacobi sweeps/calls).
python tools/run_det.py <workload> [d]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2110_04393_b200 as P
import ttsynth

name = sys.argv[1]
d = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
w = ttsynth.CONFIGS[name](device="cuda", **({"d": d} if d else {}))
ctx = P.Context(0, stream=torch.cuda.current_stream())
ctx.set_timing(True)
t0 = time.perf_counter()
r = ctx.tt_round_deterministic(w.terms, tol=w.tol if w.tol > 0 else 0.0,
                               rank=0 if w.tol > 0 else w.rank)
torch.cuda.synchronize()
print(name, d, "ranks", r.ranks[:5], "s", round(time.perf_counter() - t0, 3), "timing",
      [round(x, 1) for x in ctx.last_timing()], "status", ctx.status_words(20), flush=True)
