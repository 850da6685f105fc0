#!/usr/bin/env python
"""Benchmark of the hot path: one step = one tt_round_sum call (Alg. 7 + the
truncation to rank r) on BASELINE.json's large config (config 5, reading "C":
S=32 summands, d=50, I=256, summand rank 64, sketch rank 144 -> rank 128).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                  [--workload large|sum10|gmres|single|tiny] [--algo rand_orth|two_sided]

--algo two_sided times tt_round_sum_two_sided (Alg. 6) on the
same inputs with l = the config's target rank and rho = ceil(1.5 l).

N>1 runs under torchrun, one process per GPU; the summands are sharded across
ranks and each sweep step allreduces the partial sketched core Y_n over NCCL
(strong scaling of one rounding).  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TT sum-roundings/sec and FP64 TFLOP/s (fraction of peak) at 1/2/4/8 B200"
WORKLOADS = {
    "large": dict(cfg="config5_large", args={}, desc="config 5 (reading C): S=32, d=50, I=256, "
                  "summand rank 64 (signal 96 + 16/summand noise at 1e-6), sketch 144, rank 128"),
    "sum10": dict(cfg="config3_sum10", args={}, desc="config 3: S=10, d=20, I=100, rank 60, sketch 70"),
    "gmres": dict(cfg="config4_gmres", args={}, desc="config 4: S=20, d=12, I=128, rank 40, tol 1e-8, adaptive from 80"),
    "single": dict(cfg="config2_single", args={}, desc="config 2: S=1, d=16, I=64, rank 50 -> 25, sketch 35"),
    "tiny": dict(cfg="config1_tiny", args={}, desc="config 1: S=2, d=4, I=4, rank 3 each -> 4, sketch 6"),
}


def fp64_peak():
    """FP64 tensor (DMMA) peak: MEASURED_PEAKS.json if it has one, else this repo's
    own all-SM DMMA microbenchmark (profiles/fp64_peak.json, tools/fp64_peak.cu)."""
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        v = json.load(open(mp)).get("fp64_tflops")
        if v:
            return float(v), "MEASURED_PEAKS.json fp64_tflops"
    except Exception:
        pass
    p = os.path.join(ROOT, "profiles", "fp64_peak.json")
    try:
        v = json.load(open(p))
        return float(v["fp64_dmma_tflops"]), "measured DMMA.8x8x4 all-SM microbenchmark (profiles/fp64_peak.json)"
    except Exception:
        return 40.0, "datasheet-class FP64 tensor figure (no measurement available)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


CONFIG_SHAPES = {   # (S, d, I, sketch rank, rank, tol) of each workload (ttsynth recipes)
    "large": (32, 50, 256, 144, 128, 0.0), "sum10": (10, 20, 100, 70, 60, 0.0),
    "gmres": (20, 12, 128, 80, 0, 1e-8), "single": (1, 16, 64, 35, 25, 0.0),
    "tiny": (2, 4, 4, 6, 4, 0.0),
}


def bench_config(name, algo, world):
    """The `config` object of the JSON line; identical for both arms."""
    S, d, I, ell, r, tol = CONFIG_SHAPES[name]
    l2 = "L2 (126 MB) flushed by the inputs themselves: inputs %s than L2" % (
        "larger" if name in ("large", "sum10", "gmres") else "smaller (cache-resident; no flush)")
    if algo == "two_sided":
        a = "two_sided (Alg. 6): l = %d, rho = %d" % (r or ell, (3 * (r or ell) + 1) // 2)
    elif algo == "deterministic":
        a = "deterministic (Alg. 1 + 2 on the assembled sum)"
    else:
        a = "rand_orth (Alg. 7 + truncation)"
    return {"workload": name, "desc": WORKLOADS[name]["desc"], "summands": S, "d": d, "I": I,
            "sketch_rank": ell, "rank": r, "tol": tol, "parallelism": f"summands/{world}",
            "algo": a, "l2": l2}


def make_workload(name, device, seed_offset=0):
    import ttsynth
    w = WORKLOADS[name]
    fn = getattr(ttsynth, w["cfg"])
    return fn(device=device, **w["args"])


def two_sided_ell(wl):
    """Alg. 6's target rank for a workload: the config's rank (else its sketch rank)."""
    return int(wl.rank) if wl.rank else int(wl.ell)


def shapes_of(wl):
    """(global mode sizes, per-summand ranks) of a workload, before any sharding."""
    return (list(wl.dims),
            [[int(t[0].shape[0])] + [int(c.shape[2]) for c in t] for t in wl.terms])


def flops_of(wl, ranks_out, algo="rand_orth", shapes=None):
    from paper_2110_04393_b200 import cost
    dims, tr = shapes if shapes is not None else shapes_of(wl)
    if algo == "deterministic":
        return {"total": None, "phase1": None}, None
    sumR = [sum(r[n] for r in tr) for n in range(len(dims) + 1)]
    if algo == "two_sided":
        ell = two_sided_ell(wl)
        l = cost.caps(dims, sumR, ell)
        return cost.two_sided_flops(dims, tr, l, cost.caps(dims, sumR, (3 * ell + 1) // 2)), l
    l = cost.caps(dims, sumR, wl.ell)
    kept = ranks_out if (wl.tol > 0 or (wl.rank and any(x > wl.rank for x in l[1:-1]))) else None
    return cost.rounding_flops(dims, tr, l, kept), l


def _cores_used():
    try:
        from threadpoolctl import threadpool_info
        return max([x.get("num_threads", 1) for x in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count()


def _oracle_round(terms, wl, algo):
    import oracle
    if algo == "two_sided":
        _, lc, _ = oracle.round_sum_2s(terms, ell=two_sided_ell(wl), seed=1)
        return lc
    r = oracle.round_sum(terms, ell=wl.ell, seed=1, rank=wl.rank, tol=wl.tol,
                         adaptive=wl.adaptive)
    return list(r.ranks)


def large_bond_sample(seed=5):
    """Full-shape sample of config 5 for the oracle: the S = 32 summands cut to a
    3-mode chain whose left boundary carries the interior sketch rank
    (cores 144x256x64, 64x256x64, 64x256x1), so Alg. 3, the Alg. 7 sweep and the
    truncation each run at exactly config 5's per-bond shapes: one interior bond
    (m = 144*256 rows, sum R = 2048) plus the last bond.  Returns (terms, flops
    of the sample, flops of the full rounding)."""
    import numpy as np
    from paper_2110_04393_b200 import cost
    S, I, R, ell, r = 32, 256, 64, 144, 128
    rng = np.random.default_rng(seed)
    sd = 1.0 / math.sqrt(R * I)
    terms = [[rng.standard_normal((ell, I, R)) * sd, rng.standard_normal((R, I, R)) * sd,
              rng.standard_normal((R, I, 1)) * sd] for _ in range(S)]
    f_s = cost.rounding_flops([I] * 3, [[ell, R, R, 1]] * S, [ell, ell, ell, 1],
                              kept=[ell, r, r, 1])["total"]
    d = 50
    tr = [[1] + [R] * (d - 1) + [1]] * S
    l = cost.caps([I] * d, [sum(x[n] for x in tr) for n in range(d + 1)], ell)
    f_f = cost.rounding_flops([I] * d, tr, l, [1] + [r] * (d - 1) + [1])["total"]
    return terms, f_s, f_f


def cpu_oracle_sample(name, algo="rand_orth", reps=1):
    """The oracle (as it stands) on a bounded sample of the workload, timed on the
    host cores.  Config 5: the full-shape bond sample of large_bond_sample(),
    scaled to one rounding by the exact flop ratio; the smaller configs: complete
    roundings of the full config.  Returns (roundings/s, description, cores,
    seconds per sample)."""
    import oracle
    import ttsynth
    w = WORKLOADS[name]
    if name == "large" and algo != "two_sided":
        terms, f_s, f_f = large_bond_sample()
        t0 = time.perf_counter()
        for _ in range(reps):
            oracle.round_sum(terms, ell=144, seed=1, rank=128)
        dt = (time.perf_counter() - t0) / reps
        rate = 1.0 / (dt * f_f / f_s)
        desc = (f"oracle (NumPy fp64, BLAS/LAPACK steps) on a full-shape sample of {w['desc']}: "
                f"S=32 summands as a 3-mode chain 144x256x64 | 64x256x64 | 64x256x1 (one interior "
                f"bond + the last bond at exactly config 5's shapes; {f_s / 1e9:.1f} GFLOP), "
                f"{dt:.2f} s per sample ({f_s / dt / 1e9:.1f} GFLOP/s), scaled to one d=50 "
                f"rounding by the exact flop ratio {f_f / f_s:.2f}")
        return rate, desc, _cores_used(), dt
    if name == "large":   # Alg. 6: the same chain trick does not apply; reduced order d = 4
        wl = getattr(ttsynth, w["cfg"])(device="cpu", d=4)
    else:
        wl = getattr(ttsynth, w["cfg"])(device="cpu")
    terms = [ttsynth.to_numpy(t) for t in wl.terms]
    t0 = time.perf_counter()
    for _ in range(reps):
        ranks_s = _oracle_round(terms, wl, algo)
    dt = (time.perf_counter() - t0) / reps
    rate = 1.0 / dt
    desc = (f"oracle{' Alg. 6' if algo == 'two_sided' else ''} (NumPy fp64, BLAS/LAPACK steps): "
            f"complete rounding(s) of {w['desc']}, {dt:.2f} s each")
    if name == "large":
        fs, _ = flops_of(wl, [1] + ranks_s + [1], algo)
        full = make_workload_shapes_flops(algo)
        rate = 1.0 / (dt * full / fs["total"])
        desc += f" at d=4, scaled to d=50 by the exact flop ratio {full / fs['total']:.2f}"
    return rate, desc, _cores_used(), dt


def make_workload_shapes_flops(algo):
    from paper_2110_04393_b200 import cost
    d, S, I, R, ell = 50, 32, 256, 64, 128
    tr = [[1] + [R] * (d - 1) + [1]] * S
    sumR = [sum(x[n] for x in tr) for n in range(d + 1)]
    return cost.two_sided_flops([I] * d, tr, cost.caps([I] * d, sumR, ell),
                                cost.caps([I] * d, sumR, (3 * ell + 1) // 2))["total"]


def cpu_oracle_full(wl, algo="rand_orth"):
    """One complete rounding of the benchmarked workload (the same input bits the
    GPU rounded, copied to the host) by the oracle as it stands: a measurement of
    the full config, no scaling.  Returns (roundings/s, description, cores, s)."""
    import ttsynth
    terms = [ttsynth.to_numpy(t) for t in wl.terms]
    t0 = time.perf_counter()
    _oracle_round(terms, wl, algo)
    dt = time.perf_counter() - t0
    del terms
    return 1.0 / dt, ("oracle (NumPy fp64, BLAS/LAPACK steps): one complete rounding of the "
                      f"benchmarked inputs (full config, no scaling), {dt:.1f} s"), _cores_used(), dt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="large", choices=list(WORKLOADS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", action="store_true",
                    help="cpu_baseline from the bounded full-shape sample instead of one "
                         "complete oracle rounding of the benchmarked inputs")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--batch", type=int, default=1,
                    help="B independent roundings per step (distinct sketch seeds), spread "
                         "over --streams contexts (SURVEY 8d batched throughput of C1/C2)")
    ap.add_argument("--streams", type=int, default=1)
    ap.add_argument("--inflight", type=int, default=1,
                    help="K independent roundings in flight per GPU per step (K contexts on "
                         "K streams, one host thread each, tt_ctx_set_concurrency(--reserve-sms "
                         "or 16, 1)); each is a complete rounding of the same input sum with "
                         "its own sketch seed")
    ap.add_argument("--reserve-sms", type=int, default=-1,
                    help="--batch without --graph: tt_ctx_set_concurrency(reserve_sms, "
                         "chain_priority=1) on every context (persistent grids leave this "
                         "many SMs to the other roundings' QR/truncation chains, which run "
                         "on a highest-priority stream); -1: off")
    ap.add_argument("--graph", action="store_true",
                    help="--batch: capture the B roundings in one CUDA graph (tt_plan_create) "
                         "and replay it per step (rank mode)")
    ap.add_argument("--shard", default="summands", choices=["summands", "slab"],
                    help="N>1 partition: summands (SURVEY 8e, the default) or mode slabs "
                         "of every summand (tt_round_sum_slab, NEXT-2)")
    ap.add_argument("--algo", default="rand_orth",
                    choices=["rand_orth", "two_sided", "deterministic"],
                    help="rand_orth: tt_round_sum (Alg. 7 + truncation, the headline); "
                         "two_sided: tt_round_sum_two_sided (Alg. 6); deterministic: "
                         "tt_round_deterministic (Alg. 1 + 2 on the assembled sum, the "
                         "paper's baseline; one GPU, no flop accounting)")
    ap.add_argument("--e2e-lanes", type=int, default=2,
                    help="N=1: also report the e2e metric with this many calls in flight "
                         "(e2e.pipelined; 1 disables it)")
    ap.add_argument("--e2e-reserve-sms", type=int, default=-1,
                    help="e2e.pipelined lanes: tt_ctx_set_concurrency(reserve, chain priority) "
                         "(-1: plain contexts)")
    ap.add_argument("--nccl-one-rank", action="store_true",
                    help="N=1 only: give the context a ONE-rank NCCL communicator so the "
                         "sharded path's exchange steps (ncclAllReduce of Y_n per sweep step, "
                         "agreed validation) run on a one-GPU box; reported in config")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N` without a launcher: re-run this command under
        # torchrun with one process per GPU (the driver's own launch form)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one process per GPU")

    if args.impl == "reference":
        return reference_arm(args, world, rank)
    if args.batch > 1 or args.graph:
        return batched_run(args, world, rank, local)

    import torch
    import torch.distributed as dist
    import paper_2110_04393_b200 as P

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    wl = make_workload(args.workload, dev)
    S = len(wl.terms)
    shapes = shapes_of(wl)
    from paper_2110_04393_b200.shard import shard_bounds
    slab = args.shard == "slab"
    if slab:
        # every rank: all summands, the mode-index slab [lo_n, hi_n) of every core
        lo, hi = 0, S
        gdims = [int(c.shape[1]) for c in wl.terms[0]]
        slab_lo = [(rank * I) // world for I in gdims]
        slab_hi = [((rank + 1) * I) // world for I in gdims]
        local_terms = [[c[:, a:b, :].permute(2, 1, 0).contiguous().permute(2, 1, 0)
                        for c, a, b in zip(t, slab_lo, slab_hi)] for t in wl.terms]
        wl.terms.clear()
    else:
        lo, hi = shard_bounds(S, world, rank)
        local_terms = wl.terms[lo:hi]
        for t in wl.terms[:lo] + wl.terms[hi:]:
            t.clear()
    torch.cuda.synchronize()

    nccl_id = None
    if world > 1:
        obj = [P.tt_get_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    elif args.nccl_one_rank:
        nccl_id = P.tt_get_nccl_unique_id()
    K = max(1, args.inflight)
    if K > 1 and (args.algo != "rand_orth" or slab):
        raise SystemExit("--inflight > 1: rand_orth with summand shards only")
    if K > 1 and world > 1:
        # one communicator per lane: created in lane order on every rank
        ids = [P.tt_get_nccl_unique_id() if rank == 0 else None for _ in range(K)]
        dist.broadcast_object_list(ids, src=0)
    else:
        ids = [nccl_id] * K
    lane_streams = [torch.cuda.current_stream(dev)] if K == 1 else \
        [torch.cuda.Stream(dev) for _ in range(K)]
    ctxs = [P.Context(local, stream=lane_streams[t], nccl_id=ids[t], rank=rank, world=world)
            for t in range(K)]
    reserve = args.reserve_sms if args.reserve_sms >= 0 else 16
    for cx in ctxs:
        cx.set_timing(True)
        if K > 1:
            cx.set_concurrency(reserve, True)
    ctx = ctxs[0]
    if wl.tol > 0:
        kw = dict(mode="tol", tol=wl.tol, oversample=wl.ell, adaptive=wl.adaptive, rank=wl.rank)
    else:
        kw = dict(mode="rank", rank=wl.rank, oversample=wl.ell - wl.rank)

    two_sided = args.algo == "two_sided"
    determ = args.algo == "deterministic"
    if determ and world > 1:
        raise SystemExit("--algo deterministic runs on one GPU")

    def call(terms, cx=ctx, seed=1):
        if determ:
            return cx.tt_round_deterministic(terms, tol=wl.tol, rank=0 if wl.tol > 0 else wl.rank)
        if two_sided:
            return cx.tt_round_sum_two_sided(terms, ell=two_sided_ell(wl), rho=0, seed=seed)
        if slab:
            return cx.tt_round_sum_slab(terms, gdims, slab_lo, seed=seed, **kw)
        return cx.tt_round_sum(terms, seed=seed, **kw)

    lane_phase = [[0.0] * 8 for _ in range(K)]
    pool = None
    if K > 1:
        import concurrent.futures as cf
        pool = cf.ThreadPoolExecutor(K)

    def lane(t):
        r = call(local_terms, ctxs[t], seed=1 + t)
        for i, x in enumerate(ctxs[t].last_timing()):
            lane_phase[t][i] += x
        return r

    def step():
        return call(local_terms)

    def run_lanes(nsteps, stagger_s):
        """K host threads, each running nsteps roundings back to back on its own
        context (no barrier between steps); lane t starts t * stagger_s late, so
        one lane's latency-bound QR/truncation chain overlaps another's GEMMs."""
        def body(t):
            if t and stagger_s > 0:
                time.sleep(t * stagger_s)
            r = None
            for _ in range(nsteps):
                r = lane(t)
            return r
        return list(pool.map(body, range(K)))[0]

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    res = None
    stagger = 0.0
    if K == 1:
        for _ in range(max(3, args.warmup)):
            res = step()
    else:
        res = lane(0)                      # one rounding alone: its latency sets the stagger
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = lane(0)
        stagger = (time.perf_counter() - t0) / K
        res = run_lanes(max(3, args.warmup), stagger)
    ranks_out = res.ranks
    del res
    barrier()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    phase = [0.0] * 8
    for lp in lane_phase:
        lp[:] = [0.0] * 8
    n_l0 = P.tt_launch_count()
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for st in lane_streams[1:] if K == 1 else lane_streams:
            st.wait_event(e0)
        if K == 1:
            for _ in range(args.steps):
                r = step()
                t = ctx.last_timing()
                for i in range(len(t)):
                    phase[i] += t[i]
                del r
        else:
            del_r = run_lanes(args.steps, stagger)
            del del_r
        if K > 1:   # end after every lane stream's last work
            for st in lane_streams:
                stream.wait_event(st.record_event())
            # per-rounding phase times: the mean over the lanes (each lane's own
            # events on its own stream, so they include the sharing of the GPU)
            phase = [sum(lp[i] for lp in lane_phase) / K for i in range(8)]
        e1.record(stream)
        barrier()
    launches = P.tt_launch_count() - n_l0
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        ph = torch.tensor(phase, device=dev, dtype=torch.float64)
        dist.all_reduce(ph, op=dist.ReduceOp.MAX)
        phase = ph.tolist()
    phase = [p / args.steps for p in phase]

    fl, l = flops_of(wl, ranks_out, args.algo, shapes)
    peak, peak_src = fp64_peak()
    value = 1000.0 * K / ms                   # roundings/s (K roundings per step, all ranks)
    tflops = K * fl["total"] / (ms * 1e-3) / 1e12 if fl["total"] else None
    # dominant kernel family: the phase-1 DMMA contractions (Alg. 3), timed live
    p1_ms = phase[1]
    share = (1.0 / world) if slab else (hi - lo) / S
    p1_flops_local = fl["phase1"] * share if fl["phase1"] else None
    p1_achieved = p1_flops_local / (p1_ms * 1e-3) / 1e12 if (p1_ms > 0 and p1_flops_local) else None

    e2e = None
    if not args.no_e2e:
        e2e = e2e_run(args, call, local_terms, dev, world, dist if world > 1 else None)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not determ:
        if args.cpu_sample:
            rate, desc, cores, _ = cpu_oracle_sample(args.workload, algo=args.algo)
        else:
            rate, desc, cores, _ = cpu_oracle_full(wl, algo=args.algo)
        cpu = {"value": rate, "unit": "roundings/s", "cores": cores, "kind": "oracle",
               "sample": desc}

    if rank == 0:
        traffic = traffic_kernel = None
        prof = os.path.join(ROOT, "profiles", "traffic.json")
        try:
            tr = json.load(open(prof)).get(args.workload + ("_two_sided" if two_sided else ""))
            traffic, traffic_kernel = tr["bytes_per_launch"], tr["kernel"]
        except Exception:
            pass
        line = {
            "metric": METRIC, "value": value, "unit": "roundings/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (ttsynth, seeded; DESIGN.md input recipe)",
            "config": dict(bench_config(args.workload, args.algo, world),
                           **({"parallelism": f"mode-slabs/{world}"} if slab else {}),
                           **({"exchange": "one-rank NCCL communicator (ncclAllReduce per "
                                           "sweep step)"} if args.nccl_one_rank and world == 1
                              else {}),
                           **({"inflight": K, "concurrency": {"reserve_sms": reserve,
                                                              "chain_priority": True},
                               "step": f"{K} independent roundings of the input sum (sketch "
                                       f"seeds 1..{K}), one context + stream + host thread each; "
                                       "lanes run back to back without a barrier between steps, "
                                       "lane t started t/K of a rounding's latency late; timed from "
                                       "before the first lane's first call to after every lane's "
                                       "last"}
                              if K > 1 else {})),
            "tflops": tflops, "fp64_peak_tflops": peak, "fp64_peak_source": peak_src,
            "frac_of_fp64_peak": tflops / peak if tflops else None,
            "flops_per_rounding": fl,
            "phase_ms": ({"sketches": phase[0], "right_contractions": phase[1],
                          "left_contraction_and_assembly": phase[2], "bond_qr_svd": phase[3],
                          "collectives": phase[4], "bond_factors": phase[5], "total": phase[6]}
                         if two_sided else
                         {"sketch": phase[0], "phase1_contractions": phase[1],
                          "sweep_gemms": phase[2], "qr": phase[3], "collectives": phase[4],
                          "truncation": phase[5], "total": phase[6]}),
            "roofline": {"bound": "tensor", "kernel": "dgemm_tma_kernel + pgemm_kernel (phase-1 Alg. 3 contractions, TMA-fed DMMA.8x8x4)"
                         + (" with the right sketch (rho)" if two_sided else ""),
                         "achieved": p1_achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": (p1_achieved / peak) if p1_achieved else None,
                         "traffic": traffic, "traffic_kernel": traffic_kernel,
                         "traffic_source": "profiles/traffic.json (ncu --set full, DRAM bytes per launch)",
                         "algorithmic": "phase-1 flops = sum_j [2 R I l + sum_n (2 R^2 I l + 2 R I l^2)] (SURVEY 8d)"},
            "gpu_launches": launches,
            "ranks_out": ranks_out,
            "clocks": clk.summary(),
        }
        if e2e is not None:
            line["e2e"] = e2e
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def batched_run(args, world, rank, local):
    """B independent roundings per step on one GPU (replicas across GPUs): the
    same input sum rounded with sketch seeds 1..B by `--streams` library
    contexts (one CUDA stream each) driven from host threads, so latency-bound
    kernels of one rounding overlap with the others.  Timed by the host clock
    between device-wide synchronisations (several streams)."""
    import concurrent.futures as cf
    import torch
    import torch.distributed as dist
    import paper_2110_04393_b200 as P
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    wl = make_workload(args.workload, dev)
    ns = max(1, min(args.streams, args.batch))
    graph = args.graph and wl.tol == 0
    if graph:
        ns = 1
    lane_streams = [torch.cuda.Stream(dev) for _ in range(ns)]
    ctxs = [P.Context(local, stream=lane_streams[t]) for t in range(ns)]
    conc = args.reserve_sms >= 0 and not graph
    if conc:
        for cx in ctxs:
            cx.set_concurrency(args.reserve_sms, True)
    if wl.tol > 0:
        kw = dict(mode="tol", tol=wl.tol, oversample=wl.ell, adaptive=wl.adaptive, rank=wl.rank)
    else:
        kw = dict(mode="rank", rank=wl.rank, oversample=wl.ell - wl.rank)
    B = args.batch
    n0 = P.tt_launch_count()
    ex = cf.ThreadPoolExecutor(ns)
    plan = None
    if graph:
        torch.cuda.synchronize()
        plan = P.Plan(ctxs[0], wl.terms, [1 + b for b in range(B)],
                      branches=max(1, args.streams), **kw)
        ranks_plan = plan.result(0).ranks

    def lane(t):
        if plan is not None:
            plan.launch()
            return ranks_plan
        r = None
        for b in range(t, B, ns):
            r = ctxs[t].tt_round_sum(wl.terms, seed=1 + b, **kw)
        return r.ranks

    def step():
        return list(ex.map(lane, range(ns)))

    for _ in range(max(3, args.warmup)):
        ranks_out = step()[0]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    n0 = P.tt_launch_count()
    # device time: every lane stream starts after e0 (current stream) and the
    # current stream records e1 after every lane stream's last work
    cur = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        e0.record(cur)
        for st in lane_streams:
            st.wait_event(e0)
        for _ in range(args.steps):
            step()
        for st in lane_streams:
            cur.wait_event(st.record_event())
        e1.record(cur)
        torch.cuda.synchronize()
        dt_host = (time.perf_counter() - t0) / args.steps
        dt = e0.elapsed_time(e1) * 1e-3 / args.steps
    launches = P.tt_launch_count() - n0
    if world > 1:
        tt = torch.tensor([dt], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    fl, _ = flops_of(wl, ranks_out)
    peak, peak_src = fp64_peak()
    value = B * world / dt
    tf = fl["total"] * B * world / dt / 1e12
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "roundings/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (ttsynth, seeded; DESIGN.md input recipe)",
            "config": {"workload": args.workload, "desc": WORKLOADS[args.workload]["desc"],
                       "batch_per_gpu": B, "streams": ns, "parallelism": f"replicas/{world}",
                       "cuda_graph": bool(graph),
                       "graph_branches": max(1, args.streams) if graph else None,
                       "concurrency": ({"reserve_sms": args.reserve_sms, "chain_priority": True}
                                       if conc else None),
                       "timing": "CUDA events: start on the current stream, every lane stream "
                                 "waits on it, end after every lane stream's last work",
                       "host_ms_per_step": dt_host * 1e3},
            "tflops": tf, "fp64_peak_tflops": peak, "fp64_peak_source": peak_src,
            "roofline": {"bound": "tensor", "kernel": "whole path (batched, latency-bound)",
                         "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
                         "traffic": None},
            "gpu_launches": launches, "ranks_out": ranks_out, "clocks": clk.summary(),
        }))
    ex.shutdown()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def e2e_run(args, call, local_terms, dev, world, dist):
    """Same metric through the C-ABI with HOST (pinned) buffers: the H2D copies of
    the inputs happen inside the call (overlapped with phase 1) and the result is
    read back D2H into pinned memory, both inside the timed region."""
    import torch
    host = [[c.permute(2, 1, 0).contiguous().cpu().pin_memory().permute(2, 1, 0) for c in t]
            for t in local_terms]
    h2d = sum(c.numel() * 8 for t in host for c in t)
    r = call(host)
    outs = [torch.empty((r.ranks[n + 1], r.dims[n], r.ranks[n]), dtype=torch.float64).pin_memory()
            for n in range(r.d)]
    d2h = sum(o.numel() * 8 for o in outs)
    del r
    import ctypes
    from paper_2110_04393_b200 import _lib
    L = _lib.load_library()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    dsts = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        r = call(host)
        _lib._check(L.tt_tensor_copy_all(r._h.ptr, dsts))
        del r
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / args.e2e_steps
    if dist:
        tt = torch.tensor([dt], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    # the host link itself: a plain pinned H2D copy of 2 GiB (context for the floor)
    probe = torch.empty(2 ** 28, dtype=torch.float64).pin_memory()
    dprobe = torch.empty_like(probe, device=dev)
    dprobe.copy_(probe, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    dprobe.copy_(probe, non_blocking=True)
    torch.cuda.synchronize()
    link = probe.numel() * 8 / (time.perf_counter() - t1) / 1e9
    del probe, dprobe
    pipelined = None
    if not dist and args.e2e_lanes > 1:
        pipelined = e2e_pipelined(args, call, host, outs, dev, dt)
    del host
    return {"value": 1.0 / dt, "unit": "roundings/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
            "h2d_link_gbs": link, "h2d_floor_ms": h2d / link / 1e6,
            **({"pipelined": pipelined} if pipelined else {}),
            "note": "host-clock over the whole call incl. H2D staging and D2H of the result; "
                    "the H2D of every core precedes the sweep (phase 1 needs all of them), so "
                    "e2e >= h2d_floor + sweep + truncation"}


def e2e_pipelined(args, call, host, outs0, dev, period_s):
    """The e2e metric with `--e2e-lanes` calls in flight (N = 1): each lane is a host
    thread with its own context and stream, rounding the same HOST inputs (its own
    sketch seed) and reading its result back into its own pinned buffers, steps back
    to back.  One lane's H2D staging (copy engine) then overlaps another lane's sweep
    and truncation (SMs): throughput is bounded by max(host link, GPU time) instead
    of their sum.  Lane t starts t/K of a sequential call's time (period_s) late:
    lanes started together stay in lockstep (both staging, then both computing) and
    overlap nothing.  Every step still copies its inputs H2D and its result D2H
    inside the timed region."""
    import concurrent.futures as cf
    import ctypes
    import torch
    import paper_2110_04393_b200 as P
    from paper_2110_04393_b200 import _lib
    L = _lib.load_library()
    K = args.e2e_lanes
    n = max(4, args.e2e_steps)
    ctxs = [P.Context(dev.index, stream=torch.cuda.Stream(dev)) for _ in range(K)]
    if args.e2e_reserve_sms >= 0:     # as --inflight: leave SMs to the other lane's chain
        for cx in ctxs:
            cx.set_concurrency(args.e2e_reserve_sms, True)
    outs = [outs0] + [[torch.empty_like(o).pin_memory() for o in outs0] for _ in range(K - 1)]
    dsts = [(ctypes.c_void_p * len(o))(*[x.data_ptr() for x in o]) for o in outs]

    def one(t):
        r = call(host, ctxs[t], 1 + t)
        _lib._check(L.tt_tensor_copy_all(r._h.ptr, dsts[t]))
        del r

    for t in range(K):            # warm-up: every lane's workspaces and staging pools
        one(t)
    torch.cuda.synchronize()

    def body(t):
        if t:
            time.sleep(t * period_s / K)
        for _ in range(n):
            one(t)

    with cf.ThreadPoolExecutor(K) as pool:
        t0 = time.perf_counter()
        list(pool.map(body, range(K)))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    for cx in ctxs:
        cx.close()
    return {"value": K * n / dt, "unit": "roundings/s", "lanes": K, "steps_per_lane": n,
            **({"concurrency": {"reserve_sms": args.e2e_reserve_sms, "chain_priority": True}}
               if args.e2e_reserve_sms >= 0 else {}),
            "note": f"{K} calls in flight on {K} contexts (host threads), started "
                    f"1/{K} of a call apart; H2D of one call overlaps the sweep and "
                    "truncation of another; the timed region includes the stagger"}


def reference_arm(args, world, rank):
    """--impl reference: the oracle (as it stands) on the host cores, rank 0 only
    (other ranks exit without work).  Each step is one bounded sample of the
    workload (cpu_oracle_sample: for config 5 the full-shape bond sample, for the
    smaller configs one complete rounding); ms_per_step is the observed time of
    one such sample, value = roundings/s after the stated scaling."""
    if rank != 0:
        return
    desc = cores = None
    for _ in range(args.warmup):
        cpu_oracle_sample(args.workload, algo=args.algo)
    dts, rates = [], []
    for _ in range(args.steps):
        rate, desc, cores, dt = cpu_oracle_sample(args.workload, algo=args.algo)
        dts.append(dt)
        rates.append(rate)
    ms = 1000.0 * statistics.mean(dts)
    value = statistics.mean(rates)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "roundings/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": bench_config(args.workload, args.algo, world),
        "cpu_baseline": {"value": value, "unit": "roundings/s", "cores": cores,
                         "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": "roundings/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))


if __name__ == "__main__":
    main()
