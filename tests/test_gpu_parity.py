"""End-to-end parity of tt_round_sum (CUDA, through the C-ABI) against the oracle.

Both sides get identical input bits (ttsynth) and the same Philox sketch seed.
The metric is the relative difference ‖X_gpu − X_oracle‖ / ‖X_oracle‖ computed
in TT arithmetic by orthogonalising [X_gpu, −X_oracle] (R12), with the
north-star bar 1e-10 (BASELINE.json).  Run with -m gpu."""
import math

import numpy as np
import pytest
import torch

import oracle
import ttsynth

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def ctx():
    import paper_2110_04393_b200 as P
    return P.Context(0)


def gpu_terms(terms):
    return [[ttsynth._move(c, "cuda") for c in t] for t in terms]


def run_both(ctx, terms, ell, rank=0, tol=0.0, adaptive=False, seed=1, sketch_only=False,
             max_rank=0, host=False):
    np_terms = [ttsynth.to_numpy(t) for t in terms]
    ref = oracle.round_sum(np_terms, ell=ell, seed=seed, rank=rank, tol=tol, adaptive=adaptive,
                           max_rank=max_rank, sketch_only=sketch_only)
    if sketch_only:
        mode, r, p = "sketch_only", 0, ell
    elif tol > 0:
        mode, r, p = "tol", rank, ell
    else:
        mode, r, p = "rank", rank, ell - rank
    src = terms if host else gpu_terms(terms)
    res = ctx.tt_round_sum(src, mode=mode, rank=r, oversample=p, tol=tol, seed=seed,
                           adaptive=adaptive, max_rank=max_rank)
    return res, ref


def rel(res, ref):
    X = res.numpy()
    return oracle.rel_diff(X, ref.X), X


def check(res, ref, tol=TOL):
    assert res.ranks[1:-1] == list(ref.ranks), (res.ranks, ref.ranks)
    r, X = rel(res, ref)
    assert r <= tol, r
    return r, X


# ------------------------------------------------------------------ configs 1-4, full size
def test_config1_tiny_full(ctx):
    w = ttsynth.config1_tiny()
    res, ref = run_both(ctx, w.terms, w.ell, rank=w.rank)
    r, X = check(res, ref)
    # closed form: best rank-4 approximation of the 16x16 unfolding
    F = sum(oracle.full(ttsynth.to_numpy(t)) for t in w.terms)
    U, s, Vt = np.linalg.svd(F.reshape(16, 16))
    best = ((U[:, :4] * s[:4]) @ Vt[:4]).reshape(F.shape)
    assert np.linalg.norm(oracle.full(X) - best) <= 1e-13 * np.linalg.norm(best)


def test_config2_single_full(ctx):
    w = ttsynth.config2_single()
    res, ref = run_both(ctx, w.terms, w.ell, rank=w.rank)
    check(res, ref)


def test_config3_sum10_full(ctx):
    w = ttsynth.config3_sum10()
    res, ref = run_both(ctx, w.terms, w.ell, rank=w.rank)
    check(res, ref)


def test_config4_gmres_full(ctx):
    w = ttsynth.config4_gmres()
    res, ref = run_both(ctx, w.terms, w.ell, tol=w.tol, adaptive=True)
    check(res, ref)
    assert res.passes == ref.passes


def test_config5_reduced_depth(ctx):
    # config 5 shapes (S=32, I=256, summand rank 64, l=144 -> r=128) at d = 5
    w = ttsynth.config5_large(d=5)
    res, ref = run_both(ctx, w.terms, w.ell, rank=w.rank)
    check(res, ref)


# ------------------------------------------------------------------ modes and edge cases
def test_sketch_only_is_left_orthogonal(ctx):
    w = ttsynth.config3_sum10(d=6, I=20, S=4)
    res, ref = run_both(ctx, w.terms, 30, sketch_only=True)
    r, X = check(res, ref)
    assert oracle.left_orth_residual(X) < 1e-12
    import paper_2110_04393_b200 as P
    assert res.flags & P.FLAG_LEFT_ORTH


def test_two_modes_and_single_summand(ctx):
    terms = ttsynth.random_terms(3, [17, 9], [[1, 5, 1]])
    res, ref = run_both(ctx, terms, 4, rank=3)
    check(res, ref)


@pytest.mark.parametrize("seed", [11, 12])
def test_ragged_summand_ranks_and_dims(ctx, seed):
    dims = [3, 11, 5, 7, 2, 13]
    rng = np.random.default_rng(seed)
    tr = [[1] + [int(x) for x in rng.integers(1, 9, size=len(dims) - 1)] + [1] for _ in range(5)]
    terms = ttsynth.random_terms(seed, dims, tr)
    res, ref = run_both(ctx, terms, 9, rank=6)
    check(res, ref)
    res, ref = run_both(ctx, terms, 13, sketch_only=True)
    check(res, ref)


def test_exact_recovery_when_sketch_exceeds_rank(ctx):
    terms = ttsynth.random_terms(21, [6, 6, 6, 6], [[1, 2, 3, 2, 1], [1, 3, 2, 2, 1]])
    res, ref = run_both(ctx, terms, 8, sketch_only=True)
    r, X = check(res, ref)
    S = oracle.tt_add([ttsynth.to_numpy(t) for t in terms])
    assert oracle.rel_diff(X, S) < 1e-12


def test_zero_sum(ctx):
    import paper_2110_04393_b200 as P
    Z = [torch.zeros((1, 4, 2), dtype=torch.float64), torch.zeros((2, 4, 2), dtype=torch.float64),
         torch.zeros((2, 4, 1), dtype=torch.float64)]
    res = ctx.tt_round_sum(gpu_terms([Z, Z]), mode="rank", rank=2, oversample=2)
    assert res.ranks == [1, 1, 1, 1] and res.flags & P.FLAG_ZERO
    assert all(not np.any(c) for c in res.numpy())


def test_tolerance_mode_without_adaptivity(ctx):
    w = ttsynth.config4_gmres(d=6, I=32, R=12, S=5)
    res, ref = run_both(ctx, w.terms, 20, tol=1e-6)
    check(res, ref)


def test_host_inputs_are_staged(ctx):
    # e2e path of bench.py: host (pinned) buffers in, copies inside the call
    w = ttsynth.config3_sum10(d=6, I=40, S=3)
    pinned = [[c.permute(2, 1, 0).contiguous().pin_memory().permute(2, 1, 0) for c in t]
              for t in w.terms]
    res, ref = run_both(ctx, pinned, w.ell, rank=w.rank, host=True)
    check(res, ref)


def test_inner_product(ctx):
    terms = ttsynth.random_terms(31, [5, 6, 7, 4], [[1, 3, 4, 2, 1], [1, 2, 5, 3, 1]])
    x, y = terms
    got = ctx.tt_inner(gpu_terms([x])[0], gpu_terms([y])[0])
    want = oracle.inner(ttsynth.to_numpy(x), ttsynth.to_numpy(y))
    assert abs(got - want) <= 1e-13 * max(1.0, abs(want)) * 10


def test_user_sketch_matches_internal(ctx):
    w = ttsynth.config3_sum10(d=5, I=16, S=3)
    sumR = [1] + [sum(t[n].shape[2] for t in w.terms) for n in range(4)] + [1]
    caps = [1] + oracle.rank_caps(w.dims, sumR, 12) + [1]
    sk = ctx.tt_sketch_create(w.dims, caps, seed=9)
    a = ctx.tt_round_sum(gpu_terms(w.terms), mode="sketch_only", oversample=12, seed=9)
    b = ctx.tt_round_sum(gpu_terms(w.terms), mode="sketch_only", oversample=12, sketch=sk)
    for x, y in zip(a.numpy(), b.numpy()):
        assert np.array_equal(x, y)


def test_determinism_bitwise(ctx):
    w = ttsynth.config3_sum10(d=5, I=30, S=4)
    t = gpu_terms(w.terms)
    a = ctx.tt_round_sum(t, mode="rank", rank=20, oversample=5, seed=4).numpy()
    b = ctx.tt_round_sum(t, mode="rank", rank=20, oversample=5, seed=4).numpy()
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_errors_are_reported(ctx):
    import paper_2110_04393_b200 as P
    terms = ttsynth.random_terms(1, [4, 4, 4], [[1, 2, 2, 1], [1, 2, 2, 1]])
    bad = [terms[0], [terms[1][0], terms[1][1], torch.zeros((2, 5, 1), dtype=torch.float64)]]
    with pytest.raises(P.TTError) as e:
        ctx.tt_round_sum(gpu_terms(bad), mode="rank", rank=2, oversample=1)
    assert e.value.code == -2
    with pytest.raises(P.TTError):
        ctx.tt_round_sum(gpu_terms(terms), mode="tol", tol=0.0, oversample=3)


@pytest.mark.parametrize("bad", [float("nan"), float("inf")])
@pytest.mark.parametrize("core", [0, 2])
def test_nonfinite_input_is_reported(ctx, bad, core):
    """A NaN/Inf entry in one summand reaches every sketch Gram of the sweep: the
    call returns TT_ERR_NONFINITE (-4) instead of a tensor of NaNs, and the
    context stays usable."""
    import paper_2110_04393_b200 as P
    w = ttsynth.config3_sum10(d=4, I=12, S=3)
    terms = [[c.clone() for c in t] for t in w.terms]
    terms[1][core][0, 1, 0] = bad
    for mode in (dict(mode="rank", rank=6, oversample=3), dict(mode="tol", tol=1e-6, oversample=8),
                 dict(mode="sketch_only", rank=6, oversample=3)):
        with pytest.raises(P.TTError) as e:
            ctx.tt_round_sum(gpu_terms(terms), seed=2, **mode)
        assert e.value.code == -4, e.value
    ok = ctx.tt_round_sum(gpu_terms(w.terms), mode="rank", rank=6, oversample=3, seed=2)
    assert all(np.isfinite(c).all() for c in ok.numpy())


def test_config5_full_size_in_bench_launch_configuration():
    """Config 5 at BASELINE.json's full size (S=32, d=50, I=256, rank 64 per
    summand, sketch 144 -> rank 128), rounded through the C-ABI in the launch
    configuration bench.py times (library bound to torch's current stream), and
    compared with the oracle on the host (NumPy, ~2-3 min) in TT arithmetic."""
    import paper_2110_04393_b200 as P
    w = ttsynth.config5_large()
    c = P.Context(0, stream=torch.cuda.current_stream())
    res = c.tt_round_sum(gpu_terms(w.terms), mode="rank", rank=w.rank,
                         oversample=w.ell - w.rank, seed=1)
    ref = oracle.round_sum([ttsynth.to_numpy(t) for t in w.terms], ell=w.ell, seed=1,
                           rank=w.rank)
    r, X = check(res, ref)
    assert res.ranks == [1] + [w.rank] * (w.d - 1) + [1]


# ------------------------------------------------------------------ deterministic (NEXT-1)
def run_det(ctx, terms, tol=0.0, rank=0):
    np_terms = [ttsynth.to_numpy(t) for t in terms]
    ref = oracle.tt_round(oracle.tt_add(np_terms), tol, rank)
    res = ctx.tt_round_deterministic(gpu_terms(terms), tol=tol, rank=rank)
    X = res.numpy()
    assert res.ranks == oracle.ranks_of(ref), (res.ranks, oracle.ranks_of(ref))
    r = oracle.rel_diff(X, ref)
    assert r <= TOL, r
    return X, ref


@pytest.mark.parametrize("tol,rank", [(0.0, 4), (1e-8, 0), (1e-2, 0), (0.0, 0)])
def test_deterministic_config1(ctx, tol, rank):
    w = ttsynth.config1_tiny()
    X, ref = run_det(ctx, w.terms, tol, rank)
    assert oracle.left_orth_residual(X) < 1e-12


def test_deterministic_single_term_rank50(ctx):
    w = ttsynth.config2_single(d=6)
    run_det(ctx, w.terms, tol=1e-6)
    run_det(ctx, w.terms, rank=25)


@pytest.mark.parametrize("seed", [3, 4])
def test_deterministic_ragged(ctx, seed):
    dims = [3, 7, 5, 6, 2]
    rng = np.random.default_rng(seed)
    tr = [[1] + [int(x) for x in rng.integers(1, 7, size=len(dims) - 1)] + [1] for _ in range(4)]
    terms = ttsynth.random_terms(seed, dims, tr)
    run_det(ctx, terms, tol=1e-10)
    run_det(ctx, terms, rank=3)


def test_deterministic_sum_large_ranks(ctx):
    # assembled ranks 180 > 160: the generic Cholesky and the Jacobi with V
    w = ttsynth.config3_sum10(d=5, I=10, S=3)
    run_det(ctx, w.terms, tol=1e-9)


def test_deterministic_config3_full_size(ctx):
    """Config 3 at full size (S = 10, d = 20, I = 100, assembled rank 600 > 160,
    exactly rank-deficient: the true bond rank is 150): Alg. 1 + 2 on the
    assembled sum through the clamped-pass QRs (robust_q), the grid Jacobi and
    the generic Cholesky, against the oracle's tt_round(tt_add(...)) (LAPACK QR
    and SVD), rank 60 as in the randomized line."""
    w = ttsynth.config3_sum10()
    run_det(ctx, w.terms, rank=w.rank)


def test_deterministic_matches_randomized_when_sketch_is_exact(ctx):
    # rank-r truncation of an exactly low-rank sum: both roundings give the best
    # approximation (P:653-663 with l >= true rank), hence the same tensor
    terms = ttsynth.random_terms(41, [5, 6, 4, 5], [[1, 2, 3, 2, 1], [1, 3, 2, 2, 1]])
    a = ctx.tt_round_deterministic(gpu_terms(terms), tol=1e-12).numpy()
    b = ctx.tt_round_sum(gpu_terms(terms), mode="tol", tol=1e-12, oversample=12, seed=2).numpy()
    assert oracle.rel_diff(a, b) < 1e-10


# ------------------------------------------------------------------ more edge cases
def test_unit_mode_and_rank_one_summands(ctx):
    dims = [4, 1, 6, 1, 3]
    terms = ttsynth.random_terms(51, dims, [[1, 1, 1, 1, 1, 1]] * 3)
    res, ref = run_both(ctx, terms, 5, rank=2)
    check(res, ref)
    res, ref = run_both(ctx, terms, 5, sketch_only=True)
    check(res, ref)


def test_more_summands_than_one_gemm_batch(ctx):
    # S = 70 > kMaxGemmBatch = 64: the batched GEMMs split into several launches
    dims = [6, 5, 7, 4]
    terms = ttsynth.random_terms(52, dims, [[1, 2, 3, 2, 1]] * 70)
    res, ref = run_both(ctx, terms, 12, rank=8)
    check(res, ref)


def test_sketch_rank_above_structural_caps_is_flagged_and_exact(ctx):
    import paper_2110_04393_b200 as P
    terms = ttsynth.random_terms(53, [3, 4, 5], [[1, 2, 2, 1], [1, 3, 1, 1]])
    res, ref = run_both(ctx, terms, 50, sketch_only=True)
    check(res, ref)
    assert res.flags & P.FLAG_RANK_CAPPED
    S = oracle.tt_add([ttsynth.to_numpy(t) for t in terms])
    assert oracle.rel_diff(res.numpy(), S) < 1e-12


def test_partially_zero_summands(ctx):
    terms = ttsynth.random_terms(54, [5, 6, 5, 4], [[1, 3, 3, 3, 1]] * 3)
    terms[1] = [torch.zeros_like(c) for c in terms[1]]
    res, ref = run_both(ctx, terms, 6, rank=3)
    check(res, ref)


def test_tolerance_bound_holds(ctx):
    # truncation error of the returned TT against the input sum: the deterministic
    # part obeys eps0 ||X||; the sketch adds its own (small) error on this
    # exactly low-rank sum (l >= true rank)
    terms = ttsynth.random_terms(55, [6, 7, 6, 5], [[1, 3, 4, 3, 1], [1, 2, 2, 2, 1]])
    tol = 1e-3
    res, ref = run_both(ctx, terms, 10, tol=tol)
    check(res, ref)
    S = oracle.tt_add([ttsynth.to_numpy(t) for t in terms])
    assert oracle.rel_diff(res.numpy(), S) <= tol * (1 + 1e-10)


def test_concurrent_contexts_on_host_threads_match_sequential():
    """Several contexts (one stream each) driven from host threads, as bench.py
    --batch does: results free stream-ordered and the one-time kernel setup is
    thread-safe, so concurrent roundings give the bits of sequential ones."""
    import concurrent.futures as cf
    import paper_2110_04393_b200 as P
    w = ttsynth.config3_sum10(d=6, I=24, S=4)
    t = gpu_terms(w.terms)
    torch.cuda.synchronize()
    seq = [P.Context(0).tt_round_sum(t, mode="rank", rank=12, oversample=4, seed=s).numpy()
           for s in range(1, 9)]
    ctxs = [P.Context(0) for _ in range(4)]

    def lane(k):
        out = {}
        for s in range(1 + k, 9, 4):
            r = ctxs[k].tt_round_sum(t, mode="rank", rank=12, oversample=4, seed=s)
            out[s] = r.numpy()
            del r
        a = ctxs[k].tt_round_sum_two_sided(t, 10, seed=k + 1).numpy()
        return out, a

    with cf.ThreadPoolExecutor(4) as ex:
        res = list(ex.map(lane, range(4)))
    for k, (out, a) in enumerate(res):
        for s, X in out.items():
            for x, y in zip(X, seq[s - 1]):
                assert np.array_equal(x, y)
        b = P.Context(0).tt_round_sum_two_sided(t, 10, seed=k + 1).numpy()
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


# ------------------------------------------------------------------ ε threshold (closed form)
@pytest.mark.parametrize("N,eps0,k", [(3, 1.2e-3, 4), (3, 1.6e-3, 3), (5, 1.8e-3, 4),
                                      (5, 2.2e-3, 3)])
def test_eps_threshold_closed_form_spectra(ctx, N, eps0, k):
    """Both GPU paths keep the ranks fixed by ε = ‖X‖ε0/√(N-1) on a
    TT whose bond spectra are 10^-a exactly (tests/test_oracle_tt.py pins)."""
    from test_oracle_tt import SPECTRUM, _known_spectrum_tt
    rng = np.random.default_rng(101 + N)
    Y = _known_spectrum_tt(rng, [7] * N, SPECTRUM, left_orth=False, gauge="general")
    terms = [[torch.from_numpy(np.ascontiguousarray(c)) for c in Y]]
    exact = math.sqrt(sum(x * x for x in SPECTRUM[k:]))
    # randomized: sketch rank 6 >= true rank, so Alg. 7 is exact and only truncation cuts
    res = ctx.tt_round_sum(gpu_terms(terms), mode="tol", tol=eps0, oversample=6, seed=3)
    assert res.ranks == [1] + [k] * (N - 1) + [1]
    assert abs(oracle.diff_norm(res.numpy(), Y) - exact) < 1e-12
    det = ctx.tt_round_deterministic(gpu_terms(terms), tol=eps0)
    assert det.ranks == [1] + [k] * (N - 1) + [1]
    assert abs(oracle.diff_norm(det.numpy(), Y) - exact) < 1e-12


@pytest.mark.parametrize("seed", [21, 22])
def test_even_ragged_ranks_take_the_tma_fused_paths(ctx, seed):
    """Summand ranks all even but different (every operand TMA-addressable), so the
    fused projection-and-carry kernel and the persistent phase-1 GEMM run with
    k-tiles that straddle summand boundaries (zero-filled by TMA)."""
    dims = [6, 10, 8, 12, 4]
    rng = np.random.default_rng(seed)
    tr = [[1] + [2 * int(x) for x in rng.integers(1, 9, size=len(dims) - 1)] + [1]
          for _ in range(6)]
    terms = ttsynth.random_terms(seed, dims, tr)
    res, ref = run_both(ctx, terms, 24, rank=16)
    check(res, ref)


# ------------------------------------------------------------------ per-bond target ranks (R22)
def test_per_bond_target_ranks_match_oracle(ctx):
    """tt_round_opts.ranks: the paper's "target TT-ranks {l_n}".
    Config-3 shapes at reduced depth, a different target rank on every bond,
    sketch ranks r_n + p; the kept ranks are exactly the targets."""
    w = ttsynth.config3_sum10(d=8, I=40, S=6)
    ranks = [12, 40, 57, 60, 33, 48, 9]
    p = 10
    np_terms = [ttsynth.to_numpy(t) for t in w.terms]
    ref = oracle.round_sum(np_terms, ell=[r + p for r in ranks], seed=4, rank=ranks)
    res = ctx.tt_round_sum(gpu_terms(w.terms), mode="rank", rank=ranks, oversample=p, seed=4)
    check(res, ref)
    assert res.ranks[1:-1] == ranks


def test_per_bond_target_ranks_with_caps_and_no_truncation_needed(ctx):
    """Targets above the structural caps (R7) are capped and flagged; bonds whose
    capped sketch rank does not exceed the target are not truncated."""
    w = ttsynth.config1_tiny()
    np_terms = [ttsynth.to_numpy(t) for t in w.terms]
    ranks = [9, 5, 2]
    ref = oracle.round_sum(np_terms, ell=[r + 1 for r in ranks], seed=2, rank=ranks)
    res = ctx.tt_round_sum(gpu_terms(w.terms), mode="rank", rank=ranks, oversample=1, seed=2)
    check(res, ref)
    import paper_2110_04393_b200 as P
    assert ref.capped and res.flags & P.FLAG_RANK_CAPPED


def test_per_bond_ranks_errors(ctx):
    import paper_2110_04393_b200 as P
    w = ttsynth.config1_tiny()
    with pytest.raises(P.TTError):
        ctx.tt_round_sum(gpu_terms(w.terms), mode="rank", rank=[2, 0, 2], oversample=1)
    with pytest.raises(P.TTError):
        ctx.tt_round_deterministic(gpu_terms(w.terms), tol=0.0, rank=[2, -1, 2])


def test_deterministic_per_bond_caps(ctx):
    """tt_round_deterministic with per-bond caps against Alg. 2 with the same caps."""
    w = ttsynth.config3_sum10(d=6, I=20, S=4)
    run_det(ctx, w.terms, tol=0.0, rank=[7, 30, 22, 41, 5])
    run_det(ctx, w.terms, tol=1e-7, rank=[7, 300, 22, 300, 5])


# ------------------------------------------------------------------ bench line / pipelined e2e
def test_host_input_calls_in_flight_match_sequential():
    """bench.py's e2e.pipelined pattern: two contexts on host threads rounding the
    same pinned HOST inputs (H2D staging inside the call), results read back with
    tt_tensor_copy_all -- the bits of the same calls run one at a time."""
    import concurrent.futures as cf
    import paper_2110_04393_b200 as P
    w = ttsynth.config3_sum10(d=8, I=40, S=6)
    host = [[c.permute(2, 1, 0).contiguous().cpu().pin_memory().permute(2, 1, 0) for c in t]
            for t in w.terms]
    kw = dict(mode="rank", rank=w.rank, oversample=w.ell - w.rank)
    seq = {s: P.Context(0).tt_round_sum(host, seed=s, **kw).numpy() for s in (1, 2)}
    ctxs = [P.Context(0, stream=torch.cuda.Stream()) for _ in range(2)]

    def lane(k):
        outs = []
        for _ in range(3):
            outs.append(ctxs[k].tt_round_sum(host, seed=1 + k, **kw).numpy())
        return outs

    with cf.ThreadPoolExecutor(2) as ex:
        res = list(ex.map(lane, range(2)))
    for k, outs in enumerate(res):
        for X in outs:
            for x, y in zip(X, seq[1 + k]):
                assert np.array_equal(x, y)


def test_bench_default_line_carries_the_contract_keys():
    """python bench.py (config 3 to keep it short): one JSON line with value,
    roofline, e2e (+ pipelined), gpu_launches and clocks."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--workload", "sum10",
                          "--steps", "3", "--warmup", "3", "--no-cpu"], capture_output=True,
                         text=True, timeout=900, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["value"] > 0 and d["unit"] == "roundings/s" and d["n_gpus"] == 1
    assert d["dtype"] == "f64" and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] == "tensor" and 0 < d["roofline"]["frac"] < 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["pipelined"]["value"] > 0 and e["pipelined"]["lanes"] == 2
    assert "sm_mhz" in d["clocks"]
