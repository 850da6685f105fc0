"""GPU unit parity of the individual kernels behind the C-ABI (run with -m gpu).

Expected values: plain fp64 CPU (torch / numpy) references and the oracle."""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2110_04393_b200 as P
    return P.Context(0)


def colmajor(rows, cols, gen, device="cuda"):
    return torch.randn((cols, rows), dtype=torch.float64, generator=gen).t().to(device)


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("mnk", [(1, 1, 1), (7, 5, 3), (129, 47, 33), (64, 144, 64),
                                 (300, 35, 1000), (144, 144, 20000), (16384, 144, 64),
                                 (144, 2048, 4096), (35, 1, 2240), (144, 2048, 64),
                                 (100, 640, 33), (48, 64, 64), (97, 131, 17)])
def test_dgemm_matches_fp64_reference(ctx, ta, tb, mnk):
    m, n, k = mnk
    g = torch.Generator().manual_seed(m * 7 + n * 3 + k)
    A = colmajor(k, m, g) if ta else colmajor(m, k, g)
    B = colmajor(n, k, g) if tb else colmajor(k, n, g)
    C0 = colmajor(m, n, g)
    Cg = C0.clone()
    ctx.tt_dgemm(A, B, ta, tb, alpha=0.75, beta=-0.5, C_out=Cg)
    Ah = A.cpu().t() if ta else A.cpu()
    Bh = B.cpu().t() if tb else B.cpu()
    ref = 0.75 * (Ah @ Bh) - 0.5 * C0.cpu()
    err = (Cg.cpu() - ref).abs().max().item()
    scale = (Ah.abs() @ Bh.abs()).max().item() + C0.abs().max().item()
    assert err <= 1e-14 * max(1.0, math.sqrt(k)) * scale


def test_dgemm_batched_ldc_offsets_via_library(ctx):
    # C written into a sub-block of a larger matrix (ldc > m), beta = 0 must ignore NaNs
    g = torch.Generator().manual_seed(5)
    A, B = colmajor(50, 20, g), colmajor(20, 30, g)
    big = torch.full((40, 80), float("nan"), dtype=torch.float64, device="cuda").t()  # 80 x 40
    sub = big[10:60, 5:35]
    ctx.tt_dgemm(A, B, C_out=sub)
    assert torch.allclose(sub.cpu(), A.cpu() @ B.cpu(), rtol=1e-13, atol=1e-13)
    assert torch.isnan(big[:10]).all() and torch.isnan(big[60:]).all()


def test_sketch_matches_oracle_philox(ctx):
    import oracle
    dims = [5, 7, 3, 9]
    ranks = [1, 4, 6, 5, 1]
    sk = ctx.tt_sketch_create(dims, ranks, seed=0x123456789, tag=0)
    for n in range(2, 5):
        got = sk.core(n).cpu().numpy()
        want = oracle.sketch_core(0x123456789, n, ranks[n - 1], dims[n - 1], ranks[n])
        assert got.shape == want.shape
        # integer words identical; libm vs CUDA log/sincos may differ by a few ulp
        np.testing.assert_allclose(got, want, rtol=4 * 2.0 ** -52, atol=1e-300)
        assert np.mean(got == want) > 0.5


def test_sketch_large_count_and_odd_tail(ctx):
    import oracle
    dims = [3, 257, 3]
    ranks = [1, 3, 3, 1]
    sk = ctx.tt_sketch_create(dims, ranks, seed=77, tag=5)
    got = sk.core(2).cpu().numpy()     # 3*257*3 = 2313 entries (odd)
    want = oracle.sketch_core(77, 2, 3, 257, 3, tag=5)
    np.testing.assert_allclose(got, want, rtol=4 * 2.0 ** -52)


@pytest.mark.parametrize("m,n,cond", [(40, 7, 1e2), (2240, 35, 1e8), (7000, 70, 1e6),
                                      (36864, 144, 1e4), (500, 1, 1.0), (100, 100, 10.0),
                                      (1000, 32, 10.0), (1000, 33, 1e3), (3000, 96, 1e5),
                                      (3000, 97, 1e2), (5000, 160, 1e6), (5000, 161, 1e3),
                                      (6000, 250, 1e4)])
def test_qr_orthogonality_and_factorization(ctx, m, n, cond):
    rng = np.random.default_rng(m + n)
    U, _ = np.linalg.qr(rng.standard_normal((m, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.logspace(0, -math.log10(cond), n)
    A = (U * s) @ V.T
    Ad = torch.from_numpy(np.asfortranarray(A)).cuda()
    Ad = Ad.t().contiguous().t()
    Q, R, fb = ctx.tt_qr(Ad, want_r=True)
    Qh, Rh = Q.cpu().numpy(), R.cpu().numpy()
    assert np.linalg.norm(Qh.T @ Qh - np.eye(n)) < 1e-13 * math.sqrt(n)
    assert np.linalg.norm(Qh @ Rh - A) <= 1e-13 * np.linalg.norm(A) * max(1, math.log10(cond))
    assert np.allclose(np.tril(Rh, -1), 0)
    # same projector as LAPACK Householder (the oracle's thin_qr)
    Qo, _ = np.linalg.qr(A)
    assert np.linalg.norm(Qh @ (Qh.T @ A) - Qo @ (Qo.T @ A)) < 1e-13 * np.linalg.norm(A)


@pytest.mark.parametrize("m,n,cond", [(36864, 144, 1e10), (10240, 80, 1e12), (2240, 35, 1e8),
                                      (36864, 144, 1e13), (20000, 100, 1e14)])
def test_qr_ill_conditioned_stays_on_cholesky_routes(ctx, m, n, cond):
    """kappa up to ~1/u must be handled by CholeskyQR2/3 or shifted CholeskyQR3
    (DMMA, all SMs), never by the single-CTA Householder fallback."""
    g = torch.Generator(device="cuda").manual_seed(m + n)
    U, _ = torch.linalg.qr(torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g))
    V, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))
    s = torch.logspace(0, -math.log10(cond), n, dtype=torch.float64, device="cuda")
    A = ((U * s) @ V.T).t().contiguous().t()
    Q, R, fb = ctx.tt_qr(A, want_r=True)
    assert not fb
    eye = torch.eye(n, dtype=torch.float64, device="cuda")
    assert (Q.T @ Q - eye).norm().item() < 1e-13 * math.sqrt(n)
    assert ((Q @ R - A).norm() / A.norm()).item() < 1e-13 * math.log10(cond)
    assert torch.allclose(torch.tril(R, -1), torch.zeros_like(R))


@pytest.mark.parametrize("m,n,r", [(32768, 144, 128), (5000, 80, 3), (300, 33, 1),
                                   (32768, 144, 144), (4000, 160, 100)])
def test_qr_r_only_rank_deficient_robust(ctx, m, n, r):
    """R-only QR of a numerically rank-deficient matrix (the truncation's bond
    matrices at depth): two shifted + two clamped CholeskyQR
    passes (no TSQR, no Householder) whose R reproduces the singular values of A
    and R^T R = A^T A to O(u ||A||^2)."""
    g = torch.Generator(device="cuda").manual_seed(m + n + r)
    A = (torch.randn(m, r, dtype=torch.float64, device="cuda", generator=g)
         @ torch.randn(r, n, dtype=torch.float64, device="cuda", generator=g))
    A = (A * torch.logspace(0, -9, n, dtype=torch.float64, device="cuda")).t().contiguous().t()
    _, R, fb = ctx.tt_qr(A, want_r=True, want_q=False)
    st = ctx.status_words(17)
    assert not fb and st[14] == 0 and st[11] == 0      # no TSQR, no Householder
    assert torch.allclose(torch.tril(R, -1), torch.zeros_like(R))
    sA = torch.linalg.svdvals(A)
    sR = torch.linalg.svdvals(R)
    assert (sA - sR).abs().max().item() <= 1e-13 * sA[0].item() * math.sqrt(n)
    G = A.T @ A
    assert (R.T @ R - G).norm().item() <= 1e-13 * G.norm().item() * math.sqrt(n)


@pytest.mark.parametrize("m,n,cond", [(32768, 144, 1e15), (10000, 100, 1e3), (500, 160, 1e8)])
def test_qr_r_only_ill_conditioned(ctx, m, n, cond):
    """Full-rank but ill-conditioned (kappa up to ~1/u): the same R-only path keeps
    the small singular values to O(u ||A||) absolute."""
    g = torch.Generator(device="cuda").manual_seed(m + n)
    U, _ = torch.linalg.qr(torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g))
    V, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))
    s = torch.logspace(0, -math.log10(cond), n, dtype=torch.float64, device="cuda")
    A = ((U * s) @ V.T).t().contiguous().t()
    _, R, fb = ctx.tt_qr(A, want_r=True, want_q=False)
    assert not fb
    sR = torch.linalg.svdvals(R)
    assert (sR - s).abs().max().item() <= 1e-14 * math.sqrt(n)
    G = A.T @ A
    assert (R.T @ R - G).norm().item() <= 1e-14 * math.sqrt(n)


def test_qr_rank_deficient_uses_valid_basis(ctx):
    rng = np.random.default_rng(3)
    m, n, r = 2240, 35, 25
    A = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    Ad = torch.from_numpy(A).cuda().t().contiguous().t()
    Q, _, fb = ctx.tt_qr(Ad)
    Qh = Q.cpu().numpy()
    assert np.linalg.norm(Qh.T @ Qh - np.eye(n)) < 1e-12
    assert np.linalg.norm(Qh @ (Qh.T @ A) - A) < 1e-12 * np.linalg.norm(A)


@pytest.mark.parametrize("n", [1, 2, 5, 8, 31, 32, 33, 35, 40, 63, 64, 65, 70, 72, 96, 97, 100,
                               127, 128, 129, 136, 143, 144, 150, 159, 160, 161, 200])
@pytest.mark.parametrize("cond", [1e2, 1e7])
def test_cholesky_factor_and_inverse(ctx, n, cond):
    """The CholeskyQR passes' factorisation: L L^T = G and Rinv = L^{-T} against a
    plain fp64 reference, at every block / tile raggedness up to n = 160 (the
    blocked look-ahead kernel) and beyond (the generic kernel)."""
    rng = np.random.default_rng(n * 7 + int(math.log10(cond)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.logspace(0, -math.log10(cond), n)
    G = (V * s) @ V.T
    G = 0.5 * (G + G.T)
    Gd = torch.from_numpy(np.asfortranarray(G)).cuda().t().contiguous().t()
    Rinv, L = ctx.tt_cholesky(Gd)
    Lh, Rh = L.cpu().numpy(), Rinv.cpu().numpy()
    Lref = np.linalg.cholesky(G)
    assert np.allclose(np.triu(Lh, 1), 0) and np.allclose(np.tril(Rh, -1), 0)
    assert np.linalg.norm(Lh @ Lh.T - G) <= 1e-14 * n * np.linalg.norm(G)
    # Rinv L^T = I to the conditioning of L (sqrt(cond))
    assert np.linalg.norm(Rh.T @ Lh - np.eye(n)) <= 1e-14 * n * math.sqrt(cond)
    assert np.linalg.norm(Lh - Lref) <= 1e-12 * math.sqrt(cond) * np.linalg.norm(Lref)


@pytest.mark.parametrize("n,rank", [(150, 40), (300, 100), (600, 150)])
def test_cholesky_rank_deficient_clamped(ctx, n, rank):
    """shifted = 0 on an exactly rank-deficient Gram (the deterministic baseline's
    assembled sums): pivots below tau = 64 n u max diag G are clamped (and, in the
    generic n > 160 kernel, their columns decoupled), so the factor stays finite,
    L L^T matches G to rounding level, and Rinv L^T = I."""
    rng = np.random.default_rng(n + rank)
    B = rng.standard_normal((n, rank))
    G = B @ B.T
    Gd = torch.from_numpy(G).cuda().t().contiguous().t()
    Rinv, L = ctx.tt_cholesky(Gd)
    Lh, Rh = L.cpu().numpy(), Rinv.cpu().numpy()
    assert np.isfinite(Lh).all() and np.isfinite(Rh).all()
    tau = 64 * n * 2.0 ** -53 * np.max(np.diag(G))
    assert np.linalg.norm(Lh @ Lh.T - G) <= 1e-12 * n * np.linalg.norm(G) + n * tau
    assert np.linalg.norm(Rh.T @ Lh - np.eye(n)) <= 1e-8 * n


def test_cholesky_shifted_and_breakdown(ctx):
    """shifted = 1 factors G + 11 (m n + n (n + 1)) u tr(G) I; an indefinite G
    is reported (TT_ERR_NUMERIC), not returned."""
    import paper_2110_04393_b200 as P
    rng = np.random.default_rng(5)
    n, m = 144, 36864
    A = rng.standard_normal((n, n))
    G = A @ A.T
    Gd = torch.from_numpy(G).cuda().t().contiguous().t()
    _, L = ctx.tt_cholesky(Gd, m=m, shifted=True)
    shift = 11.0 * (m * n + n * (n + 1)) * 2.0 ** -53 * np.trace(G)
    Lh = L.cpu().numpy()
    assert np.linalg.norm(Lh @ Lh.T - (G + shift * np.eye(n))) <= 1e-13 * np.linalg.norm(G)
    Gbad = torch.from_numpy(-np.eye(n)).cuda().t().contiguous().t()
    with pytest.raises(P.TTError) as e:
        ctx.tt_cholesky(Gbad)
    assert e.value.code == -8


@pytest.mark.parametrize("m,n", [(5, 5), (144, 144), (70, 33), (300, 80), (33, 33), (400, 241),
                                 (600, 600)])
def test_jacobi_svd_matches_lapack(ctx, m, n):
    """V-accumulating one-sided Jacobi against LAPACK; m n > 26624 (the last two
    shapes) runs on the cooperative-grid kernel (one warp per pair of a round)."""
    rng = np.random.default_rng(m * n)
    A = rng.standard_normal((m, n)) * np.logspace(0, -8, n)[None, :]
    Ad = torch.from_numpy(A).cuda().t().contiguous().t()
    AV, V, s = ctx.tt_svd_jacobi(Ad)
    sh = s.cpu().numpy()
    sref = np.linalg.svd(A, compute_uv=False)
    np.testing.assert_allclose(sh, sref, rtol=1e-12, atol=1e-15 * sref[0])
    Vh, AVh = V.cpu().numpy(), AV.cpu().numpy()
    assert np.linalg.norm(Vh.T @ Vh - np.eye(n)) < 1e-13 * n
    assert np.linalg.norm(A @ Vh - AVh) < 1e-13 * np.linalg.norm(A)
    # AV has orthogonal columns with norms sigma
    G = AVh.T @ AVh
    # (each pair is left with |cos| <= m u: the off-diagonal mass grows with m and n)
    assert np.linalg.norm(G - np.diag(np.diag(G))) < 1e-13 * max(1.0, n / 100) * sref[0] ** 2
    assert np.all(np.diff(sh) <= 0)


@pytest.mark.parametrize("trans", [False, True])
@pytest.mark.parametrize("m,n", [(1, 1), (31, 7), (33, 8), (100, 9), (1000, 35), (4097, 70),
                                 (36864, 144), (36870, 143), (5000, 136), (640, 97), (64, 64)])
def test_cholqr_pass_matches_fp64_reference(ctx, m, n, trans):
    """The fused CholeskyQR pass (one launch: Q = op(A) Rinv and G = Q^T Q) against a
    plain fp64 CPU reference, at ragged chunk counts (m mod 32), ragged column
    tiles (n mod 8), the kernel's n limit (144), both input layouts, and the
    Gram-only / Q-only modes; the strictly-lower part of Rinv is garbage on
    purpose (the kernel must read only the upper triangle)."""
    g = torch.Generator().manual_seed(m * 1000 + n + int(trans))
    A = colmajor(n, m, g) if trans else colmajor(m, n, g)
    opA = A.t().cpu() if trans else A.cpu()
    Rt = torch.triu(torch.randn((n, n), dtype=torch.float64, generator=g)) + 4 * torch.eye(
        n, dtype=torch.float64)
    Rbad = Rt + torch.tril(torch.full((n, n), float("nan"), dtype=torch.float64), -1)
    Rd = Rbad.t().contiguous().t().cuda()
    Q, G = ctx.tt_cholqr_pass(A, Rd, trans=trans)
    Qref = opA @ Rt
    Gref = Qref.t() @ Qref
    scale = Qref.abs().max().item() * math.sqrt(n)
    assert torch.isfinite(Q).all() and torch.isfinite(G).all()
    assert (Q.cpu() - Qref).abs().max().item() <= 1e-14 * scale * n
    assert (G.cpu() - Gref).abs().max().item() <= 1e-14 * n * m * Qref.abs().max().item() ** 2 + 1e-300
    assert torch.equal(G.cpu(), G.cpu().t())        # both triangles, bit-symmetric
    # Gram only (Q = op(A)) and Q only
    _, G0 = ctx.tt_cholqr_pass(A, None, trans=trans, want_q=False)
    G0ref = opA.t() @ opA
    assert (G0.cpu() - G0ref).abs().max().item() <= 1e-14 * n * m * opA.abs().max().item() ** 2
    Q1, _ = ctx.tt_cholqr_pass(A, Rd, trans=trans, want_g=False)
    assert torch.equal(Q1.cpu(), Q.cpu())
    # deterministic
    Q2, G2 = ctx.tt_cholqr_pass(A, Rd, trans=trans)
    assert torch.equal(G2.cpu(), G.cpu()) and torch.equal(Q2.cpu(), Q.cpu())


def test_cholqr_pass_rejects_unsupported(ctx):
    import paper_2110_04393_b200 as P
    A = torch.zeros((145, 100), dtype=torch.float64, device="cuda").t()
    with pytest.raises(P.TTError):
        ctx.tt_cholqr_pass(A, None)
