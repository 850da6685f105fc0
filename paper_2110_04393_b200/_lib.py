"""ctypes binding of libttround.so; names mirror include/ttround.h."""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libttround.so")

SKETCH_ONLY, RANK, TOL = 0, 1, 2
FLAG_RANK_CAPPED, FLAG_LEFT_ORTH, FLAG_RIGHT_ORTH, FLAG_ZERO, FLAG_QR_FALLBACK = 1, 2, 4, 8, 16
FLAG_SLAB = 32
_MODES = {"sketch_only": SKETCH_ONLY, "rank": RANK, "tol": TOL}


class TTError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libttround error {code}: {msg}")
        self.code = code


class tt_view(C.Structure):
    _fields_ = [("d", C.c_int32), ("dims", C.POINTER(C.c_int64)),
                ("ranks", C.POINTER(C.c_int64)), ("cores", C.POINTER(C.c_void_p))]


class tt_round_opts(C.Structure):
    _fields_ = [("mode", C.c_int32), ("adaptive", C.c_int32), ("rank", C.c_int64),
                ("oversample", C.c_int64), ("tol", C.c_double), ("seed", C.c_uint64),
                ("max_rank", C.c_int64), ("ranks", C.POINTER(C.c_int64))]


def _make_opts(mode, adaptive, rank, oversample, tol, seed, max_rank):
    """tt_round_opts from Python arguments; `rank` may be a sequence of d-1
    per-bond target ranks (opts.ranks).  Returns (opts, keepalive)."""
    keep = None
    if isinstance(rank, (list, tuple)):
        keep = (C.c_int64 * len(rank))(*[int(x) for x in rank])
        opts = tt_round_opts(mode, int(adaptive), 0, int(oversample), float(tol),
                             C.c_uint64(seed).value, int(max_rank), keep)
    else:
        opts = tt_round_opts(mode, int(adaptive), int(rank), int(oversample), float(tol),
                             C.c_uint64(seed).value, int(max_rank))
    return opts, keep


class tt_kron_op(C.Structure):
    _fields_ = [("d", C.c_int32), ("nterms", C.c_int32), ("dims", C.POINTER(C.c_int64)),
                ("kinds", C.POINTER(C.c_int32)), ("mats", C.POINTER(C.c_void_p))]


class tt_gmres_opts(C.Structure):
    _fields_ = [("tol", C.c_double), ("round_tol", C.c_double), ("max_iter", C.c_int32),
                ("randomized", C.c_int32), ("precond", C.c_int32), ("oversample", C.c_int32),
                ("max_rank", C.c_int64), ("seed", C.c_uint64)]


class tt_gmres_info(C.Structure):
    _fields_ = [("iters", C.c_int32), ("converged", C.c_int32), ("roundings", C.c_int32),
                ("max_basis_rank", C.c_int32), ("residual", C.c_double)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libttround.so; raises if it is missing (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -m paper_2110_04393_b200.build`")
    L = C.CDLL(path, mode=C.RTLD_GLOBAL)
    P = C.c_void_p
    i32, i64, u64, dbl = C.c_int32, C.c_int64, C.c_uint64, C.c_double
    sig = {
        "tt_last_error": (C.c_char_p, []),
        "tt_launch_count": (u64, []),
        "tt_get_nccl_unique_id": (C.c_int, [P]),
        "tt_nccl_selftest": (C.c_int, [P, C.c_int64, P]),
        "tt_ctx_create": (C.c_int, [C.c_int, P, P, C.c_int, C.c_int, C.POINTER(P)]),
        "tt_ctx_destroy": (C.c_int, [P]),
        "tt_loopback_create": (C.c_int, [C.c_int, C.POINTER(P)]),
        "tt_loopback_destroy": (C.c_int, [P]),
        "tt_ctx_create_loopback": (C.c_int, [C.c_int, P, P, C.c_int, C.POINTER(P)]),
        "tt_ctx_set_timing": (C.c_int, [P, C.c_int]),
        "tt_ctx_set_concurrency": (C.c_int, [P, C.c_int, C.c_int]),
        "tt_ctx_last_timing": (C.c_int, [P, C.POINTER(dbl), C.c_int]),
        "tt_ctx_flags": (C.c_int, [P, C.POINTER(C.c_int), C.c_int]),
        "tt_sketch_create": (C.c_int, [P, i32, C.POINTER(i64), C.POINTER(i64), u64, C.c_uint32,
                                       C.POINTER(P)]),
        "tt_sketch_core": (C.c_int, [P, i32, C.POINTER(P)]),
        "tt_sketch_destroy": (C.c_int, [P]),
        "tt_round_sum": (C.c_int, [P, i32, C.POINTER(tt_view), C.POINTER(tt_round_opts), P,
                                   C.POINTER(P)]),
        "tt_round_sum_slab": (C.c_int, [P, i32, C.POINTER(tt_view), C.POINTER(i64),
                                        C.POINTER(i64), C.POINTER(tt_round_opts), C.POINTER(P)]),
        "tt_round_deterministic": (C.c_int, [P, i32, C.POINTER(tt_view),
                                             C.POINTER(tt_round_opts), C.POINTER(P)]),
        "tt_round_sum_two_sided": (C.c_int, [P, i32, C.POINTER(tt_view), i64, i64, u64,
                                             C.POINTER(P)]),
        "tt_inner": (C.c_int, [P, C.POINTER(tt_view), C.POINTER(tt_view), C.POINTER(dbl)]),
        "tt_tensor_info": (C.c_int, [P, C.POINTER(i32), C.POINTER(C.POINTER(i64)),
                                     C.POINTER(C.POINTER(i64)), C.POINTER(C.POINTER(P)),
                                     C.POINTER(C.c_uint32)]),
        "tt_tensor_copy_core": (C.c_int, [P, i32, P]),
        "tt_tensor_copy_all": (C.c_int, [P, C.POINTER(P)]),
        "tt_tensor_passes": (C.c_int, [P, C.POINTER(i32)]),
        "tt_tensor_destroy": (C.c_int, [P]),
        "tt_dgemm": (C.c_int, [P, C.c_int, C.c_int, i64, i64, i64, dbl, P, i64, P, i64, dbl, P,
                               i64]),
        "tt_qr": (C.c_int, [P, i64, i64, P, i64, P, P, C.POINTER(C.c_int)]),
        "tt_svd_jacobi": (C.c_int, [P, i64, i64, P, i64, P, P, P]),
        "tt_svd_nov": (C.c_int, [P, i64, i64, P, i64, P, P]),
        "tt_cholesky": (C.c_int, [P, i64, P, i64, C.c_int, P, P]),
        "tt_cholqr_pass": (C.c_int, [P, i64, i64, P, i64, C.c_int, P, P, i64, P]),
        "tt_plan_create": (C.c_int, [P, i32, C.POINTER(tt_view), C.POINTER(tt_round_opts), i32,
                                     C.POINTER(u64), i32, C.POINTER(P)]),
        "tt_plan_launch": (C.c_int, [P]),
        "tt_plan_result": (C.c_int, [P, i32, C.POINTER(P)]),
        "tt_plan_destroy": (C.c_int, [P]),
        "tt_kron_apply": (C.c_int, [P, C.POINTER(tt_kron_op), C.POINTER(tt_view), C.POINTER(P)]),
        "tt_gmres": (C.c_int, [P, C.POINTER(tt_kron_op), C.POINTER(tt_view),
                               C.POINTER(tt_gmres_opts), C.POINTER(P), C.POINTER(tt_gmres_info),
                               C.POINTER(C.c_double)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(rc):
    if rc != 0:
        raise TTError(rc, _lib.tt_last_error().decode(errors="replace"))


def tt_launch_count() -> int:
    return int(load_library().tt_launch_count())


def tt_get_nccl_unique_id() -> bytes:
    L = load_library()
    buf = (C.c_uint8 * 128)()
    _check(L.tt_get_nccl_unique_id(buf))
    return bytes(buf)


# ------------------------------------------------------------------ marshalling
def _core_layout(c: torch.Tensor) -> torch.Tensor:
    """Core of logical shape (r0, I, r1) in the a-fastest layout of ttround.h
    (strides (1, r0, r0*I)); copies only if the given strides differ."""
    if c.dtype != torch.float64 or c.dim() != 3:
        raise TypeError("TT cores must be float64 tensors of shape (R_{n-1}, I_n, R_n)")
    r0, I, r1 = c.shape
    ok = c.stride(0) == 1 and (I == 1 or c.stride(1) == r0) and (r1 == 1 or c.stride(2) == r0 * I)
    if ok:
        return c
    return c.permute(2, 1, 0).contiguous().permute(2, 1, 0)


class _View:
    """Keeps the ctypes arrays (and any layout copies) of one tt_view alive."""

    def __init__(self, cores: Sequence[torch.Tensor]):
        cores = [_core_layout(c) for c in cores]
        d = len(cores)
        self.cores = cores
        self.dims = (C.c_int64 * d)(*[int(c.shape[1]) for c in cores])
        self.ranks = (C.c_int64 * (d + 1))(*([int(cores[0].shape[0])] +
                                               [int(c.shape[2]) for c in cores]))
        self.ptrs = (C.c_void_p * d)(*[c.data_ptr() for c in cores])
        self.view = tt_view(d, self.dims, self.ranks, self.ptrs)


class _CAI:
    """__cuda_array_interface__ wrapper: zero-copy torch views of library memory
    that keep the owning handle alive."""

    def __init__(self, ptr, shape, strides, owner):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": tuple(8 * s for s in strides),
                                         "stream": None}
        self._owner = owner


class _Handle:
    def __init__(self, ptr, destroy):
        self.ptr = ptr
        self._destroy = destroy

    def __del__(self):
        if self.ptr:
            self._destroy(self.ptr)
            self.ptr = None


class TTResult:
    """A rounded TT-tensor owned by the library (tt_tensor_t)."""

    def __init__(self, handle, device: torch.device):
        L = load_library()
        self._h = _Handle(handle, L.tt_tensor_destroy)
        d = C.c_int32()
        dims = C.POINTER(C.c_int64)()
        ranks = C.POINTER(C.c_int64)()
        cores = C.POINTER(C.c_void_p)()
        flags = C.c_uint32()
        _check(L.tt_tensor_info(handle, C.byref(d), C.byref(dims), C.byref(ranks),
                                C.byref(cores), C.byref(flags)))
        self.d = d.value
        self.dims = [dims[i] for i in range(self.d)]
        self.ranks = [ranks[i] for i in range(self.d + 1)]
        self.flags = flags.value
        p = C.c_int32()
        _check(L.tt_tensor_passes(handle, C.byref(p)))
        self.passes = p.value
        self._ptrs = [cores[i] for i in range(self.d)]
        self.device = device

    @property
    def cores(self) -> List[torch.Tensor]:
        """Zero-copy views, logical shape (r0, I, r1), a-fastest layout."""
        out = []
        for n in range(self.d):
            r0, I, r1 = self.ranks[n], self.dims[n], self.ranks[n + 1]
            cai = _CAI(self._ptrs[n], (r0, I, r1), (1, r0, r0 * I), self._h)
            out.append(torch.as_tensor(cai, device=self.device))
        return out

    def numpy(self):
        """Host copies (numpy arrays of shape (r0, I, r1)) via tt_tensor_copy_core."""
        L = load_library()
        res = []
        for n in range(self.d):
            r0, I, r1 = self.ranks[n], self.dims[n], self.ranks[n + 1]
            h = torch.empty((r1, I, r0), dtype=torch.float64)
            _check(L.tt_tensor_copy_core(self._h.ptr, n + 1, C.c_void_p(h.data_ptr())))
            res.append(h.permute(2, 1, 0).numpy())
        return res


class Sketch:
    """Random Gaussian TT of Def. 3.1 (tt_sketch_t)."""

    def __init__(self, handle, dims, ranks, device):
        L = load_library()
        self._h = _Handle(handle, L.tt_sketch_destroy)
        self.dims = list(dims)
        self.ranks = list(ranks)
        self.device = device

    def core(self, n: int) -> torch.Tensor:
        """Core n (1-based, n >= 2), logical shape (l_{n-1}, I_n, l_n)."""
        L = load_library()
        p = C.c_void_p()
        _check(L.tt_sketch_core(self._h.ptr, n, C.byref(p)))
        r0, I, r1 = self.ranks[n - 1], self.dims[n - 1], self.ranks[n]
        return torch.as_tensor(_CAI(p.value, (r0, I, r1), (1, r0, r0 * I), self._h),
                               device=self.device)


class Plan:
    """tt_plan_t: B roundings of fixed inputs captured in one CUDA graph."""

    def __init__(self, ctx, terms, seeds, mode="rank", rank=0, oversample=0, branches=1):
        L = load_library()
        self._views = [_View(t) for t in terms]     # inputs stay alive with the plan
        arr = (tt_view * len(self._views))(*[v.view for v in self._views])
        opts = tt_round_opts(_MODES[mode], 0, int(rank), int(oversample), 0.0, 0, 0)
        sd = (C.c_uint64 * len(seeds))(*[int(x) for x in seeds])
        h = C.c_void_p()
        _check(L.tt_plan_create(ctx.handle, len(self._views), arr, C.byref(opts), len(seeds),
                                sd, int(branches), C.byref(h)))
        self._h = _Handle(h.value, L.tt_plan_destroy)
        self._ctx = ctx
        self.B = len(seeds)

    def launch(self):
        _check(load_library().tt_plan_launch(self._h.ptr))

    def result(self, b: int) -> "TTResult":
        h = C.c_void_p()
        _check(load_library().tt_plan_result(self._h.ptr, int(b), C.byref(h)))
        return TTResult(h.value, self._ctx.device)


class LoopbackGroup:
    """tt_loopback_t: `world` ranks as contexts of this process on one device
    (drive each from its own thread); see include/ttround.h."""

    def __init__(self, world: int):
        L = load_library()
        h = C.c_void_p()
        _check(L.tt_loopback_create(int(world), C.byref(h)))
        self._h = _Handle(h.value, L.tt_loopback_destroy)
        self.world = int(world)


class Context:
    """tt_ctx_t: one CUDA device + stream (+ NCCL communicator when world > 1).

    The stream defaults to torch's current stream of the device, so calls are
    ordered with the torch kernels that produce the inputs."""

    def __init__(self, device: int = 0, stream: Optional[torch.cuda.Stream] = None,
                 nccl_id: Optional[bytes] = None, rank: int = 0, world: int = 1,
                 loopback: Optional[LoopbackGroup] = None):
        L = load_library()
        self.device = torch.device("cuda", device)
        if stream is None:
            # order every library call after the torch work that produced its
            # inputs (and before the torch work that consumes its outputs)
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        # handle 0 is torch's legacy default stream, but NULL means "library-owned
        # stream" at the C-ABI: pass cudaStreamLegacy (0x1) for it explicitly
        sp = C.c_void_p(stream.cuda_stream or 0x1)
        idbuf = (C.c_uint8 * 128)(*nccl_id) if nccl_id is not None else None
        h = C.c_void_p()
        if loopback is not None:
            _check(L.tt_ctx_create_loopback(device, sp, loopback._h.ptr, rank, C.byref(h)))
            world = loopback.world
            self._group = loopback          # the group outlives the context
        else:
            _check(L.tt_ctx_create(device, sp, idbuf, rank, world, C.byref(h)))
        self._h = _Handle(h.value, L.tt_ctx_destroy)
        self.rank, self.world = rank, world

    @property
    def handle(self):
        return self._h.ptr

    def close(self):
        self._h.__del__()

    def nccl_selftest(self, n: int = 1 << 16) -> float:
        """tt_nccl_selftest: one-rank NCCL communicator, fp64-sum and int64
        allreduce on this context's stream; returns the largest deviation."""
        out = C.c_double(-1.0)
        _check(load_library().tt_nccl_selftest(self.handle, int(n), C.byref(out)))
        return float(out.value)

    def set_timing(self, on: bool = True):
        _check(load_library().tt_ctx_set_timing(self.handle, int(on)))

    def set_concurrency(self, reserve_sms: int = 0, chain_priority: bool = False):
        """tt_ctx_set_concurrency: size persistent grids to (SMs - reserve_sms) and
        run the QR / truncation chain on a highest-priority stream."""
        _check(load_library().tt_ctx_set_concurrency(self.handle, int(reserve_sms),
                                                     int(chain_priority)))

    def last_timing(self) -> List[float]:
        buf = (C.c_double * 8)()
        n = load_library().tt_ctx_last_timing(self.handle, buf, 8)
        return [buf[i] for i in range(n)]

    def status_words(self, n: int = 8) -> List[int]:
        buf = (C.c_int * n)()
        k = load_library().tt_ctx_flags(self.handle, buf, n)
        if k < 0:
            _check(k)
        return [buf[i] for i in range(k)]

    # ---------------------------------------------------------------- sketch
    def tt_sketch_create(self, dims, ranks, seed: int, tag: int = 0) -> Sketch:
        L = load_library()
        d = len(dims)
        dd = (C.c_int64 * d)(*dims)
        rr = (C.c_int64 * (d + 1))(*ranks)
        h = C.c_void_p()
        _check(L.tt_sketch_create(self.handle, d, dd, rr, C.c_uint64(seed), tag, C.byref(h)))
        return Sketch(h.value, dims, ranks, self.device)

    # ---------------------------------------------------------------- hot path
    def tt_round_sum(self, terms: Sequence[Sequence[torch.Tensor]], mode: str = "rank",
                     rank=0, oversample: int = 0, tol: float = 0.0, seed: int = 1,
                     adaptive: bool = False, max_rank: int = 0,
                     sketch: Optional[Sketch] = None) -> TTResult:
        """Round sum_j terms[j] (Alg. 7 + truncation); see include/ttround.h.
        `rank`: an int, or a list of d-1 per-bond target ranks (opts.ranks)."""
        L = load_library()
        views = [_View(t) for t in terms]
        arr = (tt_view * len(views))(*[v.view for v in views]) if views else None
        opts, _keep = _make_opts(_MODES[mode], adaptive, rank, oversample, tol, seed, max_rank)
        h = C.c_void_p()
        _check(L.tt_round_sum(self.handle, len(views), arr, C.byref(opts),
                              sketch._h.ptr if sketch is not None else None, C.byref(h)))
        return TTResult(h.value, self.device)

    def tt_round_sum_slab(self, terms: Sequence[Sequence[torch.Tensor]], gdims: Sequence[int],
                          slab_lo: Sequence[int], mode: str = "rank", rank: int = 0,
                          oversample: int = 0, tol: float = 0.0, seed: int = 1,
                          adaptive: bool = False, max_rank: int = 0) -> TTResult:
        """Mode-slab sharded rounding (NEXT-2): `terms` are this rank's slabs of ALL
        summands (cores (R, I_slab, R')), the slab of mode n starts at slab_lo[n] of
        gdims[n].  Returns this rank's slabs of the rounded cores."""
        L = load_library()
        views = [_View(t) for t in terms]
        arr = (tt_view * len(views))(*[v.view for v in views])
        d = len(gdims)
        g = (C.c_int64 * d)(*[int(x) for x in gdims])
        lo = (C.c_int64 * d)(*[int(x) for x in slab_lo])
        opts, _keep = _make_opts(_MODES[mode], adaptive, rank, oversample, tol, seed, max_rank)
        h = C.c_void_p()
        _check(L.tt_round_sum_slab(self.handle, len(views), arr, g, lo, C.byref(opts),
                                   C.byref(h)))
        return TTResult(h.value, self.device)

    def tt_inner(self, x: Sequence[torch.Tensor], y: Sequence[torch.Tensor]) -> float:
        L = load_library()
        vx, vy = _View(x), _View(y)
        out = C.c_double()
        _check(L.tt_inner(self.handle, C.byref(vx.view), C.byref(vy.view), C.byref(out)))
        return out.value

    def tt_round_deterministic(self, terms, tol: float, rank: int = 0) -> TTResult:
        L = load_library()
        views = [_View(t) for t in terms]
        arr = (tt_view * len(views))(*[v.view for v in views])
        opts, _keep = _make_opts(TOL, 0, rank, 0, tol, 0, 0)
        h = C.c_void_p()
        _check(L.tt_round_deterministic(self.handle, len(views), arr, C.byref(opts), C.byref(h)))
        return TTResult(h.value, self.device)

    def tt_round_sum_two_sided(self, terms, ell: int, rho: int = 0, seed: int = 1) -> TTResult:
        """Round sum_j terms[j] with Alg. 6 (two-sided randomization); rho = 0 means
        ceil(1.5 ell).  See include/ttround.h."""
        L = load_library()
        views = [_View(t) for t in terms]
        arr = (tt_view * len(views))(*[v.view for v in views]) if views else None
        h = C.c_void_p()
        _check(L.tt_round_sum_two_sided(self.handle, len(views), arr, int(ell), int(rho),
                                        C.c_uint64(seed).value, C.byref(h)))
        return TTResult(h.value, self.device)

    # ---------------------------------------------------------------- kernels
    def tt_dgemm(self, A: torch.Tensor, B: torch.Tensor, trans_a=False, trans_b=False,
                 alpha=1.0, beta=0.0, C_out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Column-major GEMM on torch tensors (matrices passed as their column-major
        storage: a torch (rows, cols) tensor with strides (1, rows))."""
        L = load_library()
        m = A.shape[1] if trans_a else A.shape[0]
        k = A.shape[0] if trans_a else A.shape[1]
        n = B.shape[0] if trans_b else B.shape[1]
        for X in (A, B):
            assert X.stride(0) == 1, "column-major operands (stride(0) == 1)"
        if C_out is None:
            C_out = torch.zeros((n, m), dtype=torch.float64, device=A.device).t()
        _check(L.tt_dgemm(self.handle, int(trans_a), int(trans_b), m, n, k, alpha,
                          A.data_ptr(), A.stride(1), B.data_ptr(), B.stride(1), beta,
                          C_out.data_ptr(), C_out.stride(1)))
        return C_out

    def tt_qr(self, A: torch.Tensor, want_r: bool = False, want_q: bool = True):
        L = load_library()
        m, n = A.shape
        assert A.stride(0) == 1
        Q = torch.empty((n, m), dtype=torch.float64, device=A.device).t() if want_q else None
        R = torch.empty((n, n), dtype=torch.float64, device=A.device).t() if want_r else None
        fb = C.c_int()
        _check(L.tt_qr(self.handle, m, n, A.data_ptr(), A.stride(1),
                       Q.data_ptr() if Q is not None else None,
                       R.data_ptr() if R is not None else None, C.byref(fb)))
        return Q, R, bool(fb.value)

    def tt_svd_jacobi(self, A: torch.Tensor):
        L = load_library()
        m, n = A.shape
        assert A.stride(0) == 1
        AV = torch.empty((n, m), dtype=torch.float64, device=A.device).t()
        V = torch.empty((n, n), dtype=torch.float64, device=A.device).t()
        s = torch.empty((n,), dtype=torch.float64, device=A.device)
        _check(L.tt_svd_jacobi(self.handle, m, n, A.data_ptr(), A.stride(1), AV.data_ptr(),
                               V.data_ptr(), s.data_ptr()))
        return AV, V, s

    def tt_cholesky(self, G: torch.Tensor, m: int = 0, shifted: bool = False):
        """One factorisation of the CholeskyQR passes: (Rinv = L^{-T}, L)."""
        L = load_library()
        n = G.shape[0]
        assert G.stride(0) == 1 and G.shape == (n, n)
        Rinv = torch.empty((n, n), dtype=torch.float64, device=G.device).t()
        Lo = torch.empty((n, n), dtype=torch.float64, device=G.device).t()
        _check(L.tt_cholesky(self.handle, n, G.data_ptr(), int(m or n), int(bool(shifted)),
                             Rinv.data_ptr(), Lo.data_ptr()))
        return Rinv, Lo

    def tt_cholqr_pass(self, A: torch.Tensor, Rinv: Optional[torch.Tensor] = None,
                       trans: bool = False, want_q: bool = True, want_g: bool = True):
        """One fused CholeskyQR pass: (Q = op(A) Rinv, G = Q^T Q); op(A) = A or A^T
        (A column-major), Rinv None means Q = op(A)."""
        L = load_library()
        assert A.stride(0) == 1 and A.dtype == torch.float64
        m, n = (A.shape[1], A.shape[0]) if trans else A.shape
        if Rinv is not None:
            assert Rinv.stride(0) == 1 and Rinv.stride(1) == n and Rinv.shape == (n, n)
        Q = torch.empty((n, m), dtype=torch.float64, device=A.device).t() if want_q else None
        G = torch.empty((n, n), dtype=torch.float64, device=A.device).t() if want_g else None
        _check(L.tt_cholqr_pass(self.handle, m, n, A.data_ptr(), A.stride(1), int(trans),
                                Rinv.data_ptr() if Rinv is not None else None,
                                Q.data_ptr() if Q is not None else None, m,
                                G.data_ptr() if G is not None else None))
        return Q, G

    def tt_svd_nov(self, A: torch.Tensor):
        """V-free one-sided Jacobi (the truncation's SVD): (U Sigma, sigma)."""
        L = load_library()
        m, n = A.shape
        assert A.stride(0) == 1
        AV = torch.empty((n, m), dtype=torch.float64, device=A.device).t()
        s = torch.empty((n,), dtype=torch.float64, device=A.device)
        _check(L.tt_svd_nov(self.handle, m, n, A.data_ptr(), A.stride(1), AV.data_ptr(),
                            s.data_ptr()))
        return AV, s

    # ---------------------------------------------------------------- TT-GMRES (NEXT-4)
    def _kron(self, op, dims):
        """Marshal a Kronecker-sum operator: op[i][n] is None (identity), a 1-D
        tensor (diagonal) or a 2-D (I, I) tensor (dense A with A[i, j] at row i)."""
        d, nt = len(dims), len(op)
        kinds = (C.c_int32 * (nt * d))()
        mats = (C.c_void_p * (nt * d))()
        keep = []
        for i, term in enumerate(op):
            if len(term) != d:
                raise ValueError("every operator term needs one factor per mode")
            for n, A in enumerate(term):
                if A is None:
                    kinds[i * d + n] = 0
                    continue
                A = torch.as_tensor(A, dtype=torch.float64, device=self.device)
                if A.dim() == 1:
                    kinds[i * d + n] = 1
                    A = A.contiguous()
                else:
                    kinds[i * d + n] = 2
                    A = A.t().contiguous()      # column-major storage of A
                keep.append(A)
                mats[i * d + n] = A.data_ptr()
        dd = (C.c_int64 * d)(*dims)
        return tt_kron_op(d, nt, dd, kinds, mats), (keep, dd, kinds, mats)

    def tt_kron_apply(self, op, x: Sequence[torch.Tensor]) -> List[TTResult]:
        """The unrounded summands of (sum_i A_{i,1} x ... x A_{i,d}) x."""
        L = load_library()
        vx = _View(x)
        k, keep = self._kron(op, [int(c.shape[1]) for c in x])
        out = (C.c_void_p * len(op))()
        _check(L.tt_kron_apply(self.handle, C.byref(k), C.byref(vx.view), out))
        return [TTResult(out[i], self.device) for i in range(len(op))]

    def tt_gmres(self, op, f: Sequence[torch.Tensor], tol: float = 1e-8, max_iter: int = 50,
                 round_tol: float = 0.0, randomized: bool = True, precond: bool = True,
                 oversample: int = 10, max_rank: int = 0, seed: int = 1):
        """Right-preconditioned TT-GMRES; returns (x, info dict)."""
        L = load_library()
        vf = _View(f)
        k, keep = self._kron(op, [int(c.shape[1]) for c in f])
        o = tt_gmres_opts(float(tol), float(round_tol), int(max_iter), int(randomized),
                          int(precond), int(oversample), int(max_rank), C.c_uint64(seed).value)
        info = tt_gmres_info()
        res = (C.c_double * (max_iter + 1))()
        h = C.c_void_p()
        _check(L.tt_gmres(self.handle, C.byref(k), C.byref(vf.view), C.byref(o), C.byref(h),
                          C.byref(info), res))
        out = {"iters": info.iters, "converged": bool(info.converged),
               "roundings": info.roundings, "max_basis_rank": info.max_basis_rank,
               "residual": info.residual, "residuals": [res[i] for i in range(info.iters + 1)]}
        return TTResult(h.value, self.device), out
