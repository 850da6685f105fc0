"""CPU-only checks of the C-ABI library: it loads and exports every function
include/ttround.h declares; argument validation paths that need no GPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ttround.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(tt_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2110_04393_b200 import build
    build.build()
    import paper_2110_04393_b200 as P
    return P.load_library()


def test_header_declares_the_boundary_calls():
    f = declared_functions()
    for name in ["tt_sketch_create", "tt_round_sum", "tt_round_deterministic", "tt_inner",
                 "tt_round_sum_two_sided",
                 "tt_ctx_create", "tt_tensor_info", "tt_last_error"]:
        assert name in f
    assert len(f) >= 20


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    so = os.path.join(ROOT, "paper_2110_04393_b200", "libttround.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tt_\w+)", out))
    assert set(declared_functions()) <= exported


def test_library_contains_sm100a_dmma_code():
    so = os.path.join(ROOT, "paper_2110_04393_b200", "libttround.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", so], capture_output=True,
                         text=True).stdout
    assert "DMMA.8x8x4" in out          # FP64 tensor-core path
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", so],
                                       capture_output=True, text=True).stdout


def test_argument_errors_without_gpu(lib):
    import paper_2110_04393_b200 as P
    # null ctx / out must fail cleanly with a message, not crash
    rc = lib.tt_round_sum(None, 1, None, None, None, None)
    assert rc == -1 and b"null" in lib.tt_last_error()
    rc = lib.tt_nccl_selftest(None, 4, None)
    assert rc == -1
    rc = lib.tt_round_sum_two_sided(None, 1, None, 4, 0, 1, None)
    assert rc == -1 and b"null" in lib.tt_last_error()
    rc = lib.tt_ctx_create(0, None, None, 2, 1, None)
    assert rc == -1
    assert lib.tt_launch_count() == 0 or lib.tt_launch_count() > 0
    with pytest.raises(P.TTError):
        P._lib._check(-2)
