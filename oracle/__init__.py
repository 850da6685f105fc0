"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 NumPy implementation of what the hot path
computes (Alg. 1, 2, 3, 5, 6, 7 and the truncation recipe of P:667-670),
written step by step in the paper's order and notation.  Library primitives
(``numpy.matmul``, ``numpy.linalg.qr`` = LAPACK Householder, ``numpy.linalg.svd``)
serve as single steps; there is no blocking, fusion or reordering beyond the
algorithms as printed.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_2110_04393_b200``) and imports nothing from it.

Parity status per function is listed in DESIGN.md §"Oracle pins"; every public
function here is pinned by a ``-m "not gpu"`` test against something other than
itself (brute force on dense tensors, closed forms, cuRAND's Philox, paper
invariants).
"""
from .philox import philox4x32_10, sketch_core, philox_normal  # noqa: F401
from .tt import *  # noqa: F401,F403
from . import gmres  # noqa: F401  (TT-GMRES)
