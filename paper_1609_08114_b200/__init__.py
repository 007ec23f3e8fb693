"""B200-native batched LP solver (Gurung & Ray, arXiv 1609.08114, hot path).

Public API (thin binding of the C ABI in include/lpb.h, kernels in csrc/):
    lpb.solve(A, b, c, ...)        batch simplex (types 1 and 2)
    lpb.hyperbox(lo, hi, dirs)     closed-form hyperbox LPs (type 3)
    lpb.Solver(...)                reusable context (device or host pipeline)
    dist.solve_sharded(...)        contiguous shards over torch.distributed ranks
Importing fails loudly when liblpb.so is missing: there is no CPU fallback.
"""
from . import lpb  # noqa: F401  (raises ImportError if liblpb.so is not built)
from .lpb import Solver, hyperbox, solve  # noqa: F401

__all__ = ["lpb", "Solver", "solve", "hyperbox"]
