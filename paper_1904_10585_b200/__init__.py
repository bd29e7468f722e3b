"""B200-native hot path of the polynomial-filtered first-order methods PFPG / PFAM
(arXiv 1904.10585): C-ABI library libpf.so (include/pf.h) + this thin binding.

The CUDA extension is required: importing `Context` / `Solver` loads libpf.so and raises if it
is missing.  There is no CPU fallback in this package.
"""
from ._lib import (Context, PFError, PF_FP64, PF_TF32, PF_OP_PSD, PF_OP_SOFT_THRESHOLD,  # noqa: F401
                   load)
from .solver import Solver, run  # noqa: F401
from .svt import SVTSolver, run_svt  # noqa: F401
