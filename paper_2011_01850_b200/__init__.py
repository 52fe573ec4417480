"""B200-native mixed-precision restarted GMRES(m) (Lindquist, Luszczek, Dongarra,
arXiv 2011.01850) — thin Python binding over the C-ABI library ``libgmres.so``.

Every step of the solve runs in the hand-written sm_100a kernels behind
``include/gmres.h``; this package only marshals arguments.  PyTorch supplies
device memory, streams and process groups.  There is no CPU fallback: if the
CUDA library is missing, importing the binding raises.
"""
from .gmres import (  # noqa: F401
    CGSR, FP64, ILU0, JACOBI, MGS, MIXED, GmresError, Solver, SolveResult, library_path, load_library,
)

__all__ = ["Solver", "SolveResult", "GmresError", "MGS", "CGSR", "FP64", "MIXED", "JACOBI", "ILU0", "load_library", "library_path"]
