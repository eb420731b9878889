"""B200-native (sm_100a) adaptive multigrid Poisson solver — the hot path of
arXiv 2512.08555 (FAS V-cycle on a block-structured multiresolution grid).

The product is `libmg.so` (include/mg.h, CUDA kernels in csrc/); `mg.Solver` is a
thin ctypes binding.  Build with `python -m paper_2512_08555_b200.build`.
"""
from .mg import (MG_BC_PERIODIC, MG_BC_UNBOUNDED, MG_CRIT_CAUCHY, MG_CRIT_RESIDUAL, MG_FIELD_F, MG_FIELD_R,
                 MG_FIELD_U, MG_FIELD_UHAT, MG_SMOOTHER_JACOBI, MG_SMOOTHER_RBGS, MgError, Solver, adapt,
                 detail, load_library)

__all__ = ["Solver", "MgError", "load_library", "detail", "adapt", "MG_BC_PERIODIC", "MG_BC_UNBOUNDED", "MG_SMOOTHER_JACOBI",
           "MG_SMOOTHER_RBGS", "MG_CRIT_RESIDUAL", "MG_CRIT_CAUCHY", "MG_FIELD_U", "MG_FIELD_F", "MG_FIELD_R",
           "MG_FIELD_UHAT"]
