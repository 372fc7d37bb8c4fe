"""B200-native matrix-free high-order FEM hot path (arXiv 2402.15940): PA
sum-factorization BP1/BP3/BP5 operators and CG, as the C-ABI library
``libhofem.so`` (include/hofem.h) plus this thin ctypes binding."""
from .hofem import (BC_DIRICHLET, BC_NONE, DIFFUSION, GAUSS, GLL, MASS, Comm, HofemError,  # noqa
                    Mesh, Operator, launch_count, launch_count_reset, lib, profile_enable,
                    profile_read)
