"""B200-native matrix-free high-order FEM hot path (arXiv 2402.15940): PA
sum-factorization BP1/BP3/BP5 operators and CG, as the C-ABI library
``libhofem.so`` (include/hofem.h) plus this thin ctypes binding."""
from .hofem import (ALWAYS, AUTO, BC_DIRICHLET, BC_NONE, DIFFUSION, GAUSS, GLL, MASS,  # noqa
                    NEVER, OPT_CG_FUSED_UPDATE, OPT_CG_PERSISTENT, OPT_INFIX, OPT_L2_PREFETCH,
                    Comm, DGMass, HofemError, LoopbackGroup, PMG, Mesh, Operator, launch_count, launch_count_reset, lib,
                    profile_enable, profile_read)
