"""Seeded synthetic input generators shared by the tests, the oracle side and the
CUDA side.  This module holds NONE of the method's arithmetic: only mesh recipes
(sizes of the BASELINE.json configs) and the counter-based random vector of
DESIGN.md reading R12.  The CUDA library implements the same generator on the
device (``hofem_fill_random``); tests check the two bit for bit.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_mix(z: np.ndarray) -> np.ndarray:
    """The standard splitmix64 output finalizer (uint64 arithmetic mod 2^64)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def random_vector(seed: int, g: np.ndarray) -> np.ndarray:
    """Reading R12: x_g = 2*((mix(seed + (g+1)*GOLDEN) >> 11) * 2^-53) - 1.

    ``g`` are GLOBAL dof indices, so every partition sees the same global vector.
    """
    g = np.asarray(g, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (g + np.uint64(1)) * GOLDEN
    u = (splitmix64_mix(z) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return 2.0 * u - 1.0


def random_lvector(mesh_dims, seed: int, z_plane0: int = 0) -> np.ndarray:
    """Random L-vector of a (window of a) structured mesh, lexicographic x fastest.

    mesh_dims = (Nx, Ny, Nz_local) lattice sizes; z_plane0 = first global plane.
    """
    Nx, Ny, Nz = mesh_dims
    n = Nx * Ny * Nz
    g = np.arange(n, dtype=np.uint64) + np.uint64(Nx * Ny * z_plane0)
    return random_vector(seed, g)


# --------------------------------------------------------------------------
# BASELINE.json configs as mesh recipes (SURVEY.md §8(d) "Concrete synthetic
# inputs"): structured unit cube, curvilinear alpha = 0.1, coefficient 1.
# --------------------------------------------------------------------------
ALPHA = 0.1


def bp1_sweep_n(p: int) -> int:
    """Config 2: BP1 on ~1M dofs, n = round(99/p) elements per axis."""
    return int(round(99.0 / p))


def bp3_sweep_n(p: int) -> int:
    """Config 3/4: BP3/BP5 on ~30M dofs per GPU, n = round(311/p)."""
    return int(round(311.0 / p))


def dg_sweep_n(p: int) -> int:
    """f4 DG mass: ~30M DG dofs, E (p+1)^3 with n = round(311/(p+1)) per axis."""
    return int(round(311.0 / (p + 1)))


def config5(n_gpus: int = 1):
    """Config 5: BP3 p=5, 200 x 200 x 25R elements (~125.5M
    dofs per GPU), weak scaling over R GPUs."""
    return dict(name=f"bp3_p5_200x200x{25 * n_gpus}", nx=200, ny=200, nz=25 * n_gpus, p=5,
                alpha=ALPHA)


CONFIG1 = dict(name="bp3_2x2x2_p2", nx=2, ny=2, nz=2, p=2, alpha=ALPHA)


def config3(p: int, n_gpus: int = 1):
    """BP3 ~30M dofs per GPU; weak scaling stacks n_gpus slabs in z."""
    n = bp3_sweep_n(p)
    return dict(name=f"bp3_p{p}_{n}x{n}x{n * n_gpus}", nx=n, ny=n, nz=n * n_gpus, p=p,
                alpha=ALPHA)


def n_dofs(nx, ny, nz, p) -> int:
    return (p * nx + 1) * (p * ny + 1) * (p * nz + 1)
