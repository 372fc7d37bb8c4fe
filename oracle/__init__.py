"""CPU FP64 oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product package
``paper_2402_15940_b200`` never imports it, and it imports nothing from the
product.  See ``oracle/oracle.c`` for what is computed and which passage of
PAPER.md / SURVEY.md §8(c) each function follows.

This module is a thin ctypes binding over ``liboracle.so`` (built from
``oracle/oracle.c`` by :func:`build`).  All arrays are numpy float64 / int64 /
uint8, C-contiguous.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

MASS, DIFFUSION = 1, 2
GAUSS, GLL = 1, 2


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (FP64, no FMA contraction, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
             "-Wall", "-Wno-unknown-pragmas", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Mesh(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("p", ctypes.c_int), ("L", ctypes.c_double * 3), ("alpha", ctypes.c_double),
                ("z0", ctypes.c_int), ("nzl", ctypes.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        d, i, ll = ctypes.c_double, ctypes.c_int, ctypes.c_longlong
        P = ctypes.c_void_p
        M = ctypes.POINTER(_Mesh)
        sig = {
            "orc_gll": (i, [i, P, P]),
            "orc_gauss": (i, [i, P, P]),
            "orc_tabulate": (i, [i, i, i, P, P]),
            "orc_dg_mass_matrices": (i, [M, i, P]),
            "orc_dg_apply": (i, [M, P, P, P]),
            "orc_dg_apply_sample": (i, [M, i, P, ll, P, P]),
            "orc_num_dofs": (ll, [M]),
            "orc_num_elems": (ll, [M]),
            "orc_mesh_coords": (i, [M, P]),
            "orc_boundary_mask": (i, [M, P]),
            "orc_qdata": (i, [M, i, i, i, P]),
            "orc_element_matrices": (i, [M, i, i, i, P]),
            "orc_apply_ea": (i, [M, P, i, P, P]),
            "orc_apply_dense": (i, [M, i, i, i, i, P, P]),
            "orc_element_apply_sample": (i, [M, i, i, i, P, ll, P, P]),
            "orc_assemble_dense": (i, [M, P, P]),
            "orc_rhs": (i, [M, i, i, i, i, P]),
            "orc_l2_error": (d, [M, P, i]),
            "orc_cg": (i, [M, P, i, P, ll, P, P, d, i, i, P, P, P]),
            "orc_num_threads": (i, []),
            "orc_diagonal": (i, [M, P, i, P]),
            "orc_prolong": (i, [M, M, P, P]),
            "orc_restrict": (i, [M, M, P, P]),
            "orc_power_lmax": (d, [M, P, i, P, P, i]),
            "orc_cheb": (i, [M, P, i, P, d, d, i, P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype, f.argtypes = res, args
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


@dataclass(frozen=True)
class Mesh:
    """Structured hex mesh window (readings R1, R3, R4, R9)."""
    nx: int
    ny: int
    nz: int
    p: int
    alpha: float = 0.1
    L: tuple = (1.0, 1.0, 1.0)
    z0: int = 0
    nzl: int | None = None

    def c(self) -> _Mesh:
        m = _Mesh()
        m.nx, m.ny, m.nz, m.p = self.nx, self.ny, self.nz, self.p
        m.L[0], m.L[1], m.L[2] = self.L
        m.alpha = self.alpha
        m.z0 = self.z0
        m.nzl = self.nz if self.nzl is None else self.nzl
        return m

    @property
    def n_dofs(self) -> int:
        nzl = self.nz if self.nzl is None else self.nzl
        return (self.p * self.nx + 1) * (self.p * self.ny + 1) * (self.p * nzl + 1)

    @property
    def n_elems(self) -> int:
        return self.nx * self.ny * (self.nz if self.nzl is None else self.nzl)


def default_q(p: int, rule: int) -> int:
    """Reading R2: Gauss Q = p+2 (BP1/BP3), GLL Q = p+1 (BP5)."""
    return p + 2 if rule == GAUSS else p + 1


def gll(p):
    x, w = np.zeros(p + 1), np.zeros(p + 1)
    assert lib().orc_gll(p, _p(x), _p(w)) == 0
    return x, w


def gauss(q):
    x, w = np.zeros(q), np.zeros(q)
    assert lib().orc_gauss(q, _p(x), _p(w)) == 0
    return x, w


def tabulate(p, Q, rule=GAUSS):
    B, G = np.zeros((Q, p + 1)), np.zeros((Q, p + 1))
    assert lib().orc_tabulate(p, Q, rule, _p(B), _p(G)) == 0
    return B, G


def mesh_coords(m: Mesh):
    xyz = np.zeros((3, m.n_dofs))
    mc = m.c()
    assert lib().orc_mesh_coords(ctypes.byref(mc), _p(xyz)) == 0
    return xyz


def boundary_mask(m: Mesh):
    mask = np.zeros(m.n_dofs, dtype=np.uint8)
    mc = m.c()
    lib().orc_boundary_mask(ctypes.byref(mc), _p(mask))
    return mask.astype(bool)


def qdata(m: Mesh, kind, rule, Q=None):
    Q = Q or default_q(m.p, rule)
    nc = 1 if kind == MASS else 6
    qd = np.zeros((m.n_elems, nc, Q ** 3))
    mc = m.c()
    st = lib().orc_qdata(ctypes.byref(mc), kind, rule, Q, _p(qd))
    if st:
        raise ValueError(f"orc_qdata status {st}")
    return qd


def element_matrices(m: Mesh, kind, rule, Q=None):
    Q = Q or default_q(m.p, rule)
    nd = (m.p + 1) ** 3
    Ae = np.zeros((m.n_elems, nd, nd))
    mc = m.c()
    st = lib().orc_element_matrices(ctypes.byref(mc), kind, rule, Q, _p(Ae))
    if st:
        raise ValueError(f"orc_element_matrices status {st}")
    return Ae


def apply_ea(m: Mesh, Ae, x, bc=0):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(m.n_dofs)
    mc = m.c()
    lib().orc_apply_ea(ctypes.byref(mc), _p(Ae), int(bc), _p(x), _p(y))
    return y


def apply_dense(m: Mesh, kind, rule, x, bc=0, Q=None):
    Q = Q or default_q(m.p, rule)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(m.n_dofs)
    mc = m.c()
    st = lib().orc_apply_dense(ctypes.byref(mc), kind, rule, Q, int(bc), _p(x), _p(y))
    if st:
        raise ValueError(f"orc_apply_dense status {st}")
    return y


def element_apply_sample(m: Mesh, kind, rule, x, elems, Q=None):
    Q = Q or default_q(m.p, rule)
    x = np.ascontiguousarray(x, dtype=np.float64)
    elems = np.ascontiguousarray(elems, dtype=np.int64)
    ye = np.zeros((len(elems), (m.p + 1) ** 3))
    mc = m.c()
    st = lib().orc_element_apply_sample(ctypes.byref(mc), kind, rule, Q, _p(x), len(elems),
                                        _p(elems), _p(ye))
    if st:
        raise ValueError(f"orc_element_apply_sample status {st}")
    return ye


def dg_mass_matrices(m: Mesh, Q=None):
    """DG (L2, Gauss-Legendre nodal) element mass matrices [E][nd][nd] (f4)."""
    Q = Q or default_q(m.p, GAUSS)
    nd = (m.p + 1) ** 3
    Me = np.zeros((m.n_elems, nd, nd))
    mc = m.c()
    st = lib().orc_dg_mass_matrices(ctypes.byref(mc), Q, _p(Me))
    if st:
        raise ValueError(f"orc_dg_mass_matrices status {st}")
    return Me


def dg_apply(m: Mesh, Me, x):
    """y_e = M_e x_e over the element-major DG vector x [E * P1^3]."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros_like(x)
    mc = m.c()
    lib().orc_dg_apply(ctypes.byref(mc), _p(Me), _p(x), _p(y))
    return y


def dg_apply_sample(m: Mesh, x, elems, Q=None):
    """y_e = M_e x_e for the listed elements of the E-vector x (sampled parity)."""
    Q = Q or default_q(m.p, GAUSS)
    x = np.ascontiguousarray(x, dtype=np.float64)
    elems = np.ascontiguousarray(elems, dtype=np.int64)
    ye = np.zeros((len(elems), (m.p + 1) ** 3))
    mc = m.c()
    st = lib().orc_dg_apply_sample(ctypes.byref(mc), Q, _p(x), len(elems), _p(elems), _p(ye))
    if st:
        raise ValueError(f"orc_dg_apply_sample status {st}")
    return ye


def assemble_dense(m: Mesh, Ae):
    A = np.zeros((m.n_dofs, m.n_dofs))
    mc = m.c()
    lib().orc_assemble_dense(ctypes.byref(mc), _p(Ae), _p(A))
    return A


def rhs(m: Mesh, kind, rule, bc=1, Q=None):
    Q = Q or default_q(m.p, rule)
    b = np.zeros(m.n_dofs)
    mc = m.c()
    assert lib().orc_rhs(ctypes.byref(mc), kind, rule, Q, int(bc), _p(b)) == 0
    return b


def l2_error(m: Mesh, uh, Qover=None):
    Qover = Qover or (m.p + 4)
    uh = np.ascontiguousarray(uh, dtype=np.float64)
    mc = m.c()
    return lib().orc_l2_error(ctypes.byref(mc), _p(uh), Qover)


def cg(b, *, m: Mesh | None = None, Ae=None, bc=0, A=None, x0=None, rel_tol=1e-12,
       max_iter=1000, fixed_iters=False, history=False):
    """Textbook CG on the EA operator (m, Ae, bc) or on a dense matrix A.

    Returns (x, status, iters, rr_hist, x_hist); x_hist is None unless history.
    status: 0 converged / fixed count done, 6 breakdown, 7 max_iter reached.
    """
    b = np.ascontiguousarray(b, dtype=np.float64)
    N = len(b)
    x = np.zeros(N) if x0 is None else np.array(x0, dtype=np.float64)
    rr = np.zeros(max_iter + 1)
    xh = np.zeros((max_iter + 1, N)) if history else None
    it = ctypes.c_int(0)
    mc = m.c() if m is not None else None
    if A is not None:
        A = np.ascontiguousarray(A, dtype=np.float64)
    st = lib().orc_cg(ctypes.byref(mc) if mc is not None else None, _p(Ae), int(bc), _p(A), N,
                      _p(b), _p(x), rel_tol, max_iter, int(fixed_iters), _p(rr), _p(xh),
                      ctypes.byref(it))
    k = it.value
    return x, st, k, rr[: k + 1], (xh[: k + 1] if history else None)


def num_threads() -> int:
    return lib().orc_num_threads()
