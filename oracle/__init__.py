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
            "orc_set_threads": (None, [i]),
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


# ----------------------------------------------------------------------------- f2
# p-multigrid preconditioned CG (§2.1;
# PAPER.md:156 BPS3).  Readings R17 (hierarchy, smoother, eigen estimate) and
# R18 (PCG) of DESIGN.md §3.  The V-cycle and PCG below follow the algorithm
# step by step in numpy, calling the C primitives (EA apply, diagonal,
# transfers, Chebyshev, power iteration) for each step.

def diagonal(m: Mesh, Ae, bc=0):
    d = np.zeros(m.n_dofs)
    mc = m.c()
    lib().orc_diagonal(ctypes.byref(mc), _p(Ae), int(bc), _p(d))
    return d


def prolong(mf: Mesh, mc_: Mesh, xc):
    xc = np.ascontiguousarray(xc, dtype=np.float64)
    xf = np.zeros(mf.n_dofs)
    a, b = mf.c(), mc_.c()
    lib().orc_prolong(ctypes.byref(a), ctypes.byref(b), _p(xc), _p(xf))
    return xf


def restrict(mf: Mesh, mc_: Mesh, rf):
    rf = np.ascontiguousarray(rf, dtype=np.float64)
    rc = np.zeros(mc_.n_dofs)
    a, b = mf.c(), mc_.c()
    lib().orc_restrict(ctypes.byref(a), ctypes.byref(b), _p(rf), _p(rc))
    return rc


def power_lmax(m: Mesh, Ae, bc, dinv, v0, iters=10):
    v0 = np.ascontiguousarray(v0, dtype=np.float64)
    mc = m.c()
    return lib().orc_power_lmax(ctypes.byref(mc), _p(Ae), int(bc), _p(dinv), _p(v0), int(iters))


def cheb(m: Mesh, Ae, bc, dinv, lmin, lmax, degree, b, x):
    """Chebyshev-Jacobi smoothing (Saad Alg. 12.1); returns the new x."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.array(x, dtype=np.float64)
    mc = m.c()
    lib().orc_cheb(ctypes.byref(mc), _p(Ae), int(bc), _p(dinv), float(lmin), float(lmax),
                   int(degree), _p(b), _p(x))
    return x


def pmg_orders(p: int):
    """Reading R17: p_{k-1} = max(1, p_k // 2) down to 1 (fine first)."""
    out = [p]
    while out[-1] > 1:
        out.append(max(1, out[-1] // 2))
    return out


CHEB_HI, CHEB_LO = 1.2, 0.3  # reading R17: [0.3 * 1.2 lam, 1.2 lam]


class PMG:
    """p-multigrid V-cycle on the BP3 (Gauss Q = p_k + 2) Dirichlet operators of
    the same element grid at orders pmg_orders(p); every level is an EA oracle."""

    def __init__(self, nx, ny, nz, p, alpha=0.1, degree=3, power_iters=10, seed=1,
                 lmax=None):
        import workloads as W
        self.orders = pmg_orders(p)
        self.degree = degree
        self.levels = []
        for k, pk in enumerate(self.orders):
            m = Mesh(nx, ny, nz, pk, alpha=alpha)
            Ae = element_matrices(m, DIFFUSION, GAUSS)
            d = diagonal(m, Ae, bc=1)
            dinv = 1.0 / d
            if lmax is not None:
                lam = lmax[k]
            else:
                v0 = W.random_vector(seed, np.arange(m.n_dofs))
                lam = power_lmax(m, Ae, 1, dinv, v0, power_iters)
            self.levels.append(dict(m=m, Ae=Ae, dinv=dinv, lam=lam, ess=boundary_mask(m),
                                    lmax=CHEB_HI * lam, lmin=CHEB_LO * CHEB_HI * lam))

    def smooth(self, k, b, x):
        L = self.levels[k]
        return cheb(L["m"], L["Ae"], 1, L["dinv"], L["lmin"], L["lmax"], self.degree, b, x)

    def vcycle(self, b, k=0):
        """Level k = 0 is the finest (orders[0] = p)."""
        L = self.levels[k]
        x = self.smooth(k, b, np.zeros_like(b))
        if k + 1 < len(self.levels):
            r = b - apply_ea(L["m"], L["Ae"], x, bc=1)
            C = self.levels[k + 1]
            rc = restrict(L["m"], C["m"], r)
            rc[C["ess"]] = 0.0  # coarse Dirichlet rows of the restricted residual (R17)
            ec = self.vcycle(rc, k + 1)
            x = x + prolong(L["m"], C["m"], ec)
        return self.smooth(k, b, x)


def pcg(b, M, *, m: Mesh, Ae, bc=1, rel_tol=1e-10, max_iter=500, history=False):
    """Preconditioned CG (reading R18): x0 = 0, z = M(r), stop at
    ||r|| <= rel_tol ||r0||.  Returns (x, status, iters, rr, x_hist)."""
    x = np.zeros_like(b)
    r = b.copy()
    rr = [float(r @ r)]
    xh = [x.copy()] if history else None
    z = M(r)
    p = z.copy()
    rz = float(r @ z)
    k = 0
    st = 7
    if rr[0] == 0.0:
        return x, 0, 0, np.array(rr), xh
    while k < max_iter:
        Ap = apply_ea(m, Ae, p, bc=bc)
        pAp = float(p @ Ap)
        if not pAp > 0:
            st = 6
            break
        a = rz / pAp
        x = x + a * p
        r = r - a * Ap
        k += 1
        rr.append(float(r @ r))
        if history:
            xh.append(x.copy())
        if np.sqrt(rr[-1]) <= rel_tol * np.sqrt(rr[0]):
            st = 0
            break
        z = M(r)
        rzn = float(r @ z)
        p = z + (rzn / rz) * p
        rz = rzn
    return x, st, k, np.array(rr), xh


def set_threads(n: int):
    lib().orc_set_threads(int(n))


def num_threads() -> int:
    return lib().orc_num_threads()
