"""Independent 1D references for the oracle pins (mpmath at 40 digits).

Nothing here is shared with oracle/ or the CUDA path: GLL nodes are the roots of
P_p' found by mpmath.polyroots on Legendre coefficients built by the Bonnet
recurrence in exact rationals, the Lagrange basis is a coefficient list, and the
integrals are exact polynomial antiderivatives evaluated in 40-digit arithmetic.
"""
from __future__ import annotations

from fractions import Fraction

import mpmath
import numpy as np

mpmath.mp.dps = 40


def _legendre_coeffs(n: int):
    """Monomial coefficients (ascending) of P_n on [-1,1], exact rationals."""
    P0, P1 = [Fraction(1)], [Fraction(0), Fraction(1)]
    if n == 0:
        return P0
    for k in range(1, n):
        # (k+1) P_{k+1} = (2k+1) s P_k - k P_{k-1}
        sP = [Fraction(0)] + P1
        Pm = P0 + [Fraction(0)] * (len(sP) - len(P0))
        P0, P1 = P1, [((2 * k + 1) * a - k * b) / (k + 1) for a, b in zip(sP, Pm)]
    return P1


def gll_nodes_mp(p: int):
    c = _legendre_coeffs(p)
    d = [i * c[i] for i in range(1, len(c))]  # P_p'
    inner = []
    if p > 1:
        roots = mpmath.polyroots([mpmath.mpf(v.numerator) / v.denominator for v in reversed(d)],
                                 maxsteps=200, extraprec=200)
        inner = sorted(mpmath.re(r) for r in roots)
    s = [mpmath.mpf(-1)] + inner + [mpmath.mpf(1)]
    return [(v + 1) / 2 for v in s]


def gll_nodes(p: int) -> np.ndarray:
    return np.array([float(v) for v in gll_nodes_mp(p)])


def _pmul(a, b):
    out = [mpmath.mpf(0)] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            out[i + j] += x * y
    return out


def _pder(a):
    return [i * a[i] for i in range(1, len(a))] or [mpmath.mpf(0)]


def _pint01(a):
    return sum(c / (i + 1) for i, c in enumerate(a))


def lagrange_polys(nodes):
    out = []
    for i, xi in enumerate(nodes):
        poly = [mpmath.mpf(1)]
        for j, xj in enumerate(nodes):
            if j != i:
                poly = _pmul(poly, [-xj / (xi - xj), 1 / (xi - xj)])
        out.append(poly)
    return out


def element_1d(p: int, h: float):
    """Exact 1D element mass and stiffness on an affine element of width h."""
    L = lagrange_polys(gll_nodes_mp(p))
    P1 = p + 1
    M = np.zeros((P1, P1))
    K = np.zeros((P1, P1))
    for i in range(P1):
        for j in range(P1):
            M[i, j] = float(_pint01(_pmul(L[i], L[j])) * h)
            K[i, j] = float(_pint01(_pmul(_pder(L[i]), _pder(L[j]))) / h)
    return M, K


def element_1d_gll_lumped(p: int, h: float):
    """GLL-collocated (Q = p+1) 1D mass: diag of the GLL weights times h; the GLL
    rule is interpolatory, so w_i = int_0^1 l_i exactly."""
    L = lagrange_polys(gll_nodes_mp(p))
    return np.diag([float(_pint01(l) * h) for l in L])


def assemble_1d(Me: np.ndarray, n: int) -> np.ndarray:
    p = Me.shape[0] - 1
    N = p * n + 1
    A = np.zeros((N, N))
    for e in range(n):
        s = slice(p * e, p * e + p + 1)
        A[s, s] += Me
    return A


def lattice_1d(p: int, n: int, L: float = 1.0) -> np.ndarray:
    xi = gll_nodes_mp(p)
    pts = [float((e + xi[a]) / n * L) for e in range(n) for a in range(p)] + [L]
    return np.array(pts)


def kron3(Az, Ay, Ax):
    """Lexicographic x-fastest ordering: index = I + Nx (J + Ny K)."""
    return np.kron(Az, np.kron(Ay, Ax))
