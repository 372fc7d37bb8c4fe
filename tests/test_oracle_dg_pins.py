"""Pins of the DG (L2) mass oracle (§2.4.1):
closed forms and identities that fix orc_dg_mass_matrices without retyping it.
1D references: numpy's Gauss-Legendre rule, tests/ref1d.py's mpmath Lagrange
polynomials."""
import numpy as np
import pytest

import oracle as O
from tests import ref1d


def gl_nodes_weights(P1):
    t, w = np.polynomial.legendre.leggauss(P1)
    return (t + 1) / 2, w / 2


def polyval(coeffs, x):
    return float(sum(c * ref1d.mpmath.mpf(float(x)) ** i for i, c in enumerate(coeffs)))


@pytest.mark.parametrize("p,dims", [(1, (2, 1, 2)), (3, (1, 2, 1)), (5, (1, 1, 2))])
def test_dg_affine_mass_is_diagonal(p, dims):
    """Affine box: psi_a are Lagrange polynomials on the P1 Gauss points, and the
    P1-point Gauss rule is exact for degree 2p, so int psi_a psi_b = w_a delta_ab:
    M_e = h_x h_y h_z diag(w_a w_b w_c) exactly (Q = p+2 integrates it exactly)."""
    L = (1.5, 1.0, 0.75)
    m = O.Mesh(*dims, p, alpha=0.0, L=L)
    Me = O.dg_mass_matrices(m)
    _, w = gl_nodes_weights(p + 1)
    h = [Lk / n for Lk, n in zip(L, dims)]
    ref = np.diag(np.kron(w * h[2], np.kron(w * h[1], w * h[0])))
    for e in range(m.n_elems):
        assert np.abs(Me[e] - ref).max() <= 1e-15 * ref.max() * 10


@pytest.mark.parametrize("nx,ny,nz,p", [(2, 2, 2, 1), (2, 2, 2, 2), (2, 3, 2, 3), (2, 2, 1, 4)])
def test_dg_volume_curved(nx, ny, nz, p):
    """Partition of unity of the DG basis: 1^T M 1 = volume = 1 on the deformed
    unit cube (Gauss Q = p+2 integrates detJ exactly for p <= 4)."""
    m = O.Mesh(nx, ny, nz, p, alpha=0.1)
    Me = O.dg_mass_matrices(m)
    assert abs(Me.sum() - 1.0) <= 1e-13


@pytest.mark.parametrize("p", [1, 2, 3])
def test_dg_mass_equals_h1_mass_on_the_same_polynomials(p):
    """Same space per element (Q_p), same geometry and quadrature: with I the 3D
    interpolation from the GLL nodal basis to the Gauss-Legendre nodal basis,
    M_H1,e = I^T M_DG,e I element by element (curved mesh) -- ties the DG oracle
    to the pinned H1 mass oracle."""
    m = O.Mesh(2, 2, 2, p, alpha=0.1)
    Me_dg = O.dg_mass_matrices(m)
    Me_h1 = O.element_matrices(m, O.MASS, O.GAUSS)
    t, _ = gl_nodes_weights(p + 1)
    Lg = ref1d.lagrange_polys(ref1d.gll_nodes_mp(p))
    I1 = np.array([[polyval(Lg[a], tg) for a in range(p + 1)] for tg in t])  # [g][a]
    I3 = np.kron(I1, np.kron(I1, I1))
    for e in range(m.n_elems):
        back = I3.T @ Me_dg[e] @ I3
        assert np.abs(back - Me_h1[e]).max() <= 1e-14 * np.abs(Me_h1[e]).max() * 10


def test_dg_symmetric_positive_definite_and_block_apply():
    m = O.Mesh(2, 2, 1, 2, alpha=0.1)
    Me = O.dg_mass_matrices(m)
    nd = 27
    for e in range(m.n_elems):
        assert np.abs(Me[e] - Me[e].T).max() <= 1e-16 * 10
        assert np.linalg.eigvalsh(Me[e]).min() > 0
    x = np.random.default_rng(0).standard_normal(m.n_elems * nd)
    y = O.dg_apply(m, Me, x)
    ref = np.concatenate([Me[e] @ x[e * nd:(e + 1) * nd] for e in range(m.n_elems)])
    assert np.abs(y - ref).max() <= 1e-14 * np.abs(ref).max()


def test_dg_sample_matches_full_apply():
    m = O.Mesh(3, 2, 2, 3, alpha=0.1)
    Me = O.dg_mass_matrices(m)
    x = np.random.default_rng(1).standard_normal(m.n_elems * 64)
    y = O.dg_apply(m, Me, x)
    elems = np.array([0, 5, 11, 7])
    ye = O.dg_apply_sample(m, x, elems)
    for k, e in enumerate(elems):
        assert np.abs(ye[k] - y[e * 64:(e + 1) * 64]).max() <= 1e-15 * np.abs(y).max() * 10
