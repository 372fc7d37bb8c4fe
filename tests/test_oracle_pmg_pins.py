"""Pins of the f2 oracle pieces: the
matrix-free diagonal, the p-transfer operators, Chebyshev-Jacobi smoothing, the
power-iteration eigen estimate, the V-cycle and PCG -- against dense linear
algebra, closed forms and the already-pinned EA oracle."""
import numpy as np
import pytest

import oracle as O
import workloads as W


def dense_bc(m, Ae):
    """Assembled A with the identity-row/zero-column Dirichlet convention (R6)."""
    A = O.assemble_dense(m, Ae)
    ess = O.boundary_mask(m)
    A[ess, :] = 0.0
    A[:, ess] = 0.0
    A[ess, ess] = 1.0
    return A


@pytest.mark.parametrize("p,bc", [(2, 1), (3, 0), (1, 1)])
def test_diagonal_is_diag_of_assembled(p, bc):
    m = O.Mesh(2, 3, 2, p, alpha=0.1)
    Ae = O.element_matrices(m, O.DIFFUSION, O.GAUSS)
    A = dense_bc(m, Ae) if bc else O.assemble_dense(m, Ae)
    d = O.diagonal(m, Ae, bc=bc)
    assert np.abs(d - np.diag(A)).max() <= 1e-14 * np.abs(A).max()


@pytest.mark.parametrize("pc,pf", [(1, 2), (2, 4), (2, 5), (3, 7), (4, 8)])
def test_prolong_reproduces_coarse_polynomials(pc, pf):
    """Nested spaces: a coarse function of degree <= pc per variable
    is represented exactly on the fine order (affine mesh, so the reference and
    physical coordinates are the lattice)."""
    mc = O.Mesh(3, 2, 2, pc, alpha=0.0, L=(1.5, 1.0, 0.5))
    mf = O.Mesh(3, 2, 2, pf, alpha=0.0, L=(1.5, 1.0, 0.5))
    Xc, Xf = O.mesh_coords(mc), O.mesh_coords(mf)
    f = lambda X: X[0] ** pc * X[1] + X[2] ** min(pc, 2) - 0.5 * X[1] ** pc
    xf = O.prolong(mf, mc, f(Xc))
    assert np.abs(xf - f(Xf)).max() <= 1e-13


def test_restrict_is_prolong_transpose_and_galerkin_affine():
    """R = P^T (<P u, v> = <u, R v>), and on an affine mesh the Galerkin product
    P^T A_f P equals the coarse operator A_c (exact quadrature on both orders)."""
    mc = O.Mesh(2, 2, 2, 2, alpha=0.0)
    mf = O.Mesh(2, 2, 2, 4, alpha=0.0)
    rng = np.random.default_rng(0)
    u, v = rng.standard_normal(mc.n_dofs), rng.standard_normal(mf.n_dofs)
    assert abs(O.prolong(mf, mc, u) @ v - u @ O.restrict(mf, mc, v)) <= 1e-12 * np.abs(v).sum()
    P = np.stack([O.prolong(mf, mc, e) for e in np.eye(mc.n_dofs)], axis=1)
    Af = O.assemble_dense(mf, O.element_matrices(mf, O.DIFFUSION, O.GAUSS))
    Ac = O.assemble_dense(mc, O.element_matrices(mc, O.DIFFUSION, O.GAUSS))
    assert np.abs(P.T @ Af @ P - Ac).max() <= 1e-12 * np.abs(Ac).max()
    Rv = O.restrict(mf, mc, v)
    assert np.abs(Rv - P.T @ v).max() <= 1e-13 * np.abs(v).max() * 10


@pytest.mark.parametrize("degree", [1, 2, 3, 5])
def test_chebyshev_error_polynomial(degree):
    """Saad Alg. 12.1 with D = diag(A): from x0 = 0 the error is
    e_m = T_m((theta - D^-1 A)/delta) / T_m(theta/delta) e_0 (closed form through
    the eigendecomposition of D^-1/2 A D^-1/2)."""
    m = O.Mesh(2, 2, 2, 2, alpha=0.1)
    Ae = O.element_matrices(m, O.DIFFUSION, O.GAUSS)
    A = dense_bc(m, Ae)
    d = O.diagonal(m, Ae, bc=1)
    b = O.rhs(m, O.DIFFUSION, O.GAUSS, bc=1) + 0.1 * W.random_vector(2, np.arange(m.n_dofs)) * \
        (~O.boundary_mask(m))
    Dh = 1.0 / np.sqrt(d)
    lam, V = np.linalg.eigh(Dh[:, None] * A * Dh[None, :])
    lmax, lmin = 1.2 * lam.max(), 0.36 * lam.max()
    x = O.cheb(m, Ae, 1, 1.0 / d, lmin, lmax, degree, b, np.zeros(m.n_dofs))
    xs = np.linalg.solve(A, b)
    th, de = 0.5 * (lmax + lmin), 0.5 * (lmax - lmin)
    T = lambda k, t: np.cosh(k * np.arccosh(t)) if t >= 1 else np.cos(k * np.arccos(np.clip(t, -1, 1)))
    g = np.array([T(degree, (th - l) / de) if abs((th - l) / de) <= 1 else
                  np.sign((th - l) / de) ** degree * T(degree, abs((th - l) / de)) for l in lam])
    g /= T(degree, th / de)
    e0 = V.T @ (xs / Dh)          # e in D^{1/2} coordinates
    em = V @ (g * e0) * Dh
    assert np.abs((xs - x) - em).max() <= 1e-12 * np.abs(xs).max()


def test_power_iteration_reaches_lambda_max():
    m = O.Mesh(2, 2, 2, 2, alpha=0.1)
    Ae = O.element_matrices(m, O.DIFFUSION, O.GAUSS)
    A = dense_bc(m, Ae)
    d = O.diagonal(m, Ae, bc=1)
    Dh = 1.0 / np.sqrt(d)
    lmax = np.linalg.eigvalsh(Dh[:, None] * A * Dh[None, :]).max()
    v0 = W.random_vector(1, np.arange(m.n_dofs))
    lam = O.power_lmax(m, Ae, 1, 1.0 / d, v0, 3000)
    assert abs(lam - lmax) <= 1e-6 * lmax
    lam10 = O.power_lmax(m, Ae, 1, 1.0 / d, v0, 10)
    assert 0.5 * lmax < lam10 < 1.5 * lmax


@pytest.mark.parametrize("dims,p", [((2, 2, 2), 2), ((2, 2, 1), 4)])
def test_vcycle_is_symmetric_positive_definite(dims, p):
    """Same Chebyshev polynomial before and after the coarse correction, R = P^T:
    the V-cycle is a symmetric positive definite operator (a valid PCG
    preconditioner)."""
    M = O.PMG(*dims, p, degree=2)
    n = M.levels[0]["m"].n_dofs
    B = np.stack([M.vcycle(e) for e in np.eye(n)], axis=1)
    assert np.abs(B - B.T).max() <= 1e-12 * np.abs(B).max()
    assert np.linalg.eigvalsh(0.5 * (B + B.T)).min() > 0


def test_pcg_reduces_to_cg_and_exact_preconditioner():
    m = O.Mesh(2, 2, 2, 2, alpha=0.1)
    Ae = O.element_matrices(m, O.DIFFUSION, O.GAUSS)
    b = O.rhs(m, O.DIFFUSION, O.GAUSS, bc=1)
    x1, st1, k1, rr1, _ = O.pcg(b, lambda r: r.copy(), m=m, Ae=Ae, rel_tol=1e-12)
    x2, st2, k2, rr2, _ = O.cg(b, m=m, Ae=Ae, bc=1, rel_tol=1e-12, max_iter=500)
    assert st1 == st2 == 0 and k1 == k2
    assert np.abs(x1 - x2).max() <= 1e-13 * np.abs(x2).max()
    A = dense_bc(m, Ae)
    x3, st3, k3, _, _ = O.pcg(b, lambda r: np.linalg.solve(A, r), m=m, Ae=Ae, rel_tol=1e-12)
    assert st3 == 0 and k3 == 1


def test_pmg_pcg_converges_faster_than_cg():
    """BPS3-style solve: p-MG-preconditioned CG reaches 1e-10 in
    far fewer iterations than CG, to the same solution."""
    M = O.PMG(3, 3, 3, 4, degree=3)
    L = M.levels[0]
    b = O.rhs(L["m"], O.DIFFUSION, O.GAUSS, bc=1)
    x, st, k, _, _ = O.pcg(b, M.vcycle, m=L["m"], Ae=L["Ae"], rel_tol=1e-10)
    xc, stc, kc, _, _ = O.cg(b, m=L["m"], Ae=L["Ae"], bc=1, rel_tol=1e-10, max_iter=2000)
    assert st == 0 and stc == 0
    assert k * 3 < kc, (k, kc)
    assert np.linalg.norm(x - xc) <= 1e-8 * np.linalg.norm(xc)
