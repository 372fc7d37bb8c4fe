"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test states the passage / closed form it checks.  None of them retypes the
oracle's formula: 1D references come from tests/ref1d.py (mpmath, 40 digits),
closed forms from tests/golden/*.json, and the rest are invariants (volume,
K*1 = 0, X_i^T K X_j = delta_ij vol, symmetry, polynomial exactness, CG closed
forms, convergence order).  These run without a GPU.
"""
import math

import numpy as np
import pytest

import oracle as O
import workloads as W
from tests.conftest import closed, golden
from tests import ref1d


# --------------------------------------------------------------------------- 1D tables
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_gll_golden(p):
    g = golden("gll_nodes.json")
    x, w = O.gll(p)
    np.testing.assert_allclose(x, [closed(s) for s in g["nodes"][str(p)]], rtol=0, atol=1e-15)
    np.testing.assert_allclose(w, [closed(s) for s in g["weights"][str(p)]], rtol=0, atol=1e-15)


@pytest.mark.parametrize("p", range(1, 13))
def test_gll_vs_numpy_legendre(p):
    x, w = O.gll(p)
    np.testing.assert_allclose(x, ref1d.gll_nodes(p), rtol=0, atol=2e-15)
    assert x[0] == 0.0 and x[-1] == 1.0
    np.testing.assert_allclose(x, 1.0 - x[::-1], atol=1e-15)  # symmetric about 1/2
    assert abs(w.sum() - 1.0) < 1e-14
    # GLL with p+1 points is exact to degree 2p-1
    for k in range(2 * p):
        assert abs(w @ x ** k - 1.0 / (k + 1)) < 1e-14


@pytest.mark.parametrize("q", [1, 2, 3])
def test_gauss_golden(q):
    g = golden("gauss.json")
    x, w = O.gauss(q)
    np.testing.assert_allclose(x, [closed(s) for s in g["points"][str(q)]], atol=1e-15)
    np.testing.assert_allclose(w, [closed(s) for s in g["weights"][str(q)]], atol=1e-15)
    if q == 2:
        assert abs(w @ x ** 3 - closed(g["integral_x3_q2"])) <= 1e-15


@pytest.mark.parametrize("q", range(1, 17))
def test_gauss_vs_numpy_leggauss(q):
    x, w = O.gauss(q)
    s, ws = np.polynomial.legendre.leggauss(q)
    np.testing.assert_allclose(x, (s + 1) / 2, atol=2e-15)
    np.testing.assert_allclose(w, ws / 2, atol=2e-15)
    for k in range(2 * q):
        assert abs(w @ x ** k - 1.0 / (k + 1)) < 1e-14


def test_tabulate_p1q1_golden():
    g = golden("tabulate_p1q1.json")
    B, G = O.tabulate(1, 1, O.GAUSS)
    np.testing.assert_array_equal(B, g["B"])
    np.testing.assert_array_equal(G, g["G"])


@pytest.mark.parametrize("p,rule", [(p, r) for p in range(1, 9) for r in (O.GAUSS, O.GLL)])
def test_tabulate_reproduction(p, rule):
    """rows of B sum to 1, rows of G to 0, and B/G
    reproduce x^m and m x^(m-1) at the quadrature points for m <= p."""
    Q = O.default_q(p, rule)
    B, G = O.tabulate(p, Q, rule)
    t = ((np.polynomial.legendre.leggauss(Q)[0] + 1) / 2 if rule == O.GAUSS
         else ref1d.gll_nodes(Q - 1))
    xi = ref1d.gll_nodes(p)
    np.testing.assert_allclose(B.sum(1), 1.0, atol=1e-13)
    np.testing.assert_allclose(G.sum(1), 0.0, atol=1e-12 * (p + 1) ** 2)
    for m in range(p + 1):
        np.testing.assert_allclose(B @ xi ** m, t ** m, atol=1e-12)
        np.testing.assert_allclose(G @ xi ** m, m * t ** max(m - 1, 0) if m else 0 * t, atol=1e-11)
    if rule == O.GLL:  # collocated: B = I (reading R2)
        np.testing.assert_allclose(B, np.eye(p + 1), atol=1e-14)


# --------------------------------------------------------------------------- element / Kronecker
def test_p1_closed_form_3d_element():
    """North-star pin: p=1 1D element matrices h/6[2 1;1 2] and 1/h[1 -1;-1 1];
    on one affine box element the 3D matrices are their Kronecker combinations."""
    g = golden("element_1d_p1.json")
    Lx, Ly, Lz = 2.0, 0.5, 1.25
    m = O.Mesh(1, 1, 1, 1, alpha=0.0, L=(Lx, Ly, Lz))
    Mm = lambda h: h * np.array([[closed(s) for s in r] for r in g["mass_over_h"]])
    Km = lambda h: np.array([[closed(s) for s in r] for r in g["stiffness_times_h"]]) / h
    Mg = lambda h: h * np.array([[closed(s) for s in r] for r in g["gll_mass_over_h"]])
    M3 = ref1d.kron3(Mm(Lz), Mm(Ly), Mm(Lx))
    K3 = (ref1d.kron3(Km(Lz), Mm(Ly), Mm(Lx)) + ref1d.kron3(Mm(Lz), Km(Ly), Mm(Lx))
          + ref1d.kron3(Mm(Lz), Mm(Ly), Km(Lx)))
    np.testing.assert_allclose(O.element_matrices(m, O.MASS, O.GAUSS)[0], M3, atol=1e-15)
    np.testing.assert_allclose(O.element_matrices(m, O.DIFFUSION, O.GAUSS)[0], K3, atol=2e-15)
    # GLL collocated p=1: lumped mass, exact stiffness with lumped transverse masses
    MG3 = ref1d.kron3(Mg(Lz), Mg(Ly), Mg(Lx))
    KG3 = (ref1d.kron3(Km(Lz), Mg(Ly), Mg(Lx)) + ref1d.kron3(Mg(Lz), Km(Ly), Mg(Lx))
           + ref1d.kron3(Mg(Lz), Mg(Ly), Km(Lx)))
    np.testing.assert_allclose(O.element_matrices(m, O.MASS, O.GLL)[0], MG3, atol=1e-15)
    np.testing.assert_allclose(O.element_matrices(m, O.DIFFUSION, O.GLL)[0], KG3, atol=2e-15)


@pytest.mark.parametrize("dims,p,rule", [((3, 2, 2), 1, O.GAUSS), ((2, 3, 2), 2, O.GAUSS),
                                         ((2, 2, 1), 3, O.GAUSS), ((1, 2, 1), 4, O.GAUSS),
                                         ((2, 2, 2), 2, O.GLL), ((2, 1, 2), 3, O.GLL)])
def test_affine_kronecker_structure(dims, p, rule):
    """On an affine box mesh M = Mz (x) My (x) Mx and K = Kz My Mx + Mz Ky Mx + Mz My Kx
    with the GLOBAL assembled 1D matrices (exact 1D integrals, tests/ref1d.py).
    For GLL (BP5) the 1D masses are the lumped GLL masses (reading R2)."""
    nx, ny, nz = dims
    L = (1.5, 1.0, 0.75)
    m = O.Mesh(nx, ny, nz, p, alpha=0.0, L=L)
    ms, ks = [], []
    for n, Lk in zip((nx, ny, nz), L):
        Me, Ke = ref1d.element_1d(p, Lk / n)
        if rule == O.GLL:
            Me = ref1d.element_1d_gll_lumped(p, Lk / n)
        ms.append(ref1d.assemble_1d(Me, n))
        ks.append(ref1d.assemble_1d(Ke, n))
    Mx, My, Mz = ms
    Kx, Ky, Kz = ks
    M3 = ref1d.kron3(Mz, My, Mx)
    K3 = ref1d.kron3(Kz, My, Mx) + ref1d.kron3(Mz, Ky, Mx) + ref1d.kron3(Mz, My, Kx)
    Ma = O.assemble_dense(m, O.element_matrices(m, O.MASS, rule))
    Ka = O.assemble_dense(m, O.element_matrices(m, O.DIFFUSION, rule))
    assert np.abs(Ma - M3).max() <= 1e-14 * np.abs(M3).max()
    assert np.abs(Ka - K3).max() <= 1e-13 * np.abs(K3).max()


def test_affine_coords_are_lattice():
    """Reading R4: alpha=0 nodes are the lattice (e + xi_a)/n * L."""
    m = O.Mesh(3, 2, 2, 3, alpha=0.0, L=(2.0, 1.0, 0.5))
    xyz = O.mesh_coords(m)
    gx = ref1d.lattice_1d(3, 3, 2.0)
    gy = ref1d.lattice_1d(3, 2, 1.0)
    gz = ref1d.lattice_1d(3, 2, 0.5)
    Z, Y, X = np.meshgrid(gz, gy, gx, indexing="ij")
    np.testing.assert_allclose(xyz[0], X.ravel(), atol=1e-15)
    np.testing.assert_allclose(xyz[1], Y.ravel(), atol=1e-15)
    np.testing.assert_allclose(xyz[2], Z.ravel(), atol=1e-15)


def test_deformation_fixes_boundary_and_moves_interior():
    """Reading R4: Phi is the identity on the boundary of the cube and moves
    interior nodes by O(alpha)."""
    m = O.Mesh(2, 2, 2, 2, alpha=0.1)
    m0 = O.Mesh(2, 2, 2, 2, alpha=0.0)
    d = O.mesh_coords(m) - O.mesh_coords(m0)
    bnd = O.boundary_mask(m)
    assert np.abs(d[:, bnd]).max() < 1e-16
    assert 0.01 < np.abs(d[:, ~bnd]).max() < 0.1


# --------------------------------------------------------------------------- invariants
CURVED = [(2, 2, 2, 1), (2, 2, 2, 2), (2, 3, 2, 3), (2, 2, 1, 4)]


@pytest.mark.parametrize("nx,ny,nz,p", CURVED)
def test_volume_and_mass_of_one(nx, ny, nz, p):
    """1^T M 1 = volume = 1 (Phi fixes the unit cube's boundary), exact when
    2Q-1 >= 3p-1 (Gauss Q = p+2 covers p <= 4)."""
    m = O.Mesh(nx, ny, nz, p, alpha=0.1)
    Me = O.element_matrices(m, O.MASS, O.GAUSS)
    one = np.ones(m.n_dofs)
    assert abs(one @ O.apply_ea(m, Me, one) - 1.0) < 1e-13
    qd = O.qdata(m, O.MASS, O.GAUSS)
    assert abs(qd.sum() - 1.0) < 1e-13
    assert (qd > 0).all()


@pytest.mark.parametrize("nx,ny,nz,p", CURVED)
def test_diffusion_kernel_and_coordinate_identity(nx, ny, nz, p):
    """K 1 = 0 and X_i^T K X_j = delta_ij 1^T M 1 on curved meshes,
    from J adj(J) = detJ I (exercises adj/detJ)."""
    m = O.Mesh(nx, ny, nz, p, alpha=0.1)
    Ke = O.element_matrices(m, O.DIFFUSION, O.GAUSS)
    Me = O.element_matrices(m, O.MASS, O.GAUSS)
    one = np.ones(m.n_dofs)
    K1 = O.apply_ea(m, Ke, one)
    assert np.linalg.norm(K1) <= 1e-13 * np.abs(Ke).max() * np.sqrt(m.n_dofs)
    vol = one @ O.apply_ea(m, Me, one)
    X = O.mesh_coords(m)
    KX = [O.apply_ea(m, Ke, X[i]) for i in range(3)]
    for i in range(3):
        for j in range(3):
            val = X[i] @ KX[j]
            assert abs(val - (vol if i == j else 0.0)) < 1e-12, (i, j, val)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_polynomial_exactness_affine(p):
    """Affine box, Gauss Q=p+2: v^T M u = int uv and v^T K u = int grad u . grad v
    exactly for u, v in Q_p (BASELINE north star)."""
    L = (1.5, 1.0, 0.5)
    m = O.Mesh(2, 2, 2, p, alpha=0.0, L=L)
    xyz = O.mesh_coords(m)
    Me = O.element_matrices(m, O.MASS, O.GAUSS)
    Ke = O.element_matrices(m, O.DIFFUSION, O.GAUSS)
    rng = np.random.default_rng(0)

    def mono_int(e):  # int_box x^e0 y^e1 z^e2
        return np.prod([L[d] ** (e[d] + 1) / (e[d] + 1) for d in range(3)])

    for _ in range(6):
        a = rng.integers(0, p + 1, 3)
        b = rng.integers(0, p + 1, 3)
        u = np.prod([xyz[d] ** a[d] for d in range(3)], axis=0)
        v = np.prod([xyz[d] ** b[d] for d in range(3)], axis=0)
        exact_m = mono_int(a + b)
        exact_k = 0.0
        for d in range(3):
            if a[d] and b[d]:
                e = a + b
                e[d] -= 2
                exact_k += a[d] * b[d] * mono_int(e)
        assert abs(v @ O.apply_ea(m, Me, u) - exact_m) <= 1e-13 * max(1, abs(exact_m))
        assert abs(v @ O.apply_ea(m, Ke, u) - exact_k) <= 1e-12 * max(1, abs(exact_k))


@pytest.mark.parametrize("kind", [O.MASS, O.DIFFUSION])
def test_symmetry_and_definiteness(kind):
    """|<Ax,y> - <x,Ay>| <= 1e-12 |A||x||y|; x^T M x > 0; x^T K x >= 0."""
    m = O.Mesh(2, 2, 2, 3, alpha=0.1)
    Ae = O.element_matrices(m, kind, O.GAUSS)
    nrm = np.abs(Ae).max() * 8
    for s in range(1, 4):
        x = W.random_vector(s, np.arange(m.n_dofs))
        y = W.random_vector(s + 100, np.arange(m.n_dofs))
        Ax, Ay = O.apply_ea(m, Ae, x), O.apply_ea(m, Ae, y)
        assert abs(Ax @ y - x @ Ay) <= 1e-12 * nrm * np.linalg.norm(x) * np.linalg.norm(y)
        assert x @ Ax > 0 if kind == O.MASS else x @ Ax >= 0


def test_qdata_affine_single_element():
    """3D analogue of SPEC.md:285-287: box [0,a]x[0,b]x[0,c], 1 element: J = diag(a,b,c),
    mass D = W abc, diffusion D = W abc diag(1/a^2, 1/b^2, 1/c^2), off-diagonals 0."""
    a, b, c = 2.0, 0.5, 1.25
    p = 3
    m = O.Mesh(1, 1, 1, p, alpha=0.0, L=(a, b, c))
    Q = p + 2
    s, ws = np.polynomial.legendre.leggauss(Q)
    w = ws / 2
    Wq = np.einsum("k,j,i->kji", w, w, w).ravel()  # qz, qy, qx with qx fastest
    qm = O.qdata(m, O.MASS, O.GAUSS)[0, 0]
    np.testing.assert_allclose(qm, Wq * a * b * c, rtol=1e-14)
    qd = O.qdata(m, O.DIFFUSION, O.GAUSS)[0]
    np.testing.assert_allclose(qd[0], Wq * a * b * c / a ** 2, rtol=1e-14)
    np.testing.assert_allclose(qd[3], Wq * a * b * c / b ** 2, rtol=1e-14)
    np.testing.assert_allclose(qd[5], Wq * a * b * c / c ** 2, rtol=1e-14)
    for k in (1, 2, 4):
        assert np.abs(qd[k]).max() < 1e-15


def test_qdata_count_golden():
    g = golden("counts.json")["qdata_count"]
    m = O.Mesh(2, 2, 2, g["p"], alpha=0.1)
    qd = O.qdata(m, O.DIFFUSION, O.GAUSS, Q=g["q"])
    assert qd.size == g["count"]


def test_restriction_multiplicity_and_counts():
    """R^T 1 = multiplicity 1/2/4/8, boundary-dof count
    N - (Nx-2)(Ny-2)(Nz-2) (config 1: 98 of 125)."""
    g = golden("counts.json")["config1"]
    m = O.Mesh(g["nx"], g["ny"], g["nz"], g["p"])
    assert m.n_dofs == g["dofs"] and m.n_elems == g["elements"]
    nd = (m.p + 1) ** 3
    Id = np.broadcast_to(np.eye(nd), (m.n_elems, nd, nd)).copy()
    mult = O.apply_ea(m, Id, np.ones(m.n_dofs)).reshape(5, 5, 5)  # K, J, I
    cnt = lambda i: 2 if i == 2 else 1  # lattice index 2 is the shared element face
    for K in range(5):
        for J in range(5):
            for I in range(5):
                assert mult[K, J, I] == cnt(I) * cnt(J) * cnt(K)
    mask = O.boundary_mask(m)
    assert mask.sum() == g["boundary"] and (~mask).sum() == g["free"]


def test_dense_b_form_equals_element_assembly():
    """The dense-B form B^T D B (PAPER.md:595 with B written densely) equals the
    EA form for every kind/rule, constrained and unconstrained."""
    for kind, rule, p in [(O.MASS, O.GAUSS, 3), (O.DIFFUSION, O.GAUSS, 3), (O.DIFFUSION, O.GLL, 4)]:
        m = O.Mesh(2, 2, 2, p, alpha=0.1)
        Ae = O.element_matrices(m, kind, rule)
        for bc in (0, 1):
            x = W.random_vector(7, np.arange(m.n_dofs))
            y1 = O.apply_ea(m, Ae, x, bc=bc)
            y2 = O.apply_dense(m, kind, rule, x, bc=bc)
            assert np.linalg.norm(y1 - y2) <= 1e-14 * np.linalg.norm(y1)


def test_element_sample_matches_interior_dofs():
    """Sampled-element parity: an element-interior dof of y gets
    a contribution from that element only."""
    p = 3
    m = O.Mesh(3, 2, 2, p, alpha=0.1)
    x = W.random_vector(3, np.arange(m.n_dofs))
    y = O.apply_dense(m, O.DIFFUSION, O.GAUSS, x)
    elems = np.array([0, 5, 11])
    ye = O.element_apply_sample(m, O.DIFFUSION, O.GAUSS, x, elems)
    Nx, Ny = p * 3 + 1, p * 2 + 1
    for k, e in enumerate(elems):
        ex, ey, ez = e % 3, (e // 3) % 2, e // 6
        for c in range(1, p):
            for b in range(1, p):
                for a in range(1, p):
                    g = (p * ex + a) + Nx * ((p * ey + b) + Ny * (p * ez + c))
                    assert abs(ye[k, a + (p + 1) * (b + (p + 1) * c)] - y[g]) < 1e-14 * np.abs(y).max()


# --------------------------------------------------------------------------- CG
def test_cg_closed_forms():
    """A = I converges in 1 iteration; [[4,1],[1,3]] b=(1,2) ->
    (1/11, 7/11) in <= 2 iterations."""
    g = golden("cg_small.json")
    x, st, k, _, _ = O.cg(np.array([3.0, -1.0, 2.0]), A=np.eye(3), rel_tol=1e-15)
    assert st == 0 and k == 1
    np.testing.assert_allclose(x, [3.0, -1.0, 2.0], rtol=0, atol=0)
    x, st, k, _, _ = O.cg(np.array(g["b"]), A=np.array(g["A"]), rel_tol=1e-15)
    assert st == 0 and k <= g["max_iters"]
    np.testing.assert_allclose(x, [closed(s) for s in g["x"]], atol=1e-16)


def test_cg_config1_vs_direct_solve():
    """Config 1 (BP3 2x2x2 p=2, 27 free dofs): CG on the constrained operator agrees
    with a dense direct solve (numpy.linalg.solve) of the assembled system."""
    m = O.Mesh(2, 2, 2, 2, alpha=0.1)
    Ke = O.element_matrices(m, O.DIFFUSION, O.GAUSS)
    b = O.rhs(m, O.DIFFUSION, O.GAUSS, bc=1)
    x, st, k, rr, _ = O.cg(b, m=m, Ae=Ke, bc=1, rel_tol=1e-14, max_iter=200)
    assert st == 0 and k <= 27
    K = O.assemble_dense(m, Ke)
    free = ~O.boundary_mask(m)
    xd = np.zeros(m.n_dofs)
    xd[free] = np.linalg.solve(K[np.ix_(free, free)], b[free])
    assert np.abs(x - xd).max() <= 1e-13 * np.abs(xd).max()


def test_linear_exactness_nonhomogeneous_dirichlet():
    """Dirichlet data u = x_1 is reproduced on affine meshes: solve
    K_ff u_f = -K_fb u_b with the assembled oracle matrix."""
    m = O.Mesh(3, 2, 2, 2, alpha=0.0, L=(1.0, 2.0, 1.5))
    K = O.assemble_dense(m, O.element_matrices(m, O.DIFFUSION, O.GAUSS))
    X = O.mesh_coords(m)
    bnd = O.boundary_mask(m)
    u = np.zeros(m.n_dofs)
    u[bnd] = X[0][bnd]
    free = ~bnd
    u[free] = np.linalg.solve(K[np.ix_(free, free)], -K[np.ix_(free, bnd)] @ u[bnd])
    assert np.abs(u - X[0]).max() < 1e-12


@pytest.mark.parametrize("p,ns", [(1, (4, 8)), (2, (4, 8)), (3, (4, 8))])
def test_convergence_rate_manufactured_poisson(p, ns):
    """BASELINE north star / SPEC.md:656-657, 700: manufactured Poisson (reading R11)
    on curved meshes, CG-solved: L2 rate >= p + 0.9."""
    errs = []
    for n in ns:
        m = O.Mesh(n, n, n, p, alpha=0.1)
        Ke = O.element_matrices(m, O.DIFFUSION, O.GAUSS)
        b = O.rhs(m, O.DIFFUSION, O.GAUSS, bc=1)
        x, st, _, _, _ = O.cg(b, m=m, Ae=Ke, bc=1, rel_tol=1e-13, max_iter=5000)
        assert st == 0
        errs.append(O.l2_error(m, x))
    rate = math.log(errs[0] / errs[1]) / math.log(ns[1] / ns[0])
    assert rate >= p + 0.9, (errs, rate)


# --------------------------------------------------------------------------- inputs
def test_splitmix64_golden():
    g = golden("splitmix64.json")
    z = W.splitmix64_mix(np.arange(1, 4, dtype=np.uint64) * W.GOLDEN)
    assert [int(v) for v in z] == [int(h, 16) for h in g["seed0_outputs_hex"]]
    x = W.random_vector(5, np.arange(100000))
    assert x.min() >= -1.0 and x.max() < 1.0 and abs(x.mean()) < 0.01


# --------------------------------------------------------------------------- round-2 pins
def test_curved_phi_golden():
    """Reading R4, hand-evaluated (tests/golden/phi_curved.json): two nodes of the
    deformed 2x2x2 p=2 mesh.  A transposed cos argument (u_{i-1} instead of
    u_{i+1}) or a wrong amplitude moves both points by ~0.035."""
    g = golden("phi_curved.json")
    n, p, alpha = g["mesh"]["n"], g["mesh"]["p"], g["mesh"]["alpha"]
    m = O.Mesh(n, n, n, p, alpha=alpha)
    xyz = O.mesh_coords(m)
    N = p * n + 1
    for pt in g["points"]:
        I, J, K = pt["lattice"]
        l = I + N * (J + N * K)
        np.testing.assert_allclose(xyz[:, l], pt["xyz"], rtol=0, atol=2e-16)


def _rhs_1d(p, n, rule):
    """b_i = int_0^1 sin(pi x) l_i(x) dx by the SAME 1D rule the 3D oracle
    tensorises (Gauss Q = p+2 from numpy's Legendre rule, or GLL Q = p+1 with
    the mpmath nodes of tests/ref1d.py and weights int l_i), assembled over n
    affine elements.  On an affine box the 3D rule of a separable integrand is
    exactly the product of the 1D rules."""
    nodes_mp = ref1d.gll_nodes_mp(p)
    L = ref1d.lagrange_polys(nodes_mp)
    if rule == O.GAUSS:
        t, w = np.polynomial.legendre.leggauss(p + 2)
        t, w = (t + 1) / 2, w / 2
    else:
        t = np.array([float(v) for v in nodes_mp])
        w = np.array([float(ref1d._pint01(l)) for l in L])
    B = np.array([[float(mpmath_polyval(l, tq)) for l in L] for tq in t])  # [q][i]
    h = 1.0 / n
    b = np.zeros(p * n + 1)
    for e in range(n):
        xq = (e + t) * h
        b[p * e: p * e + p + 1] += B.T @ (w * h * np.sin(np.pi * xq))
    return b


def mpmath_polyval(coeffs, x):
    import mpmath
    return sum(c * mpmath.mpf(x) ** i for i, c in enumerate(coeffs))


@pytest.mark.parametrize("kind,rule,p,dims,bc", [
    (O.DIFFUSION, O.GAUSS, 2, (3, 2, 2), 1), (O.MASS, O.GAUSS, 3, (2, 2, 3), 0),
    (O.DIFFUSION, O.GLL, 3, (2, 3, 2), 1), (O.MASS, O.GAUSS, 1, (4, 3, 2), 0)])
def test_rhs_affine_kronecker(kind, rule, p, dims, bc):
    """Reading R11 on the affine unit cube: f = c * prod sin(pi x_j) with c = 3 pi^2
    (diffusion) or 1 (mass), so b = c * (b_z (x) b_y (x) b_x) with the 1D vectors
    of _rhs_1d; Dirichlet rows zeroed (reading R6).  Pins f, its constant, W,
    detJ, the basis and the assembly of orc_rhs (both branches)."""
    nx, ny, nz = dims
    m = O.Mesh(nx, ny, nz, p, alpha=0.0)
    b = O.rhs(m, kind, rule, bc=bc)
    c = 3 * np.pi ** 2 if kind == O.DIFFUSION else 1.0
    ref = c * ref1d.kron3(_rhs_1d(p, nz, rule)[:, None], _rhs_1d(p, ny, rule)[:, None],
                          _rhs_1d(p, nx, rule)[:, None]).ravel()
    if bc:
        ref[O.boundary_mask(m)] = 0.0
    assert np.abs(b - ref).max() <= 1e-14 * np.abs(ref).max()


def test_l2_error_closed_forms():
    """orc_l2_error: ||0 - u||_{L2} = ||prod sin(pi x_j)|| = (1/2)^{3/2} exactly on
    the unit cube (affine, and curved, whose discrete domain is still the cube);
    u_h = 2 u_I gives ~ ||u|| again; a missing square root or weight fails."""
    exact = 0.5 ** 1.5
    m = O.Mesh(3, 3, 3, 2, alpha=0.0)
    z = np.zeros(O.mesh_coords(m).shape[1])
    assert abs(O.l2_error(m, z, Qover=10) - exact) <= 1e-13
    mc = O.Mesh(3, 3, 3, 2, alpha=0.1)
    assert abs(O.l2_error(mc, z, Qover=12) - exact) <= 1e-6
    X = O.mesh_coords(mc)
    uI = np.sin(np.pi * X[0]) * np.sin(np.pi * X[1]) * np.sin(np.pi * X[2])
    e1 = O.l2_error(mc, uI, Qover=12)
    assert e1 < 0.02 * exact
    assert abs(O.l2_error(mc, 2 * uI, Qover=12) - exact) <= e1 + 1e-6
