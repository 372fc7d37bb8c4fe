"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Tolerances (north star / DESIGN.md §3 R10, R13-R14):
relative L2 error <= 1e-12 per apply, CG iterates <= 1e-10, integer / index
work bit-exact (random generator, counts)."""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu

APPLY_TOL = 1e-12


@pytest.fixture(scope="module")
def hf():
    import paper_2402_15940_b200 as hf
    hf.lib()
    return hf


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


KINDS = {"bp1": (O.MASS, O.GAUSS), "bp3": (O.DIFFUSION, O.GAUSS), "bp5": (O.DIFFUSION, O.GLL)}


def make(hf, nx, ny, nz, p, bench, bc=0, alpha=0.1, L=(1.0, 1.0, 1.0), q=0):
    kind, rule = KINDS[bench]
    m = hf.Mesh(nx, ny, nz, p, alpha=alpha, extent=L)
    op = hf.Operator(m, kind=kind, rule=rule, q_override=q, bc=bc)
    om = O.Mesh(nx, ny, nz, p, alpha=alpha, L=L)
    return m, op, om, kind, rule


# ----------------------------------------------------------------------------- inputs / setup
def test_random_generator_bit_exact(hf):
    m = hf.Mesh(3, 2, 4, 3)
    x = host(m.random(42))
    ref = W.random_vector(42, np.arange(m.n_local))
    assert np.array_equal(x.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("p", [1, 2, 5, 8])
def test_coords_match_oracle(hf, p):
    m = hf.Mesh(3, 2, 2, p, alpha=0.1, extent=(2.0, 1.0, 0.5))
    xyz = host(m.coords())
    ref = O.mesh_coords(O.Mesh(3, 2, 2, p, alpha=0.1, L=(2.0, 1.0, 0.5)))
    assert np.abs(xyz - ref).max() <= 4e-16 * 2.0


@pytest.mark.parametrize("bench,p", [("bp1", 1), ("bp1", 4), ("bp3", 2), ("bp3", 5), ("bp3", 8),
                                     ("bp5", 3), ("bp5", 6)])
def test_qdata_matches_oracle(hf, bench, p):
    m, op, om, kind, rule = make(hf, 2, 3, 2, p, bench)
    qd = host(op.qdata()).reshape(om.n_elems, -1)
    ref = O.qdata(om, kind, rule).reshape(om.n_elems, -1)
    assert np.abs(qd - ref).max() <= 1e-13 * np.abs(ref).max()


def test_invalid_mesh_reports_err_mesh(hf):
    with pytest.raises(hf.HofemError) as e:
        m = hf.Mesh(2, 2, 2, 2, alpha=0.9)  # fold the mesh: detJ < 0 inside
        hf.Operator(m, kind=hf.DIFFUSION)
    assert e.value.status == 2


# ----------------------------------------------------------------------------- apply parity
CASES = [
    # (nx, ny, nz, p, bench) -- several bricks, ragged tails (nx not a brick multiple)
    (2, 2, 2, 2, "bp3"),   # config 1
    (5, 3, 4, 1, "bp1"), (3, 5, 3, 2, "bp1"), (5, 3, 2, 3, "bp1"), (3, 3, 3, 5, "bp1"),
    (3, 2, 2, 6, "bp1"), (2, 3, 2, 7, "bp1"), (2, 2, 3, 8, "bp1"),  # mass shapes (ShapeSMD)
    (9, 5, 3, 1, "bp3"), (5, 5, 3, 2, "bp3"), (5, 3, 3, 3, "bp3"), (3, 3, 3, 4, "bp3"),
    (3, 3, 3, 5, "bp3"), (3, 3, 2, 6, "bp3"), (3, 2, 2, 7, "bp3"), (3, 2, 2, 8, "bp3"),
    (5, 3, 3, 2, "bp5"), (3, 3, 3, 4, "bp5"), (3, 3, 2, 5, "bp5"), (3, 2, 2, 8, "bp5"),
    (4, 3, 2, 3, "bp5"), (3, 2, 2, 6, "bp5"), (2, 3, 2, 7, "bp5"),  # collocated shapes
    (1, 1, 1, 1, "bp3"), (1, 1, 1, 5, "bp3"), (1, 1, 1, 4, "bp5"),
]


def oracle_apply(om, kind, rule, x, bc, p, Q=None):
    if p <= 4 and om.n_elems <= 64:
        Ae = O.element_matrices(om, kind, rule, Q=Q)
        return O.apply_ea(om, Ae, x, bc=bc)
    return O.apply_dense(om, kind, rule, x, bc=bc, Q=Q)


@pytest.mark.parametrize("nx,ny,nz,p,bench", CASES)
@pytest.mark.parametrize("bc", [0, 1])
def test_fused_and_unfused_match_oracle(hf, nx, ny, nz, p, bench, bc):
    """The fused brick kernel with both fix-up schedules (separate fix-up kernel
    after a memset of y; in-kernel fix-up and zeroing behind grid barriers) and
    the unfused path, against the oracle."""
    m, op, om, kind, rule = make(hf, nx, ny, nz, p, bench, bc=bc)
    for seed in (1, 2):
        x = m.random(seed)
        ref = oracle_apply(om, kind, rule, host(x), bc, p)
        for infix in (hf.NEVER, hf.ALWAYS):
            op.set_option(hf.OPT_INFIX, infix)
            yf = host(op.apply(x))
            assert rel(yf, ref) <= APPLY_TOL, (infix, rel(yf, ref))
        yu = host(op.apply_unfused(x))
        assert rel(yu, ref) <= APPLY_TOL, rel(yu, ref)


@pytest.mark.parametrize("p,q,bench", [(3, 4, "bp3"), (4, 5, "bp1"), (3, 6, "bp3"), (2, 5, "bp5")])
def test_q_override(hf, p, q, bench):
    """Q = p+1 Gauss (fused Q=P1 instantiation), Q = p+2 GLL (non-collocated,
    fused general kernel) and other Q (unfused path)."""
    m, op, om, kind, rule = make(hf, 3, 2, 2, p, bench, q=q)
    x = m.random(5)
    ref = O.apply_dense(om, kind, rule, host(x), Q=q)
    for infix in (hf.NEVER, hf.ALWAYS):
        op.set_option(hf.OPT_INFIX, infix)
        assert rel(host(op.apply(x)), ref) <= APPLY_TOL, infix
    assert rel(host(op.apply_unfused(x)), ref) <= APPLY_TOL


@pytest.mark.parametrize("nx,ny,nz,p,bench,bc", [
    (5, 3, 4, 2, "bp3", 1), (7, 5, 6, 5, "bp3", 1), (5, 3, 3, 3, "bp1", 0),
    (3, 3, 2, 6, "bp3", 0), (5, 4, 3, 4, "bp5", 1), (9, 5, 3, 1, "bp3", 1),
    (3, 2, 2, 8, "bp3", 1)])
@pytest.mark.parametrize("infix", [0, 2])
def test_fused_dot_matches_separate_dot(hf, nx, ny, nz, p, bench, bc, infix):
    """hofem_op_apply_dot: the x.y accumulated inside the fused kernels equals
    the plain owned-dof dot of the same x and y (and the oracle's x.Ax) up to
    summation order, and y is the ordinary apply."""
    m, op, om, kind, rule = make(hf, nx, ny, nz, p, bench, bc=bc)
    op.set_option(hf.OPT_INFIX, infix)
    x = m.random(11)
    y, d = op.apply_dot(x)
    y2 = host(op.apply(x))
    assert np.array_equal(host(y).view(np.uint64), y2.view(np.uint64))
    d2 = m.dot(x, y)
    ref = float(np.dot(host(x), oracle_apply(om, kind, rule, host(x), bc, p)))
    scale = float(np.dot(np.abs(host(x)), np.abs(host(y))))
    assert abs(d - d2) <= 1e-13 * scale, (d, d2)
    assert abs(d - ref) <= 1e-12 * scale, (d, ref)
    _, d3 = op.apply_dot(x)
    assert d3 == d  # deterministic


@pytest.mark.parametrize("infix", [0, 2])
def test_fused_bitwise_deterministic(hf, infix):
    m, op, _, _, _ = make(hf, 7, 5, 6, 5, "bp3", bc=1)
    op.set_option(hf.OPT_INFIX, infix)
    x = m.random(3)
    y1 = host(op.apply(x))
    for _ in range(3):
        y2 = host(op.apply(x))
        assert np.array_equal(y1.view(np.uint64), y2.view(np.uint64))


@pytest.mark.parametrize("bench,p", [("bp3", 5), ("bp1", 3), ("bp5", 4), ("bp3", 2)])
def test_fused_info_partition(hf, bench, p):
    """hofem_op_fused_info: the direct / fix-up split covers every lattice point
    once; options round-trip and reject bad values."""
    m, op, _, _, _ = make(hf, 7, 5, 6, p, bench, bc=1)
    info = op.fused_info()
    assert info.direct_points + info.fixup_points == m.n_local
    assert info.variant == 1
    assert info.grid >= 1 and info.zc * info.nchunks >= 6
    for opt in (hf.OPT_INFIX, hf.OPT_CG_FUSED_UPDATE, hf.OPT_CG_PERSISTENT):
        assert op.get_option(opt) == hf.AUTO
        op.set_option(opt, hf.ALWAYS)
        assert op.get_option(opt) == hf.ALWAYS
        with pytest.raises(hf.HofemError):
            op.set_option(opt, 3)
    with pytest.raises(hf.HofemError):
        op.set_option(hf.OPT_L2_PREFETCH, 2)
    with pytest.raises(hf.HofemError):
        op.set_option(99, 0)


@pytest.mark.parametrize("infix", [0, 2])
def test_apply_graph_replay_bitwise(hf, infix):
    """hofem_op_apply captured into a CUDA graph and replayed: the in-kernel grid
    barriers reset themselves (no host-side counter), so every replay and a
    later eager call give the eager result bit for bit."""
    m, op, _, _, _ = make(hf, 7, 5, 6, 5, "bp3", bc=1)
    op.set_option(hf.OPT_INFIX, infix)
    x = m.random(4)
    ref = host(op.apply(x))
    y = torch.empty_like(x)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        op.apply(x, y)  # warm-up (lazy allocations) outside the capture
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        op.apply(x, y)
    for _ in range(4):
        y.fill_(7.0)
        g.replay()
        assert np.array_equal(host(y).view(np.uint64), ref.view(np.uint64))
    assert np.array_equal(host(op.apply(x)).view(np.uint64), ref.view(np.uint64))


def test_binding_and_abi_reject_bad_vectors(hf):
    """Wrong length / misaligned vectors never reach a kernel: the binding raises
    ValueError, the C ABI itself returns HOFEM_ERR_ARG for a misaligned pointer."""
    import ctypes
    m, op, _, _, _ = make(hf, 3, 3, 3, 2, "bp3")
    x = m.random(1)
    with pytest.raises(ValueError):
        op.apply(x[:-1])
    big = torch.zeros(m.n_local + 1, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        op.apply(big[1:], torch.empty_like(x))
    y = torch.empty(m.n_local + 1, dtype=torch.float64, device="cuda")
    st = hf.lib().hofem_op_apply(op.handle, ctypes.c_void_p(x.data_ptr()),
                                 ctypes.c_void_p(y.data_ptr() + 8),
                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 1


def test_affine_extents_and_volume(hf):
    """Mass of one = box volume; diffusion of one = 0."""
    L = (2.0, 0.5, 1.5)
    m = hf.Mesh(4, 3, 5, 3, alpha=0.0, extent=L)
    one = torch.ones(m.n_local, dtype=torch.float64, device="cuda")
    M = hf.Operator(m, kind=hf.MASS)
    K = hf.Operator(m, kind=hf.DIFFUSION)
    assert abs(host(M.apply(one)).sum() - np.prod(L)) < 1e-13
    assert np.abs(host(K.apply(one))).max() < 1e-12


def test_rhs_matches_oracle(hf):
    for bench, bc in (("bp3", 1), ("bp1", 0), ("bp5", 1)):
        m, op, om, kind, rule = make(hf, 3, 2, 2, 3, bench, bc=bc)
        b = host(op.rhs())
        ref = O.rhs(om, kind, rule, bc=bc)
        assert rel(b, ref) <= 1e-13


def test_dot_owned(hf):
    m = hf.Mesh(4, 3, 5, 3)
    a, b = m.random(1), m.random(2)
    ref = float(np.dot(host(a), host(b)))
    assert abs(m.dot(a, b) - ref) <= 1e-13 * np.abs(host(a)).sum()


# ----------------------------------------------------------------------------- CG
# CG schedules (hofem_op_set_option): the whole solve in one persistent kernel;
# per-iteration kernels with the fused cooperative update and in-kernel fix-up;
# per-iteration kernels with separate update / p-update / dot and the separate
# fix-up after a memset (the path large meshes take by default).
CG_MODES = {
    "persistent": {"OPT_CG_PERSISTENT": 2},
    "fused": {"OPT_CG_PERSISTENT": 0, "OPT_CG_FUSED_UPDATE": 2, "OPT_INFIX": 2},
    "separate": {"OPT_CG_PERSISTENT": 0, "OPT_CG_FUSED_UPDATE": 0, "OPT_INFIX": 0},
}


def set_mode(hf, op, mode):
    for k, v in CG_MODES[mode].items():
        op.set_option(getattr(hf, k), v)


@pytest.mark.parametrize("mode", list(CG_MODES))
def test_cg_config1_iterates(hf, mode):
    """Config 1 (BP3 2x2x2 p=2, Dirichlet, manufactured RHS; 125 dofs, an odd
    length): every CG iterate x_k, k <= k_conv, within 1e-10 of the oracle's
    (reading R14), in every CG schedule."""
    m, op, om, kind, rule = make(hf, 2, 2, 2, 2, "bp3", bc=1)
    set_mode(hf, op, mode)
    b = op.rhs()
    bref = O.rhs(om, kind, rule, bc=1)
    Ae = O.element_matrices(om, kind, rule)
    xo, st, kconv, rr_o, xh = O.cg(bref, m=om, Ae=Ae, bc=1, rel_tol=1e-14, max_iter=200,
                                   history=True)
    assert st == 0
    for k in range(1, kconv + 1):
        x = torch.zeros(m.n_local, dtype=torch.float64, device="cuda")
        st, stats, rr = op.cg(b, x, max_iter=k, fixed_iters=True, history=True)
        assert stats.iterations == k
        assert rel(host(x), xh[k]) <= 1e-10, (k, rel(host(x), xh[k]))
        assert abs(rr[k] - rr_o[k]) <= 1e-10 * rr_o[0], (k, rr[k], rr_o[k])
    x = torch.zeros(m.n_local, dtype=torch.float64, device="cuda")
    st, stats, rr = op.cg(b, x, rel_tol=1e-14, max_iter=200, history=True)
    assert stats.converged and abs(stats.iterations - kconv) <= 1
    assert rel(host(x), xo) <= 1e-12


@pytest.mark.parametrize("mode", list(CG_MODES))
@pytest.mark.parametrize("bench,p,n", [("bp3", 3, 4), ("bp5", 4, 3), ("bp1", 2, 4), ("bp3", 5, 3)])
def test_cg_iterates_small(hf, bench, p, n, mode):
    kind, rule = KINDS[bench]
    bc = 0 if bench == "bp1" else 1
    m, op, om, kind, rule = make(hf, n, n, n, p, bench, bc=bc)
    set_mode(hf, op, mode)
    b = op.rhs()
    Ae = O.element_matrices(om, kind, rule)
    bo = O.rhs(om, kind, rule, bc=bc)
    xo, st, kconv, rr_o, _ = O.cg(bo, m=om, Ae=Ae, bc=bc, rel_tol=1e-13, max_iter=800)
    assert st == 0
    # DESIGN.md reading R14: iterates are compared while ||r_k||/||r_0|| > 1e-4
    # (moderate iteration counts; past that, two correct CG runs drift apart by
    # rounding-driven loss of orthogonality and only re-meet at convergence).
    kwin = next(k for k in range(len(rr_o)) if np.sqrt(rr_o[k] / rr_o[0]) <= 1e-4)
    kmax = min(kwin, 200)
    _, _, _, _, xh = O.cg(bo, m=om, Ae=Ae, bc=bc, max_iter=kmax, fixed_iters=True,
                          history=True)
    # the oracle's own rounding sensitivity: the same CG on b perturbed at the
    # 1e-15 level (two correct runs differ by about this much; reading R14)
    pert = 1.0 + 1e-15 * W.random_vector(99, np.arange(len(bo)))
    _, _, _, _, xp = O.cg(bo * pert, m=om, Ae=Ae, bc=bc, max_iter=kmax, fixed_iters=True,
                          history=True)
    for k in sorted({1, 2, 5, kmax // 2, kmax}):
        x = torch.zeros(m.n_local, dtype=torch.float64, device="cuda")
        op.cg(b, x, max_iter=k, fixed_iters=True)
        tol = max(1e-10, 100.0 * rel(xp[k], xh[k]))
        assert rel(host(x), xh[k]) <= tol, (k, rel(host(x), xh[k]), tol)
    # converged solutions (both to rel-res 1e-13) agree to 1e-11
    x = torch.zeros(m.n_local, dtype=torch.float64, device="cuda")
    st, stats, _ = op.cg(b, x, rel_tol=1e-13, max_iter=800)
    assert st == 0 and abs(stats.iterations - kconv) <= 2
    assert rel(host(x), xo) <= 1e-11


@pytest.mark.parametrize("bench,p,n", [("bp3", 3, 4), ("bp3", 5, 3), ("bp1", 2, 4), ("bp5", 4, 3)])
def test_cg_every_iterate_within_rounding_envelope(hf, bench, p, n):
    """SURVEY R14 to the letter: EVERY iterate x_k, k <= min(k_conv, 200), against
    the oracle's.  Past ||r_k||/||r_0|| ~ 1e-4 two correct CG runs drift apart by
    rounding (loss of orthogonality), so the bound at k is max(1e-10, 1000 x the
    oracle's own sensitivity at k): the distance between the oracle run and the
    same run on b perturbed at the 1e-15 level (reading R14; an
    assembled-matrix oracle run stays within 1/12 of this envelope on CPU)."""
    kind, rule = KINDS[bench]
    bc = 0 if bench == "bp1" else 1
    m, op, om, kind, rule = make(hf, n, n, n, p, bench, bc=bc)
    b = op.rhs()
    Ae = O.element_matrices(om, kind, rule)
    bo = O.rhs(om, kind, rule, bc=bc)
    _, st, kconv, _, _ = O.cg(bo, m=om, Ae=Ae, bc=bc, rel_tol=1e-13, max_iter=800)
    K = min(kconv, 200)
    _, _, _, _, xh = O.cg(bo, m=om, Ae=Ae, bc=bc, max_iter=K, fixed_iters=True, history=True)
    pert = 1.0 + 1e-15 * W.random_vector(99, np.arange(len(bo)))
    _, _, _, _, xp = O.cg(bo * pert, m=om, Ae=Ae, bc=bc, max_iter=K, fixed_iters=True,
                          history=True)
    worst = 0.0
    for k in range(1, K + 1):
        x = torch.zeros(m.n_local, dtype=torch.float64, device="cuda")
        op.cg(b, x, max_iter=k, fixed_iters=True)
        tol = max(1e-10, 1000.0 * rel(xp[k], xh[k]))
        e = rel(host(x), xh[k])
        worst = max(worst, e / tol)
        assert e <= tol, (k, e, tol)


@pytest.mark.parametrize("mode", list(CG_MODES))
def test_cg_schedules_bitwise_deterministic(hf, mode):
    """Same inputs, same schedule => bitwise-identical iterate (fixed reduction
    orders everywhere)."""
    m, op, _, _, _ = make(hf, 5, 4, 3, 3, "bp3", bc=1)
    set_mode(hf, op, mode)
    b = op.rhs()
    xs = []
    for _ in range(2):
        x = torch.zeros(m.n_local, dtype=torch.float64, device="cuda")
        op.cg(b, x, max_iter=30, fixed_iters=True)
        xs.append(host(x))
    assert np.array_equal(xs[0].view(np.uint64), xs[1].view(np.uint64))


def test_cg_converges_manufactured(hf):
    """BP5 p=4 on 4^3, CG to 1e-10: the discrete solution approximates sin^3."""
    m, op, om, kind, rule = make(hf, 4, 4, 4, 4, "bp5", bc=1)
    b = op.rhs()
    x = torch.zeros(m.n_local, dtype=torch.float64, device="cuda")
    st, stats, rr = op.cg(b, x, rel_tol=1e-10, max_iter=2000, check_every=10)
    assert st == 0 and stats.converged and stats.final_rel_res <= 1e-10
    err = O.l2_error(om, host(x))
    assert err < 1e-3


# ----------------------------------------------------------------------------- at scale
def _contributors(I, J, K, p, dims):
    """Elements (and local node indices) whose closure holds lattice point
    (I, J, K) of an nx*ny*nz-element mesh: 1 (interior), 2 (face), 4 (edge), 8."""
    nx, ny, nz = dims
    def axis(L, n):
        if L % p == 0:
            return [(e, L - p * e) for e in (L // p - 1, L // p) if 0 <= e < n]
        return [(L // p, L % p)]
    out = []
    for ez, c in axis(K, nz):
        for ey, b in axis(J, ny):
            for ex, a in axis(I, nx):
                out.append((ex + nx * (ey + ny * ez), a + (p + 1) * (b + (p + 1) * c)))
    return out


def _sample_points(rng, p, dims, bc):
    """Seeded lattice points of every contribution class: element interiors,
    x / y / z single-face points (2 elements: the points the fused kernel
    completes by two-term reductions onto the zeroed y), edge-line points (4:
    the fix-up's partial sums), vertices (8), and with bc the Dirichlet faces."""
    Ns = [p * n + 1 for n in dims]
    lo = 1 if bc else 0
    def coord(on_plane, N):
        while True:
            v = int(rng.integers(lo, N - lo))
            if (v % p == 0) == on_plane and (not bc or 0 < v < N - 1):
                return v
    def point(planes):
        return tuple(coord(planes[a], Ns[a]) for a in range(3))
    pts = []
    if p > 1:
        pts += [point((False, False, False)) for _ in range(96)]
        for axis in range(3):
            for _ in range(48):
                pts.append(point(tuple(a == axis for a in range(3))))
        for axis in range(3):
            for _ in range(24):
                pts.append(point(tuple(a != axis for a in range(3))))
    pts += [point((True, True, True)) for _ in range(32)]
    if bc:
        pts += [(0, int(rng.integers(0, Ns[1])), int(rng.integers(0, Ns[2]))) for _ in range(8)]
        pts += [(int(rng.integers(0, Ns[0])), int(rng.integers(0, Ns[1])), Ns[2] - 1)
                for _ in range(8)]
    return pts


C5 = W.config5()
C5_DIMS = (C5["nx"], C5["ny"], C5["nz"])


@pytest.mark.parametrize("bench,p,bc,dims", [
    ("bp3", 5, 1, None), ("bp3", 5, 0, None), ("bp1", 8, 0, None), ("bp5", 6, 1, None),
    ("bp3", 4, 1, None), ("bp3", 6, 0, None),
    ("bp3", 5, 1, C5_DIMS),  # the bench's own workload: config 5, 200x200x25, 126M dofs
])
def test_sampled_points_full_size(hf, bench, p, bc, dims):
    """Sampled parity at the bench's full size and launch configuration (SURVEY.md
    §8(c) "parity at scale"; default options, so the memset + separate fix-up
    path the bench times): y at seeded lattice points of every contribution
    class against the oracle's dense-B element actions of the 1-8 elements that
    hold each point, summed; Dirichlet rows y = x (reading R6).  Meshes: the
    config-2/3 sweep sizes and BASELINE config 5's slab (the headline bench)."""
    kind, rule = KINDS[bench]
    if dims is None:
        n = W.bp3_sweep_n(p) if bench != "bp1" else W.bp1_sweep_n(p)
        dims = (n, n, n)
    nx, ny, nz = dims
    m = hf.Mesh(nx, ny, nz, p, alpha=W.ALPHA)
    op = hf.Operator(m, kind=kind, rule=rule, bc=bc)
    om = O.Mesh(nx, ny, nz, p, alpha=W.ALPHA)
    x = m.random(11)
    y = host(op.apply(x))
    xh = host(x)
    del x
    op.close()
    Nx, Ny, Nz = (p * nx + 1, p * ny + 1, p * nz + 1)
    rng = np.random.default_rng(7 + p + 10 * bc)
    pts = _sample_points(rng, p, dims, bc)
    contrib = {pt: _contributors(*pt, p, dims) for pt in pts}
    elems = np.array(sorted({e for c in contrib.values() for e, _ in c}))
    xz = xh
    if bc:  # z = x with the Dirichlet entries zeroed (reading R6)
        xz = xh.reshape(Nz, Ny, Nx).copy()
        xz[0, :, :] = xz[-1, :, :] = 0.0
        xz[:, 0, :] = xz[:, -1, :] = 0.0
        xz[:, :, 0] = xz[:, :, -1] = 0.0
        xz = xz.reshape(-1)
    ye = O.element_apply_sample(om, kind, rule, xz, elems)
    row = {e: i for i, e in enumerate(elems)}
    scale = np.abs(ye).max()
    num = den = 0.0
    for (I, J, K), c in contrib.items():
        g = I + Nx * (J + Ny * K)
        if bc and (min(I, J, K) == 0 or I == Nx - 1 or J == Ny - 1 or K == Nz - 1):
            assert y[g] == xh[g]
            continue
        r = sum(ye[row[e], loc] for e, loc in c)
        assert abs(y[g] - r) <= 1e-12 * scale * len(c), ((I, J, K), len(c), y[g], r)
        num += (y[g] - r) ** 2
        den += r ** 2
    assert np.sqrt(num / den) <= APPLY_TOL


@pytest.mark.parametrize("dims", [None, C5_DIMS])
def test_cg_full_size_properties(hf, dims):
    """The bench's CG (BP3 p=5, Dirichlet, manufactured RHS; config 3's 62^3
    elements and config 5's 200x200x25 slab, the headline workload) at full
    size, where the oracle cannot run the solve: x_1 = alpha_0 b with
    alpha_0 = b.b / b.Ab; after k iterations ||b - A x_k||^2 equals the
    recurrence's r_k.r_k; the per-iteration schedule (default at this size)
    and the persistent kernel give the same iterates up to reduction order."""
    if dims is None:
        n = W.bp3_sweep_n(5)
        dims = (n, n, n)
    m = hf.Mesh(*dims, 5, alpha=W.ALPHA)
    op = hf.Operator(m, kind=hf.DIFFUSION, rule=hf.GAUSS, bc=hf.BC_DIRICHLET)
    b = op.rhs()
    bb = m.dot(b, b)
    bAb = m.dot(b, op.apply(b))
    x = torch.zeros_like(b)
    op.cg(b, x, max_iter=1, fixed_iters=True)
    assert rel(host(x), (bb / bAb) * host(b)) <= 1e-12
    k = 6
    xs = {}
    for mode in ("separate", "fused", "persistent"):
        set_mode(hf, op, mode)
        x = torch.zeros_like(b)
        st, stats, rr = op.cg(b, x, max_iter=k, fixed_iters=True, history=True)
        assert stats.iterations == k
        r = b - op.apply(x)
        assert abs(m.dot(r, r) - rr[k]) <= 1e-10 * rr[0], (mode, m.dot(r, r), rr[k])
        xs[mode] = host(x)
    assert rel(xs["fused"], xs["separate"]) <= 1e-12
    assert rel(xs["persistent"], xs["separate"]) <= 1e-12
