"""The multi-rank CUDA data path on ONE GPU:
R = 2, 3 ranks as host threads with the in-process loopback transport
(hofem_loopback_group_create / hofem_comm_init_loopback), each on its own
stream, drive comm.cu's plane exchange (with Dirichlet re-imposition on the
interface planes), the owned-dof dot products / allreduce, the fused kernel's
owned-dof p.Ap and the multi-rank CG -- compared with the GLOBAL single-mesh
oracle.  Both exchange transports: the collective (loopback copies standing
in for NCCL) and the kernel-initiated peer puts (hofem_mesh_set_exchange).
The peer-put exchange is also hammered by many back-to-back applies without
any other collective in between (run-ahead bounded by the consumed flags)."""
import threading

import numpy as np
import pytest
import torch

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hf():
    import paper_2402_15940_b200 as hf
    hf.lib()
    return hf


def run_ranks(hf, R, fn):
    group = hf.LoopbackGroup(R)
    out, err = [None] * R, [None] * R

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                comm = hf.Comm.loopback(group, r)
                out[r] = fn(r, comm, s)
                s.synchronize()
        except Exception as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=worker, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    group.close()
    for e in err:
        if e is not None:
            raise e
    # every rank synchronized its stream and left: host copies are safe now
    return [to_host(o) for o in out]


def host(t):
    # Inside a rank's function results stay on the device: a copy into pageable
    # host memory may wait on the whole device, i.e. on a neighbour's put kernel
    # that spins until this rank's next exchange (deadlock).  run_ranks copies
    # them to the host after every rank finished.
    return t


def to_host(o):
    if isinstance(o, torch.Tensor):
        return o.detach().cpu().numpy()
    if isinstance(o, dict):
        return {k: to_host(v) for k, v in o.items()}
    if isinstance(o, (list, tuple)):
        return type(o)(to_host(v) for v in o)
    return o


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def slab(v, plane, p, nzl, r):
    return v[plane * p * nzl * r: plane * (p * nzl * (r + 1) + 1)]


CFG = [(2, "bp3", 3, (3, 2, 4), 1), (3, "bp3", 2, (4, 3, 6), 1), (2, "bp1", 4, (2, 3, 2), 0),
       (3, "bp5", 3, (3, 3, 3), 1), (2, "bp3", 5, (3, 2, 4), 0)]
KINDS = {"bp1": (1, 1), "bp3": (2, 1), "bp5": (2, 2)}


@pytest.mark.parametrize("xmode", [0, 1])
@pytest.mark.parametrize("R,bench,p,dims,bc", CFG)
def test_loopback_apply_rhs_dot_match_global(hf, R, bench, p, dims, bc, xmode):
    kind, rule = KINDS[bench]
    nx, ny, nz = dims
    nzl = nz // R
    plane = (p * nx + 1) * (p * ny + 1)

    def fn(r, comm, s):
        # every object and output buffer exists before the kernel-initiated
        # exchange is switched on: an allocation or object creation between two
        # exchanges may synchronize the whole (shared) device while a
        # neighbour's put kernel spins on this rank (hofem.h, set_exchange)
        m = hf.Mesh(nx, ny, nz, p, alpha=0.1, comm=comm, stream=s)
        op = hf.Operator(m, kind=kind, rule=rule, bc=bc, stream=s)
        dg = hf.DGMass(m, stream=s)
        x = m.random(5, stream=s)
        y, yd, yu, b, diag, ymf = (torch.empty_like(x) for _ in range(6))
        xdg = dg.random(4, stream=s)
        ydg = torch.empty_like(xdg)
        s.synchronize()
        m.set_exchange(xmode, stream=s)
        op.apply(x, y, stream=s)
        _, d = op.apply_dot(x, yd, stream=s)
        op.apply_unfused(x, yu, stream=s)
        op.rhs(b, stream=s)
        xx = m.dot(x, x, stream=s)
        op.diagonal(diag, stream=s)
        if bench == "bp3":
            op.apply_mf(x, ymf, stream=s)
        else:
            ymf = None
        dg.apply(xdg, ydg, stream=s)
        s.synchronize()
        return dict(x=host(x), y=host(y), yd=host(yd), yu=host(yu), b=host(b), d=d, xx=xx,
                    n_owned=m.n_owned, diag=host(diag),
                    ymf=None if ymf is None else host(ymf), xdg=host(xdg), ydg=host(ydg))

    res = run_ranks(hf, R, fn)
    om = O.Mesh(nx, ny, nz, p, alpha=0.1)
    xg = W.random_vector(5, np.arange(om.n_dofs))
    Ae = O.element_matrices(om, kind, rule)
    yg = O.apply_ea(om, Ae, xg, bc=bc)
    bg = O.rhs(om, kind, rule, bc=bc)
    for r in range(R):
        R_ = res[r]
        assert np.array_equal(R_["x"], slab(xg, plane, p, nzl, r))
        assert rel(R_["y"], slab(yg, plane, p, nzl, r)) <= 1e-12
        assert rel(R_["yu"], slab(yg, plane, p, nzl, r)) <= 1e-12
        assert np.array_equal(R_["yd"].view(np.uint64), R_["y"].view(np.uint64))
        assert rel(R_["b"], slab(bg, plane, p, nzl, r)) <= 1e-13
        # allreduced dots: identical on every rank, equal to the global values
        assert R_["d"] == res[0]["d"] and R_["xx"] == res[0]["xx"]
        if r + 1 < R:  # duplicated interface plane: bitwise equal on both ranks
            top = R_["y"][-plane:]
            bot = res[r + 1]["y"][:plane]
            assert np.array_equal(top.view(np.uint64), bot.view(np.uint64))
    dg_ref = O.diagonal(om, Ae, bc=bc)
    nd = (p + 1) ** 3
    Me = O.dg_mass_matrices(om)
    xdg = W.random_vector(4, np.arange(om.n_elems * nd))
    ydg = O.dg_apply(om, Me, xdg)
    eslab = nx * ny * nzl * nd
    for r in range(R):
        R_ = res[r]
        # matrix-free diagonal with the interface sums and Dirichlet rows = 1
        assert rel(R_["diag"], slab(dg_ref, plane, p, nzl, r)) <= 1e-13
        if R_["ymf"] is not None:  # fully matrix-free apply through the exchange
            assert rel(R_["ymf"], slab(yg, plane, p, nzl, r)) <= 1e-12
        # DG: rank r holds elements [r nx ny nzl, (r+1) nx ny nzl), global DG index
        assert np.array_equal(R_["xdg"], xdg[r * eslab:(r + 1) * eslab])
        assert rel(R_["ydg"], ydg[r * eslab:(r + 1) * eslab]) <= 1e-12
    assert sum(res[r]["n_owned"] for r in range(R)) == om.n_dofs
    scale = float(np.abs(xg) @ np.abs(yg))
    assert abs(res[0]["d"] - float(xg @ yg)) <= 1e-12 * scale
    assert abs(res[0]["xx"] - float(xg @ xg)) <= 1e-12 * float(xg @ xg)


@pytest.mark.parametrize("xmode,persist", [(0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("R,bench,p,dims", [(2, "bp3", 3, (3, 2, 4)), (3, "bp3", 2, (3, 3, 6))])
def test_loopback_cg_iterates_match_global(hf, R, bench, p, dims, xmode, persist):
    """Multi-rank CG against the global oracle CG iterates: per-iteration kernels
    with the scalars through the loopback allreduce (either exchange transport),
    and -- with the kernel-initiated exchange and the auto setting -- the
    persistent kernel with the in-kernel exchange and chain allreduce."""
    kind, rule = KINDS[bench]
    nx, ny, nz = dims
    nzl = nz // R
    plane = (p * nx + 1) * (p * ny + 1)
    om = O.Mesh(nx, ny, nz, p, alpha=0.1)
    Ae = O.element_matrices(om, kind, rule)
    bg = O.rhs(om, kind, rule, bc=1)
    ks = [1, 4, 12]
    _, _, _, _, xh = O.cg(bg, m=om, Ae=Ae, bc=1, max_iter=max(ks), fixed_iters=True, history=True)
    xo, st, kconv, _, _ = O.cg(bg, m=om, Ae=Ae, bc=1, rel_tol=1e-13, max_iter=1000)

    def fn(r, comm, s):
        m = hf.Mesh(nx, ny, nz, p, alpha=0.1, comm=comm, stream=s)
        op = hf.Operator(m, kind=kind, rule=rule, bc=1, stream=s)
        op.set_option(hf.OPT_CG_PERSISTENT, persist)  # 0 never, 1 auto
        xs = {k: torch.zeros(m.n_local, dtype=torch.float64, device="cuda")
              for k in ks + ["conv"]}
        b = torch.empty_like(xs["conv"])
        s.synchronize()
        m.set_exchange(xmode, stream=s)  # after every allocation (see the test above)
        op.rhs(b, stream=s)
        out = {}
        for k in ks:
            op.cg(b, xs[k], max_iter=k, fixed_iters=True, stream=s)
            out[k] = host(xs[k])
        x = xs["conv"]
        st, stats, _ = op.cg(b, x, rel_tol=1e-13, max_iter=1000, check_every=1, stream=s)
        out["conv"] = (st, stats.iterations, host(x))
        return out

    res = run_ranks(hf, R, fn)
    for r in range(R):
        for k in ks:
            assert rel(res[r][k], slab(xh[k], plane, p, nzl, r)) <= 1e-10, (r, k)
        st_r, it_r, x_r = res[r]["conv"]
        assert st_r == 0 and abs(it_r - kconv) <= 2
        assert rel(x_r, slab(xo, plane, p, nzl, r)) <= 1e-11


def test_loopback_peer_puts_back_to_back(hf):
    """30 applies per rank with no collective between them: the double-buffered
    receive slots and the consumed counters keep a fast rank from overwriting a
    slot its neighbour has not added yet; every result equals the collective
    transport's bit for bit (both sum a + b on each plane)."""
    R, p, dims = 3, 3, (3, 2, 6)

    def fn(r, comm, s):
        m = hf.Mesh(*dims, p, alpha=0.1, comm=comm, stream=s)
        op = hf.Operator(m, kind=hf.DIFFUSION, rule=hf.GAUSS, bc=1, stream=s)
        x = m.random(3, stream=s)
        ref = host(op.apply(x, stream=s))
        ys = [torch.empty_like(x) for _ in range(30)]
        s.synchronize()
        m.set_exchange(1, stream=s)
        for y in ys:
            op.apply(x, y, stream=s)
        s.synchronize()
        return ref, [host(y) for y in ys]

    res = run_ranks(hf, R, fn)
    for ref, ys in res:
        for y in ys:
            assert np.array_equal(y.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("R,bench,p,dims", [(2, "bp3", 3, (3, 2, 4)), (3, "bp3", 2, (3, 3, 6)),
                                            (2, "bp3", 5, (2, 3, 4)), (2, "bp5", 4, (3, 2, 4)),
                                            (3, "bp1", 3, (2, 3, 3)), (4, "bp3", 3, (2, 2, 8))])
def test_loopback_persistent_cg_in_kernel_exchange(hf, R, bench, p, dims):
    """The whole multi-rank CG in ONE persistent kernel per rank (§8(f) f1;
    PAPER.md:177-182, 197): the interface planes of Ap are put into the z
    neighbours' slots and p.Ap / r.r are allreduced (chain over the ranks) inside
    the kernel.  Iterates and the converged solution against the global oracle;
    afterwards a host-driven apply and a second solve still agree (the kernel
    continues the mesh's exchange and reduction sequence numbers)."""
    kind, rule = KINDS[bench]
    bc = 0 if bench == "bp1" else 1
    nx, ny, nz = dims
    nzl = nz // R
    plane = (p * nx + 1) * (p * ny + 1)
    om = O.Mesh(nx, ny, nz, p, alpha=0.1)
    Ae = O.element_matrices(om, kind, rule)
    bg = O.rhs(om, kind, rule, bc=bc)
    ks = [1, 3, 9]
    _, _, _, _, xh = O.cg(bg, m=om, Ae=Ae, bc=bc, max_iter=max(ks), fixed_iters=True,
                          history=True)
    xo, st, kconv, _, _ = O.cg(bg, m=om, Ae=Ae, bc=bc, rel_tol=1e-13, max_iter=1000)
    xg = W.random_vector(5, np.arange(om.n_dofs))
    yg = O.apply_ea(om, Ae, xg, bc=bc)

    def fn(r, comm, s):
        m = hf.Mesh(nx, ny, nz, p, alpha=0.1, comm=comm, stream=s)
        op = hf.Operator(m, kind=kind, rule=rule, bc=bc, stream=s)
        op.set_option(hf.OPT_CG_PERSISTENT, hf.ALWAYS)
        xs = {k: torch.zeros(m.n_local, dtype=torch.float64, device="cuda")
              for k in ks + ["conv", "again"]}
        b = torch.empty_like(xs["conv"])
        xa = m.random(5, stream=s)
        ya = torch.empty_like(xa)
        s.synchronize()
        m.set_exchange(1, stream=s)
        op.rhs(b, stream=s)
        out = {}
        for k in ks:
            st, stats, _ = op.cg(b, xs[k], max_iter=k, fixed_iters=True, stream=s)
            out[k] = (st, stats.iterations, host(xs[k]))
        st, stats, _ = op.cg(b, xs["conv"], rel_tol=1e-13, max_iter=1000, stream=s)
        out["conv"] = (st, stats.iterations, host(xs["conv"]))
        op.apply(xa, ya, stream=s)  # host-driven peer-put exchange after the kernels
        out["y"] = host(ya)
        st, stats, _ = op.cg(b, xs["again"], max_iter=ks[-1], fixed_iters=True, stream=s)
        out["again"] = host(xs["again"])
        return out

    res = run_ranks(hf, R, fn)
    for r in range(R):
        for k in ks:
            st_k, it_k, x_k = res[r][k]
            assert st_k == 0 and it_k == k
            assert rel(x_k, slab(xh[k], plane, p, nzl, r)) <= 1e-10, (r, k)
        st_r, it_r, x_r = res[r]["conv"]
        assert st_r == 0 and abs(it_r - kconv) <= 2
        assert rel(x_r, slab(xo, plane, p, nzl, r)) <= 1e-11
        assert rel(res[r]["y"], slab(yg, plane, p, nzl, r)) <= 1e-12
        assert np.array_equal(res[r]["again"].view(np.uint64), res[r][ks[-1]][2].view(np.uint64))
        if r + 1 < R:  # duplicated interface plane: the same iterate on both ranks
            assert np.array_equal(res[r]["conv"][2][-plane:].view(np.uint64),
                                  res[r + 1]["conv"][2][:plane].view(np.uint64))


def test_loopback_persistent_cg_needs_kernel_exchange(hf):
    """Several ranks with the collective exchange (mode 0): the persistent CG
    schedule needs mode 1's peer pointers, so forcing it runs the per-iteration
    kernels instead -- bitwise the same iterate as asking for them."""
    R, p, dims = 2, 2, (2, 2, 4)

    def fn(r, comm, s):
        m = hf.Mesh(*dims, p, alpha=0.1, comm=comm, stream=s)
        op = hf.Operator(m, kind=hf.DIFFUSION, rule=hf.GAUSS, bc=1, stream=s)
        b = op.rhs(stream=s)
        xs = []
        for mode in (hf.ALWAYS, hf.NEVER):
            op.set_option(hf.OPT_CG_PERSISTENT, mode)
            x = torch.zeros_like(b)
            op.cg(b, x, max_iter=5, fixed_iters=True, stream=s)
            xs.append(x)
        s.synchronize()
        return xs

    for xa, xn in run_ranks(hf, R, fn):
        assert np.array_equal(xa.view(np.uint64), xn.view(np.uint64))
