"""N>1 host logic on CPU (gloo, world_size 2 and 3): the z-slab partition,
ownership, the interface-plane exchange and the allreduced dot products
reproduce the global operator.  Per-slab local operators come from the oracle's
window mode (elements of the slab only); the exchange is
tests/partition_mirror.py (exchange_planes), the same logic comm.cu
implements with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import workloads as W
from tests import partition_mirror as partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cfg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz, p, kind, bc = cfg
        s = partition.slab(nx, ny, nz, p, rank, world)
        om = O.Mesh(nx, ny, nz, p, alpha=0.1, z0=s.z0, nzl=s.nzl)
        assert om.n_dofs == s.n_local
        # global random vector restricted to this slab (R12 indexes global dofs)
        x = W.random_lvector((s.Nx, s.Ny, s.Nzl), 3, z_plane0=s.K0)
        Ae = O.element_matrices(om, kind, O.GAUSS)
        # local apply WITHOUT the Dirichlet post-step on the interface planes
        # (mirrors the library: BC is re-imposed after the exchange)
        y = O.apply_ea(om, Ae, x, bc=bc)
        mask = O.boundary_mask(om).reshape(s.Nzl, s.plane)
        yt = torch.from_numpy(y.copy())
        xt = torch.from_numpy(x)

        def send(t, peer):
            dist.send(t.contiguous(), peer)

        def recv(t, peer):
            dist.recv(t, peer)
            return t

        def ess_fix(which, view):
            k = 0 if which == "lo" else s.Nzl - 1
            m = torch.from_numpy(mask[k])
            xs = xt[k * s.plane:(k + 1) * s.plane]
            view[m] = xs[m]

        partition.exchange_planes(s, yt, send, recv, ess_fix if bc else None)
        # owned-dof dot products, allreduced
        d = torch.tensor([float(np.dot(x[: s.n_owned], yt.numpy()[: s.n_owned]))],
                         dtype=torch.float64)
        dist.all_reduce(d)
        q.put((rank, s.K0, s.n_local, s.n_owned, yt.numpy().copy(), float(d.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg", [
    (2, (3, 2, 4, 2, O.DIFFUSION, 1)),
    (2, (2, 3, 2, 3, O.MASS, 0)),
    (3, (2, 2, 3, 2, O.DIFFUSION, 1)),
])
def test_slab_exchange_matches_global(world, cfg):
    nx, ny, nz, p, kind, bc = cfg
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in range(world)])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    gm = O.Mesh(nx, ny, nz, p, alpha=0.1)
    xg = W.random_vector(3, np.arange(gm.n_dofs))
    yg = O.apply_ea(gm, O.element_matrices(gm, kind, O.GAUSS), xg, bc=bc)
    plane = (p * nx + 1) * (p * ny + 1)
    owned_total = 0
    for rank, K0, n_local, n_owned, y, dot in res:
        g0 = K0 * plane
        np.testing.assert_allclose(y, yg[g0:g0 + n_local], rtol=0, atol=1e-13 * np.abs(yg).max())
        owned_total += n_owned
        assert abs(dot - float(np.dot(xg, yg))) <= 1e-12 * np.abs(xg).sum() * np.abs(yg).max()
    assert owned_total == gm.n_dofs
    # duplicated interface planes are bitwise identical on both neighbours
    for (r0, K0a, na, _, ya, _), (r1, K0b, nb, _, yb, _) in zip(res, res[1:]):
        top = ya[na - plane:]
        bot = yb[:plane]
        assert np.array_equal(top.view(np.uint64), bot.view(np.uint64))


def test_slab_counts():
    s = [partition.slab(62, 62, 62 * 8, 5, r, 8) for r in range(8)]
    assert sum(x.n_owned for x in s) == (5 * 62 + 1) ** 2 * (5 * 62 * 8 + 1)
    assert all(x.n_local == (5 * 62 + 1) ** 2 * (5 * 62 + 1) for x in s)
    with pytest.raises(ValueError):
        partition.slab(4, 4, 5, 2, 0, 2)
