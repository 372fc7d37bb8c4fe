"""GPU parity of the DG (L2) mass operator
against the CPU oracle's brute-force element matrices, through the C ABI.
Tolerance: relative L2 <= 1e-12 per apply (north star, FP64)."""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module")
def hf():
    import paper_2402_15940_b200 as hf
    hf.lib()
    return hf


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ragged batch tails: element counts not a multiple of the per-p batch size
CASES = [(3, 2, 2, 1, 0.1), (5, 3, 3, 1, 0.1), (3, 3, 2, 2, 0.1), (5, 3, 2, 3, 0.1),
         (3, 3, 3, 4, 0.1), (3, 2, 3, 5, 0.1), (2, 3, 2, 6, 0.1), (3, 2, 2, 7, 0.0),
         (2, 2, 3, 8, 0.1), (1, 1, 1, 5, 0.1), (1, 1, 1, 2, 0.0)]


@pytest.mark.parametrize("nx,ny,nz,p,alpha", CASES)
def test_dg_mass_matches_oracle(hf, nx, ny, nz, p, alpha):
    m = hf.Mesh(nx, ny, nz, p, alpha=alpha)
    dg = hf.DGMass(m)
    om = O.Mesh(nx, ny, nz, p, alpha=alpha)
    Me = O.dg_mass_matrices(om)
    assert dg.n_local == om.n_elems * (p + 1) ** 3
    for seed in (1, 2):
        x = dg.random(seed)
        y = host(dg.apply(x))
        ref = O.dg_apply(om, Me, host(x))
        assert rel(y, ref) <= TOL, rel(y, ref)


def test_dg_random_is_global_index_r12(hf):
    m = hf.Mesh(3, 2, 4, 2)
    dg = hf.DGMass(m)
    x = host(dg.random(9))
    ref = W.random_vector(9, np.arange(dg.n_local))
    assert np.array_equal(x.view(np.uint64), ref.view(np.uint64))


def test_dg_deterministic_and_graph_replay(hf):
    m = hf.Mesh(7, 5, 6, 5, alpha=0.1)
    dg = hf.DGMass(m)
    x = dg.random(3)
    ref = host(dg.apply(x))
    assert np.array_equal(host(dg.apply(x)).view(np.uint64), ref.view(np.uint64))
    y = torch.empty_like(x)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        dg.apply(x, y)
    for _ in range(3):
        y.zero_()
        g.replay()
        assert np.array_equal(host(y).view(np.uint64), ref.view(np.uint64))


def test_dg_rejects_unsupported_q(hf):
    m = hf.Mesh(2, 2, 2, 3)
    with pytest.raises(hf.HofemError):
        hf.DGMass(m, q_override=6)


@pytest.mark.parametrize("p", [2, 5, 8])
def test_dg_sampled_full_size(hf, p):
    """Bench size (~30M DG dofs): 192 seeded elements (plus the first and last,
    i.e. the ragged tail batch) against the oracle's element matrices."""
    n = W.dg_sweep_n(p)
    m = hf.Mesh(n, n, n, p, alpha=W.ALPHA)
    dg = hf.DGMass(m)
    om = O.Mesh(n, n, n, p, alpha=W.ALPHA)
    x = dg.random(5)
    y = host(dg.apply(x))
    xh = host(x)
    rng = np.random.default_rng(p)
    E = om.n_elems
    elems = np.unique(np.concatenate([rng.choice(E, 192, replace=False), [0, E - 1]]))
    ye = O.dg_apply_sample(om, xh, elems)
    nd = (p + 1) ** 3
    got = np.stack([y[e * nd:(e + 1) * nd] for e in elems])
    assert rel(got, ye) <= TOL
