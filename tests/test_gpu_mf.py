"""GPU parity of the fully matrix-free BP3 apply (
PAPER.md:145 "Fully Matrix-Free"): the same operator as PA with the geometric
factors recomputed from the nodal coordinates on every apply, against the CPU
oracle's brute-force element matrices (relative L2 <= 1e-12)."""
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


CASES = [(2, 2, 2, 2), (5, 3, 4, 1), (3, 4, 3, 2), (3, 3, 2, 3), (3, 2, 3, 4), (3, 3, 2, 5),
         (2, 3, 2, 6), (3, 2, 2, 7), (2, 2, 2, 8), (1, 1, 1, 3)]


@pytest.mark.parametrize("nx,ny,nz,p", CASES)
@pytest.mark.parametrize("bc", [0, 1])
def test_mf_matches_oracle_and_pa(hf, nx, ny, nz, p, bc):
    m = hf.Mesh(nx, ny, nz, p, alpha=0.1)
    op = hf.Operator(m, kind=hf.DIFFUSION, rule=hf.GAUSS, bc=bc)
    om = O.Mesh(nx, ny, nz, p, alpha=0.1)
    for seed in (1, 2):
        x = m.random(seed)
        if p <= 4:
            ref = O.apply_ea(om, O.element_matrices(om, O.DIFFUSION, O.GAUSS), host(x), bc=bc)
        else:
            ref = O.apply_dense(om, O.DIFFUSION, O.GAUSS, host(x), bc=bc)
        y = host(op.apply_mf(x))
        assert rel(y, ref) <= TOL, rel(y, ref)
        assert rel(y, host(op.apply(x))) <= TOL
    # deterministic run to run
    y1, y2 = host(op.apply_mf(x)), host(op.apply_mf(x))
    assert np.array_equal(y1.view(np.uint64), y2.view(np.uint64))


def test_mf_rejects_non_bp3(hf):
    m = hf.Mesh(2, 2, 2, 3)
    for kind, rule in ((hf.MASS, hf.GAUSS), (hf.DIFFUSION, hf.GLL)):
        op = hf.Operator(m, kind=kind, rule=rule)
        with pytest.raises(hf.HofemError):
            op.apply_mf(m.random(1))


@pytest.mark.parametrize("p", [3, 5])
def test_mf_sampled_full_size(hf, p):
    """Bench size (~30M dofs): MF apply equals the PA apply (itself sampled against
    the oracle at this size in test_gpu_parity) to 1e-12, and element-interior
    dofs of 128 seeded elements equal the oracle's element actions."""
    n = W.bp3_sweep_n(p)
    m = hf.Mesh(n, n, n, p, alpha=W.ALPHA)
    op = hf.Operator(m, kind=hf.DIFFUSION, rule=hf.GAUSS, bc=hf.BC_DIRICHLET)
    x = m.random(7)
    y = host(op.apply_mf(x))
    assert rel(y, host(op.apply(x))) <= TOL
    om = O.Mesh(n, n, n, p, alpha=W.ALPHA)
    rng = np.random.default_rng(p)
    N = p * n + 1
    elems = rng.choice(np.arange(n * n * n).reshape(n, n, n)[1:-1, 1:-1, 1:-1].ravel(), 128,
                       replace=False)
    ye = O.element_apply_sample(om, O.DIFFUSION, O.GAUSS, host(x), elems)
    num = den = 0.0
    for k, e in enumerate(elems):
        ex, ey, ez = e % n, (e // n) % n, e // (n * n)
        for c in range(1, p):
            for b in range(1, p):
                for a in range(1, p):
                    g = (p * ex + a) + N * ((p * ey + b) + N * (p * ez + c))
                    r = ye[k, a + (p + 1) * (b + (p + 1) * c)]
                    num += (y[g] - r) ** 2
                    den += r ** 2
    assert np.sqrt(num / den) <= TOL
