"""GPU parity of the f2 pieces:
matrix-free diagonal, p-transfers, power iteration, Chebyshev-Jacobi smoothing,
the V-cycle and p-MG preconditioned CG, against the CPU oracle (readings
R17-R18) through the C ABI."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hf():
    import paper_2402_15940_b200 as hf
    hf.lib()
    return hf


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


KINDS = {"bp1": (1, 1), "bp3": (2, 1), "bp5": (2, 2)}


@pytest.mark.parametrize("bench,p,bc,dims", [("bp3", 1, 1, (4, 3, 2)), ("bp3", 2, 0, (3, 2, 2)),
                                             ("bp3", 3, 1, (3, 3, 2)), ("bp3", 5, 1, (2, 2, 2)),
                                             ("bp1", 3, 0, (3, 2, 2)), ("bp5", 4, 1, (2, 3, 2)),
                                             ("bp3", 8, 0, (2, 1, 1))])
def test_diagonal_matches_oracle(hf, bench, p, bc, dims):
    kind, rule = KINDS[bench]
    m = hf.Mesh(*dims, p, alpha=0.1)
    op = hf.Operator(m, kind=kind, rule=rule, bc=bc)
    om = O.Mesh(*dims, p, alpha=0.1)
    ref = O.diagonal(om, O.element_matrices(om, kind, rule), bc=bc)
    d = host(op.diagonal())
    assert rel(d, ref) <= 1e-13, rel(d, ref)


@pytest.fixture(scope="module")
def hier(hf):
    """A 3-level hierarchy (orders 4, 2, 1) on a curved 3x2x2 mesh, GPU and oracle."""
    dims, p = (3, 2, 2), 4
    m = hf.Mesh(*dims, p, alpha=0.1)
    P = hf.PMG(m, degree=3, power_iters=10, seed=1)
    OP = O.PMG(*dims, p, degree=3, power_iters=10, seed=1)
    return m, P, OP


def test_hierarchy_orders_and_lambdas(hf, hier):
    m, P, OP = hier
    assert P.orders == O.pmg_orders(4) == [4, 2, 1]
    for k, lam in enumerate(P.lambdas()):
        assert abs(lam - OP.levels[k]["lam"]) <= 1e-10 * lam, (k, lam, OP.levels[k]["lam"])


def test_transfers_match_oracle(hf, hier):
    m, P, OP = hier
    rng = np.random.default_rng(3)
    for k in range(len(P.levels) - 1):
        F, C = OP.levels[k], OP.levels[k + 1]
        xc = rng.standard_normal(C["m"].n_dofs)
        xf0 = rng.standard_normal(F["m"].n_dofs)
        got = host(P.prolong_add(k, dev(xc), dev(xf0)))
        assert rel(got, xf0 + O.prolong(F["m"], C["m"], xc)) <= 1e-14
        rf = rng.standard_normal(F["m"].n_dofs)
        ref = O.restrict(F["m"], C["m"], rf)
        ref[C["ess"]] = 0.0
        assert rel(host(P.restrict(k, dev(rf))), ref) <= 1e-14


def test_smoother_matches_oracle(hf, hier):
    m, P, OP = hier
    rng = np.random.default_rng(4)
    for k, L in enumerate(OP.levels):
        P.set_lambda(k, L["lam"])
        b = rng.standard_normal(L["m"].n_dofs)
        x0 = rng.standard_normal(L["m"].n_dofs)
        got = host(P.smooth(k, dev(b), dev(x0)))
        ref = O.cheb(L["m"], L["Ae"], 1, L["dinv"], L["lmin"], L["lmax"], 3, b, x0)
        assert rel(got, ref) <= 1e-12, (k, rel(got, ref))


def test_vcycle_matches_oracle(hf, hier):
    m, P, OP = hier
    for k, L in enumerate(OP.levels):
        P.set_lambda(k, L["lam"])
    r = O.rhs(OP.levels[0]["m"], O.DIFFUSION, O.GAUSS, bc=1)
    got = host(P.vcycle(dev(r)))
    ref = OP.vcycle(r)
    assert rel(got, ref) <= 1e-12, rel(got, ref)


def test_pcg_matches_oracle(hf, hier):
    """p-MG PCG (reading R18): residual history and solution against the oracle's
    PCG with the same eigenvalue estimates; far fewer iterations than CG."""
    m, P, OP = hier
    for k, L in enumerate(OP.levels):
        P.set_lambda(k, L["lam"])
    L0 = OP.levels[0]
    bo = O.rhs(L0["m"], O.DIFFUSION, O.GAUSS, bc=1)
    xo, st, ko, rro, _ = O.pcg(bo, OP.vcycle, m=L0["m"], Ae=L0["Ae"], rel_tol=1e-12)
    assert st == 0
    b = dev(bo)
    x = torch.zeros_like(b)
    st, stats, rr = P.pcg(b, x, rel_tol=1e-12, max_iter=200, history=True)
    assert st == 0 and stats.converged and abs(stats.iterations - ko) <= 1
    for k in range(min(ko, stats.iterations) + 1):
        if rro[k] > 1e-16 * rro[0]:
            assert abs(rr[k] - rro[k]) <= 1e-8 * rro[k] + 1e-20, (k, rr[k], rro[k])
    assert rel(host(x), xo) <= 1e-10
    op = hf.Operator(m, kind=hf.DIFFUSION, rule=hf.GAUSS, bc=hf.BC_DIRICHLET)
    xc = torch.zeros_like(b)
    _, cstats, _ = op.cg(b, xc, rel_tol=1e-12, max_iter=2000)
    assert stats.iterations * 3 < cstats.iterations


def test_pcg_bench_size_properties(hf):
    """BPS3 at a larger size (BP3 p=5, 20^3 elements, ~1M dofs): PCG reaches
    1e-10 with a mesh-independent-ish handful of iterations and the true residual
    b - A x matches."""
    m = hf.Mesh(20, 20, 20, 5, alpha=0.1)
    P = hf.PMG(m, degree=3)
    op = hf.Operator(m, kind=hf.DIFFUSION, rule=hf.GAUSS, bc=hf.BC_DIRICHLET)
    b = op.rhs()
    x = torch.zeros_like(b)
    st, stats, rr = P.pcg(b, x, rel_tol=1e-10, max_iter=300, history=True)
    assert st == 0 and stats.final_rel_res <= 1e-10
    r = b - op.apply(x)
    assert np.sqrt(m.dot(r, r) / m.dot(b, b)) <= 2e-10
    assert stats.iterations < 100
