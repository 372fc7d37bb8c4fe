"""Small fused applies (BP1/BP3/BP5, several p, Dirichlet) for compute-sanitizer
(racecheck / synccheck / memcheck) runs on the GPU box:
    compute-sanitizer --tool racecheck python scripts/sanitize_apply.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_15940_b200 as hf  # noqa: E402

for bench, p, n in (("bp3", 5, 3), ("bp3", 4, 3), ("bp3", 6, 2), ("bp5", 6, 2), ("bp1", 8, 2)):
    kind = hf.MASS if bench == "bp1" else hf.DIFFUSION
    rule = hf.GLL if bench == "bp5" else hf.GAUSS
    m = hf.Mesh(n, n, n + 1, p)
    op = hf.Operator(m, kind=kind, rule=rule, bc=hf.BC_NONE if bench == "bp1" else hf.BC_DIRICHLET)
    x = m.random(1)
    y = op.apply(x)
    b = op.rhs()
    xs = torch.zeros_like(b)
    op.cg(b, xs, max_iter=3, fixed_iters=True)
    torch.cuda.synchronize()
    print(bench, p, n, float(y.norm()))
    op.close()
    m.close()
