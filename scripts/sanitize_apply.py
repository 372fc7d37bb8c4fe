"""Small runs of every kernel family for compute-sanitizer (racecheck /
synccheck / memcheck) on the GPU box:
    compute-sanitizer --tool racecheck python scripts/sanitize_apply.py
Fused applies (BP1/BP3/BP5, both fix-up schedules), all three CG schedules
(per-iteration, fused cooperative update, persistent whole-solve kernel), the
fully matrix-free apply, the DG mass kernel (bulk copies in and out, ragged
tail), the p-MG diagonal / transfers / V-cycle / PCG, and a loopback 2-rank apply."""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_15940_b200 as hf  # noqa: E402

for bench, p, n in (("bp3", 5, 3), ("bp3", 4, 3), ("bp3", 6, 2), ("bp5", 6, 2), ("bp1", 8, 2),
                    ("bp3", 2, 3), ("bp1", 5, 3), ("bp1", 1, 3), ("bp1", 4, 3)):
    kind = hf.MASS if bench == "bp1" else hf.DIFFUSION
    rule = hf.GLL if bench == "bp5" else hf.GAUSS
    m = hf.Mesh(n, n, n + 1, p)
    op = hf.Operator(m, kind=kind, rule=rule, bc=hf.BC_NONE if bench == "bp1" else hf.BC_DIRICHLET)
    x = m.random(1)
    for infix in (hf.NEVER, hf.ALWAYS):
        op.set_option(hf.OPT_INFIX, infix)
        y = op.apply(x)
    b = op.rhs()
    for mode in ((0, 0), (0, 2), (2, 0)):  # (persistent, fused update)
        op.set_option(hf.OPT_CG_PERSISTENT, mode[0])
        op.set_option(hf.OPT_CG_FUSED_UPDATE, mode[1])
        xs = torch.zeros_like(b)
        op.cg(b, xs, max_iter=3, fixed_iters=True)
    if bench == "bp3":
        op.apply_mf(x)
        op.diagonal()
    torch.cuda.synchronize()
    print(bench, p, n, float(y.norm()), flush=True)
    op.close()
    m.close()
for p in (2, 5, 7):
    m = hf.Mesh(3, 2, 3, p)
    dg = hf.DGMass(m)
    x = dg.random(1)
    dg.apply(x)
    torch.cuda.synchronize()
    print("dg", p, flush=True)
m = hf.Mesh(3, 3, 2, 4)
P = hf.PMG(m, degree=2)
op = hf.Operator(m, kind=hf.DIFFUSION, rule=hf.GAUSS, bc=hf.BC_DIRICHLET)
b = op.rhs()
xs = torch.zeros_like(b)
P.pcg(b, xs, rel_tol=1e-8, max_iter=5)
torch.cuda.synchronize()
print("pmg", flush=True)
group = hf.LoopbackGroup(2)


def rank(r):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        c = hf.Comm.loopback(group, r)
        mm = hf.Mesh(3, 2, 4, 3, comm=c, stream=s)
        oo = hf.Operator(mm, kind=hf.DIFFUSION, rule=hf.GAUSS, bc=hf.BC_DIRICHLET, stream=s)
        oo.apply(mm.random(1, stream=s), stream=s)
        s.synchronize()


ts = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
for t in ts:
    t.start()
for t in ts:
    t.join()
print("loopback", flush=True)
