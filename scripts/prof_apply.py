"""Profiling driver (for ncu): a few applies of one operator.

    python scripts/prof_apply.py [--bench bp3|bp1|bp5|dg] [--p 5] [--slab nx,ny,nz | --n n]
                                 [--unfused | --mf] [--reps 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_15940_b200 as hf  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bench", default="bp3")
ap.add_argument("--p", type=int, default=5)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--slab", default="")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--unfused", action="store_true")
ap.add_argument("--mf", action="store_true")
a = ap.parse_args()
if a.slab:
    nx, ny, nz = (int(v) for v in a.slab.split(","))
else:
    n = a.n or (W.bp1_sweep_n(a.p) if a.bench == "bp1" else
                W.dg_sweep_n(a.p) if a.bench == "dg" else W.bp3_sweep_n(a.p))
    nx = ny = nz = n
m = hf.Mesh(nx, ny, nz, a.p)
if a.bench == "dg":
    dg = hf.DGMass(m)
    x = dg.random(1)
    y = torch.empty_like(x)
    for _ in range(a.reps):
        dg.apply(x, y)
else:
    kind = hf.MASS if a.bench == "bp1" else hf.DIFFUSION
    rule = hf.GLL if a.bench == "bp5" else hf.GAUSS
    op = hf.Operator(m, kind=kind, rule=rule,
                     bc=hf.BC_DIRICHLET if a.bench != "bp1" else hf.BC_NONE)
    x = m.random(1)
    y = torch.empty_like(x)
    fn = op.apply_unfused if a.unfused else (op.apply_mf if a.mf else op.apply)
    for _ in range(a.reps):
        fn(x, y)
torch.cuda.synchronize()
print("done", a.bench, a.p, nx, ny, nz, m.n_local)
