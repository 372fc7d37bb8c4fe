"""Profiling driver: a few fused applies of one operator (for ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_15940_b200 as hf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bench", default="bp3")
ap.add_argument("--p", type=int, default=5)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--unfused", action="store_true")
a = ap.parse_args()
kind = hf.MASS if a.bench == "bp1" else hf.DIFFUSION
rule = hf.GLL if a.bench == "bp5" else hf.GAUSS
n = a.n or int(round((99.0 if a.bench == "bp1" else 311.0) / a.p))
m = hf.Mesh(n, n, n, a.p)
op = hf.Operator(m, kind=kind, rule=rule, bc=hf.BC_DIRICHLET if a.bench != "bp1" else hf.BC_NONE)
x = m.random(1)
y = torch.empty_like(x)
for _ in range(a.reps):
    (op.apply_unfused if a.unfused else op.apply)(x, y)
torch.cuda.synchronize()
print("done", a.bench, a.p, n, m.n_local)
