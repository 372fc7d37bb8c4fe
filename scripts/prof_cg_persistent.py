"""One persistent-CG launch (BP3, fixed iterations) for ncu.
usage: python scripts/prof_cg_persistent.py [--p 5] [--n 16] [--iters 20]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2402_15940_b200 as hf  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=5)
ap.add_argument("--n", type=int, default=16)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
m = hf.Mesh(a.n, a.n, a.n, a.p, alpha=0.1)
op = hf.Operator(m, kind=hf.DIFFUSION, rule=hf.GAUSS, bc=hf.BC_DIRICHLET)
op.set_option(hf.OPT_CG_PERSISTENT, hf.ALWAYS)
b = op.rhs()
x = torch.zeros_like(b)
op.cg(b, x, max_iter=a.iters, fixed_iters=True)
torch.cuda.synchronize()
