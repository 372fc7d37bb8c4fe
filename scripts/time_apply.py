"""Time the fused apply (brick kernel via the library's event hooks) for one op."""
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
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--tag", default="")
ap.add_argument("--slab", default="", help="nx,ny,nz instead of --n")
ap.add_argument("--opt", action="append", default=[], help="OPTION=VALUE (hofem_op_set_option)")
a = ap.parse_args()
kind = hf.MASS if a.bench == "bp1" else hf.DIFFUSION
rule = hf.GLL if a.bench == "bp5" else hf.GAUSS
n = a.n or int(round((99.0 if a.bench == "bp1" else 311.0) / a.p))
nx = ny = nz = n
if a.slab:
    nx, ny, nz = (int(v) for v in a.slab.split(","))
m = hf.Mesh(nx, ny, nz, a.p)
op = hf.Operator(m, kind=kind, rule=rule, bc=hf.BC_DIRICHLET if a.bench != "bp1" else hf.BC_NONE)
for kv in a.opt:
    k, v = kv.split("=")
    op.set_option(getattr(hf, "OPT_" + k), int(v))
x = m.random(1)
y = torch.empty_like(x)
for _ in range(3):
    op.apply(x, y)
torch.cuda.synchronize()
hf.profile_enable(True)
for _ in range(a.reps):
    op.apply(x, y)
s = hf.profile_read()
hf.profile_enable(False)
Q = op.Q
nc = 1 if kind == hf.MASS else 6
bytes_ = 16 * m.n_local + 8 * nc * nx * ny * nz * Q ** 3
t = s.brick_ms / s.brick_launches
info = op.fused_info()
print(f"{a.tag:10s} {a.bench} p={a.p} mesh={nx}x{ny}x{nz} chunks={info.nchunks}x{info.zc} brick {t:.4f} ms fixup {s.fixup_ms / max(s.fixup_launches, 1):.4f} ms"
      f"  apply-alg {bytes_ / (t + s.fixup_ms / max(s.fixup_launches,1)) / 1e6:.0f} GB/s  {m.n_local / t / 1e6:.2f} GDOF/s(brick)")
