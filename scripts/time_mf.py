"""Fully matrix-free (f3) vs partial-assembly BP3 apply at ~30M dofs, p = 1..8:
ms per apply, GDOF/s; MF algorithmic bytes 8 (x) + 24 (coords) + 8 (y) B/DOF +
16 B per E-vector entry (write + scatter read)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2402_15940_b200 as hf  # noqa: E402
import workloads as W  # noqa: E402


def timed(fn, x, y, reps=20):
    for _ in range(3):
        fn(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn(x, y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


ps = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else range(1, 9)
for p in ps:
    n = W.bp3_sweep_n(p)
    m = hf.Mesh(n, n, n, p)
    op = hf.Operator(m, kind=hf.DIFFUSION, rule=hf.GAUSS, bc=hf.BC_DIRICHLET)
    x = m.random(1)
    y = torch.empty_like(x)
    t_mf = timed(op.apply_mf, x, y)
    t_pa = timed(op.apply, x, y)
    E = n ** 3
    print(json.dumps({"p": p, "n": n, "dofs": m.n_local, "mf_ms": 1e3 * t_mf, "pa_ms": 1e3 * t_pa,
                      "mf_gdof_s": m.n_local / t_mf / 1e9, "pa_gdof_s": m.n_local / t_pa / 1e9,
                      "mf_alg_gbs": (40.0 * m.n_local + 16.0 * E * (p + 1) ** 3) / t_mf / 1e9}),
          flush=True)
    op.close()
    m.close()
    torch.cuda.empty_cache()
