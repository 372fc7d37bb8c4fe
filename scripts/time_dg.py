"""DG (L2) mass apply throughput vs p at ~30M DG dofs (f4): GDOF/s and the
fraction of the measured HBM copy bandwidth for the algorithmic bytes
16 B/DOF (x, y) + 8 Q^3 B/element (W detJ)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2402_15940_b200 as hf  # noqa: E402
import workloads as W  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 7700.0
ps = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else range(1, 9)
for p in ps:
    n = W.dg_sweep_n(p)
    m = hf.Mesh(n, n, n, p)
    dg = hf.DGMass(m)
    x = dg.random(1)
    y = torch.empty_like(x)
    for _ in range(3):
        dg.apply(x, y)
    torch.cuda.synchronize()
    reps = 30
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        dg.apply(x, y)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    Q = p + 2
    E = n ** 3
    bts = 16.0 * dg.n_local + 8.0 * E * Q ** 3
    print(json.dumps({"p": p, "n": n, "dofs": dg.n_local, "ms": 1e3 * t,
                      "gdof_s": dg.n_local / t / 1e9, "alg_gbs": bts / t / 1e9,
                      "frac": bts / t / 1e9 / peak, "grid": dg.get_info().grid}), flush=True)
    dg.close()
    m.close()
    torch.cuda.empty_cache()
