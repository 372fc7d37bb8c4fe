"""A/B timing of the CG schedules (hofem_op_set_option): persistent whole-solve
kernel vs per-iteration kernels (fused cooperative update / separate kernels).

    python scripts/cg_modes.py [--bench bp1] [--ps 1,2,...] [--iters 100]

Prints one JSON line per (bench, p, size, mode): G[DOF*it]/s of a fixed-iteration
solve timed with CUDA events (median of 3)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2402_15940_b200 as hf  # noqa: E402

MODES = {
    "persistent": {hf.OPT_CG_PERSISTENT: 2},
    "fused": {hf.OPT_CG_PERSISTENT: 0, hf.OPT_CG_FUSED_UPDATE: 2, hf.OPT_INFIX: 2},
    "separate": {hf.OPT_CG_PERSISTENT: 0, hf.OPT_CG_FUSED_UPDATE: 0, hf.OPT_INFIX: 0},
    "infix_only": {hf.OPT_CG_PERSISTENT: 0, hf.OPT_CG_FUSED_UPDATE: 0, hf.OPT_INFIX: 2},
    "upd_only": {hf.OPT_CG_PERSISTENT: 0, hf.OPT_CG_FUSED_UPDATE: 2, hf.OPT_INFIX: 0},
    "auto": {hf.OPT_CG_PERSISTENT: 1, hf.OPT_CG_FUSED_UPDATE: 1, hf.OPT_INFIX: 1},
}


def time_cg(op, b, iters):
    x = torch.zeros_like(b)
    op.cg(b, x, max_iter=3, fixed_iters=True)
    ts = []
    for _ in range(3):
        x.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.cg(b, x, max_iter=iters, fixed_iters=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return sorted(ts)[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bench", default="bp1")
    ap.add_argument("--ps", default="1,2,3,4,5,6,7,8")
    ap.add_argument("--ns", default="", help="elements per axis (default: the config-2/3 size)")
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--modes", default="persistent,fused,separate")
    ap.add_argument("--slab", default="", help="nx,ny,nz (one mesh; overrides --ns)")
    a = ap.parse_args()
    kind = hf.MASS if a.bench == "bp1" else hf.DIFFUSION
    rule = hf.GLL if a.bench == "bp5" else hf.GAUSS
    bc = hf.BC_NONE if a.bench == "bp1" else hf.BC_DIRICHLET
    for p in [int(v) for v in a.ps.split(",")]:
        ns = [int(v) for v in a.ns.split(",")] if a.ns else \
            [int(round((99.0 if a.bench == "bp1" else 311.0) / p))]
        dims = [tuple(int(v) for v in a.slab.split(","))] if a.slab else [(n, n, n) for n in ns]
        for dd in dims:
            n = dd[0]
            m = hf.Mesh(*dd, p, alpha=0.1)
            op = hf.Operator(m, kind=kind, rule=rule, bc=bc)
            b = op.rhs()
            for mode in a.modes.split(","):
                for k, v in MODES[mode].items():
                    op.set_option(k, v)
                t = time_cg(op, b, a.iters)
                print(json.dumps({"bench": a.bench, "p": p, "n": n, "dofs": m.n_local,
                                  "mode": mode, "us_per_it": 1e6 * t / a.iters,
                                  "gdof_it_s": m.n_local * a.iters / t / 1e9}), flush=True)
            op.close()
            m.close()
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
