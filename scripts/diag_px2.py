"""Loopback multi-rank persistent CG stress: R ranks, repeated solves + a host
apply, per-rank timestamps.  usage: python scripts/diag_px2.py R bench p nx ny nz"""
import os, sys, threading, time
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2402_15940_b200 as hf
hf.lib()
R, bench, p = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
dims = tuple(int(v) for v in sys.argv[4:7])
kind = hf.MASS if bench == "bp1" else hf.DIFFUSION
rule = hf.GLL if bench == "bp5" else hf.GAUSS
bc = 0 if bench == "bp1" else 1
T0 = time.time()
def log(r, w): print(f"{time.time()-T0:8.3f} r{r} {w}", flush=True)
group = hf.LoopbackGroup(R)
def worker(r):
    try:
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            comm = hf.Comm.loopback(group, r)
            m = hf.Mesh(*dims, p, alpha=0.1, comm=comm, stream=s)
            op = hf.Operator(m, kind=kind, rule=rule, bc=bc, stream=s)
            op.set_option(hf.OPT_CG_PERSISTENT, hf.ALWAYS)
            xs = [torch.zeros(m.n_local, dtype=torch.float64, device="cuda") for _ in range(6)]
            b = torch.empty_like(xs[0]); xa = m.random(5, stream=s); ya = torch.empty_like(xa)
            s.synchronize()
            m.set_exchange(1, stream=s)
            op.rhs(b, stream=s)
            for i, k in enumerate((1, 3, 9)):
                log(r, f"cg {k}")
                op.cg(b, xs[i], max_iter=k, fixed_iters=True, stream=s)
                s.synchronize()
            log(r, "cg conv")
            op.cg(b, xs[3], rel_tol=1e-13, max_iter=1000, stream=s)
            log(r, "apply")
            op.apply(xa, ya, stream=s)
            log(r, "cg again")
            op.cg(b, xs[4], max_iter=9, fixed_iters=True, stream=s)
            log(r, "done")
    except Exception as e:
        log(r, f"ERROR {e}")
th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(R)]
[t.start() for t in th]; [t.join(timeout=90) for t in th]
print("alive:", [t.is_alive() for t in th], flush=True)
os._exit(0)
