"""Loopback multi-rank persistent CG (R = 2) with per-rank host timestamps."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2402_15940_b200 as hf
T0 = time.time()
def log(r, w): print(f"{time.time()-T0:8.3f} r{r} {w}", flush=True)
R, p, dims = 2, 3, (3, 2, 4)
group = hf.LoopbackGroup(R)
def worker(r):
    try:
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            comm = hf.Comm.loopback(group, r)
            m = hf.Mesh(*dims, p, alpha=0.1, comm=comm, stream=s)
            op = hf.Operator(m, kind=hf.DIFFUSION, rule=hf.GAUSS, bc=1, stream=s)
            op.set_option(hf.OPT_CG_PERSISTENT, hf.ALWAYS)
            x = torch.zeros(m.n_local, dtype=torch.float64, device="cuda")
            b = torch.empty_like(x)
            s.synchronize()
            m.set_exchange(1, stream=s)
            op.rhs(b, stream=s)
            log(r, "cg begin")
            st, stats, _ = op.cg(b, x, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 1,
                                 fixed_iters=True, stream=s)
            log(r, f"cg end {st} {stats.iterations}")
    except Exception as e:
        log(r, f"ERROR {e}")
th = [threading.Thread(target=worker, args=(r,)) for r in range(R)]
[t.start() for t in th]; [t.join() for t in th]
