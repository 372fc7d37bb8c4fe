"""TEST INFRASTRUCTURE: a Python mirror of the host-side z-slab partition logic
(reading R9) for the gloo multi-rank tests on CPU; the product
path is csrc/comm.cu (exercised on the GPU by tests/test_gpu_loopback.py).

Mirrors what ``hofem_mesh_create`` (capi.cu) and ``exchange_planes`` (comm.cu)
do for the multi-GPU path, in plain Python over ``torch.distributed`` so the
N>1 logic can be exercised on CPU with the gloo backend (tests) and so bench.py
can size the weak-scaling problem.  No compute of the method happens here.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Slab:
    rank: int
    nranks: int
    z0: int          # first element layer of this rank
    nzl: int         # element layers on this rank
    Nx: int
    Ny: int
    Nzl: int         # local lattice planes = p*nzl + 1
    plane: int       # Nx*Ny
    n_local: int
    n_owned: int     # planes [0, Nzl-1) (+ the top plane on the last rank)
    K0: int          # global index of local plane 0


def slab(nx: int, ny: int, nz: int, p: int, rank: int, nranks: int) -> Slab:
    if nz % nranks:
        raise ValueError(f"nranks={nranks} must divide nz={nz}")
    nzl = nz // nranks
    z0 = rank * nzl
    Nx, Ny, Nzl = p * nx + 1, p * ny + 1, p * nzl + 1
    plane = Nx * Ny
    n_local = plane * Nzl
    n_owned = n_local if rank == nranks - 1 else n_local - plane
    return Slab(rank, nranks, z0, nzl, Nx, Ny, Nzl, plane, n_local, n_owned, p * z0)


def exchange_planes(s: Slab, y, send, recv, ess_fix=None):
    """Sum the duplicated interface planes of the local L-vector ``y`` (1D
    array-like supporting slicing and +=) with the neighbours: send the bottom
    plane to rank-1 and the top plane to rank+1, receive theirs, add.  ``send``
    and ``recv`` are callables (tensor, peer) -> None.  a+b == b+a in IEEE, so
    both copies end bitwise identical.  ``ess_fix(lo_or_hi, plane_view)``
    re-imposes Dirichlet rows afterwards (optional)."""
    P = s.plane
    lo = y[0:P].clone()
    hi = y[(s.Nzl - 1) * P: s.Nzl * P].clone()
    got_lo = got_hi = None
    # order sends/recvs to avoid deadlock with blocking point-to-point
    if s.rank % 2 == 0:
        if s.rank < s.nranks - 1:
            send(hi, s.rank + 1)
            got_hi = recv(hi.clone(), s.rank + 1)
        if s.rank > 0:
            send(lo, s.rank - 1)
            got_lo = recv(lo.clone(), s.rank - 1)
    else:
        if s.rank > 0:
            got_lo = recv(lo.clone(), s.rank - 1)
            send(lo, s.rank - 1)
        if s.rank < s.nranks - 1:
            got_hi = recv(hi.clone(), s.rank + 1)
            send(hi, s.rank + 1)
    if got_lo is not None:
        y[0:P] += got_lo
        if ess_fix:
            ess_fix("lo", y[0:P])
    if got_hi is not None:
        y[(s.Nzl - 1) * P: s.Nzl * P] += got_hi
        if ess_fix:
            ess_fix("hi", y[(s.Nzl - 1) * P: s.Nzl * P])
    return y
