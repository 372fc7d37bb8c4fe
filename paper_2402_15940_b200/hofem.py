"""Thin Python binding of the C ABI in ``include/hofem.h`` (ctypes).

Argument marshalling only: every step of the hot path runs in libhofem.so's
CUDA kernels.  Vectors are torch.float64 CUDA tensors (device memory and
streams come from PyTorch); their ``data_ptr()`` is passed straight through.
There is no CPU fallback: if the library or a CUDA device is missing, every
call raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# HOFEM_LIB_PATH: load a tuning build (scripts/build_pvariant.py) instead of the
# in-tree library; the default is the in-tree libhofem.so.
LIB_PATH = os.environ.get("HOFEM_LIB_PATH") or os.path.join(_PKG, "libhofem.so")

MASS, DIFFUSION = 1, 2
GAUSS, GLL = 1, 2
BC_NONE, BC_DIRICHLET = 0, 1

# hofem_option
OPT_INFIX, OPT_CG_FUSED_UPDATE, OPT_CG_PERSISTENT, OPT_L2_PREFETCH = 1, 2, 3, 4
NEVER, AUTO, ALWAYS = 0, 1, 2

OK, ERR_ARG, ERR_MESH, ERR_CUDA, ERR_NCCL, ERR_OOM, ERR_BREAKDOWN, NOT_CONVERGED = range(8)
_NAMES = ["OK", "ERR_ARG", "ERR_MESH", "ERR_CUDA", "ERR_NCCL", "ERR_OOM", "ERR_BREAKDOWN",
          "NOT_CONVERGED"]


class HofemError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_NAMES[status] if 0 <= status < 8 else status}: {msg}")
        self.status = status


class MeshDesc(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz_global", ctypes.c_int),
                ("p", ctypes.c_int), ("extent", ctypes.c_double * 3), ("alpha", ctypes.c_double)]


class MeshInfo(ctypes.Structure):
    _fields_ = [("n_local", ctypes.c_longlong), ("n_owned", ctypes.c_longlong),
                ("n_global", ctypes.c_longlong), ("elems_local", ctypes.c_longlong),
                ("plane", ctypes.c_longlong), ("rank", ctypes.c_int), ("nranks", ctypes.c_int),
                ("z0", ctypes.c_int), ("nz_local", ctypes.c_int)]


class ProfileStats(ctypes.Structure):
    _fields_ = [("brick_launches", ctypes.c_longlong), ("brick_ms", ctypes.c_double),
                ("fixup_launches", ctypes.c_longlong), ("fixup_ms", ctypes.c_double)]


class FusedInfo(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int), ("bx", ctypes.c_int), ("by", ctypes.c_int),
                ("zc", ctypes.c_int), ("nchunks", ctypes.c_int), ("grid", ctypes.c_int),
                ("direct_points", ctypes.c_longlong), ("fixup_points", ctypes.c_longlong)]


class DGInfo(ctypes.Structure):
    _fields_ = [("n_local", ctypes.c_longlong), ("n_global", ctypes.c_longlong),
                ("elems_local", ctypes.c_longlong), ("p", ctypes.c_int), ("Q", ctypes.c_int),
                ("dofs_per_elem", ctypes.c_int), ("grid", ctypes.c_int)]


class PMGInfo(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int), ("orders", ctypes.c_int * 8),
                ("lambda_", ctypes.c_double * 8), ("degree", ctypes.c_int)]


class CGStats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("converged", ctypes.c_int),
                ("r0_norm", ctypes.c_double), ("final_rel_res", ctypes.c_double)]


# name -> (restype, argtypes); the names are exactly those of include/hofem.h
_V, _I, _LL, _D = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_double
_PV = ctypes.POINTER(ctypes.c_void_p)
SIGNATURES = {
    "hofem_last_error": (ctypes.c_char_p, []),
    "hofem_comm_unique_id": (_I, [_V]),
    "hofem_comm_init": (_I, [_V, _I, _I, _I, _PV]),
    "hofem_comm_destroy": (None, [_V]),
    "hofem_loopback_group_create": (_I, [_I, _PV]),
    "hofem_comm_init_loopback": (_I, [_V, _I, _PV]),
    "hofem_loopback_group_destroy": (None, [_V]),
    "hofem_mesh_create": (_I, [ctypes.POINTER(MeshDesc), _V, _V, _PV]),
    "hofem_mesh_info_get": (_I, [_V, ctypes.POINTER(MeshInfo)]),
    "hofem_mesh_coords": (_I, [_V, _V, _V]),
    "hofem_mesh_destroy": (None, [_V]),
    "hofem_mesh_set_exchange": (_I, [_V, _I, _V]),
    "hofem_op_create": (_I, [_V, _I, _I, _I, _I, _V, _PV]),
    "hofem_op_apply": (_I, [_V, _V, _V, _V]),
    "hofem_op_apply_unfused": (_I, [_V, _V, _V, _V]),
    "hofem_op_apply_mf": (_I, [_V, _V, _V, _V]),
    "hofem_op_qdata": (_I, [_V, ctypes.POINTER(_V), ctypes.POINTER(_LL)]),
    "hofem_op_nq1d": (_I, [_V, ctypes.POINTER(_I)]),
    "hofem_rhs_manufactured": (_I, [_V, _V, _V]),
    "hofem_fill_random": (_I, [_V, ctypes.c_ulonglong, _V, _V]),
    "hofem_op_destroy": (None, [_V]),
    "hofem_dg_create": (_I, [_V, _I, _V, _PV]),
    "hofem_dg_info_get": (_I, [_V, ctypes.POINTER(DGInfo)]),
    "hofem_dg_apply": (_I, [_V, _V, _V, _V]),
    "hofem_dg_fill_random": (_I, [_V, ctypes.c_ulonglong, _V, _V]),
    "hofem_dg_destroy": (None, [_V]),
    "hofem_op_diagonal": (_I, [_V, _V, _V]),
    "hofem_pmg_create": (_I, [_V, _I, _I, ctypes.c_ulonglong, _V, _PV]),
    "hofem_pmg_info_get": (_I, [_V, ctypes.POINTER(PMGInfo)]),
    "hofem_pmg_set_lambda": (_I, [_V, _I, _D]),
    "hofem_pmg_level": (_I, [_V, _I, _PV, _PV]),
    "hofem_pmg_vcycle": (_I, [_V, _V, _V, _V]),
    "hofem_pmg_smooth": (_I, [_V, _I, _V, _V, _V]),
    "hofem_pmg_transfer": (_I, [_V, _I, _I, _V, _V, _V]),
    "hofem_pmg_pcg": (_I, [_V, _V, _V, _D, _I, _V, ctypes.POINTER(CGStats), _V]),
    "hofem_pmg_destroy": (None, [_V]),
    "hofem_cg": (_I, [_V, _V, _V, _D, _I, _I, _I, _V, ctypes.POINTER(CGStats), _V]),
    "hofem_dot": (_I, [_V, _V, _V, ctypes.POINTER(_D), _V]),
    "hofem_op_apply_dot": (_I, [_V, _V, _V, ctypes.POINTER(_D), _V]),
    "hofem_op_fused_info": (_I, [_V, ctypes.POINTER(FusedInfo)]),
    "hofem_op_set_option": (_I, [_V, _I, _I]),
    "hofem_op_get_option": (_I, [_V, _I, ctypes.POINTER(_I)]),
    "hofem_profile_enable": (_I, [_I]),
    "hofem_profile_read": (_I, [ctypes.POINTER(ProfileStats)]),
    "hofem_launch_count": (_LL, []),
    "hofem_launch_count_reset": (None, []),
}

_lib = None


def lib():
    """Load libhofem.so (built by paper_2402_15940_b200.build).  Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run python -m paper_2402_15940_b200.build "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _check(st: int):
    if st != OK:
        raise HofemError(st, lib().hofem_last_error().decode())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor, n: int | None = None):
    """Device pointer of a vector argument, after the checks the C ABI relies on:
    contiguous float64 on the current CUDA device, n elements (when given) and
    16-byte aligned (hofem.h conventions).  Raises ValueError otherwise."""
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError("expected a contiguous torch.float64 CUDA tensor")
    if t.device.index != torch.cuda.current_device():
        raise ValueError(f"tensor on {t.device}, library calls run on cuda:{torch.cuda.current_device()}")
    if n is not None and t.numel() != n:
        raise ValueError(f"expected {n} elements, got {t.numel()}")
    if t.data_ptr() % 16:
        raise ValueError("tensor data must be 16-byte aligned (e.g. not a view at an odd offset)")
    return ctypes.c_void_p(t.data_ptr())


def _cudart():
    import glob
    import nvidia.cuda_runtime  # type: ignore
    for d in nvidia.cuda_runtime.__path__:
        for f in glob.glob(os.path.join(d, "lib", "libcudart.so*")):
            return ctypes.CDLL(f)
    return ctypes.CDLL("libcudart.so.12")


def copy_device_to_tensor(dev_ptr: int, n: int, device=None) -> torch.Tensor:
    """Copy n FP64 values from a library-owned device pointer into a new tensor."""
    out = torch.empty(n, dtype=torch.float64, device=device or "cuda")
    rt = _cudart()
    rt.cudaMemcpyAsync.argtypes = [_V, _V, ctypes.c_size_t, _I, _V]
    st = rt.cudaMemcpyAsync(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(dev_ptr), n * 8, 3,
                            _stream())
    if st != 0:
        raise RuntimeError(f"cudaMemcpyAsync failed: {st}")
    return out


class LoopbackGroup:
    """In-process loopback transport: nranks ranks as threads on one GPU
    (hofem_loopback_group_create); see Comm.loopback."""

    def __init__(self, nranks: int):
        h = ctypes.c_void_p()
        _check(lib().hofem_loopback_group_create(nranks, ctypes.byref(h)))
        self.handle = h
        self.nranks = nranks

    def close(self):
        if self.handle:
            lib().hofem_loopback_group_destroy(self.handle)
            self.handle = None


class Comm:
    """NCCL communicator for the z-slab partition (one process per GPU), or the
    in-process loopback transport (Comm.loopback)."""

    def __init__(self, rank: int, nranks: int, device: int, nccl_id: bytes, _handle=None):
        if _handle is not None:
            self.handle = _handle
            return
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(nccl_id, 128)
        _check(lib().hofem_comm_init(buf, rank, nranks, device, ctypes.byref(h)))
        self.handle = h

    @classmethod
    def loopback(cls, group: "LoopbackGroup", rank: int) -> "Comm":
        h = ctypes.c_void_p()
        _check(lib().hofem_comm_init_loopback(group.handle, rank, ctypes.byref(h)))
        return cls(rank, group.nranks, 0, b"", _handle=h)

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(lib().hofem_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def from_torch_distributed(cls):
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(rank, world, torch.cuda.current_device(), obj[0])

    def close(self):
        if self.handle:
            lib().hofem_comm_destroy(self.handle)
            self.handle = None


class Mesh:
    def __init__(self, nx, ny, nz, p, alpha=0.1, extent=(1.0, 1.0, 1.0), comm: Comm | None = None,
                 stream=None):
        d = MeshDesc(nx, ny, nz, p, (ctypes.c_double * 3)(*extent), alpha)
        h = ctypes.c_void_p()
        _check(lib().hofem_mesh_create(ctypes.byref(d), comm.handle if comm else None,
                                       _stream(stream), ctypes.byref(h)))
        self.handle = h
        self.p = p
        info = MeshInfo()
        _check(lib().hofem_mesh_info_get(h, ctypes.byref(info)))
        self.info = info
        self.n_local = info.n_local
        self.n_owned = info.n_owned
        self.n_global = info.n_global
        self.dims = (p * nx + 1, p * ny + 1, p * info.nz_local + 1)

    def coords(self, stream=None) -> torch.Tensor:
        out = torch.empty(3 * self.n_local, dtype=torch.float64, device="cuda")
        _check(lib().hofem_mesh_coords(self.handle, _ptr(out, 3 * self.n_local), _stream(stream)))
        return out.view(3, self.n_local)

    def random(self, seed: int, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        out = torch.empty(self.n_local, dtype=torch.float64, device="cuda") if out is None else out
        _check(lib().hofem_fill_random(self.handle, ctypes.c_ulonglong(seed), _ptr(out, self.n_local),
                                       _stream(stream)))
        return out

    def set_exchange(self, mode: int, stream=None):
        """Interface exchange: 0 collective (NCCL / loopback copies), 1 kernel-
        initiated peer puts (collective call)."""
        _check(lib().hofem_mesh_set_exchange(self.handle, int(mode), _stream(stream)))

    def dot(self, a: torch.Tensor, b: torch.Tensor, stream=None) -> float:
        v = ctypes.c_double()
        _check(lib().hofem_dot(self.handle, _ptr(a, self.n_local), _ptr(b, self.n_local),
                               ctypes.byref(v), _stream(stream)))
        return v.value

    def close(self):
        if self.handle:
            lib().hofem_mesh_destroy(self.handle)
            self.handle = None


class Operator:
    def __init__(self, mesh: Mesh, kind=DIFFUSION, rule=GAUSS, q_override=0, bc=BC_NONE,
                 stream=None):
        h = ctypes.c_void_p()
        _check(lib().hofem_op_create(mesh.handle, kind, rule, q_override, bc, _stream(stream),
                                     ctypes.byref(h)))
        self.handle = h
        self.mesh = mesh
        q = ctypes.c_int()
        _check(lib().hofem_op_nq1d(h, ctypes.byref(q)))
        self.Q = q.value
        self.kind, self.rule, self.bc = kind, rule, bc

    def apply(self, x: torch.Tensor, y: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        y = torch.empty_like(x) if y is None else y
        n = self.mesh.n_local
        _check(lib().hofem_op_apply(self.handle, _ptr(x, n), _ptr(y, n), _stream(stream)))
        return y

    def fused_info(self) -> FusedInfo:
        """How apply() runs: fused kernel variant (1 SIMT brick kernel, -1
        unfused), brick shape, chunking, direct vs fix-up lattice points."""
        s = FusedInfo()
        _check(lib().hofem_op_fused_info(self.handle, ctypes.byref(s)))
        return s

    def set_option(self, opt: int, value: int):
        """hofem_op_set_option: OPT_* schedule option, value NEVER/AUTO/ALWAYS."""
        _check(lib().hofem_op_set_option(self.handle, int(opt), int(value)))

    def get_option(self, opt: int) -> int:
        v = ctypes.c_int()
        _check(lib().hofem_op_get_option(self.handle, int(opt), ctypes.byref(v)))
        return v.value

    def apply_dot(self, x: torch.Tensor, y: torch.Tensor | None = None, stream=None):
        """y = A x and x.y over owned dofs (fused into the operator kernels)."""
        y = torch.empty_like(x) if y is None else y
        v = ctypes.c_double()
        n = self.mesh.n_local
        _check(lib().hofem_op_apply_dot(self.handle, _ptr(x, n), _ptr(y, n), ctypes.byref(v),
                                        _stream(stream)))
        return y, v.value

    def apply_unfused(self, x: torch.Tensor, y: torch.Tensor | None = None, stream=None):
        y = torch.empty_like(x) if y is None else y
        n = self.mesh.n_local
        _check(lib().hofem_op_apply_unfused(self.handle, _ptr(x, n), _ptr(y, n), _stream(stream)))
        return y

    def apply_mf(self, x: torch.Tensor, y: torch.Tensor | None = None, stream=None):
        """Fully matrix-free apply (geometry recomputed from the nodal coordinates)."""
        y = torch.empty_like(x) if y is None else y
        n = self.mesh.n_local
        _check(lib().hofem_op_apply_mf(self.handle, _ptr(x, n), _ptr(y, n), _stream(stream)))
        return y

    def qdata(self) -> torch.Tensor:
        p, n = ctypes.c_void_p(), ctypes.c_longlong()
        _check(lib().hofem_op_qdata(self.handle, ctypes.byref(p), ctypes.byref(n)))
        return copy_device_to_tensor(p.value, n.value)

    def rhs(self, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        out = torch.empty(self.mesh.n_local, dtype=torch.float64, device="cuda") if out is None else out
        _check(lib().hofem_rhs_manufactured(self.handle, _ptr(out, self.mesh.n_local),
                                            _stream(stream)))
        return out

    def cg(self, b: torch.Tensor, x: torch.Tensor, rel_tol=1e-10, max_iter=1000,
           fixed_iters=False, check_every=1, history=False, stream=None):
        """Returns (status, stats, rr_history or None).  x is updated in place."""
        stats = CGStats()
        hist = (ctypes.c_double * (max_iter + 1))() if history else None
        n = self.mesh.n_local
        st = lib().hofem_cg(self.handle, _ptr(b, n), _ptr(x, n), rel_tol, max_iter, int(fixed_iters),
                            check_every, hist, ctypes.byref(stats), _stream(stream))
        if st not in (OK, NOT_CONVERGED):
            _check(st)
        rr = list(hist[: stats.iterations + 1]) if history else None
        return st, stats, rr

    def diagonal(self, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """diag(A) by sum factorization (hofem_op_diagonal); Dirichlet rows 1."""
        out = torch.empty(self.mesh.n_local, dtype=torch.float64, device="cuda") if out is None else out
        _check(lib().hofem_op_diagonal(self.handle, _ptr(out, self.mesh.n_local), _stream(stream)))
        return out

    def close(self):
        if self.handle:
            lib().hofem_op_destroy(self.handle)
            self.handle = None


class _Borrowed:
    """A level's mesh / operator owned by a PMG handle (never destroyed here)."""


class PMG:
    """p-multigrid V-cycle and preconditioned CG on a fine BP3 mesh (hofem_pmg_*;
    §8(f) f2).  Level 0 is the finest; level k vectors have levels[k].n_local."""

    def __init__(self, mesh: Mesh, degree=3, power_iters=10, seed=1, stream=None):
        h = ctypes.c_void_p()
        _check(lib().hofem_pmg_create(mesh.handle, degree, power_iters, ctypes.c_ulonglong(seed),
                                      _stream(stream), ctypes.byref(h)))
        self.handle = h
        self.mesh = mesh
        info = self.info()
        self.orders = list(info.orders[: info.levels])
        self.levels = []
        for k in range(info.levels):
            mh, oh = ctypes.c_void_p(), ctypes.c_void_p()
            _check(lib().hofem_pmg_level(h, k, ctypes.byref(mh), ctypes.byref(oh)))
            mi = MeshInfo()
            _check(lib().hofem_mesh_info_get(mh, ctypes.byref(mi)))
            lv = _Borrowed()
            lv.mesh_handle, lv.op_handle, lv.n_local, lv.p = mh, oh, mi.n_local, self.orders[k]
            self.levels.append(lv)

    def info(self) -> PMGInfo:
        s = PMGInfo()
        _check(lib().hofem_pmg_info_get(self.handle, ctypes.byref(s)))
        return s

    def lambdas(self):
        i = self.info()
        return list(i.lambda_[: i.levels])

    def set_lambda(self, level: int, lam: float):
        _check(lib().hofem_pmg_set_lambda(self.handle, level, float(lam)))

    def vec(self, level: int) -> torch.Tensor:
        return torch.zeros(self.levels[level].n_local, dtype=torch.float64, device="cuda")

    def apply(self, level: int, x: torch.Tensor, y: torch.Tensor | None = None, stream=None):
        y = torch.empty_like(x) if y is None else y
        n = self.levels[level].n_local
        _check(lib().hofem_op_apply(self.levels[level].op_handle, _ptr(x, n), _ptr(y, n),
                                    _stream(stream)))
        return y

    def vcycle(self, r: torch.Tensor, z: torch.Tensor | None = None, stream=None):
        z = torch.empty_like(r) if z is None else z
        n = self.levels[0].n_local
        _check(lib().hofem_pmg_vcycle(self.handle, _ptr(r, n), _ptr(z, n), _stream(stream)))
        return z

    def smooth(self, level: int, b: torch.Tensor, x: torch.Tensor, stream=None):
        n = self.levels[level].n_local
        _check(lib().hofem_pmg_smooth(self.handle, level, _ptr(b, n), _ptr(x, n), _stream(stream)))
        return x

    def prolong_add(self, level: int, xc: torch.Tensor, xf: torch.Tensor, stream=None):
        _check(lib().hofem_pmg_transfer(self.handle, level, 0, _ptr(xc, self.levels[level + 1].n_local),
                                        _ptr(xf, self.levels[level].n_local), _stream(stream)))
        return xf

    def restrict(self, level: int, rf: torch.Tensor, rc: torch.Tensor | None = None, stream=None):
        rc = self.vec(level + 1) if rc is None else rc
        _check(lib().hofem_pmg_transfer(self.handle, level, 1, _ptr(rf, self.levels[level].n_local),
                                        _ptr(rc, self.levels[level + 1].n_local), _stream(stream)))
        return rc

    def pcg(self, b: torch.Tensor, x: torch.Tensor, rel_tol=1e-10, max_iter=500, history=False,
            stream=None):
        stats = CGStats()
        hist = (ctypes.c_double * (max_iter + 1))() if history else None
        n = self.levels[0].n_local
        st = lib().hofem_pmg_pcg(self.handle, _ptr(b, n), _ptr(x, n), rel_tol, max_iter, hist,
                                 ctypes.byref(stats), _stream(stream))
        if st not in (OK, NOT_CONVERGED):
            _check(st)
        rr = list(hist[: stats.iterations + 1]) if history else None
        return st, stats, rr

    def close(self):
        if self.handle:
            lib().hofem_pmg_destroy(self.handle)
            self.handle = None


class DGMass:
    """Matrix-free DG (L2) mass operator on a Mesh (hofem_dg_*; §8(f) f4).
    Vectors are element-major E-vectors of n_local doubles."""

    def __init__(self, mesh: Mesh, q_override=0, stream=None):
        h = ctypes.c_void_p()
        _check(lib().hofem_dg_create(mesh.handle, q_override, _stream(stream), ctypes.byref(h)))
        self.handle = h
        self.mesh = mesh
        self.info = self.get_info()
        self.n_local = self.info.n_local

    def get_info(self) -> DGInfo:
        s = DGInfo()
        _check(lib().hofem_dg_info_get(self.handle, ctypes.byref(s)))
        return s

    def random(self, seed: int, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        out = torch.empty(self.n_local, dtype=torch.float64, device="cuda") if out is None else out
        _check(lib().hofem_dg_fill_random(self.handle, ctypes.c_ulonglong(seed),
                                          _ptr(out, self.n_local), _stream(stream)))
        return out

    def apply(self, x: torch.Tensor, y: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        y = torch.empty_like(x) if y is None else y
        _check(lib().hofem_dg_apply(self.handle, _ptr(x, self.n_local), _ptr(y, self.n_local),
                                    _stream(stream)))
        return y

    def close(self):
        if self.handle:
            lib().hofem_dg_destroy(self.handle)
            self.handle = None


def profile_enable(on: bool = True):
    _check(lib().hofem_profile_enable(int(on)))


def profile_read() -> ProfileStats:
    s = ProfileStats()
    _check(lib().hofem_profile_read(ctypes.byref(s)))
    return s


def launch_count() -> int:
    return lib().hofem_launch_count()


def launch_count_reset():
    lib().hofem_launch_count_reset()
