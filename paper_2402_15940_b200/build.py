"""Build libhofem.so in-tree (nvcc, sm_100a only).

    python -m paper_2402_15940_b200.build [--force] [--verbose]

Every .cu is compiled with ``-gencode arch=compute_100a,code=sm_100a -lineinfo``;
``fused_p.cu`` is compiled once per P1 = p+1 in 2..9 (-DHOFEM_P1) so the
template-heavy fused kernels build in parallel.  NCCL is the torch-bundled
libnccl.so.2 (found via the nvidia.nccl package), linked with an rpath.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libhofem.so")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
P1S = list(range(2, 10))


def _nccl_dir() -> str | None:
    try:
        import nvidia.nccl  # type: ignore
        for d in nvidia.nccl.__path__:
            lib = os.path.join(d, "lib")
            if os.path.exists(os.path.join(lib, "libnccl.so.2")):
                return lib
    except Exception:
        pass
    for d in ("/usr/lib/x86_64-linux-gnu",):
        if os.path.exists(os.path.join(d, "libnccl.so.2")):
            return d
    return None


def _common_flags():
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE,
                   "-I", CSRC, "--expt-relaxed-constexpr"]


def _jobs():
    jobs = []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        name = os.path.splitext(os.path.basename(src))[0]
        if name.endswith("_p"):  # per-P1 instantiation units (fused_p.cu, dg_p.cu)
            for p1 in P1S:
                jobs.append((src, os.path.join(BUILD, f"{name}{p1}.o"), [f"-DHOFEM_P1={p1}"]))
        else:
            jobs.append((src, os.path.join(BUILD, f"{name}.o"), []))
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cpp"))):
        name = os.path.splitext(os.path.basename(src))[0]
        jobs.append((src, os.path.join(BUILD, f"{name}_cpp.o"), []))
    return jobs


def _deps_mtime():
    files = glob.glob(os.path.join(CSRC, "*")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    return max(os.path.getmtime(f) for f in files)


def _compile(job, verbose):
    src, obj, extra = job
    cmd = [NVCC] + _common_flags() + extra + ["-c", src, "-o", obj]
    if verbose and "_p" in os.path.basename(obj):
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src} {extra}:\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps_mtime():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    jobs = _jobs()
    logs = []
    with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
        for obj, log in ex.map(lambda j: _compile(j, verbose), jobs):
            if log.strip():
                logs.append(f"== {os.path.basename(obj)}\n{log}")
    nccl = _nccl_dir()
    if nccl is None:
        raise RuntimeError("libnccl.so.2 not found")
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + [j[1] for j in jobs] + [
        f"-L{nccl}", "-l:libnccl.so.2", "-Xlinker", f"-rpath={nccl}", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
    sys.exit(0)
