"""Fast kernel-tuning variant: recompile only one per-P1 unit (fused_p.cu, or
dg_p.cu with --src dg_p) for one P1 with extra -D flags and relink against the
in-tree objects (run the normal build first).

    python scripts/build_pvariant.py [--src dg_p] NAME P1 -DFLAG=... [...]
        ->  scratch/libhofem_NAME.so   (load it with HOFEM_LIB_PATH=...)
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_15940_b200 import build as B  # noqa: E402

args = sys.argv[1:]
unit = "fused_p"
if args and args[0] == "--src":
    unit, args = args[1], args[2:]
name, p1, flags = args[0], int(args[1]), args[2:]
B.build()
os.makedirs("scratch/obj", exist_ok=True)
src = os.path.join(B.CSRC, f"{unit}.cu")
per_p1 = unit.endswith("_p")  # per-P1 units get -DHOFEM_P1; host units (e.g. fused) do not
obj = os.path.abspath(f"scratch/obj/{unit}{p1 if per_p1 else ''}_{name}.o")
cmd = [B.NVCC] + B._common_flags() + ([f"-DHOFEM_P1={p1}"] if per_p1 else []) + flags + [
    "-c", src, "-o", obj]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
target = f"{unit}{p1}.o" if per_p1 else f"{unit}.o"
objs = [obj if os.path.basename(j[1]) == target else j[1] for j in B._jobs()]
nccl = B._nccl_dir()
out = os.path.abspath(f"scratch/libhofem_{name}.so")
cmd = [B.NVCC] + B.ARCH + ["-shared", "-o", out] + objs + [
    f"-L{nccl}", "-l:libnccl.so.2", "-Xlinker", f"-rpath={nccl}", "-lcudart"]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
print(name, p1, flags)
