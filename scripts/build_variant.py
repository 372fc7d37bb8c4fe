"""Build libhofem.so with extra -D flags into scratch/ (kernel tuning experiments)."""
import shutil
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_15940_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
orig = B._common_flags
B._common_flags = lambda: orig() + flags
B.build(force=True)
os.makedirs("scratch", exist_ok=True)
shutil.copy(B.LIB, f"scratch/libhofem_{name}.so")
print(name, flags)
