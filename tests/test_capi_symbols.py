"""CPU-side checks of the C-ABI boundary: the library builds, loads without a
GPU, exports every entry point include/hofem.h declares, and the Python
binding uses exactly those names.  No compute calls (no GPU here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hofem.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hofem_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2402_15940_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["hofem_mesh_create", "hofem_op_create", "hofem_op_apply", "hofem_op_apply_unfused",
                 "hofem_cg", "hofem_dot", "hofem_comm_init", "hofem_fill_random",
                 "hofem_rhs_manufactured", "hofem_op_qdata", "hofem_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath], text=True)
    exported = set(re.findall(r" T (hofem_[a-z0-9_]+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_library_loads_and_binding_matches_header(libpath):
    from paper_2402_15940_b200 import hofem
    L = hofem.lib()
    for name in declared_functions():
        assert hasattr(L, name)
    assert set(hofem.SIGNATURES) == set(declared_functions())
    assert isinstance(L.hofem_last_error(), bytes)


def test_sm100a_code_only(libpath):
    """The fused kernels are compiled for sm_100a (cuobjdump lists the arch)."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath],
                         capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_no_oracle_in_product():
    """The product package never imports, links or reads oracle/."""
    pkg = os.path.join(ROOT, "paper_2402_15940_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "oracle.c" not in txt and "liboracle" not in txt, f
