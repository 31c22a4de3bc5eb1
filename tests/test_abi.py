"""The C-ABI library loads and exports every function include/ddqd.h declares (CPU only:
no compute calls without a GPU)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "ddqd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s*([A-Za-z_][A-Za-z0-9_]*)\s*\(",
                       src, flags=re.M)
    return sorted(set(n for n in names if n not in ("if", "while")))


def test_header_declares_the_boundary():
    names = declared_functions()
    for f in ("dd_gemm", "qd_gemm", "dd_lu_solve", "ddqd_gemm_ex", "ddqd_pre_add", "ddqd_post_add"):
        assert f in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1510_08642_b200", "libddqd.so"))
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_binding_names_match_header():
    import paper_1510_08642_b200 as ddqd
    assert set(ddqd.EXPORTED) <= set(declared_functions())
    assert ddqd.lib.ddqd_version() == 100
    assert ddqd.lib.ddqd_last_error() == b""


def test_sm100a_code_in_library():
    """The library carries sm_100a SASS (cuobjdump lists the arch)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          os.path.join(ROOT, "paper_1510_08642_b200", "libddqd.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_in_product_path():
    """The product package never imports the oracle (test infrastructure only)."""
    pkg = os.path.join(ROOT, "paper_1510_08642_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            txt = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in txt and "from oracle" not in txt, fn
