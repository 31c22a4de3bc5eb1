"""The C ABI used from plain C (examples/abi_demo.c): compiled with gcc against
include/ddqd.h and libddqd.so, no Python in the compute path."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_uses_the_abi(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = tmp_path / "abi_demo"
    subprocess.check_call([
        "gcc", "-std=c11", "-O2", "-ffp-contract=off", os.path.join(ROOT, "examples", "abi_demo.c"),
        "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include",
        "-L" + os.path.join(ROOT, "paper_1510_08642_b200"), "-lddqd", "-L/usr/local/cuda/lib64", "-lcudart", "-lm",
        "-Wl,-rpath," + os.path.join(ROOT, "paper_1510_08642_b200"), "-o", str(exe)])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 mismatching entries" in r.stdout
    assert "negative size -> -1" in r.stdout
