import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a) and the built libddqd.so")
    config.addinivalue_line("markers", "slow: longer CPU oracle runs")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


def _ensure_native_built():
    """Build libddqd.so (nvcc cross-compiles for sm_100a without a GPU) if it is missing, so
    the CPU suite can load it and check its exports."""
    so = os.path.join(ROOT, "paper_1510_08642_b200", "libddqd.so")
    if not os.path.exists(so):
        import importlib.util
        spec = importlib.util.spec_from_file_location(
            "_ddqd_build", os.path.join(ROOT, "paper_1510_08642_b200", "build.py"))
        nb = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(nb)
        nb.build()


_ensure_native_built()
