"""Build libddqd.so in-tree with nvcc for sm_100a (B200). No torch extension machinery:
the library is a plain C-ABI shared object (include/ddqd.h)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libddqd.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",            # never contract a*b+c: DD/QD error-free transforms need it
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
    "-I" + os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "ddqd.h")]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every .cu to an object in parallel (no cross-file device code), then link."""
    if not force and not needs_build():
        return SO
    from concurrent.futures import ThreadPoolExecutor
    extra = os.environ.get("DDQD_NVCC_EXTRA", "").split()   # tuning experiments only
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    flags = [f for f in NVCC_FLAGS if f != "-shared"]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *flags, *extra, "-c", "-o", obj, src]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return obj, " ".join(cmd) + "\n" + r.stdout + r.stderr, r.returncode

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, sources()))
    objs = [o for o, _, _ in results]
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", SO, *objs]
    logtxt = "".join(t for _, t, _ in results)
    failed = [t for _, t, rc in results if rc != 0]
    if not failed:
        r = subprocess.run(link, capture_output=True, text=True)
        logtxt += " ".join(link) + "\n" + r.stdout + r.stderr
        if r.returncode != 0:
            failed.append(r.stdout + r.stderr)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(logtxt)
    if failed:
        sys.stderr.write("".join(failed))
        raise RuntimeError("nvcc failed building libddqd.so (see %s)" % log)
    if verbose:
        sys.stderr.write(logtxt)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(SO)
