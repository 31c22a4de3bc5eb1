"""bench.py's reference arm (the oracle timed on the host cores) runs without a GPU: it must
print one JSON line with the same metric/config keys as our arm (CPU only)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_gemm_line():
    d = _run("--impl", "reference", "--workload", "c1", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference"
    assert d["metric"] == "DD/QD GEMM effective GFLOPS (2mln/s) and % FP64-pipe roofline"
    assert d["unit"] == "GFLOP/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["m"] == d["config"]["l"] == d["config"]["n"] == 1024
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_custom_workload():
    d = _run("--impl", "reference", "--custom", "100,90,80", "--prec", "qd", "--algo", "strassen",
             "--threshold", "16", "--steps", "1", "--warmup", "0")
    assert d["config"]["algo"] == "strassen" and d["value"] > 0


def test_reference_arm_under_torchrun_two_ranks():
    """The driver launches the reference arm like ours (torchrun, one rank per GPU): rank 0
    alone runs the oracle sample and prints the one line; the other rank exits 0 without work."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29547", os.path.join(ROOT, "bench.py"),
                        "--impl", "reference", "--workload", "c1", "--gpus", "2", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["config"]["m"] == 1024


import pytest  # noqa: E402


@pytest.mark.gpu
@pytest.mark.parametrize("wl", ["c0", "c4"])
def test_our_arm_contract_keys(wl):
    """Our arm's JSON line carries the contract keys (GPU): roofline with achieved/peak/frac,
    e2e with the copied bytes, clocks, gpu_launches > 0, cpu_baseline from the oracle."""
    d = _run("--workload", wl, "--steps", "2", "--warmup", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and r["peak"] > 0 and 0 < r["frac"] <= 1.0
    assert abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
