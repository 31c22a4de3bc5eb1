#!/usr/bin/env python
"""bench.py -- DD/QD GEMM effective GFLOPS (2mln/s) and FP64-pipe roofline on B200 (BJ:2).

Step = one C := A B through the library's public C ABI (dd_gemm/qd_gemm) for the named
workload: pre-additions, the batched leaf GEMM and post-additions of every recursion level
(all SURVEY.md s.8(a) GEMM rows). Default workload: BASELINE.json configs[3] -- DD Winograd
8191 x 8193 x 8190, threshold 256 (depth 5) -- the config the metric's 1/2/4/8-GPU numbers
are quoted on (DESIGN.md s.7 explains the choice). Inputs are the seeded synthetic matrices
of BJ:10 (ddqd_inputs), resident in HBM before the timed region; each operand (1.07 GB) is
larger than L2 (126 MB), so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c1|c2|c3] [--impl reference]

N > 1 runs under torchrun (one process per GPU, NCCL) with the multi-GPU schedule of
paper_1510_08642_b200.mgpu; rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# the paper's own CPU numbers closest to each workload (context only)
PAPER_CONTEXT = {
    "c1": {"value": 0.693, "unit": "GFLOP/s", "seconds": 3.1, "what": "DD Strassen(32), n = 1024, 8 threads",
           "cpu": "Intel Xeon E5-2620 v2 2.1 GHz, qd 2.3.15", "source": "PAPER.md:74-76 (Table 1)"},
    "c2": {"value": 0.125, "unit": "GFLOP/s", "seconds": 17.2, "what": "QD Winograd(32), n = 1024, 8 threads",
           "cpu": "Intel Xeon E5-2620 v2 2.1 GHz, qd 2.3.15", "source": "PAPER.md:103-105 (Table 2)"},
    "c3": {"value": 0.693, "unit": "GFLOP/s", "seconds": None,
           "what": "no paper run at this size; its best DD rate: Strassen/Winograd(32), n = 1024, 8 threads",
           "cpu": "Intel Xeon E5-2620 v2 2.1 GHz, qd 2.3.15", "source": "PAPER.md:74-76 (Table 1)"},
    "c4": {"value": 2.0 / 3.0 * 1024 ** 3 / 4.3 / 1e9, "unit": "GFLOP/s", "seconds": 4.3,
           "what": "DD pivot-free LU, n = 1024 (inferred), Winograd(32) update, alpha = 2, 8 threads",
           "cpu": "Intel Xeon E5-2620 v2 2.1 GHz, qd 2.3.15", "source": "PAPER.md:164"},
}

GEMM_METRIC = "DD/QD GEMM effective GFLOPS (2mln/s) and % FP64-pipe roofline"
LU_METRIC = "DD LU effective GFLOPS (2n^3/3 per solve / s)"

WORKLOADS = {
    "c0": dict(W=2, algo="block", T=128, m=128, l=128, n=128, seed=1,
               name="BJ configs[0]: DD Block GEMM 128^3, seed 1 (latency-bound; split-k variants)"),
    "c1": dict(W=2, algo="strassen", T=128, m=1024, l=1024, n=1024, seed=2,
               name="BJ configs[1]: DD Strassen GEMM 1024^3, threshold 128 (depth 3), seed 2"),
    "c2": dict(W=4, algo="winograd", T=128, m=1024, l=1024, n=1024, seed=3,
               name="BJ configs[2]: QD Winograd GEMM 1024^3, threshold 128 (depth 3), seed 3"),
    "c3": dict(W=2, algo="winograd", T=256, m=8191, l=8193, n=8190, seed=4,
               name="BJ configs[3]: DD Winograd GEMM 8191x8193x8190, threshold 256 (depth 5), seed 4"),
    "c4": dict(W=2, algo="strassen", T=128, n=4096, panel=256, seed=5, lu=True,
               name="BJ configs[4]: DD blocked right-looking LU with partial pivoting, n=4096, panel 256, "
                    "Strassen update (threshold 128), A = R + nI, b = A*1, seed 5"),
}
# FP64-pipe lane-instructions per multiply-add (docs/numerics.md: DD 3 DMUL + 1 DFMA + 16 DADD;
# QD common path 118 (qd_mul) + 82 (qd_add)).
OPS_PER_MADD = {2: 20, 4: 200}
MAD_DTYPE = {2: "f64", 4: "f64"}          # arithmetic type of the path (FP64 pipe)
REPR = {2: "double-double (2 x f64, ~106-bit)", 4: "quad-double (4 x f64, ~212-bit)"}


def rec_shapes(m, l, n, T):
    shapes = [(m, l, n)]
    while min(m, l, n) > T:
        m, l, n = (m + 1) // 2, (l + 1) // 2, (n + 1) // 2
        shapes.append((m, l, n))
    return shapes


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default per workload: c0 200, c1 50, c2 20, c3/c4 5)")
    ap.add_argument("--warmup", type=int, default=None,
                    help="untimed warm-up steps (default per workload: c0 20, c1/c2 5, else 3)")
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--custom", default=None, metavar="M,L,N",
                    help="a custom GEMM workload instead of a BASELINE config (with --prec/--algo/--threshold/--seed)")
    ap.add_argument("--prec", default="dd", choices=["dd", "qd"])
    ap.add_argument("--algo", default="winograd", choices=["block", "strassen", "winograd"])
    ap.add_argument("--threshold", type=int, default=128)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--k", type=int, default=None, help="multi-GPU product depth (default: balancer)")
    ap.add_argument("--schedule", default="auto",
                    choices=["auto", "bands", "products", "products_rows", "products_p2p", "ctiles", "auto-all"],
                    help="multi-GPU schedule: auto = whichever of the bit-identical schedules measures "
                         "fastest (BJ:5 (4)); bands = one tile of C per rank with the whole problem's "
                         "tree; products = depth-k products to rank 0 (--combine); products_p2p = "
                         "the same combined over CUDA IPC; ctiles = C row slabs (rounds differently); "
                         "auto-all = auto including ctiles")
    ap.add_argument("--combine", default="nccl", choices=["nccl", "p2p"],
                    help="multi-GPU combine: products to rank 0 over NCCL point-to-point (default), or "
                         "the fused post-additions reading peers' products over CUDA IPC / NVLink")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--staged-transport", action="store_true",
                    help="functional test of the N > 1 path on ONE GPU: every rank on cuda:0, exchanges "
                         "over gloo staged through host memory (mgpu.HostStagedGroup); not a bench number")
    ap.add_argument("--no-band-model", action="store_true",
                    help="skip the one-GPU timing of the band schedule's per-rank tiles (N = 1 line)")
    ap.add_argument("--no-variant", action="store_true",
                    help="skip the extra fused / accurate measurements reported under 'variants'")
    ap.add_argument("--madd", default="canonical", choices=["canonical", "fused", "accurate"],
                    help="arithmetic: the paper's QD-library sequences (DD madd 20 FP64 ops), the "
                         "fused multiply-add or the accurate adds of numerics.md s.2-3 (row f3)")
    args = ap.parse_args()
    # microsecond-scale steps need more of them for a stable number (and enough warm-up to
    # bring the clocks back up after the sampler's start-up idle)
    dsteps = {"c0": 200, "c1": 50, "c2": 20}.get(args.workload, 5) if args.custom is None else 5
    dwarm = {"c0": 20, "c1": 5, "c2": 5}.get(args.workload, 3) if args.custom is None else 3
    if args.steps is None:
        args.steps = dsteps
    if args.warmup is None:
        args.warmup = dwarm
    return args


# ---- clocks sampler (nvidia-smi during the timed region) ------------------------------
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.5)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0])); mx = float(f[1]); power.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# ---- CPU oracle sample (cpu_baseline and --impl reference) ----------------------------
def oracle_sample(wl, per_step=False):
    """Bounded sample of the workload for the oracle: for the cpu_baseline (one run, ~10-20 s
    of host work) the leading (m/2, l/2, n/2) block of c3 (same recipe, algorithm and
    threshold) and the full c0/c1/c2 problems; per step of the reference arm (run K + W times)
    the leading (m/4, l/4, n/4) block of c3 (~2 s). Returns (A, B, shape, description)."""
    import ddqd_inputs as gen
    m, l, n = wl["m"], wl["l"], wl["n"]
    if wl["key"] == "custom":   # keep the sample near 1024^3 (DD) / 512^3 (QD) multiply-adds
        target = (1024 if wl["W"] == 2 else 512) ** 3
        div = max(1, int(math.ceil((m * l * n / target) ** (1.0 / 3.0))))
    else:
        div = {"c3": 4 if per_step else 2, "c2": 1, "c1": 1, "c0": 1}[wl["key"]]
    ms, ls, ns = (m + div - 1) // div, (l + div - 1) // div, (n + div - 1) // div
    A = gen.matrix(wl["W"], ms, ls, wl["seed"], 0)
    B = gen.matrix(wl["W"], ls, ns, wl["seed"], 1)
    desc = (f"oracle {wl['algo']}(T={wl['T']}) on a {ms}x{ls}x{ns} problem with the workload's "
            f"input recipe ({'full problem' if div == 1 else f'1/{div} of each dimension'})")
    return A, B, (ms, ls, ns), desc


def run_oracle_once(orc, wl, A, B):
    t0 = time.perf_counter()
    orc.gemm(A, B, wl["algo"], threshold=wl["T"])
    return time.perf_counter() - t0


def ncu_leaf_traffic(workload):
    """DRAM bytes (read + write) per leaf launch from the newest committed `ncu --set full`
    capture of this workload's leaf kernel (profiles/rNN/ncu_full_leaf_<wl>_raw.csv)."""
    import csv
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", f"ncu_full_leaf_{workload}_raw.csv")))
    if not files:
        return None, None, None, ""
    rows = list(csv.reader(open(files[-1])))
    hdr, units, vals = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tot = 0.0
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(name)
        tot += float(vals[i].replace(",", "")) * scale.get(units[i], 1)
    grid = vals[hdr.index("launch__grid_size")] if "launch__grid_size" in hdr else None
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""
    return tot, f"{os.path.relpath(files[-1], ROOT)} (grid {grid})", int(grid) if grid else None, name


def leaf_tile(name):
    """Output tile (rows, cols) of one CTA of a captured leaf kernel, from its name."""
    import re
    if "leaf_small_kernel" in name:
        return 8, 16
    if "leaf_tma_kernel" in name:
        return 64, 64
    mt = re.search(r"leaf_gemm_kernel<\s*\d+\s*,\s*(\d+)\s*,\s*(\d+)", name)
    return (int(mt.group(1)), int(mt.group(2))) if mt else None


def ncu_panel_traffic():
    """DRAM bytes (read + write) of one LU panel launch from the committed `ncu --set full`
    capture (profiles/rNN/ncu_lu_raw.csv; first captured panel)."""
    import csv
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_lu_raw.csv")))
    if not files:
        return None, None
    rows = list(csv.reader(open(files[-1])))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for vals in rows[2:]:
        if "lu_panel_coop_kernel" not in vals[hdr.index("Kernel Name")]:
            continue
        tot = sum(float(vals[hdr.index(k)].replace(",", "")) * scale.get(units[hdr.index(k)], 1)
                  for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        return tot, f"{os.path.relpath(files[-1], ROOT)} (grid {vals[hdr.index('launch__grid_size')]})"
    return None, None


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


def reference_arm(args, wl, rank, world):
    if rank != 0:
        return 0
    import oracle as orc
    orc.build()
    if wl.get("lu"):
        return reference_lu(args, wl, orc)
    A, B, (ms, ls, ns), desc = oracle_sample(wl, per_step=True)
    for _ in range(args.warmup):
        run_oracle_once(orc, wl, A, B)
    tot = sum(run_oracle_once(orc, wl, A, B) for _ in range(args.steps))
    value = 2.0 * ms * ls * ns * args.steps / tot / 1e9
    cores = cpu_cores()
    line = {
        "impl": "reference", "metric": GEMM_METRIC, "value": value, "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": MAD_DTYPE[wl["W"]], "data": "synthetic (seeded SplitMix64, BASELINE.json recipe)",
        "config": {"workload": wl["name"], "m": wl["m"], "l": wl["l"], "n": wl["n"], "algo": wl["algo"],
                   "threshold": wl["T"], "madd": "canonical", "parallelism": "oracle on the host cores",
                   "sample": desc},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def reference_lu(args, wl, orc):
    """Oracle LU + solve of the c4 workload itself (n = 4096, ~10 s per solve on 16 cores)."""
    import numpy as np

    import ddqd_inputs as gen
    n = wl["n"]
    A = gen.lu_matrix(n, wl["seed"])
    ones = np.zeros((2, n, 1)); ones[0] = 1.0
    b = orc.gemm(A, ones, "block")[:, :, 0].copy()
    run = lambda: orc.solve(A, b, panel=wl["panel"], algo=wl["algo"], threshold=wl["T"])  # noqa: E731
    for _ in range(args.warmup):
        run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run()
    tot = time.perf_counter() - t0
    value = 2.0 / 3.0 * n ** 3 * args.steps / tot / 1e9
    desc = f"oracle LU+solve of the full workload, n={n} (panel {wl['panel']}, {wl['algo']} T={wl['T']})"
    print(json.dumps({
        "impl": "reference", "metric": LU_METRIC, "value": value,
        "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": MAD_DTYPE[2], "data": "synthetic (seeded SplitMix64, BASELINE.json recipe)",
        "config": {"workload": wl["name"], "n": wl["n"], "panel": wl["panel"], "algo": wl["algo"],
                   "threshold": wl["T"], "parallelism": "oracle on the host cores", "sample": desc},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cpu_cores(), "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}), flush=True)
    return 0


# ---- LU (c4) ----------------------------------------------------------------------------
def lu_bench(args, wl, rank, world, local):
    """c4: one step = dd_lu_solve (factor + solve) of a fresh copy of A. Multi-GPU: replicas
    only (DESIGN.md s.8: the LU's panel chain does not shard at this size); value = total
    work of all replicas / max-over-ranks time."""
    import numpy as np
    import torch

    import ddqd_inputs as gen
    import paper_1510_08642_b200 as ddqd

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    n, K, algo, T = wl["n"], wl["panel"], wl["algo"], wl["T"]
    A0 = torch.from_numpy(gen.lu_matrix(n, wl["seed"])).to(dev)
    ones = torch.zeros((2, n, 1), dtype=torch.float64, device=dev)
    ones[0] = 1.0
    b = ddqd.dd_gemm(A0, ones, "block")[:, :, 0].contiguous()     # b = A*1 on the device
    A = torch.empty_like(A0)
    x = torch.empty_like(b)
    ipiv = torch.empty(n, dtype=torch.int64, device=dev)

    def step():
        A.copy_(A0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ddqd._set_stream(A)
        info = ddqd.lib.dd_lu_solve(n, A.data_ptr(), b.data_ptr(), x.data_ptr(), ipiv.data_ptr(),
                                     K, ddqd._algo(algo), T)
        e1.record()
        torch.cuda.synchronize()
        assert info == 0, info
        return e0.elapsed_time(e1)

    peak = max(ddqd.fp64_peak("dadd")[0], ddqd.fp64_peak("dfma")[0])
    # the sampler starts before the warm-up: its 0.5 s start-up idles the GPU, which must not
    # sit right before the timed region (the clocks would ramp inside it)
    clocks = Clocks(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = ddqd.launch_count()
    ddqd.profile_start()
    ms = sum(step() for _ in range(args.steps))
    prof = ddqd.profile_stop()
    kern = ddqd.profile_kernels()
    launches = ddqd.launch_count() - n0
    clk = clocks.stop()
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    flops = 2.0 / 3.0 * n ** 3
    value = flops * world * args.steps / (ms * 1e-3) / 1e9
    xx = x.cpu().numpy()
    err = float(np.abs((xx[0] - 1.0) + xx[1]).max())
    leaf_ms, leaf_n, leaf_madds = prof["leaf"]
    achieved = 20.0 * leaf_madds / (leaf_ms * 1e-3) / 1e12 if leaf_ms else 0.0
    shares = {k: v[0] / ms for k, v in prof.items()}
    dominant = max(shares, key=shares.get)
    roof_leaf = {"bound": "alu", "achieved": achieved, "peak": peak / 1e12, "unit": "TFLOP/s",
                 "frac": achieved / (peak / 1e12) if peak else None,
                 "kernel": (max((k for k, v in kern.items() if v[0] == 0), key=lambda k: kern[k][1], default="leaf")
                            + " (Schur update leaves, Strassen d = 1)"),
                 "share_of_step": shares["leaf"], "traffic": None}
    # the dominant kernel: the panel factorisation (FP64 work = its rank-1 updates, R K^2 / 2 DD
    # madds per panel of R rows, 20 FP64 lane-ops each) -- far below the pipe: it is bound by
    # the latency of its 4096 dependent pivot steps, not by an execution unit
    pan_ms, pan_n, pan_madds = prof["lu_panel"]
    pan_ach = 20.0 * pan_madds / (pan_ms * 1e-3) / 1e12 if pan_ms else 0.0
    roof_pan = {"bound": "alu", "achieved": pan_ach, "peak": peak / 1e12, "unit": "TFLOP/s",
                "frac": pan_ach / (peak / 1e12) if peak else None,
                "kernel": max((k for k, v in kern.items() if v[0] == 3), key=lambda k: kern[k][1],
                              default="lu panel"), "launches": int(pan_n),
                "share_of_step": shares["lu_panel"], "traffic": None,
                "latency_bound": "the 4096-column pivot chain (l = a * r, u = a - l * u, r = 1 / u: ~0.8k "
                                 "cycles per column in the one-CTA diagonal blocks of the 32-column "
                                 "sub-panels) and the 32-step row-elimination chains (DESIGN.md s.7)",
                "work_def": "rank-1 panel updates R*K^2/2 DD madds x 20 FP64 lane-ops",
                "algorithmic_bytes_per_launch": 16.0 * K * (n - K * (n // K - 1) / 2.0) * 2,
                "traffic_note": "one panel launch reads its slab once (R x K DD) and writes it back "
                                "(the write stays in the 126 MB L2 within the launch)"}
    tr, src = ncu_panel_traffic() if "coop" in roof_pan["kernel"] else (None, None)
    if tr is not None:
        roof_pan["traffic"] = tr
        roof_pan["traffic_source"] = src
    roof_dom = roof_pan if shares["lu_panel"] >= shares["leaf"] else roof_leaf

    e2e = None
    if not args.no_e2e and world == 1:
        # the same solve through the public API from pinned HOST data: H2D of A and b, the
        # dd_lu_solve call, D2H of x -- all inside the timed region
        hA = A0.cpu().pin_memory()
        hb = b.cpu().pin_memory()
        hx = torch.empty_like(hb).pin_memory()

        def e2e_step():
            A.copy_(hA, non_blocking=True)
            bb = hb.to(dev, non_blocking=True)
            ddqd._set_stream(A)
            info = ddqd.lib.dd_lu_solve(n, A.data_ptr(), bb.data_ptr(), x.data_ptr(), ipiv.data_ptr(),
                                         K, ddqd._algo(algo), T)
            hx.copy_(x, non_blocking=True)
            return info

        e2e_step()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            assert e2e_step() == 0
        f1.record()
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1)
        e2e = {"value": flops * args.steps / (ems * 1e-3) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(hA.numel() * 8 + hb.numel() * 8),
               "d2h_bytes_per_step": int(hx.numel() * 8), "ms_per_step": ems / args.steps,
               "path": "pinned host A, b -> dd_lu_solve (device pointers, the public C ABI) -> pinned host x"}

    cpu = None
    if not args.no_cpu and world == 1 and rank == 0:
        import oracle as orc
        orc.build()
        ns = n   # the full c4 problem: the oracle LU at n = 4096 takes ~10 s on 16 cores
        As = gen.lu_matrix(ns, wl["seed"])
        on = np.zeros((2, ns, 1)); on[0] = 1.0
        bs = orc.gemm(As, on, "block")[:, :, 0].copy()
        t0 = time.perf_counter()
        orc.solve(As, bs, panel=K, algo=algo, threshold=T)
        t = time.perf_counter() - t0
        cpu = {"value": 2.0 / 3.0 * ns ** 3 / t / 1e9, "unit": "GFLOP/s", "cores": cpu_cores(), "kind": "oracle",
               "sample": f"oracle LU+solve of the full workload (n = {ns}, panel {K}, {algo} T = {T}), one solve",
               "seconds": t}
    if rank == 0:
        line = {
            "metric": LU_METRIC, "value": value, "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak" if world > 1 else "strong", "vs_baseline": None,
            "dtype": MAD_DTYPE[2], "representation": REPR[2], "data": "synthetic (seeded SplitMix64, BASELINE.json recipe)",
            "config": {"workload": wl["name"], "n": n, "panel": K, "algo": algo, "threshold": T,
                       "parallelism": f"{world} GPU replica(s)",
                       "l2": "A (268 MB) exceeds L2; fresh copy of A before each step, outside the events"},
            "roofline": roof_dom,
            "roofline_schur_leaf": roof_leaf,
            "time_shares": shares,
            "kernel_shares": {k: v[1] / ms for k, v in sorted(kern.items(), key=lambda kv: -kv[1][1])},
            "max_abs_err_x_minus_1": err,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk,
            "paper_context": PAPER_CONTEXT["c4"],
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


# ---- multi-GPU ---------------------------------------------------------------------
def make_schedule(args, W, algo, T, m, l, n, dist, dev, replicated_inputs=False):
    from paper_1510_08642_b200 import mgpu
    if args.schedule in ("auto", "auto-all"):
        cands = None if args.schedule == "auto" else ("bands", "products_rows", "products", "products_p2p", "ctiles")
        return mgpu.AutoDistributedGemm(W, algo, T, m, l, n, dist, dev, candidates=cands, k=args.k,
                                        replicated_inputs=replicated_inputs)
    if args.schedule == "bands":
        return mgpu.BandGemm(W, algo, T, m, l, n, dist, dev, replicated_inputs=replicated_inputs)
    combine = {"products_p2p": "p2p", "products_rows": "rows"}.get(args.schedule, args.combine)
    return mgpu.DistributedGemm(W, algo, T, m, l, n, dist, dev, k=0 if args.schedule == "ctiles" else args.k,
                                combine=combine, replicated_inputs=replicated_inputs)


def schedule_desc(args, sched, world):
    if world == 1:
        return "1 GPU"
    d = f"{world} GPUs, schedule {args.schedule}"
    if getattr(sched, "choice", None):
        d += f" (chose {sched.choice})"
    inner = sched.cands[sched.choice] if getattr(sched, "choice", None) else sched
    if hasattr(inner, "gr"):
        d += f", band grid {inner.gr} x {inner.gc}"
    elif getattr(inner, "k", None) is not None:
        d += f", product depth k = {inner.k}, {inner.combine} combine" if inner.k else ", C row slabs"
    return d


def mgpu_e2e(args, wl, A_h, B_h, A, B, C, dist, dev, rank, W, flops_per_step, choice=None):
    """End to end at N GPUs: pinned host A, B on rank 0 -> H2D overlapped with the NCCL broadcast
    (chunks) -> the schedule (the device-timed run's choice) -> C gathered on rank 0 -> D2H,
    every step inside the timed region; device events on each rank, max over ranks."""
    import argparse

    import torch

    from paper_1510_08642_b200 import mgpu
    m, l, n = wl["m"], wl["l"], wl["n"]
    a2 = argparse.Namespace(**vars(args))
    if choice:
        a2.schedule = choice
    sched = make_schedule(a2, W, wl["algo"], wl["T"], m, l, n, dist, dev, replicated_inputs=True)
    hA = A_h.pin_memory() if rank == 0 else None
    hB = B_h.pin_memory() if rank == 0 else None
    hC = torch.empty((W, m, n), dtype=torch.float64).pin_memory() if rank == 0 else None

    def e2e_step():
        mgpu.host_broadcast(hA, A, dist)
        mgpu.host_broadcast(hB, B, dist)
        sched(A, B, C)
        if rank == 0:
            hC.copy_(C, non_blocking=True)

    e2e_step()       # the auto schedule measures its candidates here
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        e2e_step()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ems = float(t.item())
    return {"value": flops_per_step * args.steps / (ems * 1e-3) / 1e9, "unit": "GFLOP/s",
            "h2d_bytes_per_step": int((A.numel() + B.numel()) * 8),
            "d2h_bytes_per_step": int(C.numel() * 8), "ms_per_step": ems / args.steps,
            "path": "pinned host A, B on rank 0 -> H2D overlapped with the NCCL broadcast (8 chunks each) "
                    "-> " + schedule_desc(a2, sched, dist.get_world_size()) + " -> C on rank 0 -> "
                    "pinned host C (D2H); device events, max over ranks"}


def band_model(args, wl, A, B, C, peak):
    """One-GPU measurement of the band schedule's per-rank compute at 2, 4 and 8 GPUs: the
    largest tile of each grid (pack + DDQD_DEPTH GEMM + unpack, the exact kernels a rank runs)
    timed on this GPU. The N-GPU step is that plus the operand broadcast and the tile gather,
    modelled at the measured NVLink rates of B200_PROFILING.md (no multi-GPU box here)."""
    import torch

    from paper_1510_08642_b200 import mgpu
    W, m, l, n = wl["W"], wl["m"], wl["l"], wl["n"]
    out = {}
    for G in (2, 4, 8):
        bg = mgpu.BandGemm(W, wl["algo"], wl["T"], m, l, n, None, world=G)
        # tile 0 holds the largest bands (balanced_slices gives the extra rows to the first)
        for _ in range(2):
            bg.run_tile(0, A, B, C)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 3
        for _ in range(reps):
            bg.run_tile(0, A, B, C)
        e1.record()
        torch.cuda.synchronize()
        tile_ms = e0.elapsed_time(e1) / reps
        bcast_ms = (A.numel() + B.numel()) * 8 / 725e9 * 1e3       # NCCL bus bandwidth, 1 GiB class
        rows, cols = bg.tile(0)
        gather_ms = (G - 1) / G * C.numel() * 8 / 770e9 * 1e3      # tiles into rank 0 (peer copy rate)
        ent = {"grid": [bg.gr, bg.gc], "tile_rows": len(rows), "tile_cols": len(cols),
               "tile_ms_measured": tile_ms, "broadcast_ms_model": bcast_ms,
               "gather_ms_model": gather_ms, "step_ms_model": tile_ms + bcast_ms + gather_ms}
        # the product schedule with the row-band combine: rank 0 (the largest slice) measured
        # the same way; plus the all-to-all of product row bands, modelled
        dg = mgpu.DistributedGemm(W, wl["algo"], wl["T"], m, l, n, None, combine="rows", world=G, rank=0)
        dg.compute_share(A, B)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            dg.compute_share(A, B)
        e1.record()
        torch.cuda.synchronize()
        share_ms = e0.elapsed_time(e1) / reps
        mk, _, nk = dg.shapes[dg.k]
        lo, hi = dg.slices[0]
        a2a_bytes = (hi - lo) * W * mk * nk * 8 * (G - 1) / G         # sent = received per rank
        a2a_ms = a2a_bytes / 770e9 * 1e3
        # each chunk's row bands are exchanged while the next chunk computes: only the last
        # chunk's exchange is exposed
        last = (hi - lo) - ((hi - lo - 1) // dg.chunk) * dg.chunk
        a2a_exposed = a2a_ms * last / (hi - lo)
        ent["products_rows"] = {"k": dg.k, "products_rank0": hi - lo, "share_ms_measured": share_ms,
                                "all_to_all_bytes_per_rank": a2a_bytes, "all_to_all_ms_model": a2a_ms,
                                "all_to_all_exposed_ms_model": a2a_exposed,
                                "rank0_receive_bytes": (G - 1) / G * C.numel() * 8,
                                "step_ms_model": share_ms + bcast_ms + a2a_exposed + gather_ms}
        del dg
        out[str(G)] = ent
    return out


# ---- our arm ------------------------------------------------------------------------
def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.custom:
        m_, l_, n_ = (int(v) for v in args.custom.split(","))
        W_ = 2 if args.prec == "dd" else 4
        args.workload = "custom"
        wl = dict(W=W_, algo=args.algo, T=args.threshold, m=m_, l=l_, n=n_, seed=args.seed,
                  name=f"custom: {args.prec.upper()} {args.algo} GEMM {m_}x{l_}x{n_}, threshold {args.threshold}, "
                       f"seed {args.seed}")
    else:
        wl = dict(WORKLOADS[args.workload])
    wl["key"] = args.workload
    if args.impl == "reference":
        return reference_arm(args, wl, rank, world)
    if wl.get("lu"):
        return lu_bench(args, wl, rank, world, local)

    import numpy as np
    import torch

    import ddqd_inputs as gen
    import paper_1510_08642_b200 as ddqd

    if args.staged_transport:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.staged_transport:
            from paper_1510_08642_b200.mgpu import HostStagedGroup
            dist.init_process_group("gloo")
            dist = HostStagedGroup(dist)
        else:
            dist.init_process_group("nccl", device_id=dev)

    W, algo, T, m, l, n = wl["W"], wl["algo"], wl["T"], wl["m"], wl["l"], wl["n"]
    flops_per_step = 2.0 * m * l * n

    # inputs: every rank builds the same seeded matrices (rank 0's are the ones broadcast in
    # the multi-GPU schedule); resident in HBM before the timed region
    A_h = torch.from_numpy(gen.matrix(W, m, l, wl["seed"], 0))
    B_h = torch.from_numpy(gen.matrix(W, l, n, wl["seed"], 1))
    A = A_h.to(dev)
    B = B_h.to(dev)
    C = torch.empty((W, m, n), dtype=torch.float64, device=dev)

    peak_dadd, _ = ddqd.fp64_peak("dadd")
    peak_dfma, _ = ddqd.fp64_peak("dfma")
    peak = max(peak_dadd, peak_dfma)

    sched = None
    if world > 1:
        sched = make_schedule(args, W, algo, T, m, l, n, dist, dev)

        def step():
            sched(A, B, C)
    else:
        def step():
            ddqd.gemm(A, B, algo, T, out=C, madd=args.madd)

    clocks = Clocks(local)      # before the warm-up (see the LU path)
    clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = ddqd.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    launches = ddqd.launch_count() - n0
    ms = ev0.elapsed_time(ev1)
    # the roofline's per-kernel event timing runs over a second timed pass of the same K steps:
    # its two event records per launch add host time, which a launch-bound step (c0) would
    # otherwise carry into the headline
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ddqd.profile_start()
    pr0, pr1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pr0.record()
    for _ in range(args.steps):
        step()
    pr1.record()
    torch.cuda.synchronize()
    prof = ddqd.profile_stop()
    kern = ddqd.profile_kernels()
    ms_prof = pr0.elapsed_time(pr1)
    if dist:
        dist.barrier()
    clk = clocks.stop()
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = flops_per_step * args.steps / (ms * 1e-3) / 1e9     # whole job, GFLOP/s

    # roofline of the dominant kernel: the batched leaf GEMM (FP64-pipe bound). The profile names
    # every leaf variant separately (TMA / cp.async / tail tiles / flat strips): the dominant one
    # by device time is the roofline kernel, with its own launches and work
    leaf_kern = {k: v for k, v in kern.items() if v[0] == 0}
    dom = max(leaf_kern, key=lambda k: leaf_kern[k][1]) if leaf_kern else None
    if dom is not None:
        leaf_ms, leaf_n, leaf_madds = leaf_kern[dom][1], leaf_kern[dom][2], leaf_kern[dom][3]
    else:
        leaf_ms, leaf_n, leaf_madds = prof["leaf"]
    # FP64 lane-ops per madd of the selected arithmetic (the QD variants' common-path counts
    # are not fixed numbers; they are reported against the canonical 200)
    ops = {"canonical": OPS_PER_MADD[W], "fused": 15 if W == 2 else OPS_PER_MADD[W],
           "accurate": 29 if W == 2 else OPS_PER_MADD[W]}[args.madd]
    leaf_avg_s = (leaf_ms / leaf_n) * 1e-3 if leaf_n else float("nan")
    leaf_ops_per_launch = ops * leaf_madds / leaf_n if leaf_n else 0.0
    achieved = leaf_ops_per_launch / leaf_avg_s / 1e12 if leaf_n else 0.0
    roofline = {
        "bound": "alu", "achieved": achieved, "peak": peak / 1e12, "unit": "TFLOP/s",
        "frac": achieved / (peak / 1e12),
        "flop_def": f"one FP64-pipe lane op (DADD/DMUL/DFMA); {ops} per {'DD' if W == 2 else 'QD'} madd",
        "peak_source": "measured live by ddqd_fp64_peak (DADD/DFMA stream, 148 SMs); "
                       "MEASURED_PEAKS.json has no FP64 figure",
        "peak_dadd": peak_dadd / 1e12, "peak_dfma": peak_dfma / 1e12,
        "kernel": dom or "leaf", "launches": int(leaf_n),
        "leaf_kernels": {k: {"ms_per_step": v[1] / args.steps, "launches": v[2],
                             "share_of_step": v[1] / ms_prof if ms_prof else None,
                             "frac": (ops * v[3] / (v[1] * 1e-3) / peak) if v[1] else None}
                         for k, v in leaf_kern.items()},
        "avg_launch_ms": leaf_avg_s * 1e3, "share_of_step": leaf_ms / ms_prof if ms_prof else None,
        "profiled_pass_ms_per_step": ms_prof / args.steps,
        "traffic": None,
        "algorithmic_bytes_per_launch": None,
        "pre_add": {"ms": prof["pre"][0], "launches": int(prof["pre"][1]),
                    "GB_per_s": prof["pre"][2] / (prof["pre"][0] * 1e-3) / 1e9 if prof["pre"][0] else None},
        "post_add": {"ms": prof["post"][0], "launches": int(prof["post"][1]),
                     "GB_per_s": prof["post"][2] / (prof["post"][0] * 1e-3) / 1e9 if prof["post"][0] else None},
    }
    shapes = rec_shapes(m, l, n, T)
    d = len(shapes) - 1
    if leaf_n:
        lm, ll, ln = shapes[-1]
        per_launch_leaves = leaf_madds / leaf_n / (lm * ll * ln)
        roofline["algorithmic_bytes_per_launch"] = per_launch_leaves * W * 8.0 * (lm * ll + ll * ln + lm * ln)
        tr, src, grid, kname = ncu_leaf_traffic(args.workload)
        if tr is not None:
            roofline["traffic"] = tr
            roofline["traffic_source"] = src
            tile = leaf_tile(kname)
            if tile and grid:
                # the captured launch's own algorithmic bytes (a tail-split step has launches of
                # different sizes, so the per-step average above is not its denominator)
                leaves = grid / (((lm + tile[0] - 1) // tile[0]) * ((ln + tile[1] - 1) // tile[1]))
                cap_alg = leaves * W * 8.0 * (lm * ll + ll * ln + lm * ln)
                roofline["traffic_captured_launch_algorithmic_bytes"] = cap_alg
                roofline["traffic_over_algorithmic"] = tr / cap_alg
    leaf_madds_step = (7 ** d) * shapes[-1][0] * shapes[-1][1] * shapes[-1][2]
    # whole-step algorithmic roofline: the leaf's FP64 work at the FP64 peak plus the additions'
    # algorithmic bytes at the HBM peak, over the measured step time
    hbm_peak, hbm_src = 6550.7e9, "MEASURED_PEAKS.json (driver copy benchmark)"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm_peak = float(json.load(f)["hbm_gbs"]) * 1e9
    except Exception:
        hbm_src = "the driver's last measured copy bandwidth (file absent)"
    add_bytes_step = (prof["pre"][2] + prof["post"][2]) / args.steps
    step_alg = ((ops * leaf_madds_step / peak + add_bytes_step / hbm_peak) / (ms_per_step * 1e-3)
                if world == 1 else None)   # per-rank profiles do not add up to the whole job
    classical = ops * m * l * n / (ms_per_step * 1e-3) / peak   # BJ:5's literal formula (may be > 1)

    variants = None
    if args.madd == "canonical" and world == 1 and not args.no_variant:
        # the arithmetic variants of SURVEY s.8(f) row f3 on the same inputs: different
        # (documented, oracle-mirrored) roundings, reported beside the paper-faithful headline
        variants = {}
        notes = {"fused": ("DDQD_MADD_FUSED", {2: 15, 4: None}, "fused", 1),
                 "accurate": ("DDQD_ADD_ACCURATE", {2: 29, 4: None}, "accurate", 1)}
        if args.workload == "c0":   # small shapes: the split-k cluster leaf (row a4)
            for sk in (2, 4, 8):
                notes["splitk%d" % sk] = ("DDQD_SPLITK(%d)" % sk, {2: 20, 4: 200}, "canonical", sk)
        for v, (flag, opc, mv, sk) in notes.items():
            def vstep():
                ddqd.gemm(A, B, algo, T, out=C, madd=mv, splitk=sk)
            vstep()
            torch.cuda.synchronize()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record()
            for _ in range(args.steps):
                vstep()
            f1.record()
            torch.cuda.synchronize()
            fms = f0.elapsed_time(f1)
            variants[("madd_" + v) if sk == 1 else v] = {
                "value": flops_per_step * args.steps / (fms * 1e-3) / 1e9, "unit": "GFLOP/s",
                "ms_per_step": fms / args.steps, "fp64_ops_per_madd": opc[W],
                "note": flag + ": bit-exact vs the oracle's " + v + " variant, not the canonical"}

        if args.workload == "c0":
            # c0's per-call time is set by the host (Python + ctypes launch, ~15 us) rather than
            # the ~9.5 us leaf kernel: the same canonical call captured into a CUDA graph
            # (20 calls per graph) shows the device-side rate
            cs = torch.cuda.Stream()
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cs):
                step()
            torch.cuda.current_stream().wait_stream(cs)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(20):
                    step()
            g.replay()
            torch.cuda.synchronize()
            reps = max(1, args.steps // 20)
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record()
            for _ in range(reps):
                g.replay()
            f1.record()
            torch.cuda.synchronize()
            gms = f0.elapsed_time(f1) / (20 * reps)
            variants["cuda_graph"] = {
                "value": flops_per_step / (gms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": gms,
                "fp64_ops_per_madd": OPS_PER_MADD[W],
                "note": "canonical arithmetic; 20 dd_gemm calls captured in one CUDA graph and replayed "
                        "(removes the host launch overhead; same kernels, same bits)"}
            del g

    bitwise = None
    if world > 1:
        # the multi-GPU result against one GPU's dd_gemm/qd_gemm of the same inputs on rank 0
        if rank == 0:
            C1 = ddqd.gemm(A, B, algo, T, madd=args.madd)
            torch.cuda.synchronize()
            inner = sched.cands[sched.choice] if getattr(sched, "choice", None) else sched
            bitwise = {"equal": bool(torch.equal(C1.view(torch.int64), C.view(torch.int64))),
                       "schedule": getattr(sched, "choice", None) or args.schedule,
                       "expected_bitwise": not (getattr(inner, "k", 1) == 0 and algo != "block")}
            del C1
        dist.barrier()

    e2e = None
    if not args.no_e2e and world > 1:
        e2e = mgpu_e2e(args, wl, A_h, B_h, A, B, C, dist, dev, rank, W, flops_per_step,
                       choice=getattr(sched, "choice", None))
    if not args.no_e2e and world == 1:
        hA = A_h.pin_memory()
        hB = B_h.pin_memory()
        hC = torch.empty((W, m, n), dtype=torch.float64).pin_memory()
        ddqd.gemm(hA, hB, algo, T, out=hC, madd=args.madd)   # warm the staging buffers
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            ddqd.gemm(hA, hB, algo, T, out=hC, madd=args.madd)   # H2D + compute + D2H, synchronous
        e1.record()
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        e2e = {"value": flops_per_step * args.steps / (ems * 1e-3) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(hA.numel() * 8 + hB.numel() * 8),
               "d2h_bytes_per_step": int(hC.numel() * 8),
               "ms_per_step": ems / args.steps,
               "path": "dd_gemm/qd_gemm with pinned HOST pointers (library stages H2D/D2H inside the call)"}
        del hA, hB, hC

    bandm = None
    if world == 1 and algo != "block" and not args.no_band_model and args.custom is None \
            and args.workload in ("c3", "c2", "c1"):
        bandm = band_model(args, wl, A, B, C, peak)

    cpu = None
    if rank == 0 and not args.no_cpu:
        import oracle as orc
        orc.build()
        sA, sB, (ms_, ls_, ns_), desc = oracle_sample(wl)
        t = run_oracle_once(orc, wl, sA, sB)
        cpu = {"value": 2.0 * ms_ * ls_ * ns_ / t / 1e9, "unit": "GFLOP/s", "cores": cpu_cores(),
               "kind": "oracle", "sample": desc, "seconds": t}

    if rank == 0:
        line = {
            "metric": GEMM_METRIC,
            "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": MAD_DTYPE[W], "representation": REPR[W],
            "data": "synthetic (seeded SplitMix64, BASELINE.json recipe)",
            "config": {"workload": wl["name"], "m": m, "l": l, "n": n, "algo": algo, "threshold": T,
                       "madd": args.madd,
                       "depth": d, "leaf_shape": list(shapes[-1]), "leaf_madds_per_step": leaf_madds_step,
                       "l2": "no flush: each operand (%.2f GB) exceeds the 126 MB L2" % (A.numel() * 8 / 1e9),
                       "parallelism": schedule_desc(args, sched, world),
                       "schedule_timings_ms": ({k: (v * 1e3 if math.isfinite(v) else None)
                                                for k, v in sched.timings.items()}
                                               if getattr(sched, "timings", None) else None),
                       **({"schedules_unavailable": sched.unavailable}
                          if getattr(sched, "unavailable", None) else {}),
                       **({"transport": "FUNCTIONAL TEST ONLY: all ranks on one GPU, gloo staged through "
                                        "host memory (not a bench number)"} if args.staged_transport else {})},
            "roofline": roofline,
            "fp64_roofline_fraction": {
                "algorithmic_leaf": roofline["frac"],
                "algorithmic_step": step_alg,
                "classical_normalised": classical,
                "note": "algorithmic_step = (ops_per_madd*leaf_madds/P64 + addition_bytes/HBM_peak) / t_step "
                        "(SURVEY.md s.8(d); HBM peak %.0f GB/s from %s); classical = ops_per_madd*m*l*n/(P64*t) "
                        "(BJ:5 literal; > 1 possible for Strassen/Winograd)" % (hbm_peak / 1e9, hbm_src)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "bitwise_vs_1gpu": bitwise,
            "band_schedule_model": bandm,
            "variants": variants,
            "paper_context": PAPER_CONTEXT.get(args.workload),
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()   # rank 0's oracle sample and print are done before anyone tears down
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
