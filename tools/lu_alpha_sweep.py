"""The paper's LU experiment (PAPER.md s.4) on one B200.

Random matrix with entries in [-1, 1] (the seeded DD/QD recipe of BJ:7/BJ:9, no
shift), n = 1024, true solution x = [0, 1, ..., n-1]^T and b := A x (b formed by the
library's Block GEMM), pivot-free blocked LU with block size K = alpha * n_min,
alpha = 1..10, n_min = 32, trailing update by Winograd(n_min);
DD and QD. Reports the time (CUDA events, median of 3) and the maximum relative error of
x (components with x_i = 0 are normalised by ||x||_inf), next to the paper's
8-thread times: DD 4.3 s at alpha = 2 (row-wise 13.0 s), QD 23.4 s at alpha = 5
(row-wise 56 s). Also runs the pivoted variant at the best alpha for comparison, and the
row-wise parallel (unblocked) LU the paper compares against: one panel K = n, i.e.
every column's pivot/scale/rank-1 update over all rows in parallel with no GEMM (DESIGN.md
reading R20).

    python tools/lu_alpha_sweep.py [--n 1024] [--out profiles/r01/lu_alpha_sweep.md]
"""
import argparse
import json
import os
import statistics
import sys
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def max_rel_err(xw, n):
    """max_i |x_i - i| / |i| (|x_i - 0| / ||x||_inf for i = 0), exact over the words."""
    import numpy as np
    worst = Fraction(0)
    norm = Fraction(n - 1)
    for i in range(n):
        v = sum((Fraction(float(w)) for w in xw[:, i]), Fraction(0))
        e = abs(v - i) / (Fraction(i) if i else norm)
        worst = max(worst, e)
    return float(worst)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "lu_alpha_sweep.md"))
    args = ap.parse_args()
    import numpy as np
    import torch

    import ddqd_inputs as gen
    import paper_1510_08642_b200 as ddqd

    n, nmin = args.n, 32
    rows, recs = [], []
    for W, prec in ((2, "DD"), (4, "QD")):
        A0 = torch.from_numpy(gen.matrix(W, n, n, 6, 0)).cuda()
        xt = torch.zeros((W, n, 1), dtype=torch.float64, device="cuda")
        xt[0, :, 0] = torch.arange(n, dtype=torch.float64)
        b = ddqd.gemm(A0, xt, "block")[:, :, 0].contiguous()
        runs = [(alpha, False) for alpha in range(1, 11)] + [(2 if W == 2 else 5, True), ("row-wise", False)]
        for alpha, pivot in runs:
            K = n if alpha == "row-wise" else alpha * nmin
            ts = []
            for rep in range(4):
                A = A0.clone()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                x, LU, piv, info = ddqd.lu_solve(A, b, panel=K, algo="winograd", threshold=nmin,
                                                 pivot=pivot, overwrite=True)
                e1.record()
                torch.cuda.synchronize()
                if rep:
                    ts.append(e0.elapsed_time(e1) * 1e-3)
            t = statistics.median(ts)
            err = max_rel_err(x.cpu().numpy(), n) if info == 0 else float("nan")
            rec = {"prec": prec, "n": n, "alpha": alpha, "K": K, "pivot": pivot, "info": info,
                   "seconds": t, "gflops": 2.0 / 3.0 * n ** 3 / t / 1e9, "max_rel_err": err}
            recs.append(rec)
            print(json.dumps(rec), flush=True)
            rows.append(f"| {prec} | {alpha} | {K} | {'partial' if pivot else 'none (paper)'} | "
                        f"{t * 1e3:.2f} | {rec['gflops']:.1f} | {err:.2e} |")
    txt = (f"# Paper s.4 LU experiment on one B200 (n = {n}, random matrix, x = [0..n-1], "
           "Winograd(32) update)\n\n"
           "Paper (Xeon E5-2620 v2, 8 threads, P:164): DD 4.3 s at alpha = 2 (row-wise LU 13.0 s); "
           "QD 23.4 s at alpha = 5 (row-wise 56 s). Error = max_i |x_i - i| / i (x_0 by ||x||_inf).\n\n"
           "| prec | alpha | K | pivoting | B200 ms | GFLOP/s (2n^3/3) | max rel err |\n"
           "|---|---|---|---|---|---|---|\n" + "\n".join(rows) + "\n")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        f.write(txt)
    print(txt)


if __name__ == "__main__":
    main()
