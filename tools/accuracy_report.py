"""Accuracy of the device results against the EXACT product (run on a B200): for every
BASELINE config the max-norm error of sampled (or all) entries, computed with the oracle's
exact long accumulator, and its ratio to the BJ:5 bound (2^-96 l |A||B| for DD Block,
2^-200 l |A||B| for QD, widened by 18^d for depth-d Strassen/Winograd; SURVEY.md s.8(c.2)
asks for the measured error-to-bound ratio, not just pass/fail). Also the c4 solution error.

    python tools/accuracy_report.py [--out profiles/r01/accuracy.md]
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def depth(m, l, n, T):
    d = 0
    while min(m, l, n) > T:
        m, l, n = (m + 1) // 2, (l + 1) // 2, (n + 1) // 2
        d += 1
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "accuracy.md"))
    args = ap.parse_args()
    import numpy as np
    import torch

    import ddqd_inputs as gen
    import oracle as orc
    import paper_1510_08642_b200 as ddqd

    def cu(a):
        return torch.from_numpy(np.ascontiguousarray(a)).cuda()

    rows = []
    cases = [
        ("c0", 2, "block", 128, 128, 128, 128, 1, None),
        ("c1", 2, "strassen", 128, 1024, 1024, 1024, 2, 8192),
        ("c1 (Block)", 2, "block", 128, 1024, 1024, 1024, 2, 8192),
        ("c2", 4, "winograd", 128, 1024, 1024, 1024, 3, 1024),
        ("c3", 2, "winograd", 256, 8191, 8193, 8190, 4, 4096),
    ]
    rng = np.random.default_rng(5)
    for name, W, algo, T, m, l, n, seed, samples in cases:
        A = gen.matrix(W, m, l, seed, 0)
        B = gen.matrix(W, l, n, seed, 1)
        C = ddqd.gemm(cu(A), cu(B), algo, T).cpu().numpy()
        if samples is None:
            r, c = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
            r, c = r.ravel(), c.ravel()
        else:
            r = np.concatenate([rng.integers(0, m, samples), [0, m - 1]])
            c = np.concatenate([rng.integers(0, n, samples), [n - 1, 0]])
        _, err = orc.exact_entries(A, B, C, r, c)
        d = 0 if algo == "block" else depth(m, l, n, T)
        nA, nB = float(np.abs(A[0]).max()), float(np.abs(B[0]).max())
        bound = 18.0 ** d * 2.0 ** (-96 if W == 2 else -200) * l * nA * nB
        e = float(np.abs(err).max())
        rows.append(f"| {name} | {'DD' if W == 2 else 'QD'} {algo}(T={T}) {m}x{l}x{n} | d = {d} | "
                    f"{r.size} | {e:.3e} (2^{math.log2(e):.1f}) | {bound:.3e} | 2^{math.log2(e / bound):.1f} |")
        print(rows[-1], flush=True)
    # c4: the solution of A x = A 1
    n = 4096
    L = gen.lu_matrix(n, 5)
    gA = cu(L)
    ones = torch.zeros((2, n, 1), dtype=torch.float64, device="cuda"); ones[0] = 1.0
    b = ddqd.dd_gemm(gA, ones, "block")[:, :, 0].contiguous()
    x, LU, piv, info = ddqd.dd_lu_solve(gA, b, panel=256, algo="strassen", threshold=128)
    xx = x.cpu().numpy()
    xe = float(np.abs((xx[0] - 1.0) + xx[1]).max())
    xb = 2.0 ** -96 * n * 3 * 18
    rows.append(f"| c4 | DD LU n = 4096, panel 256, Strassen(128) update | x vs 1 | {n} | {xe:.3e} "
                f"(2^{math.log2(xe):.1f}) | {xb:.3e} (2^-96 n kappa 18, kappa <= 3) | 2^{math.log2(xe / xb):.1f} |")
    print(rows[-1])
    txt = ("# Accuracy of the B200 results against the exact product (BJ:5 bounds)\n\n"
           "Exact errors from the oracle's long accumulator (`oracle/exact.c`) on the device output; "
           "bound = 18^d 2^-96 l |A|max |B|max (DD) / 2^-200 (QD), SURVEY.md s.8(c.2).\n\n"
           "| config | problem | depth | entries checked | max exact error | BJ:5 bound | error / bound |\n"
           "|---|---|---|---|---|---|---|\n" + "\n".join(rows) + "\n")
    with open(args.out, "w") as f:
        f.write(txt)
    print(txt)


if __name__ == "__main__":
    main()
