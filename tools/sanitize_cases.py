"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family once on small shapes -- TMA leaf (aligned), cp.async leaf (odd ld),
32x32 leaf, QD leaf, Strassen/Winograd pre/post adds, batched gemm_ex with beta = 1, the
cooperative LU panel (DD and QD, pivoted and pivot-free), the per-column LU path, solves."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import ddqd_inputs as gen
    import paper_1510_08642_b200 as d

    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()   # noqa: E731
    A = cu(gen.dd_matrix(130, 96, 1, 0)); B = cu(gen.dd_matrix(96, 200, 1, 1))
    d.dd_gemm(A, B, "block")                                  # TMA leaf (even strides)
    A2 = cu(gen.dd_matrix(131, 97, 2, 0)); B2 = cu(gen.dd_matrix(97, 199, 2, 1))
    d.dd_gemm(A2, B2, "block")                                # cp.async leaf (odd ld)
    d.dd_gemm(A2, B2, "winograd", 16)
    d.dd_gemm(A2, B2, "strassen", 16, madd="fused")
    d.dd_gemm(cu(gen.dd_matrix(20, 20, 3, 0)), cu(gen.dd_matrix(20, 20, 3, 1)), "block")   # 32x32 leaf
    Q = cu(gen.qd_matrix(70, 50, 4, 0)); Q2 = cu(gen.qd_matrix(50, 66, 4, 1))
    d.qd_gemm(Q, Q2, "winograd", 16)
    for W, piv in ((2, True), (2, False), (4, True)):
        n = 160
        M = gen.matrix(W, n, n, 5, 0)
        M[0, np.arange(n), np.arange(n)] += n
        b = gen.matrix(W, 1, n, 5, 1)[:, 0, :].copy()
        d.lu_solve(cu(M), cu(b), panel=48, algo="strassen", threshold=16, pivot=piv)
    torch.cuda.synchronize()
    print("sanitize cases done; kernels launched:", d.launch_count())


if __name__ == "__main__":
    main()
