"""One c4-recipe LU solve (n = 4096, panel 256, Strassen(128)) for ncu captures of single LU kernels."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ddqd_inputs as gen  # noqa: E402
import paper_1510_08642_b200 as d  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
A = torch.from_numpy(gen.lu_matrix(n, 5)).cuda()
b = torch.zeros((2, n), dtype=torch.float64, device="cuda")
b[0] = 1.0
x, LU, piv, info = d.lu_solve(A, b, panel=256, algo="strassen", threshold=128)
torch.cuda.synchronize()
print("info", int(info), "x0", float(x[0, 0].cpu()))
