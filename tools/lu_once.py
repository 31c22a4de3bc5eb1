"""One c4-shaped LU solve (n = 4096 by default, panel 256, Strassen T = 128) after one warm-up:
a small driver for ncu captures of the LU kernels."""
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ddqd_inputs as gen
import paper_1510_08642_b200 as d

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
A0 = torch.from_numpy(gen.lu_matrix(n, 5)).cuda()
b = torch.ones((2, n), dtype=torch.float64, device="cuda")
b[1] = 0
for _ in range(2):
    x, LU, piv, info = d.lu_solve(A0, b)
torch.cuda.synchronize()
print("info", info, "max|x-1|", float((x[0] - 1).abs().max()))
