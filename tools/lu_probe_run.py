"""One c4-shaped DD LU solve (n = 4096, panel 256, Strassen(128) update) on cuda:0, for
profiler runs (DDQD_LU_PROBE=1 phase report, ncu captures of the LU kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ddqd_inputs as gen  # noqa: E402
import paper_1510_08642_b200 as ddqd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
A = torch.from_numpy(gen.lu_matrix(n, 5)).cuda()
b = torch.zeros(2, n, dtype=torch.float64, device="cuda")
b[0] = 1
x, LU, piv, info = ddqd.dd_lu_solve(A.clone(), b, panel=256, algo="strassen", threshold=128)
torch.cuda.synchronize()
print("info", info)
