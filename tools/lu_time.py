"""Time one LU solve configuration on the GPU (device events, after warm-up): W n panel algo T.
Used for A/B measurements of the panel schedules (DDQD_LU_SPLIT, DDQD_LU_SUB_OVERLAP, ...)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ddqd_inputs as gen  # noqa: E402
import paper_1510_08642_b200 as d  # noqa: E402

W, n, K, algo, T = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
A = gen.matrix(W, n, n, 5, 0)
A[0, np.arange(n), np.arange(n)] += n
A0 = torch.from_numpy(A).cuda()
b = torch.zeros((W, n), dtype=torch.float64, device="cuda")
b[0] = 1.0
for _ in range(2):
    x, LU, piv, info = d.lu_solve(A0.clone(), b, panel=K, algo=algo, threshold=T)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    Ac = A0.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, LU, piv, info = d.lu_solve(Ac, b, panel=K, algo=algo, threshold=T, overwrite=True)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"W={W} n={n} K={K} {algo}({T}) split={os.environ.get('DDQD_LU_SPLIT', '1')}: "
      f"{min(ts):.3f} ms (info {info})")
