"""Per-class LU times (live profile) of the c4 matrix (n = 4096, Strassen T = 128) for several
panel widths: how the panel factorisation's cost depends on its width (different bits for
different widths; a measurement aid, not a parity case)."""
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
for K in (256, 128, 64, 32):
    for _ in range(2):
        d.lu_solve(A0, b, panel=K)
    torch.cuda.synchronize()
    d.profile_start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        d.lu_solve(A0, b, panel=K)
    e1.record()
    torch.cuda.synchronize()
    d.profile_stop()
    pk = d.profile_kernels()
    print(K, "ms/solve", round(e0.elapsed_time(e1) / 3, 3),
          {k[:40]: round(v[1] / 3, 3) for k, v in sorted(pk.items(), key=lambda kv: -kv[1][1])[:6]})
