import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import ddqd_inputs as gen, paper_1510_08642_b200 as ddqd
n = 4096
L = gen.lu_matrix(n, 5)
A = torch.from_numpy(L).cuda()
b = torch.zeros(2, n, dtype=torch.float64, device='cuda'); b[0] = 1
x, LU, piv, info = ddqd.dd_lu_solve(A.clone(), b, panel=256, algo="strassen", threshold=128)
torch.cuda.synchronize()
