"""Times the DD (or QD: second argument 4) n = 1025 threshold-32 Strassen/Winograd GEMM (fused last level, 17^3 leaves)
under the DDQD_FUSED_S variant in the environment and writes C for a bitwise comparison.
    DDQD_FUSED_S=v python tools/fused_s_case.py out.npy"""
import sys
import numpy as np
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import ddqd_inputs as gen
import paper_1510_08642_b200 as d

outs = []
W = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cases = (("strassen", 1025), ("winograd", 1025), ("strassen", 1100), ("winograd", 1500), ("strassen", 1900))
for algo, n in (cases if W == 2 else cases[:3]):
    A, B = gen.bench_pair(n, W)
    a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    C = d.gemm(a, b, algo, 32)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        d.gemm(a, b, algo, 32, out=C)
    d.profile_start()
    e0.record()
    for _ in range(10):
        d.gemm(a, b, algo, 32, out=C)
    e1.record()
    torch.cuda.synchronize()
    d.profile_stop()
    pk = d.profile_kernels()
    leaf = {k: round(v[1] / 10, 4) for k, v in pk.items() if v[0] == 0}
    print(algo, n, "ms/step", round(e0.elapsed_time(e1) / 10, 4), leaf)
    outs.append(C.cpu().numpy().ravel())
np.save(sys.argv[1], np.concatenate(outs))
