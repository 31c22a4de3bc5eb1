import sys, torch
sys.path.insert(0, "/root/repo")
import ddqd_inputs as gen, paper_1510_08642_b200 as d
n, T, W = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
A, B = gen.bench_pair(n, W)
a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
for _ in range(3):
    C = d.gemm(a, b, "strassen", T)
torch.cuda.synchronize()
d.profile_start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    C = d.gemm(a, b, "strassen", T, out=C)
e1.record(); torch.cuda.synchronize()
pr = d.profile_stop()
pk = max(d.fp64_peak("dadd")[0], d.fp64_peak("dfma")[0])
ops = 20 if W == 2 else 200
print("ms/step", e0.elapsed_time(e1) / 5, {k: (round(v[0] / 5, 3), int(v[1] / 5)) for k, v in pr.items() if v[1]},
      "leaf frac", ops * pr["leaf"][2] / (pr["leaf"][0] * 1e-3) / pk)
