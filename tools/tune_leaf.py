"""Leaf-GEMM tile-configuration sweep (run on a B200): times ddqd_gemm_ex Block on a batch of
c3-sized DD leaves (256x257x256) and c2-sized QD leaves (128^3) for each DDQD_LEAF_CFG in a
fresh process, checks every configuration against the default bits, prints TFLOP/s (FP64 ops)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, sys, torch, numpy as np
sys.path.insert(0, %(root)r)
import ddqd_inputs as gen, paper_1510_08642_b200 as d
W, batch, m, l, n = %(W)d, %(batch)d, %(m)d, %(l)d, %(n)d
A = torch.from_numpy(gen.matrix(W, batch * m, l, 1, 0)).cuda().reshape(W, batch, m, l).permute(1, 0, 2, 3).contiguous()
B = torch.from_numpy(gen.matrix(W, batch * l, n, 1, 1)).cuda().reshape(W, batch, l, n).permute(1, 0, 2, 3).contiguous()
C = torch.empty((batch, W, m, n), dtype=torch.float64, device="cuda")
for _ in range(3): d.gemm_batched(A, B, C, "block", 1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): d.gemm_batched(A, B, C, "block", 1)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
ops = {2: 20, 4: 200}[W] * batch * m * l * n
peak = d.fp64_peak("dadd")[0]
np.save(%(out)r, C[:4].cpu().numpy())
print(json.dumps({"ms": ms, "tops": ops / ms / 1e9, "frac": ops / (ms * 1e-3) / peak}))
'''


def run(cfg, W, batch, m, l, n):
    out = f"/tmp/tune_{W}_{cfg}.npy"
    code = CHILD % dict(root=ROOT, W=W, batch=batch, m=m, l=l, n=n, out=out)
    env = dict(os.environ)
    if cfg is not None:
        env["DDQD_LEAF_CFG"] = str(cfg)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    if r.returncode:
        return {"error": r.stderr[-400:]}, None
    import numpy as np
    return json.loads(r.stdout.strip().splitlines()[-1]), np.load(out)


def main():
    import numpy as np
    res = {}
    for W, cfgs, shape in ((2, [None, 0, 1, 2, 3, 4, 5, 6], (686, 256, 257, 256)),
                           (4, [None, 10, 11, 12, 13], (343, 128, 128, 128))):
        ref = None
        for c in cfgs:
            r, C = run(c, W, *shape)
            if C is not None:
                if ref is None:
                    ref = C
                r["bitwise_equal_default"] = bool(np.array_equal(C.view(np.int64), ref.view(np.int64)))
            res[f"W{W}_cfg{c}"] = r
            print(W, c, r, flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
