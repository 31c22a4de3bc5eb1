"""Mutation check of the oracle's pins (test infrastructure; CPU only).

Each mutation is a plausible mistake in an oracle function; the pinned -m "not gpu" tests
must fail on every one of them. The oracle source is restored (and rebuilt) afterwards.
    python tools/oracle_mutation_check.py   -> one line per mutation: CAUGHT / MISSED
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "ddqd_oracle.c")
TESTS = ["tests/test_oracle_lu.py", "tests/test_oracle_arith.py", "tests/test_oracle_gemm.py"]

MUTATIONS = [
    ("qd_abs_gt: no sign fold",
     "qd_t ax = x.w[0] >= 0.0 ? x : qd_neg(x);\n    qd_t ay = y.w[0] >= 0.0 ? y : qd_neg(y);",
     "qd_t ax = x; qd_t ay = y;"),
    ("qd_abs_gt: per-word fabs instead of a fold",
     "qd_t ax = x.w[0] >= 0.0 ? x : qd_neg(x);\n    qd_t ay = y.w[0] >= 0.0 ? y : qd_neg(y);",
     "qd_t ax = x, ay = y; for (int k_ = 0; k_ < 4; k_++) { ax.w[k_] = fabs(x.w[k_]); "
     "ay.w[k_] = fabs(y.w[k_]); }"),
    ("qd_abs_gt: only the two leading words compared",
     "for (int i = 0; i < 4; i++)\n        if (ax.w[i] != ay.w[i])",
     "for (int i = 0; i < 2; i++)\n        if (ax.w[i] != ay.w[i])"),
    ("dd_abs_gt: no sign fold",
     "dd_t ax = x.hi >= 0.0 ? x : dd_neg(x);\n    dd_t ay = y.hi >= 0.0 ? y : dd_neg(y);",
     "dd_t ax = x; dd_t ay = y;"),
    ("qd_mul: a3*b0 dropped from the O(eps^3) tail",
     "    tail = tail + a.w[3] * b.w[0];\n    tail = tail + q0;",
     "    tail = tail + q0;"),
    ("qd_mul: q4 (error of a1*b1) dropped",
     "    tail = tail + q4;\n    tail = tail + q5;\n    s1 = s1 + tail;\n    return qd_renorm(p0, p1, s0, s1, s2);\n}\n\nstatic qd_t qd_madd(",
     "    tail = tail + q5;\n    s1 = s1 + tail;\n    return qd_renorm(p0, p1, s0, s1, s2);\n}\n\nstatic qd_t qd_madd("),
    ("qd_mul: second ThreeSum fed the wrong operand (q1 -> q0)",
     "    three_sum(&p2, &q1, &q2);\n    three_sum(&p3, &p4, &p5);\n    two_sum(p2, p3, &s0, &t0);\n    two_sum(q1, p4, &s1, &t1);\n    s2 = q2 + p5;\n    two_sum(s1, t0, &s1, &t0);\n    s2 = s2 + (t0 + t1);\n    tail = a.w[0] * b.w[3];",
     "    three_sum(&p2, &q0, &q2);\n    three_sum(&p3, &p4, &p5);\n    two_sum(p2, p3, &s0, &t0);\n    two_sum(q1, p4, &s1, &t1);\n    s2 = q2 + p5;\n    two_sum(s1, t0, &s1, &t0);\n    s2 = s2 + (t0 + t1);\n    tail = a.w[0] * b.w[3];"),
    ("qd_add: t3 dropped from the final tail",
     "    t0 = (t0 + t1) + t3;\n    return qd_renorm(s0, s1, s2, s3, t0);",
     "    t0 = (t0 + t1);\n    return qd_renorm(s0, s1, s2, s3, t0);"),
    ("qd_add: ThreeSum2 with a sign error",
     "    *b = t2 + t3;",
     "    *b = t2 - t3;"),
    ("qd_renorm: last word's t4 fold dropped",
     "            if (s3 != 0.0) s3 = s3 + t4;",
     "            if (s3 != 0.0) s3 = s3;"),
    ("dd_mul: cross term x.lo*y.hi dropped",
     "    t = (x.hi * y.lo) + (x.lo * y.hi);\n    e = e + t;\n    fast_two_sum(p, e, &r.hi, &r.lo);",
     "    t = (x.hi * y.lo);\n    e = e + t;\n    fast_two_sum(p, e, &r.hi, &r.lo);"),
    ("dd_add: low words not added",
     "    t = x.lo + y.lo;\n    e = e + t;",
     "    t = x.lo;\n    e = e + t;"),
    ("or_lu_solve: y := P b with the swaps in reverse order",
     "    for (int64_t k = 0; k < n; k++) {\n        int64_t r = ipiv[k];\n        if (r != k)",
     "    for (int64_t k = n - 1; k >= 0; k--) {\n        int64_t r = ipiv[k];\n        if (r != k)"),
    ("or_lu_solve: no permutation of b",
     "        int64_t r = ipiv[k];\n        if (r != k)\n            for (int w = 0; w < W; w++) {",
     "        int64_t r = ipiv[k];\n        if (0 && r != k)\n            for (int w = 0; w < W; w++) {"),
]


def main() -> int:
    orig = open(SRC).read()
    missed = 0
    try:
        for name, old, new in MUTATIONS:
            assert orig.count(old) >= 1, name
            open(SRC, "w").write(orig.replace(old, new, 1))     # the first (canonical) occurrence
            subprocess.check_call([sys.executable, "-c", "import oracle; oracle.build(force=True)"],
                                  cwd=ROOT)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", *TESTS], cwd=ROOT,
                               capture_output=True, text=True)
            caught = r.returncode != 0
            missed += not caught
            first = next((ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")), "")
            print(f"{'CAUGHT' if caught else 'MISSED'}  {name}  {first}")
    finally:
        open(SRC, "w").write(orig)
        subprocess.check_call([sys.executable, "-c", "import oracle; oracle.build(force=True)"], cwd=ROOT)
    return 1 if missed else 0


if __name__ == "__main__":
    sys.exit(main())
