"""Golden worked examples (tests/golden/spec_examples.json, each with its SPEC/PAPER citation)."""
import json
import os

import numpy as np

import ddqd_inputs as gen

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_golden_efts(orc):
    for a, b, s, e in G["two_sum"]["cases"]:
        S, E = orc.two_sum(np.array([a]), np.array([b]))
        assert (S[0], E[0]) == (s, e)
    for a, b, p, e in G["two_prod"]["cases"]:
        P, E = orc.two_prod(np.array([a]), np.array([b]))
        assert (P[0], E[0]) == (p, e)


def test_golden_int_product(orc):
    g = G["int_product_2x2"]
    for W in (2, 4):
        A = np.zeros((W, 2, 2)); A[0] = g["A"]
        B = np.zeros((W, 2, 2)); B[0] = g["B"]
        for algo in ("block", "strassen", "winograd"):
            assert orc.gemm(A, B, algo, 1)[0].tolist() == g["C"]


def test_golden_bench_pair():
    for n, i, S in G["bench_pair_S"]["cases"]:
        assert gen.bench_pair_exact(n, i) == S


def test_golden_count_law(orc):
    for n, T, madds in G["count_law"]["cases"]:
        A = gen.dd_matrix(n, n, 1, 0)
        orc.reset_counters()
        orc.gemm(A, A, "winograd", T)
        assert orc.counters()[0] == madds
