"""Host logic of the band schedule (paper_1510_08642_b200/mgpu.py BandGemm; DESIGN.md reading
R21), checked with the oracle alone (CPU, no processes): a (row band x column band) tile of C,
computed from the packed operands with the whole problem's recursion depth, equals those rows
and columns of the whole product bit for bit -- for every band of every grid."""
import numpy as np
import pytest

import ddqd_inputs as gen
from paper_1510_08642_b200.mgpu import balanced_slices, band_grid, band_index_map, rec_shapes


def test_index_map_structure():
    """11 -> 6 -> 3 -> 2: the two depth-3 bands partition the rows, each level-0 set is the
    quadrant map of numerics.md s.4 applied upward, and the padded row (6 + 5 = 11) is absent."""
    dims = [11, 6, 3, 2]
    maps = [band_index_map(dims, a, b) for a, b in balanced_slices(2, 2)]
    assert sorted(maps[0] + maps[1]) == list(range(11))
    # leaf row 0 -> {0, 2} -> {0, 2, 3, 5} -> {0, 2, 3, 5, 6, 8, 9} (5 + 6 = 11 is the padding);
    # leaf row 1 -> {1} (1 + 2 = 3 is padding) -> {1, 4} -> {1, 4, 7, 10}
    assert maps[0] == [0, 2, 3, 5, 6, 8, 9] and maps[1] == [1, 4, 7, 10]
    for a, b in ((0, 1), (1, 2), (0, 2)):
        idx = band_index_map(dims, a, b)
        lev = set(range(a, b))
        for j in range(len(dims) - 2, -1, -1):
            lev = lev | {dims[j + 1] + r for r in lev if dims[j + 1] + r < dims[j]}
        assert set(idx) == lev and len(idx) == len(lev)


def test_compact_sizes_halve_with_ceil():
    """The compact size of a band at level j halves with ceil to its size at level j+1, so the
    forced-depth recursion of the compact problem visits exactly the band at every level."""
    for m in (1, 2, 7, 37, 64, 100, 8191):
        for d in range(0, 6):
            dims = [m]
            for _ in range(d):
                dims.append((dims[-1] + 1) // 2)
            for G in (1, 2, 3, 4, 8):
                for a, b in balanced_slices(dims[-1], G):
                    for j in range(d):
                        hj = len(band_index_map(dims[j:], a, b))
                        hj1 = len(band_index_map(dims[j + 1:], a, b))
                        assert (hj + 1) // 2 == hj1


def test_band_grid():
    assert band_grid(1) == (1, 1) and band_grid(2) == (1, 2) and band_grid(4) == (2, 2)
    assert band_grid(8) == (2, 4) and band_grid(6) == (2, 3) and band_grid(7) == (1, 7)


@pytest.mark.parametrize("W,algo,T,m,l,n,grid", [
    (2, "winograd", 4, 37, 29, 33, (2, 2)),
    (2, "strassen", 3, 40, 41, 42, (1, 3)),
    (2, "winograd", 2, 23, 19, 29, (3, 2)),
    (4, "strassen", 3, 21, 18, 25, (2, 2)),
    (2, "winograd", 8, 70, 65, 66, (2, 4)),     # 2 x 4: the 8-GPU grid
])
def test_tiles_equal_whole_product_bitwise(orc, W, algo, T, m, l, n, grid):
    A, B = gen.matrix(W, m, l, 41, 0), gen.matrix(W, l, n, 41, 1)
    ref = orc.gemm(A, B, algo, threshold=T)
    shapes = rec_shapes(m, l, n, T)
    d = len(shapes) - 1
    assert d >= 2
    mdims, ndims = [s[0] for s in shapes], [s[2] for s in shapes]
    C = np.full_like(ref, np.nan)
    for a, b in balanced_slices(mdims[-1], grid[0]):
        rows = band_index_map(mdims, a, b)
        for c0, c1 in balanced_slices(ndims[-1], grid[1]):
            cols = band_index_map(ndims, c0, c1)
            if not rows or not cols:
                continue
            tile = orc.gemm(np.ascontiguousarray(A[:, rows, :]), np.ascontiguousarray(B[:, :, cols]), algo,
                            threshold=1, depth=d)
            C[:, np.array(rows)[:, None], np.array(cols)[None, :]] = tile
    assert np.array_equal(C.view(np.int64), ref.view(np.int64))


def test_forced_depth_equals_stop_rule(orc):
    """DDQD_DEPTH(d) with d = the stop rule's depth is the stop rule's recursion, bitwise; a
    different depth is a different (still exact-within-bound) tree."""
    A, B = gen.matrix(2, 30, 27, 42, 0), gen.matrix(2, 27, 29, 42, 1)
    d = len(rec_shapes(30, 27, 29, 4)) - 1
    ref = orc.gemm(A, B, "winograd", threshold=4)
    assert np.array_equal(orc.gemm(A, B, "winograd", threshold=999, depth=d).view(np.int64), ref.view(np.int64))
    assert not np.array_equal(orc.gemm(A, B, "winograd", threshold=4, depth=d - 1), ref)
