"""The CPU oracle (oracle/tsg_oracle.c) is pinned to the reference: every
output below was produced by the reference package itself
(tests/golden/make_golden.py) and must be reproduced bit for bit, including
first-touch column order and fp64 summation order."""

import numpy as np

from conftest import gcm, gcsr, golden
from oracle import oracle as O


def test_compress_symbolic_numeric_match_reference():
    _, meta = golden()
    arrs, _ = golden()
    for k in range(meta["pairs"]):
        a, b = gcsr("pair%d/a" % k), gcsr("pair%d/b" % k)
        cb = O.compress(b)
        for got, want in zip(cb, gcm("pair%d/cb" % k)):
            assert np.array_equal(got, want)
        counts = O.symbolic(a, cb, workers=3)
        assert np.array_equal(counts, arrs["pair%d/counts" % k])
        c = gcsr("pair%d/c" % k)
        ptr, col, val = O.numeric(a, b, counts, workers=2)
        assert np.array_equal(ptr, c.row_ptr)
        assert np.array_equal(col, c.col_idx)                      # first-touch order
        assert np.array_equal(val.view(np.uint64), c.values.view(np.uint64))


def test_fused_sequence_matches_reference():
    from paper_1804_00695_b200.csr import CsrMatrix, slice_rows
    _, meta = golden()
    for k in range(meta["fused"]):
        a, b = gcsr("fused%d/a" % k), gcsr("fused%d/b" % k)
        lo_a, hi_a = meta["fused%d" % k]["a_rows"]
        cuts = meta["fused%d" % k]["cuts"]
        part = CsrMatrix.empty(hi_a - lo_a, b.num_cols)
        for j in range(3):
            lo, hi = cuts[j], cuts[j + 1]
            ptr, col, val = O.fused(a, slice_rows(b, lo, hi), part, lo_a, hi_a, lo, hi)
            want = gcsr("fused%d/step%d" % (k, j))
            assert np.array_equal(ptr, want.row_ptr)
            assert np.array_equal(col, want.col_idx)
            assert np.array_equal(val.view(np.uint64), want.values.view(np.uint64))
            part = CsrMatrix(hi_a - lo_a, b.num_cols, ptr, col, val)


def test_masked_count_matches_reference():
    _, meta = golden()
    for k, want in enumerate(meta["triangles"]):
        l = gcsr("tri%d/l" % k)
        assert O.masked_count(l, gcm("tri%d/cl" % k), workers=4) == want
        assert O.masked_count(l, O.compress(l)) == want
        assert want == meta["triangles_total"][k]


def test_config_shaped_products_match_reference():
    lap = gcsr("stencil/laplace2d")
    c = gcsr("config1_32/c")
    ptr, col, val = O.multiply(lap, lap)
    assert np.array_equal(ptr, c.row_ptr) and np.array_equal(col, c.col_idx)
    assert np.array_equal(val, c.values)
    a, p, ra, rap = (gcsr("config2_8/" + n) for n in ("a", "p", "ra", "rap"))
    from paper_1804_00695_b200.csr import transpose
    r = transpose(p)
    got = O.multiply(r, a)
    assert np.array_equal(got[1], ra.col_idx) and np.array_equal(got[2], ra.values)
    got = O.multiply(ra, p)
    assert np.array_equal(got[1], rap.col_idx) and np.array_equal(got[2], rap.values)


def test_count_multiplications():
    _, meta = golden()
    for k in range(meta["pairs"]):
        a, b = gcsr("pair%d/a" % k), gcsr("pair%d/b" % k)
        want = int(np.diff(b.row_ptr)[a.col_idx].sum()) if a.nnz else 0
        assert O.count_multiplications(a, b) == want


def test_worker_independence():
    a, b = gcsr("pair3/a"), gcsr("pair3/b")
    cb = O.compress(b)
    c1 = O.numeric(a, b, O.symbolic(a, cb, 1), 1)
    c7 = O.numeric(a, b, O.symbolic(a, cb, 7), 7)
    for x, y in zip(c1, c7):
        assert np.array_equal(x, y)
