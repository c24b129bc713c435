"""GPU parity: the sm_100a path through the C ABI vs the CPU oracle.

Bar (BASELINE.json north_star): row pointers and per-row sorted columns
bit-exact; fp64 values bit-exact for the thread-group tier (the reference's
summation order is replayed) and within rtol 1e-12 for CTA/global-tier rows;
integer results (triangle counts) exact.
"""

import numpy as np
import pytest

import paper_1804_00695_b200 as tsg
from paper_1804_00695_b200 import generators as gen
from paper_1804_00695_b200.csr import CsrMatrix, canonicalize, slice_rows
from oracle import oracle as O
from conftest import assert_same_product, random_csr

pytestmark = pytest.mark.gpu


def test_compress_matches_reference_first_touch_order(rng):
    for unsorted in (False, True):
        for _ in range(5):
            b = random_csr(rng, 300, 700, 40)
            if not unsorted:
                b = canonicalize(b)
            cm = tsg.compress(b)
            rp, s, bits = O.compress(b)
            assert np.array_equal(cm.row_ptr, rp)
            assert np.array_equal(cm.set_idx, s)
            assert np.array_equal(cm.set_bits, bits)


def test_compress_many_blocks_and_long_runs(rng):
    # > 8192 entries per compression block: runs crossing word and block
    # boundaries, a dense row spanning many blocks, empty rows between
    for dense in (False, True):
        b = canonicalize(random_csr(rng, 20000, 5000, 30))
        if dense:
            rows = np.concatenate([np.full(4000, 7), np.full(3000, 9)])
            cols = np.concatenate([np.arange(4000), rng.choice(5000, 3000, replace=False)])
            b = canonicalize(CsrMatrix.from_coo(rows, cols, np.ones(7000), 20, 5000))
        cm = tsg.compress(b)
        rp, s, bits = O.compress(b)
        assert np.array_equal(cm.row_ptr, rp)
        assert np.array_equal(cm.set_idx, s)
        assert np.array_equal(cm.set_bits, bits)


def test_compress_kats():
    def rows(rs, n):
        r = [i for i, cs in enumerate(rs) for _ in cs]
        c = [x for cs in rs for x in cs]
        return CsrMatrix.from_coo(r, c, np.ones(len(c)), len(rs), n)
    cm = tsg.compress(rows([[0, 63]], 64))
    assert cm.n_sets == 1 and cm.set_idx[0] == 0 and int(cm.set_bits[0]) == (1 | (1 << 63))
    cm = tsg.compress(rows([[0, 64]], 65))
    assert sorted(cm.set_idx.tolist()) == [0, 1]
    cm = tsg.compress(rows([[], [3]], 8))
    assert cm.row_ptr.tolist() == [0, 0, 1]


def test_symbolic_and_numeric_random_pairs(rng):
    for it in range(80):
        n = int(rng.integers(4, 120))
        a = random_csr(rng, n, n, 8 if it % 3 else 40)
        b = random_csr(rng, n, n, 8 if it % 4 else 90)
        if it % 2:   # row-sorted B: symbolic rows with <= 32 A entries take the merge tier
            b = canonicalize(b)
        cb = tsg.compress(b)
        counts = tsg.spgemm_symbolic(a, cb)
        want_counts = O.symbolic(a, O.compress(b))
        assert np.array_equal(counts, want_counts)
        c = tsg.spgemm_numeric(a, b, counts)
        assert_same_product(c, O.numeric(a, b, want_counts), exact=True)


def test_multiply_rectangular_and_empty_rows(rng):
    for _ in range(20):
        a = random_csr(rng, 90, 140, 12)
        b = random_csr(rng, 140, 3000, 30)
        assert_same_product(tsg.multiply(a, b), O.multiply(a, b), exact=True)


def test_multiply_many_rows_multi_tile_scans(rng):
    # > 16 K rows: the single-pass look-back scans run over many tiles
    a = random_csr(rng, 150000, 3000, 4)
    b = random_csr(rng, 3000, 4000, 6)
    assert_same_product(tsg.multiply(a, b), O.multiply(a, b), exact=True)


def test_numeric_with_host_counts(rng):
    a = random_csr(rng, 200, 200, 10)
    b = random_csr(rng, 200, 500, 10)
    want = O.symbolic(a, O.compress(b))
    c = tsg.spgemm_numeric(a, b, np.array(want))   # plain ndarray: no device set counts
    assert_same_product(c, O.numeric(a, b, want), exact=True)


def test_wrong_counts_raise_kernel_error(rng):
    a = random_csr(rng, 10, 10, 3, exact_delta=True)
    b = random_csr(rng, 10, 10, 3, exact_delta=True)
    counts = tsg.spgemm_symbolic(a, tsg.compress(b))
    bad = np.array(counts).copy()
    bad[0] += 1
    with pytest.raises(tsg.KernelError):
        tsg.spgemm_numeric(a, b, bad)


def test_dimension_and_value_errors():
    a = CsrMatrix(1, 3, [0, 1], [0], [1.0])
    b = CsrMatrix(2, 2, [0, 1, 2], [0, 0], [1.0, 1.0])
    with pytest.raises(tsg.DimensionError):
        tsg.spgemm_symbolic(a, tsg.compress(b))
    p = CsrMatrix(1, 1, [0, 1], [0], None)
    with pytest.raises(tsg.MatrixValidationError):
        tsg.spgemm_numeric(p, p, np.array([1]))


def test_config1_laplace2d_small_full():
    a = gen.stencil(gen.LAPLACE2D, (64, 64))
    assert_same_product(tsg.multiply(a, a), O.multiply(a, a), exact=True)


def test_config2_rap_small_full():
    a = gen.stencil(gen.BRICK3D, (16, 16, 16))
    p, r = gen.aggregation((16, 16, 16))
    ra = tsg.multiply(r, a)
    ra_o = O.multiply(r, a)
    assert_same_product(ra, ra_o, exact=True)
    rap = tsg.multiply(ra, p)
    ra_host = CsrMatrix(r.num_rows, a.num_cols, *ra_o)
    assert_same_product(rap, O.multiply(ra_host, p), exact=True)


def test_fused_full_range_equals_plain(rng):
    a = random_csr(rng, 30, 40, 5)
    b = random_csr(rng, 40, 35, 5)
    plain = tsg.multiply(a, b)
    fused = tsg.spgemm_numeric_fused(a, b, CsrMatrix.empty(30, 35), tsg.RowRange(0, 30),
                                     tsg.RowRange(0, 40))
    assert np.array_equal(fused.row_ptr, plain.row_ptr)
    assert np.array_equal(fused.col_idx, plain.col_idx)
    assert np.array_equal(fused.values, plain.values)


def test_fused_chunk_sequence_matches_oracle(rng):
    for _ in range(10):
        a = random_csr(rng, 80, 90, 9)
        b = random_csr(rng, 90, 120, 9)
        part = CsrMatrix.empty(50, 120)
        opart = part
        for lo, hi in ((0, 31), (31, 60), (60, 90)):
            chunk = slice_rows(b, lo, hi)
            part = tsg.spgemm_numeric_fused(a, chunk, part, tsg.RowRange(20, 70),
                                            tsg.RowRange(lo, hi))
            o = O.fused(a, chunk, opart, 20, 70, lo, hi)
            assert_same_product(part, o, exact=True)
            opart = CsrMatrix(50, 120, *o)


def test_fused_empty_a_rows_returns_partial():
    a = CsrMatrix(2, 2, [0, 1, 2], [0, 1], [1.0, 1.0])
    empty_partial = CsrMatrix.empty(0, 2)
    out = tsg.spgemm_numeric_fused(a, slice_rows(a, 0, 1), empty_partial, tsg.RowRange(0, 0),
                                   tsg.RowRange(0, 1))
    assert out is empty_partial


def test_large_rows_cta_and_global_tiers(rng):
    # rows with thousands of outputs exercise the CTA tier; a dense-ish hub row
    # the global-memory tier.  Values stay within 1e-12 (order-free adds).
    n = 6000
    a_rows = [rng.choice(n, size=k, replace=False) for k in (3, 40, 400, 2500)]
    r = np.concatenate([np.full(len(x), i) for i, x in enumerate(a_rows)])
    a = CsrMatrix.from_coo(r, np.concatenate(a_rows), rng.uniform(0.1, 1, len(r)), 4, n)
    b = random_csr(rng, n, 200000, 60)
    for bb in (b, canonicalize(b)):   # row-sorted B: hub rows also take the dense numeric tier
        c = tsg.multiply(a, bb)
        assert_same_product(c, O.multiply(a, bb), exact=False, rtol=1e-12)


def test_integer_valued_big_rows_exact(rng):
    n = 3000
    b = random_csr(rng, n, 100000, 50)
    b = CsrMatrix(b.num_rows, b.num_cols, b.row_ptr, b.col_idx, np.round(b.values * 8))
    a = CsrMatrix.from_coo(np.zeros(n, np.int64), np.arange(n), np.ones(n), 1, n)
    assert_same_product(tsg.multiply(a, b), O.multiply(a, b), exact=True)


def test_masked_count_random_graphs(rng):
    for _ in range(10):
        n = int(rng.integers(20, 300))
        up = np.triu(rng.random((n, n)) < 0.1, 1)
        rows, cols = np.nonzero(up | up.T)
        keep = rows > cols
        l = CsrMatrix.from_coo(rows[keep], cols[keep], None, n, n)
        want = O.masked_count(l, O.compress(l))
        assert tsg.masked_row_intersect_count(l, tsg.compress(l)) == want


def test_masked_count_kats_and_lower_check():
    def lower(edges, n):
        return CsrMatrix.from_coo([max(u, v) for u, v in edges], [min(u, v) for u, v in edges],
                                  None, n, n)
    k4 = lower([(i, j) for i in range(4) for j in range(i + 1, 4)], 4)
    assert tsg.masked_row_intersect_count(k4, tsg.compress(k4)) == 4
    path = lower([(0, 1), (1, 2), (2, 3)], 4)
    assert tsg.masked_row_intersect_count(path, tsg.compress(path)) == 0
    bad = CsrMatrix.from_coo([0], [1], None, 2, 2)
    with pytest.raises(tsg.MatrixValidationError):
        tsg.masked_row_intersect_count(bad, tsg.compress(bad))


def test_masked_count_rmat_scale12():
    g = gen.rmat_graph(12)
    deg = np.diff(g.row_ptr)
    perm = np.lexsort((np.arange(g.num_rows), deg))
    pos = np.empty_like(perm)
    pos[perm] = np.arange(g.num_rows)
    rows = pos[np.repeat(np.arange(g.num_rows), deg)]
    cols = pos[g.col_idx]
    keep = rows > cols
    l = CsrMatrix.from_coo(rows[keep], cols[keep], None, g.num_rows, g.num_rows)
    want = O.masked_count(l, O.compress(l), workers=8)
    assert tsg.masked_row_intersect_count(l, tsg.compress(l)) == want


def test_count_multiplications(rng):
    a = random_csr(rng, 25, 30, 5)
    b = random_csr(rng, 30, 20, 5)
    assert tsg.count_multiplications(a, b) == O.count_multiplications(a, b)


def test_placement_policies_same_product(rng):
    """Data placement (memory.py:193-223): every operand placement gives the
    same product; slow-tier operands are read/written in mapped host memory."""
    from paper_1804_00695_b200.memory import PlacementPolicy
    a = random_csr(rng, 300, 400, 12)
    b = random_csr(rng, 400, 500, 12)
    want = O.multiply(a, b)
    for name in ("all_fast", "b_in_fast", "all_slow"):
        assert_same_product(tsg.multiply(a, b, placement=name), want, exact=True)
    pol = PlacementPolicy("c_pin", {"A": "fast", "B": "fast", "C": "slow"})
    assert_same_product(tsg.multiply(a, b, placement=pol), want, exact=True)


def test_sharded_b_gather_matches_replicated(rng):
    """B sharded (§8e): the rows A selects are gathered straight from the
    shards' device memory (peer HBM on multi-GPU, three local shards here);
    the product equals the one with a replicated B, bit for bit."""
    import torch
    from paper_1804_00695_b200 import _lib, distributed as D
    a = random_csr(rng, 500, 900, 12)
    a_sub = random_csr(rng, 50, 900, 3)          # selects only some of B's rows
    b = random_csr(rng, 900, 700, 20)
    bounds = D.shard_bounds(np.diff(b.row_ptr), 3)
    shards = [(int(bounds[s]), int(bounds[s + 1])) +
              D.local_shard_tensors(b, int(bounds[s]), int(bounds[s + 1]), "cuda") for s in range(3)]
    torch.cuda.synchronize()
    for aa in (a, a_sub):
        da = _lib.DeviceCsr.upload(aa)
        db = D.gather_sharded(da, shards, b.num_cols)
        got = _lib.d_multiply(da, db).download()
        assert_same_product(got, O.multiply(aa, b), exact=True)


def test_masked_count_dense_hub_rows(rng):
    # hubs with thousands of lower neighbours take the dense bitmap tier
    n = 6000
    up = np.triu(rng.random((n, n)) < 0.002, 1)
    up[:3, 3:] = True                      # three hubs adjacent to everyone
    rows, cols = np.nonzero(up | up.T)
    g = CsrMatrix.from_coo(rows, cols, None, n, n)
    low = tsg.lower_triangle(g, tsg.degree_sort_permutation(g))
    want = O.masked_count(low, O.compress(low), workers=8)
    assert tsg.masked_row_intersect_count(low, tsg.compress(low)) == want
    assert tsg.count_triangles(g) == want


def test_masked_count_dense_rows_with_repeated_columns(rng):
    # L rows that repeat a column: the reference ORs L_j's columns into sets
    # (a repeat counts once inside L_j, but every entry of L_i counts), so the
    # dense tier must not test L_j's raw columns here
    n = 3000
    up = np.triu(rng.random((n, n)) < 0.01, 1)
    up[:2, 2:] = True
    rows, cols = np.nonzero(up | up.T)
    g = CsrMatrix.from_coo(rows, cols, None, n, n)
    low = tsg.lower_triangle(g, tsg.degree_sort_permutation(g))
    rp, ci = np.asarray(low.row_ptr), np.asarray(low.col_idx)
    r = np.repeat(np.arange(n), np.diff(rp))
    dup = rng.random(len(ci)) < 0.3                 # repeat 30 % of the entries
    r2 = np.concatenate([r, r[dup]])
    c2 = np.concatenate([ci, ci[dup]])
    order = np.lexsort((c2, r2))
    rp2 = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(r2, minlength=n), out=rp2[1:])
    ld = CsrMatrix(n, n, rp2, c2[order].astype(np.int64), None)
    want = O.masked_count(ld, O.compress(ld), workers=8)
    assert tsg.masked_row_intersect_count(ld, tsg.compress(ld)) == want


def test_empty_and_degenerate_shapes(rng):
    """Zero rows / columns / entries behave like the reference (empty results,
    no device errors), through every public entry point."""
    empty = CsrMatrix.empty
    cases = [(empty(0, 5), random_csr(rng, 5, 7, 3)),
             (random_csr(rng, 4, 5, 3), empty(5, 0)),
             (empty(3, 4), empty(4, 6)),
             (CsrMatrix.from_coo([0], [0], [2.5], 1, 1), CsrMatrix.from_coo([0], [0], [-4.0], 1, 1))]
    for a, b in cases:
        want = O.multiply(a, b)
        assert_same_product(tsg.multiply(a, b), want, exact=True)
        counts = tsg.spgemm_symbolic(a, tsg.compress(b))
        assert np.array_equal(np.asarray(counts), np.diff(want[0]))
        assert_same_product(tsg.spgemm_numeric(a, b, counts), want, exact=True)
        assert tsg.count_multiplications(a, b) == O.count_multiplications(a, b)
    z = empty(0, 0, pattern=True)
    assert tsg.count_triangles(z) == 0
    assert tsg.masked_row_intersect_count(empty(3, 3, pattern=True), tsg.compress(empty(3, 3, pattern=True))) == 0


def test_duplicate_columns_in_b_rows(rng):
    """Repeated columns inside a B row (legal in the reference: compress ORs
    them, numeric sums them in order) must not race in the lane-split mode."""
    a = random_csr(rng, 200, 300, 10)
    base = canonicalize(random_csr(rng, 300, 400, 30))
    rows = np.repeat(np.arange(300), np.diff(base.row_ptr))
    dup_r = np.concatenate([rows, rows[::3]])
    dup_c = np.concatenate([base.col_idx, base.col_idx[::3]])
    dup_v = np.concatenate([base.values, base.values[::3] * 0.5])
    b = CsrMatrix.from_coo(dup_r, dup_c, dup_v, 300, 400)   # sorted rows with adjacent repeats
    want = O.multiply(a, b)
    assert_same_product(tsg.multiply(a, b), want, exact=True)
    counts = tsg.spgemm_symbolic(a, tsg.compress(b))
    assert_same_product(tsg.spgemm_numeric(a, b, counts), want, exact=True)


# ---------------------------------------------------------------- input builders on the device

def _same_csr(got, want):
    assert (got.num_rows, got.num_cols) == (want.num_rows, want.num_cols)
    assert np.array_equal(got.row_ptr, want.row_ptr)
    assert np.array_equal(got.col_idx, want.col_idx)
    if want.values is None:
        assert got.values is None
    else:
        assert np.array_equal(got.values, want.values)


@pytest.mark.parametrize("kind,dims", [
    (gen.LAPLACE2D, (7, 5)), (gen.LAPLACE3D, (4, 5, 3)), (gen.BIGSTAR2D, (6, 7)),
    (gen.BRICK3D, (5, 4, 3)), (gen.BRICK3D, (1, 1, 1)), (gen.ELASTICITY3D, (3, 4, 2)),
    (gen.BIGSTAR2D, (2, 1))])
def test_device_stencil_equals_host_builder(kind, dims):
    _same_csr(gen.stencil_device(kind, dims).download(), gen.stencil(kind, dims))


def test_device_stencil_row_range_equals_stencil_rows():
    dims = (6, 5, 4)
    for lo, hi in ((17, 83), (0, 120), (119, 120), (40, 40)):
        _same_csr(gen.stencil_device(gen.BRICK3D, dims, lo, hi).download(),
                  gen.stencil_rows(gen.BRICK3D, dims, lo, hi))


def test_device_stencil_bad_dims_raise_like_host():
    with pytest.raises(tsg.GridError):
        gen.stencil_device(gen.BRICK3D, (4, 4))
    with pytest.raises(tsg.GridError):
        gen.stencil_device(gen.LAPLACE2D, (0, 3))


@pytest.mark.parametrize("dims,factor", [((5, 4, 3), 2), ((8, 8, 8), 2), ((5, 7), 3), ((9,), 4)])
def test_device_aggregation_equals_host_builder(dims, factor):
    p_want, r_want = gen.aggregation(dims, factor)
    dp, dr = gen.aggregation_device(dims, factor)
    _same_csr(dp.download(), p_want)
    _same_csr(dr.download(), r_want)


def test_device_transpose_equals_host():
    from paper_1804_00695_b200._lib import DeviceCsr
    from paper_1804_00695_b200.csr import transpose, transpose_device
    rng = np.random.default_rng(11)
    for rows, cols, delta in ((50, 40, 9), (300, 1000, 30), (1, 5, 5), (7, 3, 0)):
        m = random_csr(rng, rows, cols, delta)
        _same_csr(transpose_device(DeviceCsr.upload(m)).download(), transpose(m))
    pat = random_csr(rng, 60, 70, 8, values=False)
    _same_csr(transpose_device(DeviceCsr.upload(pat)).download(), transpose(pat))


def test_device_built_galerkin_product_matches_host_built():
    """R*A*P from operands built in HBM equals the product of the host-built ones."""
    from paper_1804_00695_b200 import kernel
    dims = (9, 8, 7)
    a = gen.stencil(gen.BRICK3D, dims)
    p, r = gen.aggregation(dims)
    want = kernel.multiply(kernel.multiply(r, a), p)
    da = gen.stencil_device(gen.BRICK3D, dims)
    dp, dr = gen.aggregation_device(dims)
    got = kernel.multiply_device(kernel.multiply_device(dr, da), dp).download()
    _same_csr(canonicalize(got), canonicalize(want))
    assert np.array_equal(got.values, want.values)   # same first-touch order, bit-exact


# ---------------------------------------------------------------- fused R*A*P

@pytest.mark.parametrize("dims", [(10, 9, 8), (7, 5, 3), (16, 16, 16)])
def test_fused_rap_bit_identical_to_two_multiplies(dims):
    from paper_1804_00695_b200 import kernel
    a = gen.stencil(gen.BRICK3D, dims)
    p, r = gen.aggregation(dims)
    want = kernel.multiply(kernel.multiply(r, a), p)
    dr, da, dp = kernel.upload(r), kernel.upload(a), kernel.upload(p)
    got, fused = kernel.rap_device(dr, da, dp)
    assert fused
    _same_csr(got.download(), want)
    # against the oracle restatement of the reference's two multiplies
    ra = O.multiply(r, a)
    ra_m = CsrMatrix(ra[0].shape[0] - 1, a.num_cols, ra[0], ra[1], ra[2])
    assert_same_product(canonicalize(got.download()), O.multiply(ra_m, p), exact=False)


def test_fused_rap_general_operands():
    from paper_1804_00695_b200 import kernel
    rng = np.random.default_rng(5)
    r = canonicalize(random_csr(rng, 40, 60, 5))
    a = canonicalize(random_csr(rng, 60, 70, 6))
    p = canonicalize(random_csr(rng, 70, 30, 3))
    want = kernel.multiply(kernel.multiply(r, a), p)
    got, fused = kernel.rap_device(kernel.upload(r), kernel.upload(a), kernel.upload(p))
    assert fused
    g = got.download()
    assert np.array_equal(g.row_ptr, want.row_ptr) and np.array_equal(g.col_idx, want.col_idx)
    np.testing.assert_allclose(g.values, want.values, rtol=1e-12, atol=0)


def test_fused_rap_falls_back_when_rows_do_not_fit():
    from paper_1804_00695_b200 import kernel
    rng = np.random.default_rng(6)
    r = canonicalize(random_csr(rng, 20, 300, 40, exact_delta=True))
    a = canonicalize(random_csr(rng, 300, 400, 60, exact_delta=True))
    p = canonicalize(random_csr(rng, 400, 500, 4))
    want = kernel.multiply(kernel.multiply(r, a), p)
    got, fused = kernel.rap_device(kernel.upload(r), kernel.upload(a), kernel.upload(p))
    assert not fused
    _same_csr(got.download(), want)
    # explicit two-multiply mode and the host entry point
    got2, fused2 = kernel.rap_device(kernel.upload(r), kernel.upload(a), kernel.upload(p), fused=False)
    assert not fused2
    _same_csr(got2.download(), want)
    _same_csr(kernel.rap(r, a, p), want)
    with pytest.raises(tsg.DimensionError):
        kernel.rap(r, p, a)


@pytest.mark.parametrize("knob", [{"TSG_DENSE_WIN": "777"}, {"TSG_DENSE_FLAT": "1"}])
def test_dense_numeric_small_windows(knob):
    # the windowed dense numeric tier with 777-position windows (env read once
    # per process, so in a child): many window boundaries inside set words,
    # every B row cut at precomputed points; and the opt-in flat form (fp64
    # REDs into C); compared with the oracle
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np\n"
        "import paper_1804_00695_b200 as tsg\n"
        "from paper_1804_00695_b200.csr import CsrMatrix, canonicalize\n"
        "from oracle import oracle as O\n"
        "from conftest import assert_same_product, random_csr\n"
        "rng = np.random.default_rng(7)\n"
        "n = 6000\n"
        "rows = [rng.choice(n, size=k, replace=False) for k in (3, 40, 400, 2500, 5000)]\n"
        "r = np.concatenate([np.full(len(x), i) for i, x in enumerate(rows)])\n"
        "a = CsrMatrix.from_coo(r, np.concatenate(rows), rng.uniform(0.1, 1, len(r)), len(rows), n)\n"
        "b = canonicalize(random_csr(rng, n, 150000, 60))\n"
        "assert_same_product(tsg.multiply(a, b), O.multiply(a, b), exact=False, rtol=1e-12)\n"
        "bi = CsrMatrix(b.num_rows, b.num_cols, b.row_ptr, b.col_idx, np.round(b.values * 8))\n"
        "ai = CsrMatrix(a.num_rows, a.num_cols, a.row_ptr, a.col_idx, np.ones(a.nnz))\n"
        "assert_same_product(tsg.multiply(ai, bi), O.multiply(ai, bi), exact=True)\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, **knob,
               PYTHONPATH=os.pathsep.join([root, os.path.join(root, "tests")]))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


def test_dense_tiers_beyond_shared_memory(rng):
    # B with 2.1 M columns: the symbolic bitmap (262 KB) exceeds shared memory,
    # so hub rows take the L2-slab symbolic dense tier and the windowed numeric
    # tier over a 33 K-set width; rows below the raised dense threshold take
    # the CTA / global tiers
    n, cols = 20000, 2_100_000
    rows = [rng.choice(n, size=k, replace=False) for k in (5, 300, 2000, 6000)]
    r = np.concatenate([np.full(len(x), i) for i, x in enumerate(rows)])
    a = CsrMatrix.from_coo(r, np.concatenate(rows), rng.uniform(0.1, 1, len(r)), len(rows), n)
    bu = random_csr(rng, n, cols, 60)
    b = canonicalize(bu)   # row-sorted: windowed shared-memory symbolic bitmaps
    assert_same_product(tsg.multiply(a, b), O.multiply(a, b), exact=False, rtol=1e-12)
    bi = CsrMatrix(b.num_rows, b.num_cols, b.row_ptr, b.col_idx, np.round(b.values * 8))
    ai = CsrMatrix(a.num_rows, a.num_cols, a.row_ptr, a.col_idx, np.ones(a.nnz))
    assert_same_product(tsg.multiply(ai, bi), O.multiply(ai, bi), exact=True)
    # unsorted B: the L2-slab symbolic bitmap
    assert_same_product(tsg.multiply(a, bu), O.multiply(a, bu), exact=False, rtol=1e-12)


def test_dense_tiers_many_windows():
    # the wide case with 3000-set symbolic windows and 1000-position numeric
    # windows (env read once per process, so in a child): 11 symbolic windows
    # per row, cut points at every boundary
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np\n"
        "import paper_1804_00695_b200 as tsg\n"
        "from paper_1804_00695_b200.csr import CsrMatrix, canonicalize\n"
        "from oracle import oracle as O\n"
        "from conftest import assert_same_product, random_csr\n"
        "rng = np.random.default_rng(11)\n"
        "n, cols = 20000, 2_100_000\n"
        "rows = [rng.choice(n, size=k, replace=False) for k in (5, 300, 2000, 6000)]\n"
        "r = np.concatenate([np.full(len(x), i) for i, x in enumerate(rows)])\n"
        "a = CsrMatrix.from_coo(r, np.concatenate(rows), rng.uniform(0.1, 1, len(r)), len(rows), n)\n"
        "b = canonicalize(random_csr(rng, n, cols, 60))\n"
        "assert_same_product(tsg.multiply(a, b), O.multiply(a, b), exact=False, rtol=1e-12)\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TSG_SYM_WIN_WORDS="3000", TSG_DENSE_WIN="1000",
               PYTHONPATH=os.pathsep.join([root, os.path.join(root, "tests")]))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


def test_global_tier_size_classes(rng):
    # B 134 M columns wide: the dense threshold rises to B's words / 8 (262 K
    # sets), so rows of 12 K .. 100 K sets take the global-memory tier, split
    # into table-size classes (2^15, 2^17, 2^19 slots) with their own slabs
    n, cols = 20000, 1 << 27
    rows = [rng.choice(n, size=k, replace=False) for k in (3, 400, 1700, 3400)]
    r = np.concatenate([np.full(len(x), i) for i, x in enumerate(rows)])
    a = CsrMatrix.from_coo(r, np.concatenate(rows), rng.uniform(0.1, 1, len(r)), len(rows), n)
    b = random_csr(rng, n, cols, 60)
    assert_same_product(tsg.multiply(a, b), O.multiply(a, b), exact=False, rtol=1e-12)


@pytest.mark.parametrize("seed", range(16))
def test_big_row_tiers_random_battery(seed):
    # random hub rows against random B of random width (dense tier in shared
    # memory, windowed, L2 slab; CTA and global tiers; sorted and unsorted B)
    # with small-integer values, so every tier must be exact
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2000, 12000))
    cols = int(rng.choice([5000, 200_000, 2_500_000, 40_000_000]))
    lens = [int(x) for x in rng.integers(1, 3000, size=6)] + [1, 2]
    rows = [rng.choice(n, size=min(k, n), replace=False) for k in lens]
    r = np.concatenate([np.full(len(x), i) for i, x in enumerate(rows)])
    a = CsrMatrix.from_coo(r, np.concatenate(rows), rng.integers(1, 4, len(r)).astype(np.float64), len(rows), n)
    b = random_csr(rng, n, cols, int(rng.integers(2, 80)))
    b = CsrMatrix(b.num_rows, b.num_cols, b.row_ptr, b.col_idx, np.round(b.values * 4))
    for bb in (b, canonicalize(b)):
        assert_same_product(tsg.multiply(a, bb), O.multiply(a, bb), exact=True)


def test_small_product_path_against_oracle():
    # the opt-in symbolic-free path for small products (TSG_SMALL_PATH=1,
    # read once per process: a child) on random pairs and config 1's A*A
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np\n"
        "import paper_1804_00695_b200 as tsg\n"
        "from paper_1804_00695_b200 import generators as gen\n"
        "from oracle import oracle as O\n"
        "from conftest import assert_same_product, random_csr\n"
        "rng = np.random.default_rng(3)\n"
        "for _ in range(12):\n"
        "    m, k, n = (int(x) for x in rng.integers(1, 400, 3))\n"
        "    a = random_csr(rng, m, k, int(rng.integers(1, 20)))\n"
        "    b = random_csr(rng, k, n, int(rng.integers(1, 20)))\n"
        "    assert_same_product(tsg.multiply(a, b), O.multiply(a, b), exact=True)\n"
        "a = gen.stencil(gen.LAPLACE2D, (256, 256))\n"
        "assert_same_product(tsg.multiply(a, a), O.multiply(a, a), exact=True)\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TSG_SMALL_PATH="1",
               PYTHONPATH=os.pathsep.join([root, os.path.join(root, "tests")]))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]
