"""The reference's own test suite, restated against the drop-in.

Each test below re-states one test of /root/reference/pkg/tests (cited by
file:line) with the same inputs-by-construction, the same oracles (dense
numpy products, trace(A^3)/6 for triangles, closed-form copy costs) and the
same assertions, but calls this package -- i.e. the sm_100a kernels behind
the C ABI -- through the reference's public names (INTEGRATION.md §3 shows
the one-line re-pointing).  The only intentional difference the reference
contract allows is noted where it matters: C rows come out with ascending
columns instead of first-touch order, which every comparison here (dense,
products_match) is independent of.

The oracles are restated from the reference's conftest.py:13-80 (dense
product, boolean symbolic counts, trace(A^3)/6) and use no library kernel.
"""

import numpy as np
import pytest

import paper_1804_00695_b200 as ts
from paper_1804_00695_b200.chunking import c_row_byte_sizes
from paper_1804_00695_b200.csr import CsrMatrix, slice_rows

pytestmark = pytest.mark.gpu


# ---- oracles (reference conftest.py:13-80, restated) -----------------------------

def dense(m):
    out = np.zeros((m.num_rows, m.num_cols))
    r = np.repeat(np.arange(m.num_rows), np.diff(m.row_ptr))
    out[r, m.col_idx] = 1.0 if m.values is None else m.values
    return out


def dense_counts(a, b):
    x = (dense(a) != 0).astype(np.int64) @ (dense(b) != 0).astype(np.int64)
    return (x > 0).sum(axis=1).astype(np.int64)


def matches_dense(c, want, rtol=1e-12):
    got = dense(c)
    nz = want != 0
    return bool(np.all(np.abs(got[nz] - want[nz]) <= rtol * np.abs(want[nz])) and
                np.all(np.abs(got[~nz]) <= 1e-300))


def rand_csr(rng, rows, cols, delta, exact=False):
    r, c, v = [], [], []
    for i in range(rows):
        k = min(delta if exact else int(rng.integers(0, delta + 1)), cols)
        for j in rng.choice(cols, size=k, replace=False):
            r.append(i)
            c.append(int(j))
            v.append(float(rng.uniform(0.1, 1.0)))
    return CsrMatrix.from_coo(r, c, v, rows, cols)


def rand_graph(rng, n, p):
    up = np.triu(rng.random((n, n)) < p, 1)
    rows, cols = np.nonzero(up | up.T)
    return CsrMatrix.from_coo(rows, cols, None, n, n)


def triangles_oracle(g):
    x = (dense(g) != 0).astype(np.int64)
    return int(np.trace(x @ x @ x)) // 6


def permuted(g, perm):
    perm = np.asarray(perm)
    return CsrMatrix.from_coo(perm[np.repeat(np.arange(g.num_rows), np.diff(g.row_ptr))],
                              perm[g.col_idx], None, g.num_rows, g.num_cols)


def rows_matrix(rows, ncols, values=True):
    r = [i for i, cs in enumerate(rows) for _ in cs]
    c = [j for cs in rows for j in cs]
    return CsrMatrix.from_coo(r, c, [1.0] * len(c) if values else None, len(rows), ncols)


def graph(edges, n):
    u = [e[0] for e in edges]
    v = [e[1] for e in edges]
    return CsrMatrix.from_coo(u + v, v + u, None, n, n)


# ---- kernel (reference test_kernel.py) --------------------------------------------

def test_compress_word_packing_and_empty_rows():             # test_kernel.py:27-42
    cm = ts.compress(rows_matrix([[0, 63]], 64))
    assert cm.n_sets == 1 and cm.set_idx[0] == 0 and int(cm.set_bits[0]) == (1 | (1 << 63))
    cm = ts.compress(rows_matrix([[0, 64]], 65))
    assert cm.n_sets == 2 and sorted(cm.set_idx.tolist()) == [0, 1]
    assert ts.compress(rows_matrix([[], [3]], 8)).row_ptr.tolist() == [0, 0, 1]


def test_compress_popcount_identity(rng):                    # test_kernel.py:45-52
    b = rand_csr(rng, 60, 200, 8)
    cm = ts.compress(b)
    pops = np.zeros(b.num_rows, dtype=np.int64)
    for i in range(b.num_rows):
        for t in range(int(cm.row_ptr[i]), int(cm.row_ptr[i + 1])):
            pops[i] += bin(int(cm.set_bits[t])).count("1")
    assert np.array_equal(pops, np.diff(b.row_ptr))


def test_symbolic_identity_union_and_dense(rng):             # test_kernel.py:57-79
    b = rand_csr(rng, 20, 30, 4)
    assert np.array_equal(ts.spgemm_symbolic(CsrMatrix.identity(20), ts.compress(b)), np.diff(b.row_ptr))
    a = rows_matrix([[0, 1]], 2)
    assert ts.spgemm_symbolic(a, ts.compress(rows_matrix([[0, 1], [1, 2]], 3))).tolist() == [3]
    for _ in range(5):
        a, b = rand_csr(rng, 40, 40, 6), rand_csr(rng, 40, 40, 6)
        assert np.array_equal(ts.spgemm_symbolic(a, ts.compress(b)), dense_counts(a, b))
    with pytest.raises(ts.DimensionError):
        ts.spgemm_symbolic(rows_matrix([[0]], 3), ts.compress(rows_matrix([[0], [0]], 2)))


def test_numeric_identities_and_dense_oracle(rng):           # test_kernel.py:84-114
    a = CsrMatrix.from_coo([0, 0, 1], [0, 1, 1], [1.0, 2.0, 1.0], 2, 2)
    assert matches_dense(ts.multiply(a, CsrMatrix.identity(2)), dense(a))
    b = rand_csr(rng, 25, 30, 5)
    assert matches_dense(ts.multiply(CsrMatrix.identity(25), b), dense(b))
    for _ in range(20):
        n = int(rng.integers(5, 64))
        a, b = rand_csr(rng, n, n, 8), rand_csr(rng, n, n, 8)
        counts = ts.spgemm_symbolic(a, ts.compress(b))
        c = ts.spgemm_numeric(a, b, counts)
        assert np.array_equal(np.diff(c.row_ptr), counts)
        assert matches_dense(c, dense(a) @ dense(b))


def test_numeric_unsorted_columns_and_errors(rng):           # test_kernel.py:117-140
    a = rand_csr(rng, 20, 20, 5)
    rc, rv = a.col_idx.copy(), a.values.copy()
    for i in range(a.num_rows):
        lo, hi = int(a.row_ptr[i]), int(a.row_ptr[i + 1])
        rc[lo:hi], rv[lo:hi] = rc[lo:hi][::-1], rv[lo:hi][::-1]
    b = rand_csr(rng, 20, 20, 5)
    assert matches_dense(ts.multiply(CsrMatrix(20, 20, a.row_ptr, rc, rv), b), dense(a) @ dense(b))
    a, b = rand_csr(rng, 10, 10, 3, exact=True), rand_csr(rng, 10, 10, 3, exact=True)
    bad = np.array(ts.spgemm_symbolic(a, ts.compress(b))).copy()
    bad[0] += 1
    with pytest.raises(ts.KernelError):
        ts.spgemm_numeric(a, b, bad)
    p = rows_matrix([[0]], 1, values=False)
    with pytest.raises(ts.MatrixValidationError):
        ts.spgemm_numeric(p, p, np.array([1]))


def test_worker_count_does_not_change_result(rng):           # test_kernel.py:143-152
    a, b = rand_csr(rng, 50, 50, 6), rand_csr(rng, 50, 50, 6)
    c1 = ts.spgemm_symbolic(a, ts.compress(b), workers=1)
    c4 = ts.spgemm_symbolic(a, ts.compress(b), workers=4)
    assert np.array_equal(c1, c4)
    x, y = ts.spgemm_numeric(a, b, c1, workers=1), ts.spgemm_numeric(a, b, c1, workers=4)
    assert np.array_equal(x.col_idx, y.col_idx) and np.array_equal(x.values, y.values)


def test_fused_variants(rng):                                 # test_kernel.py:157-197
    a, b = rand_csr(rng, 30, 40, 5), rand_csr(rng, 40, 35, 5)
    plain = ts.spgemm_numeric(a, b, ts.spgemm_symbolic(a, ts.compress(b)))
    fused = ts.spgemm_numeric_fused(a, b, CsrMatrix.empty(30, 35), ts.RowRange(0, 30), ts.RowRange(0, 40))
    assert np.array_equal(fused.row_ptr, plain.row_ptr)
    assert np.array_equal(fused.col_idx, plain.col_idx)
    assert np.array_equal(fused.values, plain.values)
    a, b = rand_csr(rng, 30, 40, 6), rand_csr(rng, 40, 30, 6)
    plain = ts.multiply(a, b)
    part = CsrMatrix.empty(30, 30)
    for lo, hi in ((0, 17), (17, 40)):
        part = ts.spgemm_numeric_fused(a, slice_rows(b, lo, hi), part, ts.RowRange(0, 30), ts.RowRange(lo, hi))
    assert ts.products_match(part, plain, rtol=1e-12)[0]
    a = rows_matrix([[0], [1]], 2)
    empty = CsrMatrix.empty(0, 2)
    assert ts.spgemm_numeric_fused(a, slice_rows(a, 0, 1), empty, ts.RowRange(0, 0), ts.RowRange(0, 1)) is empty
    a = CsrMatrix(1, 3, np.array([0, 2]), np.array([2, 0]), np.array([5.0, 1.0]))
    b = rows_matrix([[0], [1], [2]], 3)
    out = ts.spgemm_numeric_fused(a, slice_rows(b, 0, 1), CsrMatrix.empty(1, 3), ts.RowRange(0, 1),
                                  ts.RowRange(0, 1))
    assert dense(out).tolist() == [[1.0, 0.0, 0.0]]


def test_masked_count_cases(rng):                              # test_kernel.py:202-232
    def low(edges, n):
        return CsrMatrix.from_coo([max(e) for e in edges], [min(e) for e in edges], None, n, n)
    path = low([(0, 1), (1, 2), (2, 3)], 4)
    assert ts.masked_row_intersect_count(path, ts.compress(path)) == 0
    k4 = low([(i, j) for i in range(4) for j in range(i + 1, 4)], 4)
    assert ts.masked_row_intersect_count(k4, ts.compress(k4)) == 4
    bad = CsrMatrix.from_coo([0], [1], None, 2, 2)
    with pytest.raises(ts.MatrixValidationError):
        ts.masked_row_intersect_count(bad, ts.compress(bad))
    for _ in range(10):
        g = rand_graph(rng, 30, 0.2)
        rows = np.repeat(np.arange(30), np.diff(g.row_ptr))
        keep = rows > g.col_idx
        l = CsrMatrix.from_coo(rows[keep], g.col_idx[keep], None, 30, 30)
        assert ts.masked_row_intersect_count(l, ts.compress(l)) == triangles_oracle(g)


def test_count_multiplications_cases(rng):                    # test_kernel.py:237-256
    b = rand_csr(rng, 15, 15, 4)
    assert ts.count_multiplications(CsrMatrix.identity(15), b) == b.nnz
    assert ts.count_multiplications(rows_matrix([[2]], 3), rows_matrix([[], [], [0, 1, 2, 3, 4]], 5)) == 5
    a, b = rand_csr(rng, 25, 30, 5), rand_csr(rng, 30, 20, 5)
    bn = np.diff(b.row_ptr)
    assert ts.count_multiplications(a, b) == int(sum(bn[k] for k in a.col_idx))


# ---- chunking (reference test_chunking.py) -----------------------------------------

def loose_model(cap=1 << 40):
    return ts.MemoryModel(ts.MemorySpaceSpec("fast", cap, 400e9, 1e-7),
                          ts.MemorySpaceSpec("slow", None, 20e9, 1e-6))


def product_fixture(rng, n=30, m=40, k=35, delta=6):
    a, b = rand_csr(rng, n, m, delta), rand_csr(rng, m, k, delta)
    counts = ts.spgemm_symbolic(a, ts.compress(b))
    return a, b, counts, ts.spgemm_numeric(a, b, counts)


def sizes_of(a, b, counts):
    return a.byte_size, b.byte_size, 8 * (a.num_rows + 1) + 16 * int(np.sum(counts))


def test_knl_cases(rng):                                        # test_chunking.py:116-155
    a, b, counts, plain = product_fixture(rng)
    c, led = ts.knl_chunk_multiply(a, b, counts, b.byte_size + 100, loose_model())
    assert ts.products_match(c, plain)[0] and len(led.events) == 1 and led.total_bytes() == b.byte_size
    c, led = ts.knl_chunk_multiply(a, b, counts, int(b.byte_size / 2.1), loose_model())
    assert ts.products_match(c, plain)[0]
    assert len([e for e in led.events if e.tag == "B"]) == 3 and led.total_bytes() == b.byte_size
    fast = b.byte_size // 4
    _, led = ts.knl_chunk_multiply(a, b, counts, fast, loose_model(cap=fast))
    assert led.peak_residency("fast") <= fast
    with pytest.raises(ts.UnsplittableRowError):
        ts.knl_chunk_multiply(a, b, counts, int(b.row_byte_sizes().max()) - 1, loose_model())
    a = rand_csr(rng, 20, 30, 4, exact=True)
    b = rand_csr(rng, 30, 20, 3)
    counts = ts.spgemm_symbolic(a, ts.compress(b))
    plain = ts.spgemm_numeric(a, b, counts)
    c, led = ts.knl_chunk_multiply(a, b, counts, b.byte_size // 3 + 1, loose_model())
    assert ts.products_match(c, plain)[0] and led.total_bytes() == b.byte_size


def test_knl_multigrid_product():                               # test_chunking.py:158-180
    spec = ts.StencilSpec(ts.LAPLACE3D, (9, 9, 9))
    a = ts.generate_stencil(spec)
    _, r = ts.generate_interpolation(spec)
    counts = ts.spgemm_symbolic(r, ts.compress(a))
    plain = ts.spgemm_numeric(r, a, counts)
    c, led = ts.knl_chunk_multiply(r, a, counts, a.byte_size // 4 + 8, loose_model())
    assert ts.products_match(c, plain, rtol=1e-12)[0] and led.total_bytes() == a.byte_size


def _p_ac(a, counts, parts):
    rb = a.row_byte_sizes() + c_row_byte_sizes(a.num_rows, counts)
    return ts.binary_search_partition(rb, int(rb.sum() // parts) + 1)


def _p_b(b, parts):
    rb = b.row_byte_sizes()
    return ts.binary_search_partition(rb, int(rb.sum() // parts) + 1)


def test_chunk1_cases(rng):                                     # test_chunking.py:185-216
    a, b, counts, plain = product_fixture(rng)
    sa, sb, sc = sizes_of(a, b, counts)
    p_ac = ts.singleton_partition(a.row_byte_sizes() + c_row_byte_sizes(a.num_rows, counts))
    c, led = ts.gpu_chunk_multiply_1(a, b, counts, p_ac, ts.singleton_partition(b.row_byte_sizes()),
                                     loose_model())
    assert ts.products_match(c, plain)[0] and led.total_bytes() == sa + sb + sc
    p_ac = _p_ac(a, counts, 3)
    c, led = ts.gpu_chunk_multiply_1(a, b, counts, p_ac, ts.singleton_partition(b.row_byte_sizes()),
                                     loose_model())
    assert len(p_ac) == 3 and len(led.events_tagged("B")) == 3
    assert led.total_bytes() == ts.copy_cost_chunk1(sa, sb, sc, 3) and ts.products_match(c, plain)[0]
    for _ in range(5):
        a, b, counts, plain = product_fixture(rng, n=40, m=50, k=45, delta=5)
        p_ac, p_b = _p_ac(a, counts, int(rng.integers(2, 4))), _p_b(b, int(rng.integers(2, 4)))
        c, led = ts.gpu_chunk_multiply_1(a, b, counts, p_ac, p_b, loose_model())
        assert ts.products_match(c, plain, rtol=1e-12)[0]
        sa, sb, sc = sizes_of(a, b, counts)
        assert led.total_bytes() == ts.copy_cost_chunk1(sa, sb, sc, len(p_ac))


def test_chunk2_cases(rng):                                     # test_chunking.py:219-253
    a, b, counts, plain = product_fixture(rng)
    sa, sb, sc = sizes_of(a, b, counts)
    c, led = ts.gpu_chunk_multiply_2(a, b, counts, _p_ac(a, counts, 2),
                                     ts.singleton_partition(b.row_byte_sizes()), loose_model())
    assert ts.products_match(c, plain)[0]
    assert sum(e.bytes for e in led.events_tagged("C_in")) == 0
    assert led.total_bytes() == ts.copy_cost_chunk2(sa, sb, sc, 1) == sa + sb
    p_ac, p_b = _p_ac(a, counts, 2), _p_b(b, 2)
    c, led = ts.gpu_chunk_multiply_2(a, b, counts, p_ac, p_b, loose_model())
    assert ts.products_match(c, plain)[0]
    assert sum(e.bytes for e in led.events_tagged("A")) == 2 * sa
    assert sum(e.bytes for e in led.events_tagged("C_in")) == sc
    assert len(led.events_tagged("C_out")) == 2 * len(p_ac)
    assert led.total_bytes() == ts.copy_cost_chunk2(sa, sb, sc, 2)


def test_chunk_capacity_and_residency(rng):                    # test_chunking.py:256-281
    a, b, counts, _ = product_fixture(rng)
    p_ac, p_b = _p_ac(a, counts, 2), _p_b(b, 2)
    with pytest.raises(ts.CapacityError):
        ts.gpu_chunk_multiply_1(a, b, counts, p_ac, p_b,
                                loose_model(cap=p_ac.max_range_bytes + p_b.max_range_bytes - 1))
    p_b = _p_b(b, 3)
    cap = p_ac.max_range_bytes + p_b.max_range_bytes
    for algo in (ts.gpu_chunk_multiply_1, ts.gpu_chunk_multiply_2):
        _, led = algo(a, b, counts, p_ac, p_b, loose_model(cap=cap))
        assert led.peak_residency("fast") <= cap


def test_plan_execute_consistency_sweep(rng):                  # test_chunking.py:361-397
    for fast_divisor in (2, 3, 5):
        a, b, counts, plain = product_fixture(rng, n=50, m=60, k=40, delta=5)
        fast = sum(sizes_of(a, b, counts)) // fast_divisor
        plan = ts.plan_for_multiply(a, b, counts, fast)
        c, led = ts.execute_plan(a, b, counts, plan, loose_model(cap=fast))
        assert ts.products_match(c, plain)[0] and led.total_bytes() == plan.predicted_copy_bytes
    seen = set()
    for trial in range(25):
        a, b, counts, plain = product_fixture(rng, n=int(rng.integers(20, 90)), m=int(rng.integers(20, 90)),
                                              k=int(rng.integers(15, 70)), delta=int(rng.integers(2, 7)))
        fast = int(sum(sizes_of(a, b, counts)) / float(rng.uniform(1.3, 6.0)))
        try:
            plan = ts.plan_for_multiply(a, b, counts, fast)
        except ts.UnsplittableRowError:
            continue
        seen.add(plan.heuristic_branch)
        c, led = ts.execute_plan(a, b, counts, plan, loose_model(cap=fast))
        assert ts.products_match(c, plain, rtol=1e-12)[0], trial
        assert led.total_bytes() == plan.predicted_copy_bytes
        assert led.peak_residency("fast") <= fast
    assert len(seen) >= 2, seen


# ---- triangles (reference test_triangles.py) ------------------------------------------

K4 = graph([(i, j) for i in range(4) for j in range(i + 1, 4)], 4)
C5 = graph([(i, (i + 1) % 5) for i in range(5)], 5)
PETERSEN = graph([(i, (i + 1) % 5) for i in range(5)] + [(5 + i, 5 + (i + 2) % 5) for i in range(5)]
                 + [(i, 5 + i) for i in range(5)], 10)


def test_triangle_known_graphs_and_prep(rng):                   # test_triangles.py:24-61
    assert (ts.count_triangles(K4), ts.count_triangles(C5), ts.count_triangles(PETERSEN)) == (4, 0, 0)
    star = graph([(0, i) for i in range(1, 5)], 5)
    assert ts.degree_sort_permutation(star)[-1] == 0
    assert np.array_equal(ts.degree_sort_permutation(C5), np.arange(5))
    g = rand_graph(rng, 60, 0.1)
    assert np.all(np.diff(np.diff(g.row_ptr)[ts.degree_sort_permutation(g)]) >= 0)
    k3 = graph([(0, 1), (0, 2), (1, 2)], 3)
    l = ts.lower_triangle(k3, np.arange(3))
    assert l.nnz == 3 and np.all(l.col_idx < np.repeat(np.arange(3), np.diff(l.row_ptr)))
    assert ts.lower_triangle(CsrMatrix.empty(4, 4, pattern=True), np.arange(4)).nnz == 0
    g = rand_graph(rng, 40, 0.15)
    assert ts.lower_triangle(g, ts.degree_sort_permutation(g)).nnz == g.nnz // 2


def test_triangle_counts_random_relabelled_workers(rng):        # test_triangles.py:64-90
    for _ in range(15):
        n = int(rng.integers(10, 80))
        g = rand_graph(rng, n, float(rng.uniform(0.05, 0.3)))
        assert ts.count_triangles(g) == triangles_oracle(g)
    g = rand_graph(rng, 50, 0.15)
    want = ts.count_triangles(g)
    for _ in range(5):
        assert ts.count_triangles(permuted(g, rng.permutation(50))) == want
    g = rand_graph(rng, 70, 0.12)
    assert ts.count_triangles(g, workers=1) == ts.count_triangles(g, workers=4)
    g = rand_graph(rng, 40, 0.2)
    l_id = ts.lower_triangle(g, np.arange(40))
    assert ts.masked_row_intersect_count(l_id, ts.compress(l_id)) == ts.count_triangles(g)


def test_triangle_validation_and_cleaning():                    # test_triangles.py:93-112
    with pytest.raises(ts.GraphError):
        ts.lower_triangle(CsrMatrix.from_coo([0], [1], None, 2, 2), np.arange(2))
    with pytest.raises(ts.GraphError):
        ts.lower_triangle(CsrMatrix.from_coo([0, 0, 1, 1], [0, 1, 0, 1], None, 2, 2), np.arange(2))
    assert ts.count_triangles(graph([(0, 1)], 2)) == 0
    g = ts.to_undirected_pattern(CsrMatrix.from_coo([0, 0, 1, 2, 2], [1, 1, 1, 0, 2], None, 3, 3))
    assert g.nnz == 4 and ts.count_triangles(g) == 0


# ---- acceptance criteria (reference test_acceptance.py) --------------------------------

def test_c01_spgemm_oracle_equivalence():                       # test_acceptance.py:38-54
    rng = np.random.default_rng(101)
    for _ in range(200):
        n = int(rng.integers(4, 65))
        a, b = rand_csr(rng, n, n, 8), rand_csr(rng, n, n, 8)
        counts = ts.spgemm_symbolic(a, ts.compress(b))
        assert np.array_equal(counts, dense_counts(a, b))
        c = ts.spgemm_numeric(a, b, counts)
        assert np.array_equal(np.diff(c.row_ptr), counts)
        assert matches_dense(c, dense(a) @ dense(b))


def test_c02_c03_chunked_equals_unchunked_and_ledgers():        # test_acceptance.py:59-120
    rng = np.random.default_rng(202)
    for _ in range(50):
        n, m, k = (int(rng.integers(40, 120)), int(rng.integers(40, 120)), int(rng.integers(30, 100)))
        a, b = rand_csr(rng, n, m, 8), rand_csr(rng, m, k, 8)
        counts = ts.spgemm_symbolic(a, ts.compress(b))
        plain = ts.spgemm_numeric(a, b, counts)
        sa, sb, sc = a.byte_size, b.byte_size, 8 * (n + 1) + 16 * int(np.sum(counts))
        fast = -(-sb // int(rng.integers(2, 9)))
        for _ in range(20):
            knl = ts.knl_chunk_multiply(a, b, counts, fast, loose_model())
            parts = len(knl[1].events)
            if 2 <= parts <= 8:
                break
            fast = max(1, int(fast * (1.15 if parts > 8 else 0.85)))
        ac_rows = a.row_byte_sizes() + c_row_byte_sizes(n, counts)
        p_ac = ts.binary_search_partition(ac_rows, int(ac_rows.sum() // int(rng.integers(2, 5))) + 1)
        p_b = ts.binary_search_partition(b.row_byte_sizes(), int(sb // int(rng.integers(2, 5))) + 1)
        runs = {"knl": knl, "gpu1": ts.gpu_chunk_multiply_1(a, b, counts, p_ac, p_b, loose_model()),
                "gpu2": ts.gpu_chunk_multiply_2(a, b, counts, p_ac, p_b, loose_model())}
        for name, (c, _) in runs.items():
            assert ts.products_match(c, plain, rtol=1e-12)[0], name
        assert 2 <= len(runs["knl"][1].events) <= 8
        assert runs["knl"][1].total_bytes() == sb
        assert runs["gpu1"][1].total_bytes() == ts.copy_cost_chunk1(sa, sb, sc, len(p_ac))
        assert runs["gpu2"][1].total_bytes() == ts.copy_cost_chunk2(sa, sb, sc, len(p_b))


def test_c07_triangle_counting():                               # test_acceptance.py:270-300
    rng = np.random.default_rng(707)
    assert (ts.count_triangles(K4), ts.count_triangles(C5), ts.count_triangles(PETERSEN)) == (4, 0, 0)
    for _ in range(50):
        n = int(rng.integers(10, 101))
        g = rand_graph(rng, n, float(rng.uniform(0.03, 0.25)))
        want = triangles_oracle(g)
        assert ts.count_triangles(g) == want
        for _ in range(10):
            assert ts.count_triangles(permuted(g, rng.permutation(n))) == want
