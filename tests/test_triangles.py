"""Config 3 path: triangle counts through the device masked-count kernel are
exact and equal the reference's (golden counts computed by the reference)."""

import numpy as np
import pytest

from conftest import gcsr, golden

pytestmark = pytest.mark.gpu


def graph(edges, n):
    import paper_1804_00695_b200 as tsg
    u = [e[0] for e in edges]
    v = [e[1] for e in edges]
    return tsg.CsrMatrix.from_coo(u + v, v + u, None, n, n)


def test_known_graphs():
    import paper_1804_00695_b200 as tsg
    k4 = graph([(i, j) for i in range(4) for j in range(i + 1, 4)], 4)
    c5 = graph([(i, (i + 1) % 5) for i in range(5)], 5)
    pet = graph([(i, (i + 1) % 5) for i in range(5)] + [(5 + i, 5 + (i + 2) % 5) for i in range(5)]
                + [(i, 5 + i) for i in range(5)], 10)
    assert tsg.count_triangles(k4) == 4
    assert tsg.count_triangles(c5) == 0
    assert tsg.count_triangles(pet) == 0


def test_golden_graphs_match_reference():
    import paper_1804_00695_b200 as tsg
    _, meta = golden()
    for k, want in enumerate(meta["triangles_total"]):
        assert tsg.count_triangles(gcsr("tri%d/g" % k)) == want


def test_relabel_invariance(rng):
    import paper_1804_00695_b200 as tsg
    g = gcsr("tri3/g")
    want = tsg.count_triangles(g)
    n = g.num_rows
    for _ in range(4):
        perm = rng.permutation(n)
        rows = perm[np.repeat(np.arange(n), np.diff(g.row_ptr))]
        cols = perm[g.col_idx]
        h = tsg.CsrMatrix.from_coo(rows, cols, None, n, n)
        assert tsg.count_triangles(h) == want


def test_rmat_scale14_against_oracle():
    import paper_1804_00695_b200 as tsg
    from paper_1804_00695_b200 import generators as gen
    from oracle import oracle as O
    g = gen.rmat_graph(14)
    low = tsg.lower_triangle(g, tsg.degree_sort_permutation(g), check=False)
    assert tsg.count_triangles(g) == O.masked_count(low, O.compress(low), workers=8)


# ---- §8f rows 2-3: graph preparation on the device --------------------------

def _download(dm):
    return dm.download()


def test_device_lower_triangle_equals_host(rng):
    import paper_1804_00695_b200 as tsg
    from paper_1804_00695_b200 import _lib
    from paper_1804_00695_b200.triangles import lower_triangle_device
    graphs = [gcsr("tri%d/g" % k) for k in range(4)]
    for n, p in ((50, 0.2), (300, 0.05), (2000, 0.004)):
        up = np.triu(rng.random((n, n)) < p, 1)
        r, c = np.nonzero(up | up.T)
        graphs.append(tsg.CsrMatrix.from_coo(r, c, None, n, n))
    for g in graphs:
        want_perm = tsg.degree_sort_permutation(g)
        want = tsg.lower_triangle(g, want_perm)
        for shuffled in (False, True):
            h = g
            if shuffled:   # columns in arbitrary order inside each row
                ci = np.asarray(g.col_idx).copy()
                for i in range(g.num_rows):
                    lo, hi = g.row_ptr[i], g.row_ptr[i + 1]
                    ci[lo:hi] = rng.permutation(ci[lo:hi])
                h = tsg.CsrMatrix(g.num_rows, g.num_cols, g.row_ptr, ci, None)
            dl, perm = lower_triangle_device(_lib.DeviceCsr.upload(h), want_perm=True)
            got = _download(dl)
            assert np.array_equal(perm, want_perm)
            assert np.array_equal(got.row_ptr, want.row_ptr)
            assert np.array_equal(got.col_idx, want.col_idx)


def test_device_graph_validation_errors():
    import paper_1804_00695_b200 as tsg
    with pytest.raises(tsg.GraphError):   # self loop
        tsg.count_triangles(tsg.CsrMatrix.from_coo([0, 1, 1], [1, 0, 1], None, 2, 2))
    with pytest.raises(tsg.GraphError):   # not symmetric
        tsg.count_triangles(tsg.CsrMatrix.from_coo([0, 1, 2], [1, 2, 0], None, 3, 3))
    with pytest.raises(tsg.GraphError):   # not square
        tsg.count_triangles(tsg.CsrMatrix.from_coo([0], [1], None, 1, 2))


def test_device_rmat_equals_host_builder():
    from paper_1804_00695_b200 import generators as gen
    for scale, ef, seed in ((8, 16, 22), (11, 8, 5), (13, 16, 22)):
        want = gen.rmat_graph(scale, ef, seed)
        got = gen.rmat_graph_device(scale, ef, seed).download()
        assert np.array_equal(got.row_ptr, want.row_ptr)
        assert np.array_equal(got.col_idx, want.col_idx)


def test_device_pipeline_rmat_scale15_against_oracle():
    from paper_1804_00695_b200 import generators as gen
    from paper_1804_00695_b200.triangles import count_triangles_device
    import paper_1804_00695_b200 as tsg
    from oracle import oracle as O
    g = gen.rmat_graph(15)
    low = tsg.lower_triangle(g, tsg.degree_sort_permutation(g), check=False)
    want = O.masked_count(low, O.compress(low), workers=8)
    assert count_triangles_device(gen.rmat_graph_device(15)) == want
