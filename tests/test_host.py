"""Host-side logic pinned to the reference: generators (input builders),
SplitMix64, CSR utilities and the parity comparator."""

import numpy as np

from conftest import gcsr, golden
from paper_1804_00695_b200 import generators as gen
from paper_1804_00695_b200 import rng as R
from paper_1804_00695_b200.csr import (CsrMatrix, canonicalize, matrices_equal,
                                       products_match, slice_rows, transpose, validate)


def test_stencils_match_reference_generators():
    _, meta = golden()
    for kind in ("laplace3d", "brick3d", "bigstar2d", "elasticity3d", "laplace2d"):
        want = gcsr("stencil/%s" % kind)
        got = gen.stencil(kind, meta["stencil/%s/dims" % kind])
        assert np.array_equal(got.row_ptr, want.row_ptr), kind
        assert np.array_equal(got.col_idx, want.col_idx), kind
        assert np.array_equal(got.values, want.values), kind
        validate(got)


def test_stencil_rows_is_a_row_slice():
    full = gen.stencil(gen.BRICK3D, (6, 6, 8))
    part = gen.stencil_rows(gen.BRICK3D, (6, 6, 8), 72, 180)
    want = slice_rows(full, 72, 180)
    assert np.array_equal(part.row_ptr, want.row_ptr)
    assert np.array_equal(part.col_idx, want.col_idx)


def test_aggregation_matches_golden_and_transpose():
    p, r = gen.aggregation((8, 8, 8))
    want = gcsr("config2_8/p")
    assert np.array_equal(p.col_idx, want.col_idx)
    assert matrices_equal(r, transpose(p))
    assert r.num_rows == 64 and int(np.diff(r.row_ptr).max()) == 8


def test_splitmix_kats():
    _, meta = golden()
    g = R.PortableRng(0)
    assert [g.next_u64() for _ in range(3)] == meta["splitmix_seed0"]
    assert meta["splitmix_seed0"][0] == 0xE220A8397B1DCDAF
    g = R.PortableRng(22)
    assert [g.below(1000) for _ in range(5)] == meta["splitmix_seed22_below"]
    # the vectorised stream equals the sequential generator
    g = R.PortableRng(22)
    seq = [g.next_u64() for _ in range(50)]
    assert R.stream(22, 0, 50).tolist() == seq
    assert R.stream(22, 10, 5).tolist() == seq[10:15]


def test_rmat_is_deterministic_symmetric_loop_free():
    g1 = gen.rmat_graph(9, seed=5)
    g2 = gen.rmat_graph(9, seed=5)
    assert np.array_equal(g1.col_idx, g2.col_idx)
    rows = np.repeat(np.arange(g1.num_rows), np.diff(g1.row_ptr))
    assert not np.any(rows == g1.col_idx)
    assert matrices_equal(g1, transpose(g1))
    validate(g1)


def test_products_match_tolerance_kat():
    _, meta = golden()
    base = CsrMatrix(1, 2, [0, 2], [0, 1], [1.0, 2.0])
    assert products_match(CsrMatrix(1, 2, [0, 2], [0, 1], [1.0 + 1e-13, 2.0]), base)[0] == meta["match_kat"][0]
    assert products_match(CsrMatrix(1, 2, [0, 2], [0, 1], [1.0 + 1e-9, 2.0]), base)[0] == meta["match_kat"][1]
    # structure differences always fail
    assert not products_match(CsrMatrix(1, 2, [0, 1], [0], [1.0]), base)[0]


def test_canonicalize_and_slice():
    m = CsrMatrix(2, 5, [0, 3, 5], [4, 0, 2, 3, 1], [1., 2., 3., 4., 5.])
    c = canonicalize(m)
    assert c.col_idx.tolist() == [0, 2, 4, 1, 3]
    assert c.values.tolist() == [2., 3., 1., 5., 4.]
    s = slice_rows(m, 1, 2)
    assert s.row_ptr.tolist() == [0, 2] and s.col_idx.tolist() == [3, 1]


def test_reference_byte_convention():
    m = CsrMatrix(3, 4, [0, 2, 2, 3], [0, 1, 3], [1., 1., 1.])
    assert m.byte_size == 8 * 4 + 16 * 3
    assert int(m.row_byte_sizes().sum()) == m.byte_size
    p = CsrMatrix(3, 4, [0, 2, 2, 3], [0, 1, 3], None)
    assert p.byte_size == 8 * 4 + 8 * 3


REFERENCE_EXPORTS = (   # /root/reference/pkg/src/tiered_spgemm/__init__.py:10-39
    "HashmapAccumulator MemoryPool accumulator_capacity GPU_CHUNK1_AC_IN_PLACE GPU_CHUNK2_B_IN_PLACE "
    "KNL_CHUNK ChunkPlan RowPartition binary_search_partition copy_cost_chunk1 copy_cost_chunk2 "
    "decide_chunking execute_plan gpu_chunk_multiply_1 gpu_chunk_multiply_2 knl_chunk_multiply "
    "plan_for_multiply CsrMatrix canonicalize matrices_equal products_match slice_rows transpose validate "
    "CapacityError DimensionError GraphError GridError KernelError MatrixMarketError MatrixValidationError "
    "PlacementError TieredSpgemmError UnsplittableRowError VerifyError BIGSTAR2D BRICK3D ELASTICITY3D "
    "LAPLACE3D STENCIL_KINDS StencilSpec generate_interpolation generate_random_rhs generate_stencil "
    "grid_for_target_bytes stencil_byte_size stencil_nnz CompressedMatrix RowRange compress "
    "count_multiplications masked_row_intersect_count multiply spgemm_numeric spgemm_numeric_fused "
    "spgemm_symbolic read_matrix_market write_matrix_market AccessStats CopyLedger MemoryModel "
    "MemorySpaceSpec PlacementPolicy compute_access_stats default_model estimate_kernel_time simulate_copy "
    "validate_placement PortableRng count_triangles degree_sort_permutation load_graph lower_triangle "
    "to_undirected_pattern").split()


def test_public_surface_covers_the_reference():
    import paper_1804_00695_b200 as tsg
    missing = [n for n in REFERENCE_EXPORTS if not hasattr(tsg, n)]
    assert not missing, missing
