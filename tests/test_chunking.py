"""Chunked path.  CPU: the planner / partitioner / copy-cost host logic equals
the reference's outputs (golden plans from the reference itself).  GPU: the
three executors really stream data and return C identical to the plain
product plus ledgers identical to the reference's."""

import numpy as np
import pytest

from conftest import assert_same_product, gcsr, golden, random_csr
from paper_1804_00695_b200 import chunking as ch
from paper_1804_00695_b200.errors import CapacityError, UnsplittableRowError
from paper_1804_00695_b200.memory import MemoryModel, MemorySpaceSpec


def loose_model(cap=1 << 40):
    return MemoryModel(MemorySpaceSpec("fast", cap, 100e9, 1e-7),
                       MemorySpaceSpec("slow", None, 10e9, 1e-6))


def test_plans_match_reference():
    _, meta = golden()
    for case in meta["plans"]:
        a, b, c = (np.array(case[k], dtype=np.int64) for k in "abc")
        try:
            got = ch.decide_chunking(int(a.sum()), int(b.sum()), int(c.sum()), a, b, c,
                                     case["fast"]).to_json_dict()
        except CapacityError:
            got = {"error": "CapacityError"}
        assert got == case["plan"]


def test_partitions_match_reference():
    _, meta = golden()
    for case in meta["partitions"]:
        rb = np.array(case["rows"], dtype=np.int64)
        try:
            got = ch.binary_search_partition(rb, case["target"], case["cap"]).to_json_dict()
        except UnsplittableRowError:
            got = {"error": "UnsplittableRowError"}
        assert got == case["out"]
        try:
            bal = ch.balanced_partition(rb, max(1, int(rb.sum()) // 3 + 1)).to_json_dict()
        except UnsplittableRowError:
            bal = {"error": "UnsplittableRowError"}
        assert bal == case["balanced"]


def test_partition_kats():
    p = ch.binary_search_partition([10, 10, 10, 10], 20)
    assert [(r.begin, r.end) for r in p.ranges] == [(0, 2), (2, 4)] and p.range_bytes == [20, 20]
    p = ch.binary_search_partition([30, 10, 10, 30], 40, capacity=40)
    assert [(r.begin, r.end) for r in p.ranges] == [(0, 2), (2, 4)]
    with pytest.raises(UnsplittableRowError):
        ch.binary_search_partition([50], 25, capacity=40)
    assert len(ch.balanced_partition([10] * 10, 40)) == 3


def test_copy_cost_kats():
    gb = 10 ** 9
    assert ch.copy_cost_chunk1(2 * gb, 4 * gb, 3 * gb, 3) == 17 * gb
    assert ch.copy_cost_chunk1(2300, 4000, 5000, 2) == 15300
    assert ch.copy_cost_chunk2(2 * gb, 4 * gb, 3 * gb, 3) == 16 * gb
    assert ch.copy_cost_chunk2(3900, 250, 500, 2) == 8550
    _, meta = golden()
    assert ch.c_row_byte_sizes(4, [1, 0, 3, 2]).tolist() == meta["c_row_bytes"]


def test_heuristic_published_case_and_tie():
    unit = 10 ** 7
    plan = ch.decide_chunking(230 * unit, 400 * unit, 500 * unit, np.full(10, 23 * unit),
                              np.full(10, 40 * unit), np.full(10, 50 * unit), 800 * unit)
    assert plan.heuristic_branch == 1 and plan.algorithm == ch.GPU_CHUNK2_B_IN_PLACE
    tie = ch.decide_chunking(300, 300, 100, np.full(20, 15), np.full(20, 15), np.full(20, 5), 360)
    assert tie.algorithm == ch.GPU_CHUNK1_AC_IN_PLACE


# ---------------------------------------------------------------- GPU executors

def _partitions(meta):
    def part(d, n):
        return ch.RowPartition([ch.RowRange(a, b) for a, b in d["ranges"]], d["range_bytes"], n)
    return part


@pytest.mark.gpu
def test_executors_match_reference_ledgers_and_products():
    from oracle import oracle as O
    from paper_1804_00695_b200.csr import CsrMatrix
    _, meta = golden()
    a, b = gcsr("chunk/a"), gcsr("chunk/b")
    counts = O.symbolic(a, O.compress(b))
    want = O.numeric(a, b, counts)
    info = meta["chunk"]
    p_ac = ch.RowPartition([ch.RowRange(x, y) for x, y in info["p_ac"]["ranges"]],
                           info["p_ac"]["range_bytes"], a.num_rows)
    p_b = ch.RowPartition([ch.RowRange(x, y) for x, y in info["p_b"]["ranges"]],
                          info["p_b"]["range_bytes"], b.num_rows)
    runs = {"gpu1": ch.gpu_chunk_multiply_1(a, b, counts, p_ac, p_b, loose_model()),
            "gpu2": ch.gpu_chunk_multiply_2(a, b, counts, p_ac, p_b, loose_model()),
            "knl": ch.knl_chunk_multiply(a, b, counts, info["knl_fast"], loose_model())}
    for name, (c, led) in runs.items():
        assert [[e.bytes, e.src, e.dst, e.tag] for e in led.events] == info["ledgers"][name], name
        # the reference's own chunked result: same chunk order -> bit-identical
        ref = gcsr("chunk/%s_c" % name)
        assert_same_product(c, (ref.row_ptr, ref.col_idx, ref.values), exact=True)
        assert_same_product(c, want, exact=False)
        assert led.physical["h2d_bytes"] > 0 and led.physical["d2h_bytes"] > 0


@pytest.mark.gpu
def test_executors_random_battery(rng):
    from oracle import oracle as O
    for _ in range(12):
        n, m, k = (int(rng.integers(40, 200)) for _ in range(3))
        a = random_csr(rng, n, m, 10)
        b = random_csr(rng, m, k, 10)
        counts = O.symbolic(a, O.compress(b))
        want = O.numeric(a, b, counts)
        acr = a.row_byte_sizes() + ch.c_row_byte_sizes(n, counts)
        p_ac = ch.binary_search_partition(acr, int(acr.sum() // int(rng.integers(2, 5))) + 1)
        p_b = ch.binary_search_partition(b.row_byte_sizes(), int(b.byte_size // int(rng.integers(2, 5))) + 1)
        sa, sb = a.byte_size, b.byte_size
        sc = 8 * (n + 1) + 16 * int(counts.sum())
        c1, l1 = ch.gpu_chunk_multiply_1(a, b, counts, p_ac, p_b, loose_model())
        c2, l2 = ch.gpu_chunk_multiply_2(a, b, counts, p_ac, p_b, loose_model())
        c3, l3 = ch.knl_chunk_multiply(a, b, counts, sb // 3 + 1, loose_model())
        for c in (c1, c2, c3):   # chunking reorders sums: the reference's 1e-12 rule
            assert_same_product(c, want, exact=False, rtol=1e-12)
        assert l1.total_bytes() == ch.copy_cost_chunk1(sa, sb, sc, len(p_ac))
        assert l2.total_bytes() == ch.copy_cost_chunk2(sa, sb, sc, len(p_b))
        assert l3.total_bytes() == sb


@pytest.mark.gpu
def test_plan_execute_stencil_rap_chunked():
    from oracle import oracle as O
    from paper_1804_00695_b200 import generators as gen
    a = gen.stencil(gen.BRICK3D, (12, 12, 12))
    counts = O.symbolic(a, O.compress(a))
    want = O.numeric(a, a, counts)
    for frac in (0.3, 0.6, 2.5):
        fast = int(a.byte_size * frac)
        plan = ch.plan_for_multiply(a, a, counts, fast)
        c, led = ch.execute_plan(a, a, counts, plan, loose_model(cap=fast))
        assert_same_product(c, want, exact=True)   # integer-valued stencil: exact
        assert led.total_bytes() == plan.predicted_copy_bytes


@pytest.mark.gpu
def test_capacity_violation_raises():
    from oracle import oracle as O
    a = gcsr("chunk/a")
    b = gcsr("chunk/b")
    counts = O.symbolic(a, O.compress(b))
    p_ac = ch.singleton_partition(a.row_byte_sizes() + ch.c_row_byte_sizes(a.num_rows, counts))
    p_b = ch.singleton_partition(b.row_byte_sizes())
    with pytest.raises(CapacityError):
        ch.gpu_chunk_multiply_1(a, b, counts, p_ac, p_b, loose_model(cap=100))
