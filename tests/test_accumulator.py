"""Host accumulator API kept from the reference (accumulator.py:24-152); the
reference's test_accumulator.py is the model.  The device tables are covered
by the parity tests."""

import pytest

from paper_1804_00695_b200 import HashmapAccumulator, MemoryPool, accumulator_capacity


@pytest.mark.parametrize("bound,capacity", [(0, 1), (1, 2), (2, 4), (3, 8), (4, 8), (5, 16), (8, 16),
                                            (9, 32)])
def test_capacity_rule(bound, capacity):
    assert accumulator_capacity(bound) == capacity


def _acc(bound):
    pool = MemoryPool.for_row_bound(bound)
    return pool, HashmapAccumulator(pool.acquire(), accumulator_capacity(bound))


def test_add_or_and_first_touch_order():
    _, acc = _acc(8)
    for k, v in ((7, 1.0), (3, 2.0), (7, 0.5), (11, -1.0), (3, 0.25)):
        acc.add(k, v)
    assert list(acc.items()) == [(7, 1.5), (3, 2.25), (11, -1.0)]
    assert acc.occupied == 3
    _, sym = _acc(4)
    sym.or_bits(5, 0b0101)
    sym.or_bits(9, 1 << 63)
    sym.or_bits(5, 0b0010)
    assert list(sym.items()) == [(5, 0b0111), (9, 1 << 63)] and sym.popcount_sum() == 4


def test_reset_and_collisions():
    _, acc = _acc(4)                     # capacity 8: keys 0, 8, 16 share a home slot
    for k in (0, 8, 16, 24):
        acc.add(k, float(k))
    assert [k for k, _ in acc.items()] == [0, 8, 16, 24] and acc.live_slot_count() == 4
    acc.reset()
    assert acc.occupied == 0 and acc.live_slot_count() == 0
    acc.add(8, 1.0)
    assert list(acc.items()) == [(8, 1.0)]


def test_capacity_checks_and_pool():
    pool = MemoryPool(8)
    with pytest.raises(ValueError):
        HashmapAccumulator(pool.acquire(), 6)
    with pytest.raises(ValueError):
        HashmapAccumulator(pool.acquire(), 16)
    a, b = pool.acquire(), pool.acquire()
    assert a is not b and a.slots == b.slots == 8 and pool.slab_bytes == 192
    pool.release(a)
    assert pool.acquire() is a
    with pytest.raises(ValueError):
        pool.release(object())
    with pytest.raises(ValueError):
        MemoryPool(0)
