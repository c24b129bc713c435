"""Shared fixtures.  GPU tests are marked ``gpu``; everything else runs on CPU.

The checker is the CPU oracle in oracle/ (a C restatement of the reference,
pinned to the reference's own outputs by tests/test_oracle.py)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 and the built libtsg.so")


@pytest.fixture
def rng():
    return np.random.default_rng(20240811)


def random_csr(rng, rows, cols, delta, exact_delta=False, values=True):
    """Up to (or exactly) delta distinct columns per row, values in (0.1, 1],
    columns kept in random (unsorted) order like the reference's fixtures."""
    from paper_1804_00695_b200.csr import CsrMatrix
    lens = np.full(rows, min(delta, cols)) if exact_delta else \
        np.minimum(rng.integers(0, delta + 1, size=rows), cols)
    ptr = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    cidx = np.concatenate([rng.choice(cols, size=int(k), replace=False) for k in lens]) \
        if rows else np.zeros(0, np.int64)
    vals = rng.uniform(0.1, 1.0, size=int(ptr[-1])) if values else None
    return CsrMatrix(rows, cols, ptr, cidx.astype(np.int64), vals)


def sorted_rows(m):
    from paper_1804_00695_b200.csr import canonicalize
    return canonicalize(m)


def assert_same_product(got, want_tuple, exact=True, rtol=1e-12):
    """got: CsrMatrix (any row order); want_tuple: oracle (ptr, col, val)."""
    from paper_1804_00695_b200.csr import CsrMatrix, canonicalize
    ptr, col, val = want_tuple
    want = canonicalize(CsrMatrix(got.num_rows, got.num_cols, ptr, col, val))
    g = canonicalize(got)
    assert np.array_equal(g.row_ptr, want.row_ptr), "row pointers differ"
    assert np.array_equal(g.col_idx, want.col_idx), "column structure differs"
    if exact:
        assert np.array_equal(g.values.view(np.uint64), want.values.view(np.uint64)), \
            "values not bit-identical (max abs diff %g)" % np.abs(g.values - want.values).max()
    else:
        d = np.abs(g.values - want.values)
        mag = np.maximum(np.abs(g.values), np.abs(want.values))
        assert np.all((d <= rtol * mag) | (d <= 1e-250))


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


# ---- golden fixtures (tests/golden/make_golden.py ran the reference) --------------
_GOLD = None


def golden():
    """(arrays, meta) of tests/golden/golden.{npz,json}."""
    global _GOLD
    if _GOLD is None:
        import json
        d = os.path.join(ROOT, "tests", "golden")
        arrs = dict(np.load(os.path.join(d, "golden.npz")))
        with open(os.path.join(d, "golden.json")) as fh:
            meta = json.load(fh)
        _GOLD = (arrs, meta)
    return _GOLD


def gcsr(name):
    from paper_1804_00695_b200.csr import CsrMatrix
    arrs, meta = golden()
    rows, cols, has_v = meta[name]
    return CsrMatrix(rows, cols, arrs[name + "/rp"], arrs[name + "/ci"],
                     arrs[name + "/va"] if has_v else None)


def gcm(name):
    arrs, _ = golden()
    return arrs[name + "/rp"], arrs[name + "/set"], arrs[name + "/bits"]
