"""Drop-in replacement for the reference's hot path, tiered_spgemm.kernel.

Same names, signatures, defaults, argument checks and exceptions as
/root/reference/pkg/src/tiered_spgemm/kernel.py:37-394; every numeric call
runs hand-written sm_100a kernels through the C ABI (include/tsg.h, bound in
_lib.py).  There is no CPU fallback.

Differences a caller can observe, all inside the reference's contract:

* ``spgemm_numeric`` / ``multiply`` / ``spgemm_numeric_fused`` emit each C row
  with ascending columns instead of the accumulator's first-touch order.
  ``canonicalize`` (csr.py:145-150) of either is identical, which is what
  ``products_match`` compares.  Values are bit-identical to the reference for
  rows handled by the thread-group tier (every row of the five benchmark
  configurations) and within 1e-12 relative elsewhere.
* ``workers`` is accepted and ignored: one launch covers every row, results
  never depend on it (the reference guarantees the same, kernel.py:11-14).
* Operands stay cached in HBM while the host object is alive, so
  compress -> symbolic -> numeric on the same objects uploads each once.
"""

import weakref
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _lib
from .csr import CsrMatrix, as_csr
from .errors import CapacityError, DimensionError, MatrixValidationError

COMPRESSION_WORD_BITS = 64


def set_debug_checks(enabled: bool) -> None:
    """Accepted for compatibility (kernel.py:31-34).  Device tables are rebuilt
    per row and probe overflow always raises KernelError, so there is no
    separate debug scan to enable."""
    return None


@dataclass(frozen=True)
class RowRange:
    """Half-open row interval [begin, end) (kernel.py:37-49)."""

    begin: int
    end: int

    def __post_init__(self):
        if not (0 <= self.begin <= self.end):
            raise DimensionError("invalid row range [%d, %d)" % (self.begin, self.end))

    def __len__(self):
        return self.end - self.begin


class CompressedMatrix:
    """Per-row (set index, 64-bit mask) pairs (kernel.py:52-70).

    Produced on the device by ``compress``; the host arrays are fetched lazily
    on first access, and the device copy is reused by ``spgemm_symbolic``.
    """

    def __init__(self, num_rows, row_ptr=None, set_idx=None, set_bits=None, _device=None):
        self.num_rows = int(num_rows)
        self._dev = _device
        self._host = None
        if row_ptr is not None:
            arrs = (np.array(row_ptr, dtype=np.int64), np.array(set_idx, dtype=np.int64),
                    np.array(set_bits, dtype=np.uint64))
            for a in arrs:
                a.flags.writeable = False
            self._host = arrs

    def _fetch(self):
        if self._host is None:
            arrs = self._dev.download()
            for a in arrs:
                a.flags.writeable = False
            self._host = arrs
        return self._host

    @property
    def row_ptr(self):
        return self._fetch()[0]

    @property
    def set_idx(self):
        return self._fetch()[1]

    @property
    def set_bits(self):
        return self._fetch()[2]

    @property
    def n_sets(self) -> int:
        return int(self.set_idx.shape[0])

    def device(self, ctx=None):
        if self._dev is None:
            self._dev = _lib.DeviceCompressed.upload(self, ctx)
        return self._dev


# ---- device residency cache ---------------------------------------------------

_resident = {}


def _key(m):
    vals = None if m.values is None else m.values.__array_interface__["data"][0]
    return (id(m), m.row_ptr.__array_interface__["data"][0],
            m.col_idx.__array_interface__["data"][0], vals, m.num_rows, m.num_cols)


def _on_device(m) -> "_lib.DeviceCsr":
    """Device copy of a host CSR (cached while the host object lives)."""
    if isinstance(m, _lib.DeviceCsr):
        return m
    k = _key(m)
    hit = _resident.get(id(m))
    if hit is not None and hit[0] == k:
        return hit[1]
    d = _with_room(_lib.DeviceCsr.upload, m)
    try:
        weakref.finalize(m, _resident.pop, id(m), None)
        _resident[id(m)] = (k, d)
    except TypeError:  # not weak-referenceable: do not cache
        pass
    return d


# results keep their device copy, so a product fed straight back as an operand
# -- RA in R*A*P -- is not uploaded again.  The cache is a small LRU (a few
# results, bounded bytes); an allocation that runs out of HBM drops it and
# retries (``_with_room``), and ``release_device_cache`` empties it.
_RESULT_CACHE_BYTES = 8 << 30
_RESULT_CACHE_ENTRIES = 4
_results = OrderedDict()   # id(host) -> bytes, oldest first


def _evict(i):
    if _results.pop(i, None) is not None:
        _resident.pop(i, None)


def release_device_cache() -> None:
    """Drop every cached device copy of results and operands (their host
    objects stay valid; the next use uploads again)."""
    for i in list(_results):
        _evict(i)
    _resident.clear()


def _keep_result(host, dev):
    nbytes = 8 * (dev.num_rows + 1) + 12 * dev.nnz
    if nbytes > _RESULT_CACHE_BYTES:
        return host
    while _results and (len(_results) >= _RESULT_CACHE_ENTRIES or
                        sum(_results.values()) + nbytes > _RESULT_CACHE_BYTES):
        _evict(next(iter(_results)))
    try:
        k = _key(host)
        _resident[id(host)] = (k, dev)
        _results[id(host)] = nbytes
        weakref.finalize(host, _evict, id(host))
    except TypeError:
        pass
    return host


def _with_room(fn, *args):
    """fn(*args); on CapacityError (HBM exhausted) drop the device caches and
    retry once."""
    try:
        return fn(*args)
    except CapacityError:
        release_device_cache()
        return fn(*args)


def _counts_on_device(counts: np.ndarray) -> "_lib.DeviceVec":
    dv = getattr(counts, "_tsg_dev", None)
    snap = getattr(counts, "_tsg_snap", None)
    if dv is not None and snap is not None and np.array_equal(snap, counts):
        return dv
    return _lib.DeviceVec.upload(np.asarray(counts, dtype=np.int64))


class _Counts(np.ndarray):
    """int64 symbolic counts that remember their device copy (which also
    carries the per-row distinct-set counts the numeric phase sizes its
    tables with)."""


def _wrap_counts(host: np.ndarray, dev) -> np.ndarray:
    out = host.view(_Counts)
    out._tsg_dev = dev
    out._tsg_snap = host.copy()
    return out


# ---- the hot path ---------------------------------------------------------------

def compress(b) -> CompressedMatrix:
    """Bitmask-compress B's rows on the device (kernel.py:73-93)."""
    db = _on_device(b)
    return CompressedMatrix(b.num_rows, _device=_lib.d_compress(db))


def count_multiplications(a, b) -> int:
    """Scalar multiplications of A * B (kernel.py:96-103); flops are twice this."""
    if a.num_cols != b.num_rows:
        raise DimensionError("A is %dx%d but B has %d rows" % (a.num_rows, a.num_cols, b.num_rows))
    if a.col_idx.shape[0] == 0:
        return 0
    return _lib.d_count_multiplications(_on_device(a), _on_device(b))


def spgemm_symbolic(a, cb, workers: int = 1) -> np.ndarray:
    """Exact per-row nonzero counts of A * B (kernel.py:124-168)."""
    if a.num_cols != cb.num_rows:
        raise DimensionError("A has %d cols but compressed B has %d rows" % (a.num_cols, cb.num_rows))
    dcb = cb.device() if isinstance(cb, CompressedMatrix) else _lib.DeviceCompressed.upload(cb)
    dv = _lib.d_symbolic(_on_device(a), dcb)
    return _wrap_counts(dv.download(), dv)


def spgemm_numeric(a, b, c_counts, workers: int = 1) -> CsrMatrix:
    """C = A * B with exactly c_counts entries per row (kernel.py:171-232)."""
    if a.num_cols != b.num_rows:
        raise DimensionError("A is %dx%d but B has %d rows" % (a.num_rows, a.num_cols, b.num_rows))
    if b.values is None or a.values is None:
        raise MatrixValidationError("numeric multiply requires values on both operands")
    counts = np.asarray(c_counts)
    if counts.ndim != 1 or counts.shape[0] != a.num_rows:
        raise DimensionError("c_counts length must equal A's row count")
    dv = _counts_on_device(c_counts if isinstance(c_counts, _Counts) else counts)
    dc = _lib.d_numeric(_on_device(a), _on_device(b), None, dv)
    return _keep_result(dc.download(), dc)


def spgemm_numeric_fused(a, b_chunk, c_partial, a_rows: RowRange, b_rows: RowRange,
                         workers: int = 1) -> CsrMatrix:
    """result = c_partial + A[a_rows, b_rows] * B[b_rows, :] (kernel.py:235-340)."""
    if a_rows.end > a.num_rows:
        raise DimensionError("a_rows exceeds A's row count")
    if b_rows.end > a.num_cols:
        raise DimensionError("b_rows exceeds A's column count")
    if b_chunk.num_rows != len(b_rows):
        raise DimensionError("b_chunk must hold exactly the b_rows rows")
    if c_partial.num_rows != len(a_rows):
        raise DimensionError("c_partial must cover exactly the a_rows rows")
    if c_partial.num_cols != b_chunk.num_cols:
        raise DimensionError("c_partial and b_chunk column spaces differ")
    if len(a_rows) == 0:
        return c_partial
    if a.values is None or b_chunk.values is None or c_partial.values is None:
        raise MatrixValidationError("fused multiply requires numeric operands")
    out = _lib.d_numeric_fused(_on_device(a), _on_device(b_chunk), _on_device(c_partial),
                               a_rows.begin, a_rows.end, b_rows.begin, b_rows.end)
    return _keep_result(out.download(), out)


def multiply(a, b, workers: int = 1, placement="all_fast") -> CsrMatrix:
    """compress -> symbolic -> numeric on the device (kernel.py:343-346).

    ``placement`` (a memory.PlacementPolicy or its name, memory.py:193-223)
    places each operand in HBM ("fast") or in pinned, device-mapped host
    memory ("slow") that the kernels read and write in place over PCIe --
    the paper's data-placement experiment:
    "all_fast" (default), "b_in_fast" (A and C slow), "all_slow", or any
    PlacementPolicy with per-operand spaces.  "chunked" is the executors'
    job (chunking.execute_plan)."""
    if a.num_cols != b.num_rows:
        raise DimensionError("A has %d cols but compressed B has %d rows" % (a.num_cols, b.num_rows))
    if b.values is None or a.values is None:
        raise MatrixValidationError("numeric multiply requires values on both operands")
    from .memory import ALL_FAST, CHUNKED, FAST, PlacementPolicy
    pol = placement if isinstance(placement, PlacementPolicy) else PlacementPolicy.from_name(placement)
    if pol.name in (ALL_FAST, CHUNKED) or all(v == FAST for v in pol.spaces.values()):
        dc = _with_room(_lib.d_multiply, _on_device(a), _on_device(b))
        return _keep_result(dc.download(), dc)
    da = _on_device(a) if pol.space_of("A") == FAST else _lib.DeviceCsr.map_host(a)
    db = _on_device(b) if pol.space_of("B") == FAST else _lib.DeviceCsr.map_host(b)
    dc = _lib.d_multiply_placed(da, db, pol.space_of("C") != FAST)
    return dc.download()


def masked_row_intersect_count(l, cl, workers: int = 1) -> int:
    """Sum over L's entries (i, j) of |cols(L_j) & cols(L_i)|; L strictly
    lower triangular (kernel.py:349-394)."""
    if l.num_rows != cl.num_rows:
        raise DimensionError("matrix and compressed form disagree on row count")
    dcl = cl.device() if isinstance(cl, CompressedMatrix) else _lib.DeviceCompressed.upload(cl)
    return _lib.d_masked_count(_on_device(l), dcl)


# ---- device-resident entry points (no host round trips) ------------------------

def rap(r, a, p, fused: bool = True, workers: int = 1) -> CsrMatrix:
    """Galerkin triple product R * A * P.  The reference
    computes it as multiply(multiply(r, a), p) (kernel.py:343-346); with
    ``fused`` the device keeps each row of R * A in shared memory and never
    writes RA to HBM (csrc/tsg_rap.cu), falling back to the two multiplies
    when a row does not fit.  ``workers`` is accepted and ignored."""
    del workers
    r, a, p = as_csr(r), as_csr(a), as_csr(p)
    if r.num_cols != a.num_rows or a.num_cols != p.num_rows:
        raise DimensionError("R is %dx%d, A %dx%d, P %dx%d: inner dimensions differ"
                             % (r.num_rows, r.num_cols, a.num_rows, a.num_cols, p.num_rows, p.num_cols))
    c, _ = rap_device(upload(r), upload(a), upload(p), fused)
    return c.download()


def rap_device(dr, da, dp, fused: bool = True):
    """(C, fused_ran) for operands already in HBM; C is a DeviceCsr."""
    return _lib.d_rap(dr, da, dp, fused)


def multiply_device(da, db):
    """A * B for operands already in HBM; returns a DeviceCsr."""
    return _lib.d_multiply(da, db)


def upload(m):
    return _lib.DeviceCsr.upload(as_csr(m))
