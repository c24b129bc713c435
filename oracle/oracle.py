"""ctypes front end of the CPU oracle (tsg_oracle.c).

TEST INFRASTRUCTURE ONLY -- the parity checker and the CPU baseline.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module; the product package never does.

Results are plain numpy arrays (or tuples of them) so the checker does not
depend on the product's types.  Every function takes CSR-like objects with
``num_rows, num_cols, row_ptr, col_idx, values`` attributes.  Each call maps
1:1 to a reference function (see the citations in tsg_oracle.c) and returns
bit-identical results, including first-touch column order.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_I64 = ctypes.c_int64
_I64P = ctypes.POINTER(ctypes.c_int64)


class OracleError(Exception):
    def __init__(self, code, row):
        super().__init__("oracle status %d at row %d" % (code, row))
        self.code = code
        self.row = row


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        L.oc_compress.argtypes = [_I64, _i64p, _i64p, _i64p, _i64p, _u64p, _I64P]
        L.oc_count_multiplications.argtypes = [_I64, _i64p, _i64p]
        L.oc_count_multiplications.restype = ctypes.c_int64
        L.oc_symbolic.argtypes = [_I64, _i64p, _i64p, _i64p, _i64p, _u64p, _i64p, ctypes.c_int]
        L.oc_numeric.argtypes = [_I64, _i64p, _i64p, _f64p, _i64p, _i64p, _f64p, _i64p,
                                 _i64p, _i64p, _f64p, ctypes.c_int, _I64P]
        L.oc_fused_bounds.argtypes = [_I64, _I64, _i64p, _i64p, _I64, _I64, _i64p, _i64p, _i64p]
        L.oc_fused_bounds.restype = ctypes.c_int64
        L.oc_fused.argtypes = [_I64, _I64, _i64p, _i64p, _f64p, _I64, _I64, _i64p, _i64p,
                               _f64p, _i64p, _i64p, _f64p, _i64p, _i64p, _i64p, _i64p,
                               _f64p, ctypes.c_int]
        L.oc_masked_count.argtypes = [_I64, _i64p, _i64p, _i64p, _i64p, _u64p, ctypes.c_int,
                                      _I64P, _I64P]
        _lib = L
    return _lib


def _a(x, dt):
    return np.ascontiguousarray(np.asarray(x), dtype=dt)


def compress(b):
    """(row_ptr, set_idx, set_bits) in first-touch order (kernel.py:73-93)."""
    rp, ci = _a(b.row_ptr, np.int64), _a(b.col_idx, np.int64)
    nnz = ci.shape[0]
    out_rp = np.zeros(b.num_rows + 1, np.int64)
    s = np.zeros(max(nnz, 1), np.int64)
    bits = np.zeros(max(nnz, 1), np.uint64)
    n = ctypes.c_int64(0)
    lib().oc_compress(b.num_rows, rp, ci, out_rp, s, bits, ctypes.byref(n))
    return out_rp, s[:n.value].copy(), bits[:n.value].copy()


def count_multiplications(a, b):
    ci = _a(a.col_idx, np.int64)
    if ci.shape[0] == 0:
        return 0
    return int(lib().oc_count_multiplications(ci.shape[0], ci, _a(b.row_ptr, np.int64)))


def symbolic(a, cb, workers=1):
    """Per-row nnz of A*B from compress(B) = (row_ptr, set_idx, set_bits)."""
    crp, cs, cbits = cb
    counts = np.zeros(a.num_rows, np.int64)
    lib().oc_symbolic(a.num_rows, _a(a.row_ptr, np.int64), _a(a.col_idx, np.int64),
                      _a(crp, np.int64), _a(cs, np.int64) if len(cs) else np.zeros(1, np.int64),
                      _a(cbits, np.uint64) if len(cbits) else np.zeros(1, np.uint64),
                      counts, int(workers))
    return counts


def numeric(a, b, counts, workers=1):
    """(row_ptr, col_idx, values) of A*B in first-touch order."""
    counts = _a(counts, np.int64)
    tot = int(counts.sum())
    c_ptr = np.zeros(a.num_rows + 1, np.int64)
    c_col = np.zeros(max(tot, 1), np.int64)
    c_val = np.zeros(max(tot, 1), np.float64)
    err = ctypes.c_int64(-1)
    z64, zf = np.zeros(1, np.int64), np.zeros(1, np.float64)
    ca = _a(a.col_idx, np.int64)
    cb = _a(b.col_idx, np.int64)
    st = lib().oc_numeric(a.num_rows, _a(a.row_ptr, np.int64), ca if len(ca) else z64,
                          _a(a.values, np.float64) if len(ca) else zf,
                          _a(b.row_ptr, np.int64), cb if len(cb) else z64,
                          _a(b.values, np.float64) if len(cb) else zf,
                          counts if len(counts) else z64, c_ptr, c_col, c_val,
                          int(workers), ctypes.byref(err))
    if st:
        raise OracleError(st, err.value)
    return c_ptr, c_col[:tot].copy(), c_val[:tot].copy()


def fused(a, b_chunk, c_partial, a_lo, a_hi, b_lo, b_hi, workers=1):
    """(row_ptr, col_idx, values) of c_partial + A[a_rows, b_rows] * B[b_rows]
    (kernel.py:235-340, argument checks left to the caller)."""
    n_out = a_hi - a_lo
    z64, zf = np.zeros(1, np.int64), np.zeros(1, np.float64)

    def arr(x, dt, z):
        x = _a(x, dt)
        return x if x.shape[0] else z

    rp_a, ca, va = _a(a.row_ptr, np.int64), arr(a.col_idx, np.int64, z64), arr(a.values, np.float64, zf)
    rp_b, cbc, vbc = _a(b_chunk.row_ptr, np.int64), arr(b_chunk.col_idx, np.int64, z64), \
        arr(b_chunk.values, np.float64, zf)
    rp_c, cc, vc = _a(c_partial.row_ptr, np.int64), arr(c_partial.col_idx, np.int64, z64), \
        arr(c_partial.values, np.float64, zf)
    bounds = np.zeros(max(n_out, 1), np.int64)
    tot = lib().oc_fused_bounds(n_out, a_lo, rp_a, ca, b_lo, b_hi, rp_b, rp_c, bounds)
    sptr = np.zeros(max(n_out, 1), np.int64)
    if n_out > 1:
        np.cumsum(bounds[:n_out - 1], out=sptr[1:n_out])
    row_len = np.zeros(max(n_out, 1), np.int64)
    s_col = np.zeros(max(tot, 1), np.int64)
    s_val = np.zeros(max(tot, 1), np.float64)
    lib().oc_fused(n_out, a_lo, rp_a, ca, va, b_lo, b_hi, rp_b, cbc, vbc, rp_c, cc, vc,
                   bounds, sptr, row_len, s_col, s_val, int(workers))
    out_ptr = np.zeros(n_out + 1, np.int64)
    np.cumsum(row_len[:n_out], out=out_ptr[1:])
    take = np.concatenate([np.arange(sptr[i], sptr[i] + row_len[i]) for i in range(n_out)]) \
        if n_out else np.zeros(0, np.int64)
    take = take.astype(np.int64)
    return out_ptr, s_col[take], s_val[take]


def masked_count(l, cl, workers=1):
    """Sum over L's entries (i, j) of |cols(L_i) & cols(L_j)| (kernel.py:349-394)."""
    crp, cs, cbits = cl
    tot = ctypes.c_int64(0)
    err = ctypes.c_int64(-1)
    z64 = np.zeros(1, np.int64)
    ci = _a(l.col_idx, np.int64)
    st = lib().oc_masked_count(l.num_rows, _a(l.row_ptr, np.int64), ci if len(ci) else z64,
                               _a(crp, np.int64), _a(cs, np.int64) if len(cs) else z64,
                               _a(cbits, np.uint64) if len(cbits) else np.zeros(1, np.uint64),
                               int(workers), ctypes.byref(tot), ctypes.byref(err))
    if st:
        raise OracleError(st, err.value)
    return int(tot.value)


def multiply(a, b, workers=1):
    cb = compress(b)
    return numeric(a, b, symbolic(a, cb, workers), workers)


def count_triangles_lower(l, workers=1):
    return masked_count(l, compress(l), workers)
