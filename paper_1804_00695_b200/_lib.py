"""ctypes binding of libtsg.so (include/tsg.h) and device-resident handles.

This is the stub a maintainer would add to the reference to bind the C ABI
(INTEGRATION.md shows it next to the reference call sites).  There is no CPU
fallback: if the library or a B200 is missing, every entry point raises
KernelError.  Status codes map to the reference's exception classes
(errors.py:4-45).
"""

import ctypes
import os
import threading
import weakref

import numpy as np

from .csr import CsrMatrix
from .errors import (CapacityError, DimensionError, GridError, KernelError,
                     MatrixValidationError, UnsplittableRowError)

_HERE = os.path.dirname(os.path.abspath(__file__))
# TSG_LIB: an alternative build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("TSG_LIB") or os.path.join(_HERE, "libtsg.so")

TSG_OK, TSG_EDIM, TSG_EVALID, TSG_EKERNEL, TSG_ECAPACITY, TSG_EUNSPLIT, TSG_ECUDA, TSG_EARG = range(8)

_ERRORS = {
    TSG_EDIM: DimensionError,
    TSG_EVALID: MatrixValidationError,
    TSG_EKERNEL: KernelError,
    TSG_ECAPACITY: CapacityError,
    TSG_EUNSPLIT: UnsplittableRowError,
    TSG_ECUDA: KernelError,
    TSG_EARG: ValueError,
}

# every symbol include/tsg.h declares (checked by tests/test_boundary.py)
EXPORTS = (
    "tsg_last_error", "tsg_abi_version", "tsg_device_count", "tsg_init", "tsg_destroy",
    "tsg_sync", "tsg_mem_in_use", "tsg_probe_stats", "tsg_pool_reserved", "tsg_last_phase_ms", "tsg_set_timing", "tsg_get_stats",
    "tsg_csr_upload", "tsg_csr_info", "tsg_csr_download", "tsg_csr_slice_rows", "tsg_csr_free",
    "tsg_compress", "tsg_cmat_info", "tsg_cmat_download", "tsg_cmat_upload", "tsg_cmat_free",
    "tsg_vec_upload", "tsg_vec_download", "tsg_vec_len", "tsg_vec_free",
    "tsg_count_multiplications", "tsg_symbolic", "tsg_numeric", "tsg_multiply",
    "tsg_numeric_fused", "tsg_masked_count", "tsg_event_record", "tsg_event_elapsed",
    "tsg_csr_from_device", "tsg_csr_device_ptrs", "tsg_host_alloc", "tsg_host_free",
    "tsg_chunk_multiply", "tsg_csr_map_host", "tsg_multiply_placed",
    "tsg_graph_lower", "tsg_rmat_graph", "tsg_numeric_calls", "tsg_numeric_ms",
    "tsg_csr_set_values", "tsg_gather_sharded", "tsg_stencil", "tsg_aggregation", "tsg_transpose",
    "tsg_rap", "tsg_row_flops", "tsg_stream", "tsg_chunk_symbolic",
    "tsg_shard_granularity", "tsg_shard_alloc", "tsg_shard_free", "tsg_shard_map", "tsg_vmap_free",
    "tsg_csr_view", "tsg_mg_multiply", "tsg_memcpy", "tsg_csr_dims",
)

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PP = ctypes.POINTER(ctypes.c_void_p)

_SIGS = {
    "tsg_last_error": ([], ctypes.c_char_p),
    "tsg_probe_stats": ([_P, ctypes.POINTER(ctypes.c_int64), ctypes.c_int], ctypes.c_int),
    "tsg_abi_version": ([], ctypes.c_int),
    "tsg_device_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "tsg_init": ([ctypes.c_int, _PP], ctypes.c_int),
    "tsg_destroy": ([_P], ctypes.c_int),
    "tsg_sync": ([_P], ctypes.c_int),
    "tsg_mem_in_use": ([_P, _PI64], ctypes.c_int),
    "tsg_pool_reserved": ([_P, _PI64], ctypes.c_int),
    "tsg_last_phase_ms": ([_P, ctypes.POINTER(ctypes.c_float), ctypes.c_int], ctypes.c_int),
    "tsg_set_timing": ([_P, ctypes.c_int], ctypes.c_int),
    "tsg_get_stats": ([_P, _P], ctypes.c_int),
    "tsg_csr_upload": ([_P, _I64, _I64, _I64, _P, _P, _P, _PP], ctypes.c_int),
    "tsg_csr_info": ([_P, _PI64, _PI64, _PI64, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "tsg_csr_download": ([_P, _P, _P, _P, _P], ctypes.c_int),
    "tsg_csr_slice_rows": ([_P, _P, _I64, _I64, _PP], ctypes.c_int),
    "tsg_csr_free": ([_P, _P], ctypes.c_int),
    "tsg_compress": ([_P, _P, _PP], ctypes.c_int),
    "tsg_cmat_info": ([_P, _P, _PI64, _PI64], ctypes.c_int),
    "tsg_cmat_download": ([_P, _P, _P, _P, _P], ctypes.c_int),
    "tsg_cmat_upload": ([_P, _I64, _I64, _P, _P, _P, _PP], ctypes.c_int),
    "tsg_cmat_free": ([_P, _P], ctypes.c_int),
    "tsg_vec_upload": ([_P, _I64, _P, _PP], ctypes.c_int),
    "tsg_vec_download": ([_P, _P, _P], ctypes.c_int),
    "tsg_vec_len": ([_P, _PI64], ctypes.c_int),
    "tsg_vec_free": ([_P, _P], ctypes.c_int),
    "tsg_count_multiplications": ([_P, _P, _P, _PI64], ctypes.c_int),
    "tsg_row_flops": ([_P, _P, _P, _P, _PI64], ctypes.c_int),
    "tsg_stream": ([_P, _PP], ctypes.c_int),
    "tsg_shard_granularity": ([_P, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "tsg_shard_alloc": ([_P, ctypes.c_size_t, _PP, _PP, ctypes.POINTER(ctypes.c_int),
                         ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "tsg_shard_free": ([_P, _P], ctypes.c_int),
    "tsg_shard_map": ([_P, ctypes.c_int, _P, _P, _PP, _PP], ctypes.c_int),
    "tsg_vmap_free": ([_P, _P], ctypes.c_int),
    "tsg_csr_view": ([_P, _I64, _I64, _I64, _P, _P, _P, ctypes.c_int, _I64, _PP], ctypes.c_int),
    "tsg_mg_multiply": ([_P, _P, _P, _I64, _PP, _P], ctypes.c_int),
    "tsg_memcpy": ([_P, _P, _P, ctypes.c_size_t], ctypes.c_int),
    "tsg_csr_dims": ([_P, _PI64, _PI64, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "tsg_symbolic": ([_P, _P, _P, _PP], ctypes.c_int),
    "tsg_numeric": ([_P, _P, _P, _P, _P, _PP], ctypes.c_int),
    "tsg_multiply": ([_P, _P, _P, _PP], ctypes.c_int),
    "tsg_numeric_fused": ([_P, _P, _P, _P, _I64, _I64, _I64, _I64, _PP], ctypes.c_int),
    "tsg_masked_count": ([_P, _P, _P, _PI64], ctypes.c_int),
    "tsg_graph_lower": ([_P, _P, ctypes.c_int, _PP, _P], ctypes.c_int),
    "tsg_numeric_calls": ([_P, _PI64], ctypes.c_int),
    "tsg_csr_set_values": ([_P, _P, ctypes.c_double], ctypes.c_int),
    "tsg_stencil": ([_P, ctypes.c_int, _P, ctypes.c_int, _I64, _I64, _PP], ctypes.c_int),
    "tsg_aggregation": ([_P, _P, ctypes.c_int, ctypes.c_int, _PP, _PP], ctypes.c_int),
    "tsg_transpose": ([_P, _P, _PP], ctypes.c_int),
    "tsg_rap": ([_P, _P, _P, _P, ctypes.c_int, _PP, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "tsg_gather_sharded": ([_P, ctypes.c_int, _P, _P, _P, _P, _I64, _P, _PP], ctypes.c_int),
    "tsg_numeric_ms": ([_P, _I64, ctypes.POINTER(ctypes.c_float)], ctypes.c_int),
    "tsg_rmat_graph": ([_P, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_double,
                        ctypes.c_double, ctypes.c_double, _PP], ctypes.c_int),
    "tsg_event_record": ([_P, ctypes.c_int], ctypes.c_int),
    "tsg_event_elapsed": ([_P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)],
                          ctypes.c_int),
    "tsg_csr_from_device": ([_P, _I64, _I64, _I64, _P, _P, _P, _PP], ctypes.c_int),
    "tsg_csr_device_ptrs": ([_P, _PP, _PP, _PP], ctypes.c_int),
    "tsg_host_alloc": ([ctypes.c_size_t, _PP], ctypes.c_int),
    "tsg_host_free": ([_P], ctypes.c_int),
    "tsg_csr_map_host": ([_P, _I64, _I64, _I64, _P, _P, _P, _PP], ctypes.c_int),
    "tsg_multiply_placed": ([_P, _P, _P, ctypes.c_int, _PP], ctypes.c_int),
    "tsg_chunk_multiply": ([_P, ctypes.c_int, _I64, _I64, _P, _P, _P, _I64, _I64, _P, _P, _P,
                            _P, _P, _P, _I64, _P, _I64, _P, _I64, _P], ctypes.c_int),
    "tsg_chunk_symbolic": ([_P, _I64, _I64, _P, _P, _I64, _I64, _P, _P, _I64, _P, _P], ctypes.c_int),
}

_lib = None
_lib_lock = threading.Lock()


def load():
    """Load libtsg.so (raises KernelError if it was never built)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise KernelError("libtsg.so is not built (run __graft_entry__.build()); "
                                  "there is no CPU fallback")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def check(status):
    if status == TSG_OK:
        return
    msg = load().tsg_last_error().decode(errors="replace")
    raise _ERRORS.get(status, KernelError)(msg)


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


class _PinnedBlock:
    """Owner of one pinned host block; returns it to libtsg's pool when the
    last numpy view goes away."""

    __slots__ = ("addr", "__weakref__")

    def __init__(self, nbytes):
        p = ctypes.c_void_p()
        check(load().tsg_host_alloc(max(int(nbytes), 1), ctypes.byref(p)))
        self.addr = p.value
        weakref.finalize(self, _host_free, p.value)


def _host_free(addr):
    try:
        load().tsg_host_free(ctypes.c_void_p(addr))
    except Exception:  # interpreter shutdown
        pass


def pinned_empty(n, dtype):
    """numpy array of n elements in pinned host memory (pooled)."""
    dtype = np.dtype(dtype)
    nbytes = int(n) * dtype.itemsize
    blk = _PinnedBlock(nbytes)
    raw = (ctypes.c_char * max(nbytes, 1)).from_address(blk.addr)
    raw._owner = blk
    return np.frombuffer(raw, dtype=dtype, count=int(n))


class _Stats(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("symbolic_ms", ctypes.c_float),
                ("numeric_ms", ctypes.c_float)]


class Context:
    """One CUDA device: compute stream + copy streams inside libtsg."""

    _instances = {}

    def __init__(self, device=0):
        self.device = device
        h = ctypes.c_void_p()
        check(load().tsg_init(device, ctypes.byref(h)))
        self.h = h

    @classmethod
    def get(cls, device=None):
        if device is None:
            device = int(os.environ.get("TSG_DEVICE", os.environ.get("LOCAL_RANK", "0")))
            n = ctypes.c_int(0)
            check(load().tsg_device_count(ctypes.byref(n)))
            if n.value == 0:
                raise KernelError("no CUDA device visible; libtsg has no CPU fallback")
            device = device % n.value
        ctx = cls._instances.get(device)
        if ctx is None:
            ctx = cls._instances[device] = Context(device)
        return ctx

    def sync(self):
        check(load().tsg_sync(self.h))

    def set_timing(self, on=True):
        check(load().tsg_set_timing(self.h, 1 if on else 0))

    def phase_ms(self):
        out = (ctypes.c_float * 8)()
        check(load().tsg_last_phase_ms(self.h, out, 8))
        return list(out)

    def stats(self):
        """(launches so far, symbolic ms, numeric ms of the last multiply)."""
        st = _Stats()
        check(load().tsg_get_stats(self.h, ctypes.byref(st)))
        return st.launches, st.symbolic_ms, st.numeric_ms

    def stream(self) -> int:
        """cudaStream_t of the compute stream (for torch.cuda.ExternalStream)."""
        v = ctypes.c_void_p()
        check(load().tsg_stream(self.h, ctypes.byref(v)))
        return v.value or 0

    def record(self, slot):
        check(load().tsg_event_record(self.h, slot))

    def numeric_calls(self) -> int:
        v = ctypes.c_int64(0)
        check(load().tsg_numeric_calls(self.h, ctypes.byref(v)))
        return v.value

    def numeric_ms(self, call: int) -> float:
        v = ctypes.c_float()
        check(load().tsg_numeric_ms(self.h, int(call), ctypes.byref(v)))
        return v.value

    def elapsed_ms(self, a, b):
        v = ctypes.c_float()
        check(load().tsg_event_elapsed(self.h, a, b, ctypes.byref(v)))
        return v.value

    def pool_reserved(self):
        v = ctypes.c_int64(0)
        check(load().tsg_pool_reserved(self.h, ctypes.byref(v)))
        return v.value

    def mem_in_use(self):
        v = ctypes.c_int64(0)
        check(load().tsg_mem_in_use(self.h, ctypes.byref(v)))
        return v.value


class _Handle:
    _free_fn = None

    def __init__(self, ctx, h):
        self.ctx = ctx
        self.h = h
        self._fin = weakref.finalize(self, _Handle._release, self._free_fn, ctx, h)

    @staticmethod
    def _release(fname, ctx, h):
        try:
            getattr(load(), fname)(ctx.h, h)
        except Exception:  # interpreter shutdown
            pass

    def free(self):
        self._fin()


class DeviceCsr(_Handle):
    """CSR matrix resident in HBM (int64 offsets, int32 columns, fp64 values)."""

    _free_fn = "tsg_csr_free"

    def __init__(self, ctx, h):
        super().__init__(ctx, h)
        r, c, hv = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
        check(load().tsg_csr_dims(h, ctypes.byref(r), ctypes.byref(c), ctypes.byref(hv)))
        self.num_rows, self.num_cols, self.has_values = r.value, c.value, bool(hv.value)
        self._nnz = None

    @property
    def nnz(self) -> int:
        """Entries (a product's count is read from the device on first use:
        the multiply that made it did not wait for the device)."""
        if self._nnz is None:
            n = ctypes.c_int64()
            check(load().tsg_csr_info(self.h, None, None, ctypes.byref(n), None))
            self._nnz = n.value
        return self._nnz

    @classmethod
    def upload(cls, m, ctx=None):
        ctx = ctx or Context.get()
        rp = np.ascontiguousarray(m.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(m.col_idx, dtype=np.int64)
        va = None if m.values is None else np.ascontiguousarray(m.values, dtype=np.float64)
        if rp.shape[0] != m.num_rows + 1:
            raise MatrixValidationError("row_ptr length must be num_rows + 1")
        h = ctypes.c_void_p()
        check(load().tsg_csr_upload(ctx.h, m.num_rows, m.num_cols, ci.shape[0], _ptr(rp), _ptr(ci),
                                    _ptr(va), ctypes.byref(h)))
        return cls(ctx, h)

    @classmethod
    def map_host(cls, m, ctx=None):
        """A CSR kept in pinned, device-mapped HOST memory (placement slow tier)."""
        ctx = ctx or Context.get()
        rp = np.ascontiguousarray(m.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(m.col_idx, dtype=np.int64)
        va = None if m.values is None else np.ascontiguousarray(m.values, dtype=np.float64)
        h = ctypes.c_void_p()
        check(load().tsg_csr_map_host(ctx.h, m.num_rows, m.num_cols, ci.shape[0], _ptr(rp), _ptr(ci),
                                      _ptr(va), ctypes.byref(h)))
        return cls(ctx, h)

    def set_values(self, value: float) -> "DeviceCsr":
        """Every stored entry := value (a pattern matrix gets a value array)."""
        check(load().tsg_csr_set_values(self.ctx.h, self.h, float(value)))
        self.has_values = True
        return self

    def download(self) -> CsrMatrix:
        rp = pinned_empty(self.num_rows + 1, np.int64)
        ci = pinned_empty(self.nnz, np.int64)
        va = pinned_empty(self.nnz, np.float64) if self.has_values else None
        check(load().tsg_csr_download(self.ctx.h, self.h, _ptr(rp), _ptr(ci), _ptr(va)))
        return CsrMatrix._adopt(self.num_rows, self.num_cols, rp, ci, va)

    @classmethod
    def from_device(cls, ctx, rows, cols, nnz, rp_ptr, col_ptr, val_ptr):
        """D2D import of CSR arrays already on this device (int64/int32/fp64)."""
        h = ctypes.c_void_p()
        check(load().tsg_csr_from_device(ctx.h, rows, cols, nnz, ctypes.c_void_p(rp_ptr),
                                         ctypes.c_void_p(col_ptr),
                                         None if val_ptr is None else ctypes.c_void_p(val_ptr),
                                         ctypes.byref(h)))
        return cls(ctx, h)

    def device_ptrs(self):
        rp, ci, va = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        check(load().tsg_csr_device_ptrs(self.h, ctypes.byref(rp), ctypes.byref(ci), ctypes.byref(va)))
        return rp.value, ci.value, va.value

    def slice_rows(self, begin, end):
        h = ctypes.c_void_p()
        check(load().tsg_csr_slice_rows(self.ctx.h, self.h, begin, end, ctypes.byref(h)))
        return DeviceCsr(self.ctx, h)


class DeviceCompressed(_Handle):
    _free_fn = "tsg_cmat_free"

    def __init__(self, ctx, h, rows):
        super().__init__(ctx, h)
        self.num_rows = rows

    @classmethod
    def upload(cls, cm, ctx=None):
        ctx = ctx or Context.get()
        rp = np.ascontiguousarray(cm.row_ptr, dtype=np.int64)
        si = np.ascontiguousarray(cm.set_idx, dtype=np.int64)
        sb = np.ascontiguousarray(cm.set_bits, dtype=np.uint64)
        h = ctypes.c_void_p()
        check(load().tsg_cmat_upload(ctx.h, cm.num_rows, si.shape[0], _ptr(rp), _ptr(si), _ptr(sb),
                                     ctypes.byref(h)))
        return cls(ctx, h, cm.num_rows)

    def download(self):
        r, n = ctypes.c_int64(), ctypes.c_int64()
        check(load().tsg_cmat_info(self.ctx.h, self.h, ctypes.byref(r), ctypes.byref(n)))
        rp = np.empty(self.num_rows + 1, dtype=np.int64)
        si = np.empty(n.value, dtype=np.int64)
        sb = np.empty(n.value, dtype=np.uint64)
        check(load().tsg_cmat_download(self.ctx.h, self.h, _ptr(rp), _ptr(si), _ptr(sb)))
        return rp, si, sb


class DeviceVec(_Handle):
    _free_fn = "tsg_vec_free"

    def __init__(self, ctx, h):
        super().__init__(ctx, h)
        n = ctypes.c_int64()
        check(load().tsg_vec_len(h, ctypes.byref(n)))
        self.n = n.value

    @classmethod
    def upload(cls, arr, ctx=None):
        ctx = ctx or Context.get()
        a = np.ascontiguousarray(arr, dtype=np.int64)
        h = ctypes.c_void_p()
        check(load().tsg_vec_upload(ctx.h, a.shape[0], _ptr(a), ctypes.byref(h)))
        return cls(ctx, h)

    def download(self):
        out = np.empty(self.n, dtype=np.int64)
        check(load().tsg_vec_download(self.ctx.h, self.h, _ptr(out)))
        return out


# ---- raw calls on device handles ---------------------------------------------

def d_compress(db: DeviceCsr) -> DeviceCompressed:
    h = ctypes.c_void_p()
    check(load().tsg_compress(db.ctx.h, db.h, ctypes.byref(h)))
    return DeviceCompressed(db.ctx, h, db.num_rows)


def d_count_multiplications(da, db) -> int:
    v = ctypes.c_int64()
    check(load().tsg_count_multiplications(da.ctx.h, da.h, db.h, ctypes.byref(v)))
    return v.value


def d_row_flops(da, db):
    """(per-row multiplications of A*B as int64 numpy, total)."""
    out = np.empty(da.num_rows, dtype=np.int64)
    tot = ctypes.c_int64()
    check(load().tsg_row_flops(da.ctx.h, da.h, db.h, _ptr(out), ctypes.byref(tot)))
    return out, tot.value


class MgStats(ctypes.Structure):
    _fields_ = [("nnz", ctypes.c_int64), ("blocks", ctypes.c_int64), ("max_block_nnz", ctypes.c_int64),
                ("value_sum", ctypes.c_double), ("value_sumsq", ctypes.c_double)]


def d_mg_multiply(da, db, c_budget_bytes: int = 0, keep_c: bool = True):
    """(C block or None, stats dict): one GPU's row block of A * B
    (tsg_mg_multiply); c_budget_bytes > 0 streams C through that budget."""
    h = ctypes.c_void_p()
    st = MgStats()
    check(load().tsg_mg_multiply(da.ctx.h, da.h, db.h, int(c_budget_bytes),
                                 ctypes.byref(h) if keep_c else None, ctypes.byref(st)))
    c = DeviceCsr(da.ctx, h) if (keep_c and h.value) else None
    return c, {"nnz": st.nnz, "blocks": st.blocks, "max_block_nnz": st.max_block_nnz,
               "value_sum": st.value_sum, "value_sumsq": st.value_sumsq}


class Shard(_Handle):
    """This GPU's exported VMM physical shard (tsg_shard_alloc)."""

    _free_fn = "tsg_shard_free"

    def __init__(self, ctx, nbytes):
        h, p = ctypes.c_void_p(), ctypes.c_void_p()
        fd, size = ctypes.c_int(-1), ctypes.c_size_t(0)
        check(load().tsg_shard_alloc(ctx.h, int(nbytes), ctypes.byref(h), ctypes.byref(p),
                                     ctypes.byref(fd), ctypes.byref(size)))
        super().__init__(ctx, h)
        self.ptr, self.fd, self.size = p.value, fd.value, size.value


class VMap(_Handle):
    """Shards (own + peers', by file descriptor) mapped into one VA range."""

    _free_fn = "tsg_vmap_free"

    def __init__(self, ctx, fds, sizes):
        n = len(fds)
        fa = (ctypes.c_int * n)(*[int(x) for x in fds])
        sa = (ctypes.c_size_t * n)(*[int(x) for x in sizes])
        h, va = ctypes.c_void_p(), ctypes.c_void_p()
        check(load().tsg_shard_map(ctx.h, n, fa, sa, ctypes.byref(h), ctypes.byref(va)))
        super().__init__(ctx, h)
        self.va = va.value
        self.total = sum(int(x) for x in sizes)


def memcpy(ctx, dst: int, src: int, nbytes: int) -> None:
    """Synchronous copy between device-reachable addresses (tsg_memcpy)."""
    check(load().tsg_memcpy(ctx.h, ctypes.c_void_p(dst), ctypes.c_void_p(src), int(nbytes)))


def shard_granularity(ctx) -> int:
    g = ctypes.c_size_t(0)
    check(load().tsg_shard_granularity(ctx.h, ctypes.byref(g)))
    return g.value


def d_csr_view(ctx, rows, cols, nnz, rp_ptr, col_ptr, val_ptr, sorted_rows=False, max_row=-1,
               owners=()) -> DeviceCsr:
    """DeviceCsr over caller-owned device arrays; `owners` are kept alive
    for as long as the view."""
    h = ctypes.c_void_p()
    check(load().tsg_csr_view(ctx.h, int(rows), int(cols), int(nnz), ctypes.c_void_p(rp_ptr),
                              ctypes.c_void_p(col_ptr), ctypes.c_void_p(val_ptr) if val_ptr else None,
                              1 if sorted_rows else 0, int(max_row), ctypes.byref(h)))
    v = DeviceCsr(ctx, h)
    v._owners = tuple(owners)
    return v


def d_symbolic(da, dcb) -> DeviceVec:
    h = ctypes.c_void_p()
    check(load().tsg_symbolic(da.ctx.h, da.h, dcb.h, ctypes.byref(h)))
    return DeviceVec(da.ctx, h)


def d_numeric(da, db, dcb, dcounts) -> DeviceCsr:
    h = ctypes.c_void_p()
    check(load().tsg_numeric(da.ctx.h, da.h, db.h, None if dcb is None else dcb.h, dcounts.h,
                             ctypes.byref(h)))
    return DeviceCsr(da.ctx, h)


def d_multiply(da, db) -> DeviceCsr:
    h = ctypes.c_void_p()
    check(load().tsg_multiply(da.ctx.h, da.h, db.h, ctypes.byref(h)))
    return DeviceCsr(da.ctx, h)


def d_multiply_placed(da, db, c_in_host: bool) -> DeviceCsr:
    h = ctypes.c_void_p()
    check(load().tsg_multiply_placed(da.ctx.h, da.h, db.h, 1 if c_in_host else 0, ctypes.byref(h)))
    return DeviceCsr(da.ctx, h)


def d_numeric_fused(da, dbc, dcp, a_lo, a_hi, b_lo, b_hi) -> DeviceCsr:
    h = ctypes.c_void_p()
    check(load().tsg_numeric_fused(da.ctx.h, da.h, dbc.h, dcp.h, a_lo, a_hi, b_lo, b_hi,
                                   ctypes.byref(h)))
    return DeviceCsr(da.ctx, h)


def d_masked_count(dl, dcl) -> int:
    v = ctypes.c_int64()
    check(load().tsg_masked_count(dl.ctx.h, dl.h, dcl.h, ctypes.byref(v)))
    return v.value


check_ = check


def d_graph_lower(dg, check: bool = True, want_perm: bool = False):
    """(L, perm or None): degree-ordered strict lower triangle on the device."""
    h = ctypes.c_void_p()
    perm = np.empty(dg.num_rows, dtype=np.int64) if want_perm else None
    check_(load().tsg_graph_lower(dg.ctx.h, dg.h, 1 if check else 0, ctypes.byref(h),
                                  _ptr(perm) if want_perm else None))
    return DeviceCsr(dg.ctx, h), perm


def d_rmat_graph(scale: int, edge_factor: int, seed: int, a: float, b: float, c: float,
                 ctx=None) -> DeviceCsr:
    ctx = ctx or Context.get()
    h = ctypes.c_void_p()
    check_(load().tsg_rmat_graph(ctx.h, int(scale), int(edge_factor), int(seed) & ((1 << 64) - 1),
                                 float(a), float(b), float(c), ctypes.byref(h)))
    return DeviceCsr(ctx, h)


STENCIL_CODES = {"laplace2d": 0, "laplace3d": 1, "bigstar2d": 2, "brick3d": 3, "elasticity3d": 4}


def d_stencil(kind: str, dims, row_lo: int = -1, row_hi: int = -1, ctx=None) -> DeviceCsr:
    ctx = ctx or Context.get()
    if kind not in STENCIL_CODES:
        raise GridError("unknown stencil kind %r" % (kind,))
    d = np.ascontiguousarray(dims, dtype=np.int64)
    h = ctypes.c_void_p()
    check_(load().tsg_stencil(ctx.h, STENCIL_CODES[kind], _ptr(d), int(d.size), int(row_lo), int(row_hi),
                              ctypes.byref(h)))
    return DeviceCsr(ctx, h)


def d_aggregation(dims, factor: int = 2, ctx=None):
    ctx = ctx or Context.get()
    d = np.ascontiguousarray(dims, dtype=np.int64)
    hp, hr = ctypes.c_void_p(), ctypes.c_void_p()
    check_(load().tsg_aggregation(ctx.h, _ptr(d), int(d.size), int(factor), ctypes.byref(hp), ctypes.byref(hr)))
    return DeviceCsr(ctx, hp), DeviceCsr(ctx, hr)


def d_transpose(da) -> DeviceCsr:
    h = ctypes.c_void_p()
    check_(load().tsg_transpose(da.ctx.h, da.h, ctypes.byref(h)))
    return DeviceCsr(da.ctx, h)


def d_rap(dr, da, dp, fused: bool = True):
    """(C, fused_ran): C = R * A * P in HBM (csrc/tsg_rap.cu)."""
    h = ctypes.c_void_p()
    f = ctypes.c_int(0)
    check_(load().tsg_rap(da.ctx.h, dr.h, da.h, dp.h, 1 if fused else 0, ctypes.byref(h), ctypes.byref(f)))
    return DeviceCsr(da.ctx, h), bool(f.value)


def d_gather_sharded(da, shards, b_cols: int) -> DeviceCsr:
    """shards: [(row_lo, row_hi, rp_ptr, col_ptr, val_ptr or 0)] device
    pointers in row order (local or peer memory)."""
    n = len(shards)
    lo = np.array([s[0] for s in shards] + [shards[-1][1]], dtype=np.int64)
    arr = lambda k: (ctypes.c_void_p * n)(*[ctypes.c_void_p(int(s[k]) or None) for s in shards])
    h = ctypes.c_void_p()
    vals = arr(4) if all(s[4] for s in shards) else None
    check_(load().tsg_gather_sharded(da.ctx.h, n, _ptr(lo), arr(2), arr(3), vals, int(b_cols), da.h,
                                     ctypes.byref(h)))
    return DeviceCsr(da.ctx, h)
