"""The C ABI boundary: libtsg.so loads on a CPU-only host, exports exactly the
symbols include/tsg.h declares, and status codes map to the reference's
exception classes.  No compute calls (no GPU here)."""

import re
import os

import pytest

from conftest import ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "tsg.h")).read()
    return set(re.findall(r"^\s*(?:const\s+char\s*\*\s*|int\s+)(tsg_\w+)\s*\(", text, re.M))


def test_library_exports_every_header_symbol():
    from paper_1804_00695_b200 import _lib
    lib = _lib.load()
    declared = header_symbols()
    assert len(declared) >= 25
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_lib.EXPORTS) == declared


def test_abi_version():
    from paper_1804_00695_b200 import _lib
    assert _lib.load().tsg_abi_version() == 1


def test_error_mapping_matches_reference_classes():
    from paper_1804_00695_b200 import _lib, errors
    assert _lib._ERRORS[_lib.TSG_EDIM] is errors.DimensionError
    assert _lib._ERRORS[_lib.TSG_EVALID] is errors.MatrixValidationError
    assert _lib._ERRORS[_lib.TSG_EKERNEL] is errors.KernelError
    assert _lib._ERRORS[_lib.TSG_ECAPACITY] is errors.CapacityError
    assert _lib._ERRORS[_lib.TSG_EUNSPLIT] is errors.UnsplittableRowError
    for cls in _lib._ERRORS.values():
        if cls is not ValueError:
            assert issubclass(cls, errors.TieredSpgemmError)


def test_no_cpu_fallback_without_gpu():
    """On a host without a B200 the product path raises instead of computing."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    import paper_1804_00695_b200 as tsg
    a = tsg.CsrMatrix.identity(3)
    with pytest.raises(tsg.KernelError):
        tsg.multiply(a, a)


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1804_00695_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).lower() or f == "__init__.py", f
