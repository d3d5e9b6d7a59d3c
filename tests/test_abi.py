"""The C-ABI library loads and exports every symbol include/ibmi_b200.h
declares (no compute calls: this runs on CPU-only hosts too)."""

import ctypes
import os
import re

from conftest import ROOT


def header_functions():
    text = open(os.path.join(ROOT, "include", "ibmi_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ibmi_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header():
    from paper_2502_06377_b200 import _abi

    lib = _abi.lib()
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    bound = {n for n, _, _ in _abi.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound


def test_version_and_error_string():
    from paper_2502_06377_b200 import _abi

    lib = _abi.lib()
    assert b"sm_100a" in lib.ibmi_version()
    assert isinstance(lib.ibmi_last_error(), bytes)


def test_argument_errors_without_gpu():
    """Validation that happens before any CUDA call maps to the right codes."""
    from paper_2502_06377_b200 import _abi

    lib = _abi.lib()
    assert lib.ibmi_create(None, 0, 10, None) == _abi.ERR_INVALID
    h = ctypes.c_void_p()
    assert lib.ibmi_create(ctypes.byref(h), 0, 1, None) == _abi.ERR_DIM
    assert lib.ibmi_dgemm_nt(-1, 2, 2, 1.0, None, 2, None, 2, 0.0, None, 2, None) == _abi.ERR_DIM


def test_library_is_sm100a():
    from paper_2502_06377_b200 import _abi

    data = open(_abi.LIB_PATH, "rb").read()
    assert b"sm_100a" in data


def test_block_cache_entry_points_without_gpu():
    """The device block cache's ABI answers on a CPU-only host: nothing cached,
    release is a no-op (neither entry point touches CUDA when the cache is empty)."""
    import paper_2502_06377_b200 as pkg
    from paper_2502_06377_b200 import _abi

    assert pkg.cached_bytes() == 0
    assert pkg.cached_bytes(0) == 0
    pkg.release_cached_memory()
    assert _abi.lib().ibmi_cached_bytes(-1, None) == _abi.ERR_INVALID
