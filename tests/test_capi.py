"""The C-ABI library loads without a GPU and exports every declared symbol."""
import re
from pathlib import Path

from paper_2310_03294_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "distattn_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(da_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    decl = declared_functions()
    assert decl, "no declarations parsed"
    assert sorted(_lib.SIGNATURES) == decl


def test_library_exports_every_symbol():
    lib = _lib.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.da_abi_version() == 3


def test_status_maps_to_reference_exceptions():
    from paper_2310_03294_b200 import errors
    assert errors.STATUS[1] is errors.ShapeError
    assert errors.STATUS[2] is errors.ConfigError
    assert errors.STATUS[3] is errors.ScheduleError
    assert errors.STATUS[4] is errors.StateError
    assert errors.STATUS[5] is errors.DegenerateRowError
    for cls in errors.STATUS.values():
        assert issubclass(cls, errors.Error)


def test_argument_errors_without_device():
    """Shape/config validation happens before any device work."""
    import ctypes as C
    lib = _lib.lib()
    a = _lib.FwdArgs()
    a.d = 64
    assert lib.da_attn_fwd_chunk(C.byref(a), None) == 8  # DA_ERR_UNSUPPORTED
    a.d = 128
    a.h_q, a.h_kv = 3, 2
    assert lib.da_attn_fwd_chunk(C.byref(a), None) == 1  # ShapeError
    a.h_q, a.h_kv, a.rows_q, a.rows_kv, a.mask = 2, 2, 256, 128, 0
    assert lib.da_attn_fwd_chunk(C.byref(a), None) == 1  # diagonal needs a square chunk
    assert b"square" in lib.da_last_error()
    b = _lib.BwdArgs()
    b.d, b.h_q, b.h_kv, b.rows_q, b.rows_kv, b.mask = 128, 2, 2, 128, 128, 1
    assert lib.da_attn_bwd_chunk(C.byref(b), None) == 4  # StateError: no lse / D


def test_host_entry_points_validate_before_device_work():
    """The drop-in's host-buffer entry points (da_host_*) reject null buffers,
    d != 128 and non-square diagonal chunks without touching a device."""
    import ctypes as C

    import numpy as np
    lib = _lib.lib()
    buf = np.zeros((128, 64))
    p = C.c_void_p(buf.ctypes.data)
    assert lib.da_host_attn_update(None, 128, p, p, 128, 128, p, p, p, 0, 0.1) == 2
    assert b"null host buffer" in lib.da_last_error()
    assert lib.da_host_attn_update(p, 128, p, p, 128, 64, p, p, p, 0, 0.1) == 8  # d != 128
    assert lib.da_host_attn_update(p, 128, p, p, 64, 128, p, p, p, 0, 0.1) == 1  # diagonal
    assert lib.da_host_attn_backward(p, 128, p, p, 128, 128, p, p, None, 1, 0.1, p, p, p) == 2
    assert lib.da_host_attn_update(p, 128, p, p, 128, 128, p, p, p, 2, 0.1) == 0  # Empty: no-op
