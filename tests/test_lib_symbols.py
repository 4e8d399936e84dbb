"""The C-ABI library loads and exports every symbol include/hybrimoe.h declares (CPU only)."""
import ctypes

from paper_2504_05897_b200 import _lib


def test_every_declared_symbol_is_exported():
    names = _lib.symbols_declared()
    assert len(names) > 60
    missing = [n for n in names if not hasattr(_lib.lib, n)]
    assert not missing, missing


def test_version_and_error_channel():
    assert _lib.lib.hm_version().startswith(b"hybrimoe-b200")
    out = ctypes.c_double()
    p = _lib.Profile(1.0, 1.0, 1.0, 0.0, 256, 0.0, 1.4, 0.0, 0.0)
    assert _lib.lib.hm_gpu_time(ctypes.byref(p), 0, ctypes.byref(out)) == _lib.HM_EVALUE
    assert "load must be >= 1" in _lib.last_error()
