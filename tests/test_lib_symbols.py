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


def test_ffn_rejects_bad_groups_without_touching_the_device():
    arr = (_lib.HmGroup * 1)()
    arr[0].slot, arr[0].row_begin, arr[0].row_count = 5, 0, 1
    rc = _lib.lib.hm_expert_ffn(None, 2, 256, 256, arr, 1, None, 1, None, None, 0, None)
    assert rc == _lib.HM_EVALUE and "outside the pool" in _lib.last_error()
