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


def test_new_entry_points_validate_before_touching_the_device():
    """4-bit, expert-parallel and runtime-config entry points reject bad
    arguments with ValueError status (no CUDA device needed)."""
    nb = ctypes.c_size_t()
    assert _lib.lib.hm_q4_image_bytes(4096, 14336, ctypes.byref(nb)) == _lib.HM_OK
    assert nb.value == 3 * 4096 * 14336 // 2 + 3 * 4096 * 14336 // 64      # nibbles + bf16 scales per 128
    assert _lib.lib.hm_q4_image_bytes(100, 256, ctypes.byref(nb)) == _lib.HM_EVALUE
    assert "multiples of 128" in _lib.last_error()
    arr = (_lib.HmGroup * 1)()
    arr[0].slot, arr[0].row_begin, arr[0].row_count = 0, 0, 8
    rc = _lib.lib.hm_expert_ffn_q4(None, nb.value, 1, 256, 256, arr, 1, None, 4, None, None, None, 0, 0, None)
    assert rc == _lib.HM_EVALUE and "row range" in _lib.last_error()
    h = ctypes.c_void_p()
    _lib.lib.hm_ep_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_void_p)]
    assert _lib.lib.hm_ep_create(0, 9, 16, 256, ctypes.byref(h)) == _lib.HM_EVALUE  # world > 8
    assert _lib.lib.hm_ep_create(2, 2, 16, 256, ctypes.byref(h)) == _lib.HM_EVALUE  # rank out of range
    assert _lib.lib.hm_cpu_set_decode_grain(-1) == _lib.HM_EVALUE


def test_runtime_config_layout_matches_header():
    """The ctypes mirror of hm_runtime_config has the header's size (the
    weight_bits field was appended with explicit padding)."""
    assert ctypes.sizeof(_lib.RuntimeConfig) == 8 * 4 + 2 * 8 + 8 * 4  # 8 int32, 2 int64, 8 int32


def test_lookahead_rejects_bad_shapes_without_touching_the_device():
    """hm_lookahead (live prediction) validates its shape before any launch."""
    f = _lib.lib.hm_lookahead
    assert f(None, None, 1, 3, 1, 0, 8, 2, 256, None, None, None) == _lib.HM_EVALUE      # N = 0
    assert f(None, None, 1, 3, 1, 8, 4, 2, 256, None, None, None) == _lib.HM_EVALUE      # ld < N
    assert f(None, None, 1, 3, 1, 8, 8, 9, 256, None, None, None) == _lib.HM_EVALUE      # K > N
    assert f(None, None, 1, 3, 1, 8, 8, 2, 100, None, None, None) == _lib.HM_EVALUE      # H % 8
    assert "look-ahead shape" in _lib.last_error()
    assert f(None, None, 1, 0, 1, 8, 8, 2, 256, None, None, None) == _lib.HM_OK          # horizon 0: nothing to do
