"""Host worker (AVX-512 BF16) numerics against the fp32 oracle, CPU only."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from oracle import moe_ref as ref

from paper_2504_05897_b200 import _lib
from paper_2504_05897_b200.weights import pack_expert, unpack_expert

lib = _lib.lib
pytestmark = pytest.mark.skipif(not lib.hm_cpu_has_avx512bf16(), reason="host lacks AVX-512 BF16")


@pytest.fixture(scope="module")
def pool():
    p = C.c_void_p()
    _lib.check(lib.hm_cpu_pool_create(4, C.byref(p)))
    yield p
    lib.hm_cpu_pool_destroy(p)


def _expert(rng, H, I):
    g, u, d = (ref.f32_to_bf16(rng.standard_normal(s).astype(np.float32) * 0.02) for s in ((I, H), (I, H), (H, I)))
    return pack_expert(g, u, d), tuple(ref.bf16_to_f32(a) for a in (g, u, d))


def test_pack_unpack_roundtrip():
    rng = np.random.default_rng(0)
    img, _ = _expert(rng, 64, 256)
    g, u, d = unpack_expert(img, 64, 256)
    assert np.array_equal(pack_expert(g, u, d), img)


@pytest.mark.parametrize("H,I,M", [(256, 256, 1), (512, 384, 3), (512, 384, 17), (1024, 1408, 1), (1024, 1408, 40),
                                   (512, 256, 8), (512, 256, 33), (2048, 1408, 96), (256, 384, 300)])
def test_cpu_expert_matches_oracle(pool, H, I, M):
    rng = np.random.default_rng(H + M)
    img, ex = _expert(rng, H, I)
    x = ref.f32_to_bf16(rng.standard_normal((M, H)).astype(np.float32))
    out = np.empty((M, H), np.float32)
    _lib.check(lib.hm_cpu_expert(pool, img.ctypes.data, H, I, x.ctypes.data, M, out.ctypes.data))
    want = ref.expert(ref.bf16_to_f32(x), *ex)
    assert np.abs(out - want).max() / np.abs(want).max() <= 1e-2


@pytest.mark.parametrize("grain", [0, 5, 16, 64])
@pytest.mark.parametrize("H,I,n", [(512, 384, 3), (256, 1408, 4), (2048, 1408, 3)])
def test_cpu_experts_decode_batch(pool, grain, H, I, n):
    rng = np.random.default_rng(9 + grain)
    lib.hm_cpu_set_decode_grain.argtypes = [C.c_int]
    _lib.check(lib.hm_cpu_set_decode_grain(grain))
    exps = [_expert(rng, H, I) for _ in range(n)]
    xs = [ref.f32_to_bf16(rng.standard_normal((1, H)).astype(np.float32)) for _ in range(n)]
    outs = [np.empty((1, H), np.float32) for _ in range(n)]
    P = C.c_void_p * n
    _lib.check(lib.hm_cpu_experts_decode(pool, P(*[e[0].ctypes.data for e in exps]), P(*[x.ctypes.data for x in xs]),
                                         n, H, I, P(*[o.ctypes.data for o in outs])))
    for (img, ex), x, o in zip(exps, xs, outs):
        want = ref.expert(ref.bf16_to_f32(x), *ex)
        assert np.abs(o - want).max() / np.abs(want).max() <= 1e-2
    _lib.check(lib.hm_cpu_set_decode_grain(16))


def test_host_read_bandwidth_probe(pool):
    buf = np.zeros(1 << 24, dtype=np.uint8)
    gbs = C.c_double()
    _lib.check(lib.hm_host_read_bw(pool, buf.ctypes.data, buf.nbytes, 2, C.byref(gbs)))
    assert gbs.value > 0


def test_oracle_q4_roundtrip():
    """The 4-bit restatement: dequantize(quantize(w)) within half a scale step of w."""
    rng = np.random.default_rng(3)
    w = ref.f32_to_bf16(rng.standard_normal((6, 256)).astype(np.float32) * 0.02)
    nib, s = ref.q4_quantize_rows(w)
    back = ref.q4_dequantize_rows(nib, s)
    step = np.repeat(ref.bf16_to_f32(s), 128, axis=1)
    assert np.all(np.abs(back - ref.bf16_to_f32(w)) <= 0.5 * step * (1 + 1e-6) + 1e-12)


def _q4_expert(rng, H, I):
    img, _ = _expert(rng, H, I)
    q = ref.q4_image(img[: 2 * I * H].reshape(2 * I, H), img[2 * I * H:].reshape(H, I))
    return q, ref.q4_expert(q, H, I)


@pytest.mark.parametrize("H,I,M", [(256, 256, 1), (512, 384, 1), (256, 384, 3), (512, 256, 17), (256, 256, 40)])
def test_cpu_expert_q4_matches_oracle(pool, H, I, M):
    if M > 1 and not lib.hm_cpu_has_amx_bf16():
        pytest.skip("4-bit prefill on the host needs AMX")
    rng = np.random.default_rng(H * 7 + M)
    q, ex = _q4_expert(rng, H, I)
    x = ref.f32_to_bf16(rng.standard_normal((M, H)).astype(np.float32))
    out = np.empty((M, H), np.float32)
    _lib.check(lib.hm_cpu_expert_q4(pool, q.ctypes.data, H, I, x.ctypes.data, M, out.ctypes.data))
    want = ref.expert(ref.bf16_to_f32(x), *ex)
    assert np.abs(out - want).max() / np.abs(want).max() <= 1e-2


def test_cpu_experts_decode_q4_batch(pool):
    rng = np.random.default_rng(11)
    H, I, n = 256, 384, 3
    exps = [_q4_expert(rng, H, I) for _ in range(n)]
    xs = [ref.f32_to_bf16(rng.standard_normal((1, H)).astype(np.float32)) for _ in range(n)]
    outs = [np.empty((1, H), np.float32) for _ in range(n)]
    P = C.c_void_p * n
    _lib.check(lib.hm_cpu_experts_decode_q4(pool, P(*[e[0].ctypes.data for e in exps]),
                                            P(*[x.ctypes.data for x in xs]), n, H, I,
                                            P(*[o.ctypes.data for o in outs])))
    for (q, ex), x, o in zip(exps, xs, outs):
        want = ref.expert(ref.bf16_to_f32(x), *ex)
        assert np.abs(o - want).max() / np.abs(want).max() <= 1e-2


@pytest.mark.skipif(not lib.hm_cpu_has_amx_bf16(), reason="host lacks AMX-BF16")
@pytest.mark.parametrize("H,I,Ms", [(512, 384, [8, 33, 17]), (1024, 1408, [96, 9, 40, 128]), (256, 256, [300]),
                                    (2048, 1408, [8, 96, 200])])   # the DeepSeek-V2-Lite expert shape
def test_batched_amx_experts_equal_one_by_one(pool, H, I, Ms):
    """hm_cpu_experts_amx (a layer's prefill experts in one pass, units claimed
    across experts) gives hm_cpu_expert's bits per expert, and the oracle's
    values within 1e-2."""
    rng = np.random.default_rng(H + len(Ms))
    exps = [_expert(rng, H, I) for _ in Ms]
    xs = [ref.f32_to_bf16(rng.standard_normal((m, H)).astype(np.float32)) for m in Ms]
    one = []
    for (img, _), x, m in zip(exps, xs, Ms):
        o = np.empty((m, H), np.float32)
        _lib.check(lib.hm_cpu_expert(pool, img.ctypes.data, H, I, x.ctypes.data, m, o.ctypes.data))
        one.append(o)
    outs = [np.full((m, H), np.nan, np.float32) for m in Ms]
    P = C.c_void_p * len(Ms)
    _lib.check(lib.hm_cpu_experts_amx(pool, P(*[e[0].ctypes.data for e in exps]), P(*[x.ctypes.data for x in xs]),
                                      (C.c_int * len(Ms))(*Ms), len(Ms), H, I, P(*[o.ctypes.data for o in outs])))
    for o, o1, (_, ex), x in zip(outs, one, exps, xs):
        assert np.array_equal(o, o1)
        want = ref.expert(ref.bf16_to_f32(x), *ex)
        assert np.abs(o - want).max() / np.abs(want).max() <= 1e-2
