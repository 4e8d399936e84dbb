"""ORACLE -- test infrastructure only (tests/, bench.py's reference arm / cpu_baseline).

ctypes front end of oracle/cpu_moe.c (built by `make -C oracle`, which
__graft_entry__.build() runs): the reference's CPU expert evaluation in plain
C on all host threads.  See the C file for the arithmetic contract.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

_LIB = Path(__file__).resolve().parent / "liboracle_cpu.so"
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _LIB.exists():
            raise RuntimeError(f"{_LIB} is missing: run `make -C oracle`")
        _lib = C.CDLL(str(_LIB))
        _lib.oc_expert.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                                   C.c_void_p]
        _lib.oc_expert.restype = C.c_int
        _lib.oc_threads.restype = C.c_int
    return _lib


def threads() -> int:
    return int(lib().oc_threads())


class Scratch:
    def __init__(self) -> None:
        self.buf = np.empty(0, np.float32)

    def get(self, n: int) -> np.ndarray:
        if self.buf.size < n:
            self.buf = np.empty(n, np.float32)
        return self.buf


def expert(w13_ptr: int, w2_ptr: int, H: int, I: int, x_ptr: int, M: int, out_ptr: int, scratch: Scratch) -> None:
    """out[M][H] fp32 = SwiGLU of bf16 rows x[M][H]; weights as raw bf16 pointers."""
    s = scratch.get((H + I) * max(M, 1))
    if lib().oc_expert(w13_ptr, w2_ptr, H, I, x_ptr, M, out_ptr, s.ctypes.data) != 0:
        raise ValueError("oc_expert: bad arguments")
