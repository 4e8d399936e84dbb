"""Build libhybrimoe.so in-tree: C++ decision core + runtime, CUDA kernels for sm_100a.

The library is the only native artefact of the package; it is loaded with
ctypes by ``_lib.py``.  Objects go to ``build/`` and the shared library next to
this file so that it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build"
LIB = PKG / "libhybrimoe.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

# Decision arithmetic must not be contracted into FMAs: the reference is
# CPython fp64, one rounding per operation.
CXXFLAGS = ["-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math",
            "-Wall", "-Wextra", "-Wno-unused-parameter", "-pthread"]
HOST_ISA = ["-mavx512f", "-mavx512bw", "-mavx512vl", "-mavx512bf16", "-mavx512dq", "-mavx512vnni", "-mfma", "-mamx-tile",
            "-mamx-bf16"]
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
           "--expt-relaxed-constexpr", "-Xcompiler", "-ffp-contract=off"] + GENCODE


def _sources():
    cpp = sorted(CSRC.glob("*.cpp"))
    cu = sorted(CSRC.glob("*.cu"))
    return cpp, cu


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src] + sorted(CSRC.glob("*.hpp")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "hybrimoe.h"]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps if d.exists())


def _run(cmd, log):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write(" ".join(cmd) + "\n" + r.stdout + r.stderr + "\n")
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd)}")


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    cpp, cu = _sources()
    objs = []
    with open(BUILD / "build.log", "w") as log:
        for src in cpp:
            obj = BUILD / (src.stem + ".o")
            objs.append(obj)
            if force or _stale(obj, src):
                isa = HOST_ISA if src.stem.startswith("host_") else []
                _run(["g++", *CXXFLAGS, *isa, "-I", str(ROOT / "include"), "-I", "/usr/local/cuda/include",
                      "-c", str(src), "-o", str(obj)], log)
        for src in cu:
            obj = BUILD / (src.stem + ".cu.o")
            objs.append(obj)
            if force or _stale(obj, src):
                _run([NVCC, *NVFLAGS, "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)], log)
        newest = max(o.stat().st_mtime for o in objs)
        if force or not LIB.exists() or LIB.stat().st_mtime < newest:
            tmp = LIB.with_suffix(".so.tmp")
            _run([NVCC, "-shared", *GENCODE, "-cudart", "static", "-o", str(tmp), *map(str, objs),
                  "-Xcompiler", "-pthread", "-ldl", "-lrt"], log)
            os.replace(tmp, LIB)
    if verbose:
        print((BUILD / "build.log").read_text())
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
