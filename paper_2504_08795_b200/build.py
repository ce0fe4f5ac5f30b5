"""In-tree build of the native libraries (no torch JIT cache, so the .so files
travel to the GPU box with the repo snapshot).

* ``lib/libdaris_core.so``   — C++ dispatcher + sim/trace engines (no CUDA).
* ``lib/libdaris_gpu.so``    — sm_100a stage kernels + GPU executor.

Usage: ``python -m paper_2504_08795_b200.build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"
INCLUDE = ROOT / "include"

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CORE_SOURCES = ["core/dispatcher.cpp", "core/decide.cpp", "core/sim.cpp", "core/capi.cpp"]
GPU_SOURCES = ["kernels/conv_tc.cu", "kernels/linear_tc.cu", "kernels/aux.cu", "exec/executor.cu"]


def _run(cmd: list[str]) -> None:
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} (exit {proc.returncode})")


def _stale(target: Path, sources: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    deps = list(sources) + list(CSRC.rglob("*.h")) + list(CSRC.rglob("*.hpp")) + \
        list(CSRC.rglob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def build_core(force: bool = False) -> Path:
    """g++ build of the dispatcher; -ffp-contract=off keeps IEEE results identical
    to CPython float arithmetic (no FMA contraction, no fast-math)."""
    LIB.mkdir(exist_ok=True)
    out = LIB / "libdaris_core.so"
    srcs = [CSRC / s for s in CORE_SOURCES]
    if force or _stale(out, srcs):
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off",
               "-fno-fast-math", "-Wall", "-Wno-unused-function", f"-I{INCLUDE}", f"-I{CSRC}",
               *map(str, srcs), "-o", str(out)]
        _run(cmd)
    return out


def build_gpu(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libdaris_gpu.so"
    srcs = [CSRC / s for s in GPU_SOURCES]
    if force or _stale(out, srcs):
        objs = []
        for src in srcs:
            obj = LIB / (src.stem + ".o")
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr",
                   f"-I{INCLUDE}", f"-I{CSRC}", *os.environ.get("DARIS_NVCC_EXTRA", "").split(),
                   "-c", str(src), "-o", str(obj)]
            _run(cmd)
            objs.append(str(obj))
        cmd = [NVCC, *ARCH, "-shared", "--cudart", "shared", "-o", str(out), *objs, f"-L{LIB}", "-ldaris_core",
               "-Xlinker", "-rpath,$ORIGIN"]
        _run(cmd)
        for o in objs:
            os.remove(o)
    return out


def build_all(force: bool = False) -> None:
    build_core(force)
    build_gpu(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built", *(p.name for p in sorted(LIB.glob("*.so"))))
