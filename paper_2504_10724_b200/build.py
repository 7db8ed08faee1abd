"""In-tree build of the native libraries.

* ``paper_2504_10724_b200/libeeb.so`` — the CUDA kernels and the C ABI
  (include/eeb/eeb.h), compiled for sm_100a only.
The host C++ engine (include/eeserve/*.hpp) is header-only; its test and tool
binaries are built by host_build.py.

The build uses nvcc directly (no torch JIT cache) so the .so files live in the
repo and travel to the GPU box with the snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_build"
LIB = PKG / "libeeb.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O3,-ffp-contract=off",
    f"-I{ROOT / 'include'}",
]
SOURCES = ["synth_kernels.cu", "rows.cu", "gemm_cc.cu", "gemm_tc.cu", "attention.cu", "attention_dec.cu",
           "exit_head.cu", "eeb_api.cu"]


def _deps(src: Path) -> list[Path]:
    hdrs = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "eeb" / "eeb.h"]
    return [src] + hdrs


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.exists() and d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def build_eeb(verbose: bool = False, extra_flags: list[str] | None = None) -> Path:
    OBJ.mkdir(exist_ok=True)
    flags = NVCC_FLAGS + (extra_flags or []) + os.environ.get("EEB_NVCC_EXTRA", "").split()
    jobs = []
    objs = []
    for name in SOURCES:
        src = CSRC / name
        obj = OBJ / (name + ".o")
        objs.append(obj)
        if _stale(obj, _deps(src)):
            jobs.append([NVCC, *flags, "-c", str(src), "-o", str(obj)])
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for f in [ex.submit(_run, j) for j in jobs]:
                f.result()
    if jobs or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart", "-ldl", "-lcublasLt",
               "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
        if verbose:
            print(" ".join(cmd))
        _run(cmd)
    return LIB


def build_all(verbose: bool = False) -> None:
    build_eeb(verbose)
    from . import host_build

    host_build.build_host(verbose)


if __name__ == "__main__":
    build_all(verbose="-v" in sys.argv)
