"""Build the host C++ tests of include/eeserve (the drop-in API over the C ABI).

tests/_bin/test_host links the header-only eeserve API, libeeb.so (the C ABI,
needed for CudaBackend's symbols) and — only where it exists — the compiled
reference driver oracle/_ref/libeeref.so used as the differential checker.
"""
from __future__ import annotations

import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
JSON_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"


def build_engine_gpu(verbose: bool = False) -> Path:
    """tests/_bin/test_engine_gpu: BatchedEngine + CudaBackend end to end (needs a GPU to run)."""
    src = ROOT / "tests" / "cpp" / "test_engine_gpu.cpp"
    out = ROOT / "tests" / "_bin" / "test_engine_gpu"
    lib = ROOT / "paper_2504_10724_b200"
    deps = [src, lib / "libeeb.so", ROOT / "include" / "eeb" / "eeb.h", *(ROOT / "include" / "eeserve").glob("*.hpp")]
    if out.exists() and all(d.stat().st_mtime <= out.stat().st_mtime for d in deps):
        return out
    out.parent.mkdir(exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", "-I/usr/local/cuda/include", str(src), "-o", str(out),
           f"-L{lib}", "-leeb", f"-Wl,-rpath,{lib}", "-L/usr/local/cuda/lib64", "-lcudart"]
    if verbose:
        print(" ".join(cmd))
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"engine GPU test build failed:\n{r.stderr}")
    return out


def build_serve_c3(verbose: bool = False) -> Path:
    """paper_2504_10724_b200/_build/serve_c3: the C3 serving run (engine + CudaBackend), used by bench.py."""
    src = ROOT / "tools" / "serve_c3.cpp"
    lib = ROOT / "paper_2504_10724_b200"
    out = lib / "_build" / "serve_c3"
    deps = [src, lib / "libeeb.so", ROOT / "include" / "eeb" / "eeb.h", *(ROOT / "include" / "eeserve").glob("*.hpp")]
    if out.exists() and all(d.stat().st_mtime <= out.stat().st_mtime for d in deps):
        return out
    out.parent.mkdir(exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", "-I/usr/local/cuda/include", str(src), "-o", str(out),
           f"-L{lib}", "-leeb", f"-Wl,-rpath,{lib}", "-L/usr/local/cuda/lib64", "-lcudart"]
    if verbose:
        print(" ".join(cmd))
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"serve_c3 build failed:\n{r.stderr}")
    return out


def build_replay_gpu(verbose: bool = False) -> Path | None:
    """tests/_bin/test_replay_gpu: GPU-recorded traces replayed by the compiled reference (needs a GPU to run)."""
    ref = ROOT / "oracle" / "_ref" / "libeeref.so"
    src = ROOT / "tests" / "cpp" / "test_replay_gpu.cpp"
    out = ROOT / "tests" / "_bin" / "test_replay_gpu"
    lib = ROOT / "paper_2504_10724_b200"
    if not ref.exists() or not Path(JSON_INC).is_dir():
        return None
    deps = [src, ref, lib / "libeeb.so", ROOT / "include" / "eeb" / "eeb.h", *(ROOT / "include" / "eeserve").glob("*.hpp")]
    if out.exists() and all(d.stat().st_mtime <= out.stat().st_mtime for d in deps):
        return out
    out.parent.mkdir(exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", f"-I{JSON_INC}", "-I/usr/local/cuda/include",
           str(src), "-o", str(out), f"-L{ref.parent}", "-leeref", f"-Wl,-rpath,{ref.parent}",
           f"-L{lib}", "-leeb", f"-Wl,-rpath,{lib}", "-L/usr/local/cuda/lib64", "-lcudart"]
    if verbose:
        print(" ".join(cmd))
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"replay GPU test build failed:\n{r.stderr}")
    return out


def build_host(verbose: bool = False) -> Path | None:
    ref = ROOT / "oracle" / "_ref" / "libeeref.so"
    src = ROOT / "tests" / "cpp" / "test_host.cpp"
    out = ROOT / "tests" / "_bin" / "test_host"
    lib = ROOT / "paper_2504_10724_b200"
    if not ref.exists() or not Path(JSON_INC).is_dir():
        return None
    deps = [src, ref, lib / "libeeb.so", *(ROOT / "include" / "eeserve").glob("*.hpp")]
    if out.exists() and all(d.stat().st_mtime <= out.stat().st_mtime for d in deps):
        return out
    out.parent.mkdir(exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", f"-I{JSON_INC}", "-I/usr/local/cuda/include",
           str(src), "-o", str(out), f"-L{ref.parent}", "-leeref", f"-Wl,-rpath,{ref.parent}",
           f"-L{lib}", "-leeb", f"-Wl,-rpath,{lib}", "-L/usr/local/cuda/lib64", "-lcudart"]
    if verbose:
        print(" ".join(cmd))
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"host test build failed:\n{r.stderr}")
    return out
