"""CPU-side checks of the C ABI library: it loads, exports exactly what
include/eeb/eeb.h declares, and refuses to run without a B200 (no CPU fallback)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2504_10724_b200 import eeb

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "eeb" / "eeb.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(eeb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = eeb.load_library()
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(eeb.EXPORTED) == names


def test_exports_are_c_abi_not_mangled():
    out = subprocess.run(["nm", "-D", "--defined-only", str(eeb.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (eeb_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_abi_version():
    assert eeb.load_library().eeb_abi_version() == 1


def test_built_for_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(eeb.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu suite")
    with pytest.raises(eeb.EebError) as e:
        eeb.Context(0)
    assert e.value.kind in ("CudaError", "DomainError")
