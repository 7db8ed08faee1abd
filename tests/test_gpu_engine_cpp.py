"""GPU: the host C++ engine (include/eeserve BatchedEngine) over CudaBackend and
the C ABI — prefill, host-tier greedy loads, batched decode, HELIOS evaluation
cycles and replanning — runs end to end on the B200 (tests/cpp/test_engine_gpu.cpp)."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

BIN = Path(__file__).resolve().parent / "_bin" / "test_engine_gpu"


def test_engine_over_cuda_backend():
    if not BIN.exists():
        pytest.fail("tests/_bin/test_engine_gpu missing: run __graft_entry__.build()")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
