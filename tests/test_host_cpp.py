"""The host C++ drop-in API (include/eeserve) against the reference: re-hosted
reference KATs, randomized differential tests against the compiled reference
(oracle/_ref), and the batched engine replaying reference traces at batch 1
against the reference simulate().  Built by __graft_entry__.build()."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BIN = ROOT / "tests" / "_bin" / "test_host"


def test_host_api_against_reference():
    if not BIN.exists():
        pytest.skip("compiled reference (oracle/_ref) unavailable: it is only built where /root/reference exists")
    r = subprocess.run([str(BIN), str(ROOT / "tests" / "golden")], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
