"""GPU: decode records replayed through the unmodified reference (VERDICT r1
item 8, SURVEY §4 implication 3).  tests/cpp/test_replay_gpu.cpp records every
(request, model) on the B200 with all exit heads (EEB_PROFILE) as a
reference-format trace, runs the compiled reference simulate() over it
(oracle/_ref/libeeref.so), and checks that BatchedEngine over ProfileBackend —
the same requests decoded live on the GPU — produces the same report: exit
tables, load-more / switch counts, PHT histograms, perplexity, throughput."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

BIN = Path(__file__).resolve().parent / "_bin" / "test_replay_gpu"


def test_gpu_records_replayed_by_reference_simulate():
    if not BIN.exists():
        pytest.skip("tests/_bin/test_replay_gpu not built (needs oracle/_ref: build() where /root/reference exists)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "0 failures" in r.stdout
