"""GPU: the host C++ engine (include/eeserve BatchedEngine) over CudaBackend and
the C ABI — prefill, host-tier greedy loads, batched decode, HELIOS evaluation
cycles and replanning — runs end to end on the B200 (tests/cpp/test_engine_gpu.cpp)."""
import ctypes
import json
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

BIN = Path(__file__).resolve().parent / "_bin" / "test_engine_gpu"
REF = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "libeeref.so"


def test_engine_over_cuda_backend():
    if not BIN.exists():
        pytest.fail("tests/_bin/test_engine_gpu missing: run __graft_entry__.build()")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_gpu_event_log_rebuilds_report_through_reference_aggregate(tmp_path):
    """A real GPU serving run's events.jsonl, fed to the reference's own
    aggregate() (compiled from the unmodified reference headers, oracle/_ref),
    rebuilds the engine's report: batched steps counted once, exit table,
    perplexity, TTFT/TPOT, action counts."""
    if not REF.exists():
        pytest.skip("oracle/_ref/libeeref.so (compiled reference) not built")
    log = tmp_path / "events.jsonl"
    r = subprocess.run([str(BIN), str(log)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    mine = json.loads(next(l for l in r.stdout.splitlines() if l.startswith("REPORT "))[7:])
    lib = ctypes.CDLL(str(REF))
    lib.ref_aggregate.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int]
    buf = ctypes.create_string_buffer(1 << 24)
    assert lib.ref_aggregate(str(log).encode(), buf, len(buf)) > 0
    agg = json.loads(buf.value.decode())
    a = agg["aggregates"]
    for k in ("throughput_tok_s", "perplexity", "mean_ttft_s", "mean_tpot_s"):
        assert a[k] == pytest.approx(mine[k], rel=1e-9), k
    assert a["achieved_batch_size"] == mine["achieved_batch_size"] == 16
    assert agg["action_counts"] == {"ld": mine["ld"], "sw": mine["sw"]}
    assert sum(sum(v.values()) for v in agg["exit_table"].values()) == pytest.approx(100.0)
