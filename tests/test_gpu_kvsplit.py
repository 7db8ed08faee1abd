"""Decode attention with the KV split (flash-decoding partials, EEB_ATTN_KVSPLIT)
against the oracle.  kv_splits() caches the environment variable, so each
setting runs in its own process.  Covers a short context where some splits
own no chunk, several kv heads (GQA) and the per-(row, kv head) ticket reset
across consecutive launches (several steps)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r"""
import numpy as np
from oracle.oracle import OracleModel
from paper_2504_10724_b200 import eeb
desc = eeb.ModelDesc("kvsplit-gqa", 4, 512, 8, 2, 1024, 1000, (2, 4), mlp_kind=eeb.MLP_SWIGLU,
                     max_slots=16, max_seq_len=160, seed=41)
ctx = eeb.Context(0)
m = ctx.register(desc)
ctx.load_layers(m, desc.num_layers)
ref = OracleModel(desc)
ref.load(desc.num_layers)
rng = np.random.default_rng(9)
B = 16
slots = np.arange(B)
agree = n = 0
for p in range(70):   # contexts 1..70: 1 chunk (other splits idle) up to 3 chunks
    toks = rng.integers(0, desc.vocab, B)
    policy = eeb.PROFILE if p % 3 == 0 else eeb.INTROSPECTIVE
    g = ctx.decode_step(m, 0, policy, 0.7, slots, toks, np.full(B, p))
    r = ref.decode_step(0, policy, 0.7, slots, toks, np.full(B, p))
    agree += int((g["token_id"] == r["token_id"]).sum())
    n += B
    same = g["exit_layer"] == r["exit_layer"]
    near = np.abs(r["confidence"] - 0.7) <= 2e-2
    assert (same | near).all(), (p, g["exit_layer"], r["exit_layer"])
assert agree / n >= 0.99, agree / n
print("KVSPLIT_OK", agree / n)
"""


@pytest.mark.parametrize("splits", [2, 4])
def test_kv_split_matches_oracle(splits):
    env = dict(os.environ, EEB_ATTN_KVSPLIT=str(splits), PYTHONPATH=str(ROOT))
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600,
                       cwd=str(ROOT))
    assert r.returncode == 0 and "KVSPLIT_OK" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])
