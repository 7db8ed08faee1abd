import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from oracle.oracle import OracleModel  # noqa: E402
from paper_2504_10724_b200 import eeb  # noqa: E402

TH = 0.7
desc = eeb.PRESETS["tiny"]
ref = OracleModel(desc)
ref.load(desc.num_layers)
rng = np.random.default_rng(3)
B = 8
seq = [rng.integers(0, desc.vocab, B) for _ in range(7)]
ref_kv = None
res = []
c = eeb.Context(0)
for run in range(int(os.environ.get("RUNS", "6"))):
    m = c.register(desc.replace(name=f"t{run}"))
    c.load_layers(m, desc.num_layers)
    c.retain_logits(os.environ.get("RETAIN", "1") == "1")
    for pos in range(7):
        policy = eeb.PROFILE if pos < 6 else eeb.INTROSPECTIVE
        g = c.decode_step(m, 0, policy, TH, np.arange(B), seq[pos], np.full(B, pos))
        if run == 0:
            ref.decode_step(0, policy, TH, np.arange(B), seq[pos], np.full(B, pos))
    if ref_kv is None:
        ref_kv = {(l, b): ref.read_kv(l, b, 6)[0] for l in range(1, 13) for b in range(B)}
    bad = sum(1 for l in range(1, 13) for b in range(B)
              if g["exit_layer"][b] >= l and not np.allclose(c.read_kv(m, l, b, 6)[0], ref_kv[(l, b)], atol=1e-4, rtol=1e-3))
    res.append(bad)
    c.evict(m)
print("RESULT", os.environ.get("TAG", ""), res, flush=True)
