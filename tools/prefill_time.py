"""Wall time of one C2 batch prefill (64 prompts x 128 tokens through 24
layers, host tokens in): best of 5 after a warm-up.  Env knobs (EEB_SKIP=...)
give the A/B splits.  Run on the GPU box."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_10724_b200 import eeb  # noqa: E402

B, P = int(sys.argv[1]) if len(sys.argv) > 1 else 64, int(sys.argv[2]) if len(sys.argv) > 2 else 128
desc = eeb.PRESETS[sys.argv[3] if len(sys.argv) > 3 else "opt-1.3b-4x"].replace(max_slots=B, max_seq_len=P + 16)
ctx = eeb.Context(0)
m = ctx.register(desc)
ctx.load_layers(m, desc.num_layers)
rng = np.random.default_rng(0)
prompts = list(rng.integers(0, desc.vocab, (B, P)).astype(np.int32))
best = 1e9
for k in range(6):
    ctx.synchronize()
    t0 = time.perf_counter()
    ctx.prefill(m, desc.num_layers, np.arange(B), prompts)
    ctx.synchronize()
    if k:
        best = min(best, time.perf_counter() - t0)
print(f"prefill {B}x{P} {desc.name}: {best * 1e3:.2f} ms  ({B * P / best / 1e3:.1f}k tok/s)")
ctx.close()
