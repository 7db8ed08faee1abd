"""Batch-1 C2 decode: step time by exit layer (is the early-exit saving real?)."""
import collections
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2504_10724_b200 import eeb  # noqa: E402

desc = eeb.PRESETS["opt-1.3b-4x"].replace(max_slots=4, max_seq_len=228)
ctx = eeb.Context(0)
m = ctx.register(desc)
ctx.load_layers(m, desc.num_layers)
rng = np.random.default_rng(77)
ctx.prefill(m, desc.num_layers, [0], [rng.integers(0, desc.vocab, 128)])
stream = torch.cuda.ExternalStream(ctx.stream())
dev = torch.device("cuda")
sl = torch.zeros(1, dtype=torch.int32, device=dev)
outs = {"exit_layer": torch.zeros(1, dtype=torch.int32, device=dev)}
ptrs = {k: v.data_ptr() for k, v in outs.items()}
by = collections.defaultdict(list)
for k in range(60):
    tok = torch.tensor([int(rng.integers(0, desc.vocab))], dtype=torch.int32, device=dev)
    pos = torch.tensor([128 + k], dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.decode_step_device(m, 0, eeb.INTROSPECTIVE, 0.7, 1, sl.data_ptr(), tok.data_ptr(), pos.data_ptr(), ptrs)
    e1.record(stream)
    e1.synchronize()
    if k >= 3:
        by[int(outs["exit_layer"][0])].append(e0.elapsed_time(e1))
for l in sorted(by):
    print(f"exit {l:2d}: n={len(by[l]):2d} mean {np.mean(by[l]):.3f} ms  min {np.min(by[l]):.3f}")
