"""Persistent-kernel GEMM stream over every layer of a model preset (GPU box)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_10724_b200 import eeb  # noqa: E402

PEAK = 6650.0
name = os.environ.get("MODEL", "opt-1.3b-4x")
desc = eeb.PRESETS[name]
ctx = eeb.Context(0)
m = ctx.register(desc.replace(max_slots=128, max_seq_len=256))
ctx.load_layers(m, desc.num_layers)
by = desc.layer_weight_elems() * 2 * desc.num_layers
for B in [int(b) for b in os.environ.get("BS", "64").split(",")]:
    ms = ctx.bench_layers(m, B, 20)
    print(f"{os.environ.get('TAG','')} {name} B={B}: {ms*1e3:.1f} us/launch for {by/1e9:.3f} GB -> {by/ms/1e6:.0f} GB/s ({by/ms/1e6/PEAK:.1%} of 6650)")
