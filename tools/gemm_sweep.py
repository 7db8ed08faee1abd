"""Steady-state GEMM timing over the step's shapes (run on the GPU box)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_10724_b200 import eeb  # noqa: E402

PEAK = 6550.1
shapes = {"qkv": (6144, 2048), "o": (2048, 2048), "up": (8192, 2048), "down": (2048, 8192), "head": (50272, 2048)}
ctx = eeb.Context(0)
B = int(os.environ.get("B", "64"))
tag = os.environ.get("TAG", "")
tot_ms = tot_b = 0.0
for name, (n, k) in shapes.items():
    ms = ctx.bench_gemm(2, n, k, B, 100)
    by = n * k * 2
    if name != "head":
        tot_ms += ms
        tot_b += by
    print(f"{tag} {name:5s} N={n:6d} K={k:5d} B={B:3d} {ms*1e3:8.2f} us  {by/ms/1e6:8.1f} GB/s  {by/ms/1e6/PEAK:6.1%}")
print(f"{tag} layer GEMMs: {tot_ms*1e3:.2f} us per layer, {tot_b/tot_ms/1e6:.1f} GB/s ({tot_b/tot_ms/1e6/PEAK:.1%})")
