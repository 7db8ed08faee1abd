"""Large-batch decode GEMM timing (34B and C2 layer shapes): us, GB/s of
weights, TFLOP/s per launch (run on the GPU box).
  B=64,128,256 MODEL=34b|c2 ITERS=50 python tools/gemm_big.py"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_10724_b200 import eeb  # noqa: E402

SHAPES = {
    "34b": {"qkv": (10240, 8192), "o": (8192, 8192), "up": (44032, 8192), "down": (8192, 22016)},
    "c2": {"qkv": (6144, 2048), "o": (2048, 2048), "up": (8192, 2048), "down": (2048, 8192)},
}
ctx = eeb.Context(0)
iters = int(os.environ.get("ITERS", "50"))
only = os.environ.get("ONLY", "")
for model in os.environ.get("MODEL", "34b,c2").split(","):
    for B in [int(b) for b in os.environ.get("B", "64,128,256").split(",")]:
        tot_ms = tot_b = tot_f = 0.0
        for name, (n, k) in SHAPES[model].items():
            if only and name not in only.split(","):
                continue
            ms = ctx.bench_gemm(2, n, k, B, iters)
            by, fl = n * k * 2, 2.0 * n * k * B
            tot_ms += ms; tot_b += by; tot_f += fl
            print(f"{model} B={B:3d} {name:5s} N={n:6d} K={k:5d} {ms*1e3:8.2f} us {by/ms/1e6:7.0f} GB/s {fl/ms/1e9:7.0f} TF/s")
        print(f"{model} B={B:3d} layer: {tot_ms*1e3:.1f} us {tot_b/tot_ms/1e6:.0f} GB/s {tot_f/tot_ms/1e9:.0f} TF/s", flush=True)
