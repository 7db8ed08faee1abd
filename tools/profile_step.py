"""Profiling harness: set up the bench workload, then run a few decode steps
between cudaProfilerStart/Stop so `ncu --profile-from-start off` sees only them.

  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
      python tools/profile_step.py --steps 2
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="opt-1.3b-4x")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--policy", default="introspective")
    ap.add_argument("--depth", type=int, default=6, help="flat policy: serving depth")
    ap.add_argument("--graphs", type=int, default=-1)  # -1: library default (stream launches under ncu)
    args = ap.parse_args()
    import torch

    from paper_2504_10724_b200 import eeb

    pol = {"introspective": eeb.INTROSPECTIVE, "flat": eeb.FLAT, "profile": eeb.PROFILE,
           "full_depth": eeb.FULL_DEPTH}[args.policy]
    desc = eeb.PRESETS[args.model].replace(max_slots=args.batch, max_seq_len=args.prompt + 100)
    ctx = eeb.Context(0)
    m = ctx.register(desc)
    ctx.load_layers(m, desc.num_layers)
    if args.graphs >= 0:
        ctx.set_graphs(bool(args.graphs))
    rng = np.random.default_rng(0)
    B = args.batch
    slots = np.arange(B)
    for p in range(args.prompt):
        ctx.decode_step(m, 0, eeb.FULL_DEPTH, 0.7, slots, rng.integers(0, desc.vocab, B), np.full(B, p))
    depth = args.depth if pol == eeb.FLAT else 0
    for k in range(3):  # warm (graph capture happens here)
        ctx.decode_step(m, depth, pol, 0.7, slots, rng.integers(0, desc.vocab, B), np.full(B, args.prompt + k))
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for k in range(args.steps):
        ctx.decode_step(m, depth, pol, 0.7, slots, rng.integers(0, desc.vocab, B),
                        np.full(B, args.prompt + 3 + k))
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    ctx.close()


if __name__ == "__main__":
    main()
