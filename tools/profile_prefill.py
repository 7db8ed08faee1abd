"""Profiling harness for the prefill path: one eeb_prefill of B prompts between
cudaProfilerStart/Stop (ncu --profile-from-start off)."""
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
    ap.add_argument("--graphs", type=int, default=0)
    args = ap.parse_args()
    import torch

    from paper_2504_10724_b200 import eeb

    desc = eeb.PRESETS[args.model].replace(max_slots=args.batch, max_seq_len=args.prompt + 100)
    ctx = eeb.Context(0)
    m = ctx.register(desc)
    ctx.load_layers(m, desc.num_layers)
    ctx.set_graphs(bool(args.graphs))
    rng = np.random.default_rng(0)
    slots = np.arange(args.batch)
    prompts = list(rng.integers(0, desc.vocab, (args.batch, args.prompt)))
    ctx.prefill(m, desc.num_layers, slots, prompts)  # warm
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    ctx.prefill(m, desc.num_layers, slots, prompts)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    ctx.close()


if __name__ == "__main__":
    main()
