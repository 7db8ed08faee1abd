"""C5 shape on one B200: Llama2-70B (80 layers, d 8192, 64/8 heads, SwiGLU 28672,
exits 8/10/20/40/80) with all 8 tensor-parallel shards in one context
(tp_size 8, tp_rank -1: the same column/row/vocab-parallel shard kernels an
8-GPU rank runs, summed locally instead of over NCCL).  Prints one JSON line:
step time at batch 64 (introspective and flat at the greedy depth 10).  A TP=8
rank streams 1/8 of these weights per step plus the all-reduces."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_10724_b200 import eeb  # noqa: E402


def main():
    B, P = 64, 128
    desc = eeb.PRESETS["llama2-70b"].replace(tp_size=8, tp_rank=-1, max_slots=B, max_seq_len=P + 64,
                                            name="llama2-70b-tp8x1")
    ctx = eeb.Context(0)
    m = ctx.register(desc)
    t0 = time.perf_counter()
    ctx.load_layers(m, desc.num_layers)
    load_s = time.perf_counter() - t0
    rng = np.random.default_rng(0)
    slots = np.arange(B)
    ctx.prefill(m, desc.num_layers, slots, list(rng.integers(0, desc.vocab, (B, P))))
    out = {"workload": "C5 shape (Llama2-70B bf16, 8 TP shards in one context on one B200)", "batch": B,
           "weights_gb": None, "synth_load_s": load_s}
    stream = torch.cuda.ExternalStream(ctx.stream())
    for name, pol, depth in (("introspective", eeb.INTROSPECTIVE, 0), ("flat_depth10", eeb.FLAT, 10)):
        times = []
        for k in range(8):
            toks = rng.integers(0, desc.vocab, B)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.decode_step(m, depth, pol, 0.7, slots, toks, np.full(B, P + k))
            e1.record(stream)
            e1.synchronize()
            if k >= 3:
                times.append(e0.elapsed_time(e1))
        out[name + "_ms_per_step"] = float(np.median(times))
        out[name + "_tokens_per_s"] = B / (np.median(times) / 1000.0)
    wb = ctx.weight_bytes(m, desc.num_layers) if hasattr(ctx, "weight_bytes") else None
    out["weights_gb"] = wb / 1e9 if wb else None
    print(json.dumps(out))
    ctx.close()


if __name__ == "__main__":
    main()
