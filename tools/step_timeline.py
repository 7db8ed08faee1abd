"""In-graph per-kernel timeline of the C2 decode step (paper_2504_10724_b200.timeline).

  python tools/step_timeline.py [--batch 64] [--steps 5] [--top 60] [--json out.json]

Sets up the bench workload (prompt prefilled with eeb_prefill, warm-up
steps), then runs stamped graph steps and prints per-category critical-path
times and the first launches.  Also times the same number of unstamped steps
with CUDA events so the stamping overhead is visible.
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="opt-1.3b-4x")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--policy", default="introspective")
    ap.add_argument("--depth", type=int, default=6)
    ap.add_argument("--top", type=int, default=0)
    ap.add_argument("--json", default="")
    ap.add_argument("--cta", default="", help="launch indices whose per-CTA stamps to summarise, e.g. 2,3,4")
    args = ap.parse_args()
    import torch

    from paper_2504_10724_b200 import eeb, timeline

    pol = {"introspective": eeb.INTROSPECTIVE, "flat": eeb.FLAT, "profile": eeb.PROFILE,
           "full_depth": eeb.FULL_DEPTH}[args.policy]
    depth = args.depth if pol == eeb.FLAT else 0
    B, P = args.batch, args.prompt
    desc = eeb.PRESETS[args.model].replace(max_slots=B, max_seq_len=P + 100)
    ctx = eeb.Context(0)
    m = ctx.register(desc)
    ctx.load_layers(m, depth or desc.num_layers)
    rng = np.random.default_rng(1)
    slots = np.arange(B, dtype=np.int32)
    ctx.prefill(m, depth or desc.num_layers, slots, list(rng.integers(0, desc.vocab, (B, P)).astype(np.int32)))
    dev = torch.device("cuda")
    n = args.steps + 8
    toks = torch.from_numpy(rng.integers(0, desc.vocab, (n, B)).astype(np.int32)).to(dev)
    pos = torch.from_numpy(np.stack([np.full(B, P + k, np.int32) for k in range(n)])).to(dev)
    sl = torch.from_numpy(slots).to(dev)

    def step(k):
        ctx.decode_step_device(m, depth, pol, 0.7, B, sl.data_ptr(), toks[k].data_ptr(), pos[k].data_ptr())

    for k in range(4):
        step(k)
    ctx.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(args.steps):
        step(k)
    e1.record(stream)
    e1.synchronize()
    plain_ms = e0.elapsed_time(e1) / args.steps
    tl = timeline.run(ctx, step, args.steps)
    if args.cta:
        # one more stamped step, then per-CTA start / wait / end of the chosen launches
        ctx.stamps(1024)
        step(0)
        ctx.synchronize()
        step(1)
        rows = ctx.stamps_read()
        prev_end = 0
        for i, l in enumerate(rows):
            if str(i) in args.cta.split(","):
                c = ctx.stamps_cta(i, min(l["ctas"], 2048)) / 1e3
                c = c[c[:, 0] >= 0]
                q = lambda v: " ".join(f"{x:7.2f}" for x in np.percentile(v, [0, 10, 50, 90, 100]))
                print(f"launch {i} {timeline.kernel_kind(l['kernel'])} ctas={len(c)} (us after previous launch's end;"
                      f" percentiles 0/10/50/90/100)")
                print(f"   start {q(c[:, 0] - prev_end / 1e3)}")
                if (c[:, 2] >= 0).any():
                    print(f"   wait  {q(c[c[:, 2] >= 0][:, 2] - prev_end / 1e3)}")
                if (c[:, 3] >= 0).any():
                    print(f"   mark  {q(c[c[:, 3] >= 0][:, 3] - prev_end / 1e3)}")
                print(f"   end   {q(c[:, 1] - prev_end / 1e3)}")
            prev_end = max(prev_end, l["end_ns"])
        ctx.stamps(0)
    print(f"unstamped graph steps: {plain_ms * 1e3:.1f} us/step (CUDA events, back to back)")
    print(timeline.table(tl, args.top))
    if args.json:
        Path(args.json).parent.mkdir(parents=True, exist_ok=True)
        Path(args.json).write_text(json.dumps({"plain_ms_per_step": plain_ms, **tl}, indent=1))
    ctx.close()


if __name__ == "__main__":
    main()
