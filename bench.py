#!/usr/bin/env python3
"""Benchmark of the batched early-exit (EE) decode step on B200.

Metric (BASELINE.json): EE decode tokens/s (whole job, all GPUs) with the
exit-head / decode-GEMM fraction of HBM roofline.  One "step" = one batched
decode step: every one of the B rows advances one token through the
introspective early-exit path (exits 6/12/18/24, compaction of survivors).

Workload (BASELINE configs[1], C2): OPT-1.3B shape (24 layers, d 2048, 32
heads, ffn 8192, V 50272), exits at 6/12/18/24, random-init weights with
biased exit heads, batch 64 per GPU, bf16, prompt 128 + up to 100 decode
positions (KV context 128..227), teacher-forced synthetic tokens.  N GPUs run
N independent replicas over disjoint request shards (weak scaling); the only
collective is the profiler-histogram all-reduce after the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl eeb|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


# ----------------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.f.flush()
        rows = []
        for line in Path(self.f.name).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:7]))
            except ValueError:
                continue
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, flags in rows for i, f in enumerate(flags) if f == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------
# algorithmic bytes
# ----------------------------------------------------------------------------
def gemm_bytes_per_step(desc, batch: int, layers: int) -> int:
    """Weights of every layer GEMM read once + activations in/out."""
    bw = desc.bytes_per_el
    hd = desc.head_dim
    dq, dkv = desc.n_heads * hd, desc.n_kv_heads * hd
    up = 2 * desc.d_ffn if desc.mlp_kind == 1 else desc.d_ffn
    D, F = desc.d_model, desc.d_ffn
    shapes = [(dq + 2 * dkv, D), (D, dq), (up, D), (D, F)]
    per_layer = sum(n * k * bw + batch * k * bw + batch * n * 4 for n, k in shapes)
    return per_layer * layers


def gemm_flops_per_step(desc, batch: int, layers: int) -> float:
    """2 flop per weight per row of every layer GEMM (every row runs every layer: flat steps)."""
    hd = desc.head_dim
    dq, dkv = desc.n_heads * hd, desc.n_kv_heads * hd
    up = 2 * desc.d_ffn if desc.mlp_kind == 1 else desc.d_ffn
    D, F = desc.d_model, desc.d_ffn
    return 2.0 * batch * layers * sum(n * k for n, k in [(dq + 2 * dkv, D), (D, dq), (up, D), (D, F)])


def head_bytes(desc, batch: int) -> int:
    """K2: V x d head weights + normed activations + 17 B per row."""
    return desc.vocab * desc.d_model * desc.bytes_per_el + batch * desc.d_model * desc.bytes_per_el + 17 * batch


# ----------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle port on host cores
# ----------------------------------------------------------------------------
def cpu_port_run(desc, steps: int, warmup: int, rows: int = 64, prompt: int = 128, seed: int = 1):
    """The reference path timed on the host cores: the CPU oracle port (the
    reference itself only looks verdicts up in a trace) running the
    same workload as the GPU arm — `rows` rows of the same model, KV context
    `prompt` (the prompt's KV filled synthetically to full depth: running the
    prompt through the CPU model would dominate the sample), introspective
    steps at positions prompt, prompt+1, ..."""
    from oracle.oracle import OracleModel
    from paper_2504_10724_b200 import eeb

    cores = os.cpu_count() or 1
    d = desc.replace(max_slots=rows, max_seq_len=prompt + steps + warmup + 1)
    ref = OracleModel(d, threads=cores)
    ref.load(d.num_layers)
    for r in range(rows):
        ref.fill_kv_synthetic(r, prompt, seed + r)
    rng = np.random.default_rng(seed)
    slots = np.arange(rows)
    times = []
    for k in range(warmup + steps):
        toks = rng.integers(0, d.vocab, rows)
        t0 = time.perf_counter()
        ref.decode_step(0, eeb.INTROSPECTIVE, 0.7, slots, toks, np.full(rows, prompt + k))
        if k >= warmup:
            times.append(time.perf_counter() - t0)
    ref.close()
    total = sum(times)
    return {"value": rows * len(times) / total, "unit": "tokens/s", "cores": cores, "kind": "port",
            "sample": f"{len(times)} introspective steps x {rows} rows (the GPU arm's batch) of the same model, "
                      f"context {prompt}..{prompt + warmup + steps - 1} (prompt KV synthetic, full depth), on the "
                      f"CPU oracle (f64-accumulating restatement with the device's rounding points, {cores} threads)",
            "seconds": total}


def run_reference(args, desc):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # one warm-up step (first touch of the KV pool); every timed step is the
    # whole 64-row batch
    r = cpu_port_run(desc, args.steps, min(args.warmup, 1), rows=args.batch, prompt=args.prompt)
    line = {"metric": METRIC, "value": r["value"], "unit": "tokens/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * r["seconds"] / max(1, args.steps), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, desc),
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": r["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


METRIC = "EE decode tokens/s vs batch at 1/2/4/8 B200; exit-head/GEMM % HBM roofline"


def workload_name(args, desc):
    if desc.name.startswith("opt-1.3b") and args.policy == "introspective":
        return ("C2: OPT-1.3B-shape early-exit decode step, exits " + "/".join(map(str, desc.exit_layers)) +
                ", introspective (earliest confident head, survivors compacted), teacher-forced synthetic tokens")
    if desc.name.startswith("llama2-70b") and args.tp > 1:
        return (f"C5: Llama2-70B-shape tensor-parallel over {args.tp} GPUs, greedy first-{args.depth}-layer "
                f"loading, flat decode at depth {args.depth}, teacher-forced synthetic tokens")
    if desc.name.startswith("codellama-34b") and args.policy == "flat":
        return (f"C4: CodeLlama-34B-shape greedy first-{args.depth}-layer loading, flat decode at depth "
                f"{args.depth} (observation_for_depth), teacher-forced synthetic tokens")
    return f"{desc.name} {args.policy} decode step (depth {args.depth if args.policy == 'flat' else desc.num_layers})"


def workload_config(args, desc):
    return {"workload": workload_name(args, desc),
            "model_shape": desc.name, "layers": desc.num_layers, "d_model": desc.d_model,
            "vocab": desc.vocab, "exit_layers": list(desc.exit_layers), "batch_per_gpu": args.batch,
            "global_batch": args.batch * args.gpus, "prompt_len": args.prompt,
            "context": f"{args.prompt}..{args.prompt + args.warmup + args.steps - 1} (timed steps: "
                       f"{args.prompt + args.warmup}..{args.prompt + args.warmup + args.steps - 1})",
            "th": args.th, "policy": args.policy,
            "parallelism": ((f"tp{args.tp} (Megatron shards; row-parallel partials reduce-scattered, "
                             f"all-gathered and folded into the residual + RMSNorm by one peer-memory kernel; "
                             f"vocab-parallel head partials all-gathered by peer copies)" if args.tp_comm == "px" else
                             f"tp{args.tp} (Megatron shards; NCCL all-reduce of row-parallel partials and "
                             f"all-gather of vocab-parallel head partials inside the step)") if args.tp > 1 else
                            f"replicas x{args.gpus} (requests sharded, no data-path collective)"),
            "l2": "inputs larger than L2 (GBs of weights streamed per step > 126 MB L2)"}


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------
def batch_sweep(ctx, eeb, desc, args, stream, batches=(1, 2, 4, 16, 32, 64, 128, 256), n_steps=10):
    """The metric is 'EE decode tokens/s vs batch': the same workload at each
    batch (own model instance with a 256-slot KV pool, prompts prefilled),
    with the layer-GEMM and exit-head fractions of the HBM roofline per batch
    from the in-graph launch timeline of that batch's steps."""
    import torch

    from paper_2504_10724_b200 import timeline

    P = args.prompt
    d = desc.replace(max_slots=max(batches), max_seq_len=P + 100, name=desc.name + "-sweep")
    m = ctx.register(d)
    policy = {"introspective": eeb.INTROSPECTIVE, "flat": eeb.FLAT}.get(args.policy, eeb.INTROSPECTIVE)
    depth = args.depth if policy == eeb.FLAT else 0
    run_layers = depth if policy == eeb.FLAT else d.num_layers
    ctx.load_layers(m, run_layers)  # greedy first-k loading: only the layers the step runs
    hbm = float(peaks()[0]["hbm_gbs"])
    rng = np.random.default_rng(77)
    dev = torch.device("cuda")
    out = []
    for B in batches:
        slots = np.arange(B, dtype=np.int32)
        ctx.prefill(m, run_layers, slots, list(rng.integers(0, d.vocab, (B, P)).astype(np.int32)))
        toks = torch.from_numpy(rng.integers(0, d.vocab, (n_steps + 3, B)).astype(np.int32)).to(dev)
        pos = torch.from_numpy(np.stack([np.full(B, P + k, np.int32) for k in range(n_steps + 3)])).to(dev)
        sl = torch.from_numpy(slots).to(dev)
        torch.cuda.synchronize()

        def one(k):
            ctx.decode_step_device(m, depth, policy, args.th, B, sl.data_ptr(), toks[k].data_ptr(), pos[k].data_ptr())

        for k in range(3):
            one(k)
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(3, n_steps + 3):
            one(k)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / n_steps
        row = {"batch": B, "ms_per_step": ms, "tokens_per_s": B / (ms / 1000.0)}
        try:
            tl = timeline.run(ctx, lambda k: one(3 + k % n_steps), 4)
            g_ms = sum(l["crit_us"] for l in tl["launches"] if l["cat"] == "layer_gemm") / 1e3
            h_ms = sum(l["crit_us"] for l in tl["launches"]
                       if l["cat"] == "exit_head" and l["kernel"] in ("gemm_tc", "gemm_cc")) / 1e3
            # bytes of the launches that ran (batch <= 2: conditional graph
            # bodies skip the layers after a head when every row has exited;
            # a skipped launch records no CTA; `ran` = share of stamped steps)
            g_all = [l for l in tl["launches"] if l["cat"] == "layer_gemm"]
            g_ran = sum(l["ran"] for l in g_all)
            heads = sum(l["ran"] for l in tl["launches"] if l["cat"] == "exit_head" and l["kernel"] == "gemm_tc")
            if g_ms > 0 and g_all:
                row["layer_gemm_frac"] = (gemm_bytes_per_step(d, B, run_layers) * g_ran / len(g_all)
                                          / (g_ms / 1e3) / 1e9 / hbm)
                if policy == eeb.FLAT:
                    # at large batch the decode GEMMs reach the ridge point (2 B
                    # flop per weight byte): the binding roofline is the slower
                    # of the HBM stream and the tensor pipe (sustained bf16 peak)
                    t_hbm = gemm_bytes_per_step(d, B, run_layers) / (hbm * 1e9)
                    tf = float(peaks()[0].get("bf16_tflops_sustained", 0) or peaks()[0].get("bf16_tflops", 0))
                    if tf > 0:
                        t_tc = gemm_flops_per_step(d, B, run_layers) / (tf * 1e12)
                        row["layer_gemm_tensor_frac"] = t_tc / (g_ms / 1e3)
                        row["layer_gemm_bound"] = "tensor" if t_tc > t_hbm else "hbm"
                        row["layer_gemm_roofline_frac"] = max(t_tc, t_hbm) / (g_ms / 1e3)
                    # whole step (weights + heads + KV): the per-launch critical-path
                    # times credit a GEMM's pre-wait weight prefetch to its
                    # predecessor, so at small batch the GEMM fraction can read
                    # above 1; the step fraction is the unattributed check
                    kv = B * run_layers * (P + 3 + 0.5 * n_steps) * 2 * d.n_kv_heads * d.head_dim * d.bytes_per_el
                    w = d.layer_weight_elems() * d.bytes_per_el * run_layers + head_bytes(d, B) * heads
                    row["step_hbm_frac"] = (w + kv) / (ms / 1e3) / 1e9 / hbm
            if h_ms > 0 and heads:
                row["exit_head_frac"] = head_bytes(d, B) * heads / (h_ms / 1e3) / 1e9 / hbm
        except Exception as e:  # per-batch roofline is extra information
            row["roofline_error"] = repr(e)[:120]
        out.append(row)
    ctx.evict(m)
    return out


def measure_loader(ctx, m, eeb, step, args, stream, depth=16, n_steps=20):
    """C3's switching partner: stage OPT-2.7B to pinned host memory, then load its
    first `depth` layers (+ base weights) asynchronously while the serving model
    keeps decoding.  Reports the measured H2D rate and the decode step time with
    and without the transfer in flight."""
    import torch

    d2 = eeb.PRESETS["opt-2.7b"].replace(max_slots=8, max_seq_len=16, name="opt-2.7b-switch")
    m2 = ctx.register(d2)
    t0 = time.perf_counter()
    ctx.host_stage(m2, depth)
    stage_s = time.perf_counter() - t0

    def timed_steps():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(n_steps):
            step(k % max(1, args.warmup))
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / n_steps

    alone = timed_steps()
    ctx.load_layers_async(m2, depth)
    during = timed_steps()
    secs, nbytes = ctx.load_wait(m2)
    ctx.evict(m2)
    return {"model": "opt-2.7b shape", "layers": depth, "bytes": nbytes, "seconds": secs,
            "h2d_gbs": nbytes / secs / 1e9 if secs > 0 else None, "host_stage_s": stage_s,
            "decode_ms_per_step_alone": alone, "decode_ms_per_step_during_load": during,
            "how": "eeb_host_stage (pinned host tier) then eeb_load_layers_async on the load stream while "
                   f"{n_steps} C2 decode steps run on the decode stream; CUDA events on both streams"}



def ncu_traffic(args, desc):
    """DRAM bytes per step of the layer GEMMs and the exit-head GEMMs from the
    committed ncu launch list of this workload (profiles/r2, one serialised
    --metrics dram__bytes_read.sum,dram__bytes_write.sum capture of a C2 step;
    cold cache).  None for other workloads."""
    path = ROOT / "profiles" / "r2" / "launches_c2_b64.csv.gz"
    if not path.exists() or desc.name != "opt-1.3b-4x" or args.batch != 64 or args.policy != "introspective":
        return None
    import csv
    import gzip
    launches = {}
    with gzip.open(path, "rt") as f:
        for r in csv.DictReader(line for line in f if not line.startswith("==")):
            d = launches.setdefault(r["ID"], {"name": r["Kernel Name"], "grid": r.get("Grid Size", "")})
            d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    layer = head = 0.0
    for d in launches.values():
        if "gemm_tc" not in d["name"]:
            continue
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        if d["grid"].startswith(f"({(desc.vocab + 127) // 128},"):
            head += b
        else:
            layer += b
    return {"layer_gemm": int(layer), "exit_head": int(head), "source": str(path.relative_to(ROOT))}

def parity_sample(ctx, m, desc, eeb, args, policy, depth, toks_h, pos_h, e2e_outs, n_rows: int = 8):
    """bf16 token / exit agreement of the e2e steps (the headline e2e calls)
    with the CPU oracle on a sample of rows: the oracle is seeded with those
    rows' prompt KV read back from the GPU (prefill parity is its own test),
    then replays every decode step of the run (warm-up positions included, so
    its KV of the decode positions is its own) and each e2e step's outputs for
    the sampled rows are compared."""
    from oracle.oracle import OracleModel

    t0 = time.perf_counter()
    B, P = args.batch, args.prompt
    rows = np.linspace(0, B - 1, n_rows).astype(np.int32)
    ref = OracleModel(desc.replace(max_slots=n_rows))
    ref.load(depth or desc.num_layers)
    for i, r in enumerate(rows):
        for layer in range(1, desc.num_layers + 1):
            k, v = ctx.read_kv_span(m, layer, int(r), 0, P)
            ref.write_kv(layer, i, 0, k, v)
    tok_same = exit_same = n = 0
    conf_err = 0.0
    near_th = 0
    for k in range(len(toks_h)):
        r = ref.decode_step(depth, policy, args.th, np.arange(n_rows), toks_h[k][rows], pos_h[k][rows])
        if k < args.warmup:
            continue
        g = e2e_outs[k - args.warmup]
        tok_same += int((g["token_id"][rows] == r["token_id"]).sum())
        same = g["exit_layer"][rows] == r["exit_layer"]
        exit_same += int(same.sum())
        near_th += int((~same & ((np.abs(r["confidence"] - args.th) <= 2e-2) |
                                 (np.abs(g["confidence"][rows] - args.th) <= 2e-2))).sum())
        if same.any():
            conf_err = max(conf_err, float(np.max(np.abs(g["confidence"][rows][same] - r["confidence"][same]))))
        n += n_rows
    ref.close()
    return {"token_agreement": tok_same / max(1, n), "exit_agreement": exit_same / max(1, n),
            "exit_mismatches_within_2e-2_of_th": near_th, "exit_mismatches": n - exit_same,
            "max_abs_conf_diff_where_exits_agree": conf_err, "row_steps": n, "rows": rows.tolist(),
            "seconds": time.perf_counter() - t0,
            "how": "the e2e steps' outputs (host API) for the sampled rows vs the CPU oracle replaying every decode "
                   "step from the GPU's prompt KV; bf16 bar: token agreement >= 0.99"}


def _free_port() -> int:
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def run_eeb(args, desc):
    import torch

    from paper_2504_10724_b200 import eeb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    B, P = args.batch, args.prompt
    policy = {"introspective": eeb.INTROSPECTIVE, "flat": eeb.FLAT, "profile": eeb.PROFILE,
              "full_depth": eeb.FULL_DEPTH}[args.policy]
    depth = args.depth if policy == eeb.FLAT else 0
    desc = desc.replace(max_slots=B, max_seq_len=P + 100)
    tp = args.tp
    if tp > 1:
        # C5: one Megatron shard per rank (column-parallel QKV / up, row-parallel
        # O / down + NCCL all-reduce, vocab-parallel heads + all-gather); every
        # rank serves the same B rows
        if tp != world:
            raise SystemExit(f"--tp {tp} needs exactly {tp} ranks (got {world})")
        desc = desc.replace(tp_size=tp, tp_rank=rank)
    # rows served per step by the whole job: replicas add rows, a TP group does not
    job_rows = B if tp > 1 else world * B
    ctx = eeb.Context(local)
    if tp > 1 and args.tp_comm == "nccl":
        uid = [eeb.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.nccl_init(uid[0], world, rank)
    ctx.set_gemm_tier(args.tier)
    m = ctx.register(desc)
    if tp > 1 and args.tp_comm == "px":
        # peer-memory exchange (tp_norm / px_gather kernels over NVLink P2P):
        # every rank's exchange buffer through CUDA IPC handles
        _, h = ctx.tp_px_alloc(m)
        handles = [None] * world
        dist.all_gather_object(handles, h)
        ctx.tp_px_attach(m, world, handles=handles)
    ctx.load_layers(m, desc.num_layers)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))
    rng = np.random.default_rng(1000 if tp > 1 else 1000 + rank)  # a TP group decodes the same rows
    slots = np.arange(B, dtype=np.int32)

    # prefill (eeb_prefill, 1024-row chunked passes over all layers): the
    # prompts' KV at every layer.  Two untimed passes (eager, then the graph
    # capture), then a timed one over the same prompts (TTFT of the batch: every request's first
    # token waits for it; host->device copy of the prompts included).
    prompts = rng.integers(0, desc.vocab, (B, P)).astype(np.int32)
    for _ in range(2):  # (a chunk layout runs eagerly once, is captured on its repeat)
        ctx.prefill(m, desc.num_layers, slots, list(prompts))
    barrier()
    t_pf = time.perf_counter()
    ctx.prefill(m, desc.num_layers, slots, list(prompts))
    pf_s = max_over_ranks(time.perf_counter() - t_pf)
    prefill = {"tokens_per_gpu": B * P, "depth": desc.num_layers, "ms": 1000.0 * pf_s,
               "tokens_per_s": job_rows * P / pf_s, "ttft_ms": 1000.0 * pf_s,
               "how": "eeb_prefill of the batch's prompts (host tokens, H2D + chunked passes), wall clock "
                      "around the blocking call, max over ranks"}

    n_tok = args.warmup + args.steps
    toks_h = rng.integers(0, desc.vocab, (n_tok, B)).astype(np.int32)
    pos_h = np.stack([np.full(B, P + (k % 100), np.int32) for k in range(n_tok)])
    dev = torch.device("cuda", local)
    toks_d = torch.from_numpy(toks_h).to(dev)
    pos_d = torch.from_numpy(pos_h).to(dev)
    slots_d = torch.from_numpy(slots).to(dev)
    ne = len(desc.exit_layers)
    outs = {"exit_layer": torch.zeros(B, dtype=torch.int32, device=dev),
            "token_id": torch.zeros(B, dtype=torch.int32, device=dev),
            "confidence": torch.zeros(B, dtype=torch.float32, device=dev),
            "hist": torch.zeros(ne, dtype=torch.int64, device=dev)}
    hist_acc = torch.zeros(ne, dtype=torch.int64, device=dev)
    out_ptrs = {k: v.data_ptr() for k, v in outs.items()}
    torch.cuda.synchronize()

    hist_all = torch.zeros((n_tok, ne), dtype=torch.int64, device=dev)

    def step(k, hist_row=None):
        if hist_row is not None:
            out_ptrs["hist"] = hist_row.data_ptr()
        ctx.decode_step_device(m, depth, policy, args.th, B, slots_d.data_ptr(), toks_d[k].data_ptr(),
                               pos_d[k].data_ptr(), out_ptrs)

    # The clock sampler starts before the warm-up steps so the GPU never idles
    # between warm-up and the timed region (an idle gap lets clocks/power
    # state drop and the first timed steps pay the ramp back up).
    sampler = ClockSampler(local)
    sampler.start()
    t_w = time.perf_counter()
    k = 0
    while k < args.warmup or time.perf_counter() - t_w < 0.3:
        step(k % args.warmup)
        k += 1
    ctx.synchronize()

    # ---- timed region (device events on the eeb stream), graphs on ----------
    barrier()
    torch.cuda.synchronize()
    ctx.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for k in range(args.warmup, n_tok):
        step(k, hist_all[k])  # each step's histogram into its own row: no extra op in the timed region
    ev1.record(stream)
    ev1.synchronize()
    ctx.synchronize()
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    hist_acc = hist_all[args.warmup:].sum(dim=0)
    ms_local = ev0.elapsed_time(ev1) / args.steps
    ms = max_over_ranks(ms_local)
    value = job_rows / (ms / 1000.0)

    # ---- in-graph launch timeline of the same steps (eeb_debug_stamps) ---------
    # Every kernel of the captured PDL graph stamps its first-CTA start and
    # last-warp exit; per-launch critical-path times sum to the step span.
    from paper_2504_10724_b200 import timeline

    n_tl = min(args.steps, 8)
    tl = timeline.run(ctx, lambda k: step(args.warmup + (k % args.steps)), n_tl)
    launches_per_step = len(tl["launches"])
    pk, pk_kind = peaks()
    hbm = float(pk["hbm_gbs"])
    peak_source = ("measured MEASURED_PEAKS.json hbm_gbs (copy burst)" if pk_kind == "measured"
                   else "fallback 6650 GB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)")
    hist_np = hist_acc.cpu().numpy().astype(np.float64)
    run_layers = args.depth if policy == eeb.FLAT else desc.num_layers
    heads_run = 1 if policy in (eeb.FLAT, eeb.FULL_DEPTH) else ne
    hist_frac = hist_np / max(1.0, hist_np.sum())

    def crit_ms(pred):
        return sum(l["crit_us"] for l in tl["launches"] if pred(l)) / 1e3

    gemm_ms = crit_ms(lambda l: l["cat"] == "layer_gemm")
    head_gemm_ms = crit_ms(lambda l: l["cat"] == "exit_head" and l["kernel"] in ("gemm_tc", "gemm_cc", "head_reduce"))
    head_ms = crit_ms(lambda l: l["cat"] == "exit_head")
    attn_ms = crit_ms(lambda l: l["cat"] == "attention")
    g_bytes = gemm_bytes_per_step(desc, B, run_layers)
    h_bytes = head_bytes(desc, B) * heads_run
    tr = ncu_traffic(args, desc)
    roof = {"bound": "hbm", "kernel": "layer decode GEMMs (K1, tcgen05)",
            "achieved": g_bytes / (gemm_ms / 1000.0) / 1e9, "peak": hbm, "unit": "GB/s",
            "traffic": tr["layer_gemm"] if tr else None,
            **({"traffic_source": tr["source"] + " (DRAM bytes per step, ncu, cold cache)"} if tr else {}),
            "peak_source": peak_source, "algorithmic_bytes_per_step": g_bytes, "kernel_ms_per_step": gemm_ms,
            "time_source": "in-graph %globaltimer stamps (critical-path time per launch, captured PDL graph)",
            "step_share": gemm_ms / max(1e-9, tl["span_ms"])}
    roof["frac"] = roof["achieved"] / hbm
    exit_head = {"kernel": "fused exit-head GEMM (K2: LM head + max/argmax/sum-exp epilogue)",
                 "achieved": h_bytes / (head_gemm_ms / 1000.0) / 1e9 if head_gemm_ms > 0 else None,
                 "unit": "GB/s", "ms_per_step": head_gemm_ms, "head_path_ms_per_step": head_ms,
                 "algorithmic_bytes_per_step": h_bytes, "traffic": tr["exit_head"] if tr else None}
    if exit_head["achieved"]:
        exit_head["frac"] = exit_head["achieved"] / hbm
        exit_head["frac_incl_decide"] = h_bytes / (head_ms / 1000.0) / 1e9 / hbm
    # KV of the rows that reached each layer (introspective: survivors only)
    if policy == eeb.INTROSPECTIVE:
        row_layers = float(np.sum(hist_frac * np.asarray(desc.exit_layers))) * B
    else:
        row_layers = float(run_layers * B)
    mean_ctx = P + args.warmup + 0.5 * args.steps + 1
    kv_step = row_layers * mean_ctx * 2 * desc.n_kv_heads * desc.head_dim * desc.bytes_per_el
    attention = {"kernel": "decode attention (K1b)", "ms_per_step": attn_ms, "algorithmic_bytes_per_step": int(kv_step),
                 "achieved": kv_step / (attn_ms / 1000.0) / 1e9 if attn_ms > 0 else None, "unit": "GB/s"}
    if attention["achieved"]:
        attention["frac"] = attention["achieved"] / hbm
    w_step = desc.layer_weight_elems() * desc.bytes_per_el * run_layers + \
        desc.vocab * desc.d_model * desc.bytes_per_el * heads_run
    step_roof = {"bound": "hbm", "algorithmic_bytes_per_step": int(w_step + kv_step),
                 "weight_bytes": int(w_step), "kv_bytes": int(kv_step),
                 "achieved": (w_step + kv_step) / (ms / 1000.0) / 1e9, "peak": hbm, "unit": "GB/s"}
    step_roof["frac"] = step_roof["achieved"] / hbm
    kernel_ms = {c: v["crit_ms"] for c, v in tl["cats"].items()}
    kernel_ms["span"] = tl["span_ms"]

    # ---- e2e: public host-pointer API, H2D + D2H inside every call ------------
    # (one untimed host-API call first, like the device loop's warm-up: the
    #  host path's first call sizes its pinned staging; it replays the last
    #  warm-up position, which the timed calls do not reuse)
    kw = max(0, args.warmup - 1)
    ctx.decode_step(m, depth, policy, args.th, slots, toks_h[kw], pos_h[kw])
    ctx.synchronize()
    barrier()
    t0 = time.perf_counter()
    e2e_outs = []
    for k in range(args.warmup, n_tok):
        e2e_outs.append(ctx.decode_step(m, depth, policy, args.th, slots, toks_h[k], pos_h[k]))
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    parity = None
    if rank == 0 and not args.no_parity and tp == 1:
        try:
            parity = parity_sample(ctx, m, desc, eeb, args, policy, depth, toks_h, pos_h, e2e_outs)
        except Exception as e:  # reported, never fatal for the headline line
            parity = {"error": repr(e)[:200]}
    e2e_value = job_rows * args.steps / e2e_s
    h2d = 3 * B * 4
    d2h = B * (4 + 4 + 4 + 4 + 1 + 1) + ne * 8 + 8 + 8

    # ---- profiler histogram all-reduce across replicas (the one collective) ---
    from paper_2504_10724_b200 import replicas

    prof_counters = replicas.ProfileCounters(desc.exit_layers, hist=hist_acc.cpu().numpy())
    prof_counters.tokens = int(prof_counters.hist.sum())
    if world > 1 and tp == 1:  # (a TP group serves the same rows on every rank: nothing to merge)
        uid = [eeb.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.nccl_init(uid[0], world, rank)
        prof_counters.allreduce(replicas.eeb_allreduce(ctx))
    hist_total = prof_counters.hist
    exit_frac = {str(l): float(c) / max(1, hist_total.sum()) for l, c in zip(desc.exit_layers, hist_total)}

    # ---- greedy loader: real pinned H2D of a second model's
    # first layers on the load stream, overlapped with this model's decode steps
    loader = sweep = None
    if rank == 0 and world == 1 and (args.sweep or not args.no_secondary):
        try:
            sweep = batch_sweep(ctx, eeb, desc, args, stream)
        except Exception as e:  # reported, never fatal for the headline line
            sweep = {"error": repr(e)[:200]}
    if rank == 0 and world == 1 and not args.no_secondary:
        try:
            loader = measure_loader(ctx, m, eeb, step, args, stream)
        except Exception as e:  # reported, never fatal for the headline line
            loader = {"error": repr(e)[:200]}

    ctx.close()

    def child_bench(extra: list, timeout: float):
        """bench.py for another workload in a child process per rank (every
        rank spawns one; under torchrun the children form their own process
        group on a fresh port).  Rank 0 returns the child's JSON line."""
        env = dict(os.environ)
        if world > 1:
            port = [_free_port() if rank == 0 else None]
            dist.broadcast_object_list(port, src=0)
            env["MASTER_PORT"] = str(port[0])
            env.pop("TORCHELASTIC_USE_AGENT_STORE", None)  # the child's rank 0 hosts its own store
        cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", str(world), *extra,
               "--no-cpu-baseline", "--no-secondary", "--no-parity"]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
            lines = r.stdout.strip().splitlines()
            if rank != 0:
                return None
            if r.returncode != 0 or not lines:
                return {"error": f"rc={r.returncode}: " + (r.stderr.strip().splitlines() or [""])[-1][:200]}
            return json.loads(lines[-1])
        except Exception as e:  # reported, never fatal for the headline line
            return {"error": repr(e)[:200]} if rank == 0 else None
        finally:
            barrier()

    secondary = None
    if not args.no_secondary and tp == 1:
        # C4 beside the headline at every N: the 34B shape the north star's
        # scaling target (>= 6x from 1 to 8 GPUs) is quoted on — greedy first-12
        # layers (choose_depth, test_policy.cpp:322-327), flat decode, requests
        # sharded over the ranks; with its batch sweep at N = 1.
        d = child_bench(["--model", "codellama-34b", "--policy", "flat", "--depth", "12", "--batch", str(args.batch),
                         "--steps", "10", "--warmup", "3"] + (["--sweep"] if world == 1 else []), 600)
        if d is not None and "error" not in d:
            secondary = {"workload": d["config"]["workload"], "value": d["value"], "unit": d["unit"],
                         "n_gpus": d["n_gpus"], "ms_per_step": d["ms_per_step"], "batch_per_gpu": args.batch,
                         "e2e": d["e2e"], "layer_gemm_roofline_frac": d["roofline"]["frac"],
                         "step_roofline": d["step_roofline"],
                         "exit_head_roofline_frac": (d.get("exit_head_roofline") or {}).get("frac"),
                         "clocks": d.get("clocks"), **({"batch_sweep": d["batch_sweep"]} if "batch_sweep" in d else {})}
        else:
            secondary = d
    c5 = None
    if not args.no_secondary and tp == 1 and world > 1:
        # C5 (BASELINE configs[4]): Llama2-70B shape tensor-parallel over the
        # launched ranks (NCCL inside the step), flat at the greedy depth 10
        # (test_policy.cpp:328)
        d = child_bench(["--model", "llama2-70b", "--tp", str(world), "--policy", "flat", "--depth", "10",
                         "--batch", str(args.batch), "--steps", "10", "--warmup", "3"], 420)
        if d is not None and "error" not in d:
            c5 = {"workload": d["config"]["workload"], "value": d["value"], "unit": d["unit"], "n_gpus": d["n_gpus"],
                  "ms_per_step": d["ms_per_step"], "batch": args.batch, "e2e": d["e2e"],
                  "layer_gemm_roofline_frac": d["roofline"]["frac"], "step_roofline": d["step_roofline"],
                  "kernel_ms_per_step": d.get("kernel_ms_per_step")}
        else:
            c5 = d

    c3 = None
    serve_c3 = ROOT / "paper_2504_10724_b200" / "_build" / "serve_c3"
    if rank == 0 and world == 1 and not args.no_secondary and serve_c3.exists():
        # C3 (BASELINE configs[2]): OPT-1.3B + OPT-2.7B shapes behind the host C++
        # engine in HELIOS mode at batch 256 (eval cycles, greedy loads from a
        # pinned host tier, continuous batching), its own process.
        try:
            out = subprocess.run([str(serve_c3), "1024", "128", "64"], capture_output=True, text=True,
                                 timeout=600).stdout.strip().splitlines()
            c3 = json.loads(out[-1])
        except Exception as e:  # reported, never fatal for the headline line
            c3 = {"error": repr(e)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_port_run(desc, steps=2, warmup=0, rows=B, prompt=P + args.warmup)
        cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, biased exit heads)",
                "config": workload_config(args, desc), "roofline": roof, "step_roofline": step_roof,
                "exit_head_roofline": exit_head, "attention_roofline": attention,
                "cpu_baseline": cpu, "parity": parity,
                "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h},
                "gpu_launches": int(launches_per_step * args.steps),
                "launches_per_step": launches_per_step,
                "timeline": {"span_ms": tl["span_ms"], "steps_stamped": n_tl,
                             "how": "separate stamped replay of the timed steps' inputs; per-launch critical-path "
                                    "times (end - previous end) from in-kernel %globaltimer stamps"},
                "clocks": clocks, "exit_fractions": exit_frac, "prefill": prefill,
                "kernel_ms_per_step": kernel_ms,
                "path": "per-op kernel chain (CUDA graph, PDL)"}
        if secondary is not None:
            line["secondary_c4"] = secondary
        if c5 is not None:
            line["secondary_c5"] = c5
        if c3 is not None:
            line["secondary_c3"] = c3
        if loader is not None:
            line["loader"] = loader
        if sweep is not None:
            line["batch_sweep"] = sweep
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="eeb", choices=["eeb", "reference"])
    ap.add_argument("--model", default="opt-1.3b-4x")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--policy", default="introspective",
                    choices=["introspective", "flat", "profile", "full_depth"])
    ap.add_argument("--depth", type=int, default=6)
    ap.add_argument("--th", type=float, default=0.7)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check of sampled e2e rows")
    ap.add_argument("--no-secondary", action="store_true", help="skip the C4 (34B) line attached at N=1")
    ap.add_argument("--tier", type=int, default=0, help="0 auto, 1 CUDA-core GEMV, 2 tcgen05 GEMMs")
    ap.add_argument("--tp", type=int, default=1, help="tensor-parallel group = the launched ranks (C5)")
    ap.add_argument("--tp-comm", choices=["px", "nccl"], default="px",
                    help="C5 exchange: px = fused peer-memory reduce + residual + RMSNorm kernels (default), "
                         "nccl = NCCL all-reduce / all-gather between the step's kernels")
    ap.add_argument("--sweep", action="store_true", help="batch sweep of this workload with per-batch roofline")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    from paper_2504_10724_b200 import eeb

    desc = eeb.PRESETS[args.model]
    if args.impl == "reference":
        return run_reference(args, desc)
    return run_eeb(args, desc)


if __name__ == "__main__":
    sys.exit(main())
