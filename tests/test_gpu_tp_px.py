"""Tensor parallelism over peer memory (C5 without NCCL on the step's data
path): two rank processes, each holding one Megatron
shard (tp_size = 2, tp_rank = rank) and one exchange buffer shared through
CUDA IPC (eeb_tp_px_alloc / eeb_tp_px_attach).  Every O / down GEMM's partial
planes are reduce-scattered, all-gathered and folded into the residual +
RMSNorm by one kernel (tp_norm), and the exit-head partials are all-gathered
by a peer copy kernel.

The row owner sums the ranks' planes in rank-major, plane-minor order — the
order the all-shards-in-one-context model (tp_rank = -1, test_gpu_tp.py,
itself checked against the oracle) reduces its concatenated planes in — so
both ranks must reproduce that model bit for bit: tokens, exits and
confidences.

The two ranks share the one GPU of a gpurun box (two processes, time-sliced
contexts; on an NVLink node each rank has its own GPU and the same code runs
over P2P).  A rank that stalls traps after ~10 s instead of hanging the
device."""
import os
import tempfile
import time

import numpy as np
import pytest

from paper_2504_10724_b200 import eeb

pytestmark = pytest.mark.gpu

TH = 0.7
BASE = eeb.ModelDesc("tp-px", 6, 512, 8, 4, 1024, 1024, (2, 4, 6), dtype=eeb.BF16, mlp_kind=eeb.MLP_SWIGLU,
                     max_slots=16, max_seq_len=64, seed=321)
B, STEPS = 16, 6


def _schedule(plen):
    rng = np.random.default_rng(11)
    prompts = [rng.integers(0, BASE.vocab, plen).astype(np.int32) for _ in range(B)]
    toks = [rng.integers(0, BASE.vocab, B).astype(np.int32) for _ in range(STEPS)]
    return prompts, toks


def _decode(ctx, m, plen):
    prompts, toks = _schedule(plen)
    ctx.load_layers(m, BASE.num_layers)
    ctx.prefill(m, BASE.num_layers, np.arange(B), prompts)
    out = []
    for k, t in enumerate(toks):
        pol = eeb.PROFILE if k % 2 == 0 else eeb.INTROSPECTIVE
        r = ctx.decode_step(m, 0, pol, TH, np.arange(B), t, np.full(B, plen + k))
        out.append(np.stack([r["token_id"], r["exit_layer"]]).astype(np.int64))
        out.append(np.asarray(r["confidence"], np.float32)[None])
    return out


def _rank(rank, d, graphs, devices, plen):
    ctx = eeb.Context(devices[rank])
    if not graphs:
        ctx.set_graphs(False)
    m = ctx.register(BASE.replace(name=f"px-r{rank}", tp_size=2, tp_rank=rank))
    _, h = ctx.tp_px_alloc(m)
    with open(os.path.join(d, f"h{rank}.tmp"), "wb") as f:
        f.write(h)
    os.replace(os.path.join(d, f"h{rank}.tmp"), os.path.join(d, f"h{rank}"))
    while not all(os.path.exists(os.path.join(d, f"h{p}")) for p in range(2)):
        time.sleep(0.02)
    handles = [open(os.path.join(d, f"h{p}"), "rb").read() for p in range(2)]
    ctx.tp_px_attach(m, 2, handles=handles)
    res = _decode(ctx, m, plen)
    np.savez(os.path.join(d, f"rank{rank}.npz"), *res)
    ctx.close()


# plen 40: 16 x 40 = 640 prompt rows in one prefill chunk (cuBLASLt planes
# written into the exchange buffer, tp_norm over 640 rows)
@pytest.mark.parametrize("graphs,devices,plen", [(True, (0, 0), 8), (False, (0, 0), 8), (True, (0, 1), 8),
                                                 (True, (0, 0), 40)],
                         ids=["graph-1gpu", "eager-1gpu", "graph-2gpu", "graph-1gpu-prefill640"])
def test_tp2_peer_memory_ranks_match_all_shards_bit_for_bit(graphs, devices, plen):
    import torch
    import torch.multiprocessing as mp

    if max(devices) >= torch.cuda.device_count():
        pytest.skip("needs 2 GPUs (one shard per GPU over NVLink P2P)")
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_rank, args=(d, graphs, devices, plen), nprocs=2, join=True, start_method="spawn")
        got = []
        for r in range(2):
            z = np.load(os.path.join(d, f"rank{r}.npz"))
            got.append([z[f"arr_{i}"] for i in range(len(z.files))])
    ctx = eeb.Context(0)
    ref = _decode(ctx, ctx.register(BASE.replace(name="px-all", tp_size=2, tp_rank=-1)), plen)
    ctx.close()
    for r in range(2):
        for k in range(len(ref)):
            np.testing.assert_array_equal(got[r][k], ref[k], err_msg=f"rank {r} output {k}")
