"""Tensor parallelism over real rank contexts (C5): two
processes, one GPU each, every rank a Megatron shard (tp_size = 2, tp_rank =
rank) joined by an NCCL communicator (eeb_nccl_init) — the row-parallel O /
down partials all-reduced and the vocab-parallel head partials all-gathered
inside the step — must decode like the all-shards-in-one-context model
(test_gpu_tp.py), itself checked against the oracle.  Skips below 2 GPUs
(every gpurun box has one; the driver's multi-GPU runs execute it)."""
import os
import tempfile

import numpy as np
import pytest

from paper_2504_10724_b200 import eeb

pytestmark = pytest.mark.gpu

TH = 0.7
BASE = eeb.ModelDesc("tp-nccl", 6, 512, 8, 4, 1024, 1024, (2, 4, 6), dtype=eeb.BF16, mlp_kind=eeb.MLP_SWIGLU,
                     max_slots=16, max_seq_len=64, seed=321)
B, STEPS = 16, 6


def _schedule():
    rng = np.random.default_rng(11)
    prompts = [rng.integers(0, BASE.vocab, 8).astype(np.int32) for _ in range(B)]
    toks = [rng.integers(0, BASE.vocab, B).astype(np.int32) for _ in range(STEPS)]
    return prompts, toks


def _decode(ctx, m):
    prompts, toks = _schedule()
    ctx.load_layers(m, BASE.num_layers)
    ctx.prefill(m, BASE.num_layers, np.arange(B), prompts)
    out = []
    for k, t in enumerate(toks):
        pol = eeb.PROFILE if k % 2 == 0 else eeb.INTROSPECTIVE
        r = ctx.decode_step(m, 0, pol, TH, np.arange(B), t, np.full(B, 8 + k))
        out.append(np.stack([r["token_id"], r["exit_layer"]]).astype(np.int64))
        out.append(np.asarray(r["confidence"], np.float64)[None])
    return out


def _rank(rank, uid_path, out_path):
    import time

    ctx = eeb.Context(rank)
    if rank == 0:
        uid = eeb.Context.nccl_unique_id()
        with open(uid_path + ".tmp", "wb") as f:
            f.write(uid)
        os.replace(uid_path + ".tmp", uid_path)
    else:
        while not os.path.exists(uid_path):
            time.sleep(0.05)
        with open(uid_path, "rb") as f:
            uid = f.read()
    ctx.nccl_init(uid, 2, rank)
    m = ctx.register(BASE.replace(name=f"tp2-r{rank}", tp_size=2, tp_rank=rank))
    res = _decode(ctx, m)
    if rank == 0:
        np.savez(out_path, *res)
    ctx.close()


def test_tp2_rank_contexts_decode_like_one_context():
    import torch
    import torch.multiprocessing as mp

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (one Megatron shard per rank)")
    with tempfile.TemporaryDirectory() as d:
        uid_path, out_path = os.path.join(d, "uid"), os.path.join(d, "rank0.npz")
        mp.start_processes(_rank, args=(uid_path, out_path), nprocs=2, join=True, start_method="spawn")
        got = np.load(out_path)
        got = [got[f"arr_{i}"] for i in range(len(got.files))]
    ctx = eeb.Context(0)
    ref = _decode(ctx, ctx.register(BASE.replace(name="tp2-all", tp_size=2, tp_rank=-1)))
    ctx.close()
    agree = total = 0
    for k in range(0, len(ref), 2):
        a, b = got[k], ref[k]
        agree += int((a[0] == b[0]).sum())
        total += a.shape[1]
        far = np.abs(ref[k + 1][0] - TH) > 1e-2
        assert (a[1][far] == b[1][far]).all()
        np.testing.assert_allclose(got[k + 1][0], ref[k + 1][0], atol=2e-2)
    assert agree / total >= 0.99, agree / total
