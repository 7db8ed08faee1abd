"""The N>1 path on CPU: requests sharded over 2 replicas (gloo, world size 2),
profiler counters merged by all-reduce, every rank reaching the same greedy
depth as a single replica that served all requests.  The per-row
decode runs on the CPU oracle here; on the GPU box the same code drives
libeeb with the NCCL reduction (bench.py --gpus N)."""
import json
import os
import socket
from pathlib import Path

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_10724_b200 import eeb, replicas

GOLDEN = Path(__file__).resolve().parent / "golden" / "decision_vectors.json"
DESC = eeb.PRESETS["tiny"].replace(max_slots=16)
N_REQ, N_TOK, TH = 12, 3, 0.7


def _tokens(req: int) -> np.ndarray:
    return np.random.default_rng(1000 + req).integers(0, DESC.vocab, N_TOK)


def serve(requests) -> replicas.ProfileCounters:
    """Serve `requests` (slot = request id) with one batched step per position."""
    from oracle.oracle import OracleModel

    o = OracleModel(DESC, threads=2)
    o.load(DESC.num_layers)
    c = replicas.ProfileCounters(DESC.exit_layers)
    reqs = np.asarray(requests, np.int32)
    toks = np.stack([_tokens(r) for r in reqs]) if len(reqs) else np.zeros((0, N_TOK), np.int64)
    for pos in range(N_TOK):
        if len(reqs):
            c.add_step(o.decode_step(0, eeb.INTROSPECTIVE, TH, reqs, toks[:, pos], np.full(len(reqs), pos)))
    o.close()
    return c


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = replicas.shard(range(N_REQ), world, rank)
    c = serve(mine).allreduce(replicas.torch_allreduce())
    depth = c.choose_depth(DESC.num_layers, 0.7)
    Path(out_dir, f"r{rank}.json").write_text(json.dumps(
        {"hist": c.hist.tolist(), "n_breached": c.n_breached, "tokens": c.tokens, "snl": c.sum_neg_logprob,
         "depth": depth, "shard": mine}))
    dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_replicas_merge_to_the_single_replica_profile(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    ranks = [json.loads((tmp_path / f"r{r}.json").read_text()) for r in range(world)]
    assert sorted(ranks[0]["shard"] + ranks[1]["shard"]) == list(range(N_REQ))
    assert not set(ranks[0]["shard"]) & set(ranks[1]["shard"])
    whole = serve(range(N_REQ))
    for r in ranks:
        assert r["hist"] == whole.hist.tolist()
        assert r["n_breached"] == whole.n_breached and r["tokens"] == N_REQ * N_TOK
        assert r["snl"] == pytest.approx(whole.sum_neg_logprob, rel=1e-12)
        assert r["depth"] == whole.choose_depth(DESC.num_layers, 0.7)


def test_shard_is_a_partition():
    ids = list(range(37))
    parts = [replicas.shard(ids, 8, r) for r in range(8)]
    assert sorted(sum(parts, [])) == ids
    assert max(map(len, parts)) - min(map(len, parts)) <= 1
    with pytest.raises(ValueError):
        replicas.shard(ids, 2, 2)


def test_choose_depth_matches_compiled_reference_vectors():
    g = json.loads(GOLDEN.read_text())
    for v in g["choose_depth"]:
        assert replicas.choose_depth(v["layers"], v["counts"], v["layers"][-1], v["coverage"]) == v["depth"], v
    # test_pht.cpp:30-56: 73 / 5 / 22 at 6 / 12 / 24
    assert replicas.choose_depth([6, 12, 24], [73, 5, 22], 24, 0.70) == 6
    assert replicas.choose_depth([6, 12, 24], [73, 5, 22], 24, 0.74) == 12
    assert replicas.choose_depth([6, 12, 24], [73, 5, 22], 24, 0.79) == 24
