"""Tensor parallelism (C5: Llama2-70B shape over 8 GPUs) on one GPU.

A model registered with tp_size = N, tp_rank = -1 holds all N Megatron shards
in one context — column-parallel QKV / up, row-parallel O / down whose partial
planes are summed, vocab-parallel exit heads whose per-tile softmax partials
are merged — and runs the same kernels a rank context runs, with the
cross-rank sum / gather done locally instead of by NCCL.  It must decode like
the unsharded model (bf16 bar: token agreement >= 99 %, exits equal away from
the threshold) and like the oracle.
"""
import numpy as np
import pytest

from oracle.oracle import OracleModel
from paper_2504_10724_b200 import eeb

pytestmark = pytest.mark.gpu

TH = 0.7
BASE = eeb.ModelDesc("tp-mini", 6, 512, 8, 4, 1024, 1024, (2, 4, 6), dtype=eeb.BF16, mlp_kind=eeb.MLP_SWIGLU,
                     max_slots=32, max_seq_len=64, seed=123)


@pytest.fixture(scope="module")
def ctx():
    c = eeb.Context(0)
    yield c
    c.close()


def _run(ctx, m, steps, B, policy, depth=0):
    out = []
    for k, toks in enumerate(steps):
        out.append(ctx.decode_step(m, depth, policy, TH, np.arange(B), toks, np.full(B, k)))
    return out


@pytest.mark.parametrize("tp", [2, 4])
def test_tp_shards_decode_like_unsharded(ctx, tp):
    full = ctx.register(BASE.replace(name=f"full-{tp}"))
    ctx.load_layers(full, BASE.num_layers)
    sh = ctx.register(BASE.replace(name=f"tp{tp}", tp_size=tp, tp_rank=-1))
    ctx.load_layers(sh, BASE.num_layers)
    assert ctx.weight_bytes(sh, BASE.num_layers) == ctx.weight_bytes(full, BASE.num_layers)
    rng = np.random.default_rng(tp)
    B = 24
    steps = [rng.integers(0, BASE.vocab, B) for _ in range(8)]
    agree, exits_ok = [], []
    for policy in (eeb.PROFILE, eeb.INTROSPECTIVE):
        a = _run(ctx, full, steps[:4], B, policy) if policy == eeb.PROFILE else \
            [ctx.decode_step(full, 0, policy, TH, np.arange(B), t, np.full(B, 4 + k)) for k, t in enumerate(steps[4:])]
        b = _run(ctx, sh, steps[:4], B, policy) if policy == eeb.PROFILE else \
            [ctx.decode_step(sh, 0, policy, TH, np.arange(B), t, np.full(B, 4 + k)) for k, t in enumerate(steps[4:])]
        for x, y in zip(a, b):
            agree.extend(x["token_id"] == y["token_id"])
            far = np.abs(x["confidence"] - TH) > 1e-2
            exits_ok.extend((x["exit_layer"] == y["exit_layer"])[far])
            np.testing.assert_allclose(x["confidence"], y["confidence"], atol=2e-2)
    assert np.mean(agree) >= 0.99, np.mean(agree)
    assert all(exits_ok)
    # KV of every (global) kv head lands in the same place
    for layer in (1, BASE.num_layers):
        gk, gv = ctx.read_kv(sh, layer, 3, 5)
        rk, rv = ctx.read_kv(full, layer, 3, 5)
        np.testing.assert_allclose(gk, rk, atol=3e-2, rtol=3e-2)
        np.testing.assert_allclose(gv, rv, atol=3e-2, rtol=3e-2)
    ctx.evict(full)
    ctx.evict(sh)


@pytest.mark.parametrize("plen", [12, 40], ids=["chunk192", "chunk640"])
def test_tp_matches_oracle_and_prefill(ctx, plen):
    """Sharded model prefilled then decoded against the oracle; 16 x 40 = 640
    prompt rows put the row-parallel shards' prefill GEMMs on cuBLASLt planes
    side by side (chunks above 256 rows have no split-K tcgen05 path)."""
    desc = BASE.replace(name=f"tp2-oracle-{plen}", tp_size=2, tp_rank=-1)
    m = ctx.register(desc)
    ctx.load_layers(m, desc.num_layers)
    ref = OracleModel(BASE)
    ref.load(BASE.num_layers)
    rng = np.random.default_rng(9)
    B = 16
    prompts = [rng.integers(0, BASE.vocab, plen) for _ in range(B)]
    ctx.prefill(m, desc.num_layers, np.arange(B), prompts)
    for k in range(plen):
        ref.decode_step(0, eeb.FULL_DEPTH, TH, np.arange(B), np.array([p[k] for p in prompts]), np.full(B, k))
    agree = []
    for k in range(4):
        toks = rng.integers(0, BASE.vocab, B)
        g = ctx.decode_step(m, 0, eeb.INTROSPECTIVE, TH, np.arange(B), toks, np.full(B, plen + k))
        r = ref.decode_step(0, eeb.INTROSPECTIVE, TH, np.arange(B), toks, np.full(B, plen + k))
        agree.extend(g["token_id"] == r["token_id"])
    assert np.mean(agree) >= 0.99, np.mean(agree)
    ctx.evict(m)


def test_tp_rank_context_needs_communicator(ctx):
    m = ctx.register(BASE.replace(name="tp-rank0", tp_size=2, tp_rank=0))
    ctx.load_layers(m, BASE.num_layers)
    assert ctx.weight_bytes(m, BASE.num_layers) < ctx.weight_bytes(ctx.register(BASE.replace(name="ref-bytes")),
                                                                   BASE.num_layers)
    with pytest.raises(eeb.EebError) as e:
        ctx.decode_step(m, 0, eeb.FULL_DEPTH, TH, np.arange(16), np.zeros(16, np.int32), np.zeros(16, np.int32))
    assert e.value.kind == "DomainError"
    ctx.evict(m)
