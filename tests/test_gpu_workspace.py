"""Captured step graphs stay valid when the shared step workspace grows.

Every model of a context shares one step workspace, grown to the largest
model served.  A graph captured for a small model holds the workspace's
device pointers; when a larger model then grows (reallocates) the workspace,
that graph must be dropped and recaptured, never replayed (a
use-after-free).  Also: reconfiguring the KV pool into pages drops the
model's graphs (they hold the unpaged kernel and the old KV tensor maps).
"""
import numpy as np
import pytest

from paper_2504_10724_b200 import eeb

pytestmark = pytest.mark.gpu

SMALL = eeb.ModelDesc("ws-small", 4, 256, 4, 4, 1024, 512, (2, 4), max_slots=16, max_seq_len=64, seed=11)
LARGE = eeb.ModelDesc("ws-large", 4, 512, 8, 8, 2048, 1024, (2, 4), max_slots=32, max_seq_len=64, seed=12)
KEYS = ("exit_layer", "token_id", "confidence", "logprob", "hist")


def _run(ctx, m, desc, batch, steps, seed, policy=eeb.INTROSPECTIVE, pos0=0):
    rng = np.random.default_rng(seed)
    outs = []
    for t in range(steps):
        toks = rng.integers(0, desc.vocab, batch).astype(np.int32)
        outs.append(ctx.decode_step(m, 0, policy, 0.7, np.arange(batch), toks, np.full(batch, pos0 + t)))
    return outs


def _same(a, b):
    for x, y in zip(a, b):
        for k in KEYS:
            assert np.array_equal(x[k], y[k]), k


def test_small_large_small_graphs_equal_eager():
    # eager reference (no graphs), each model on its own context
    ref = {}
    for desc, batch in ((SMALL, 8), (LARGE, 24)):
        c = eeb.Context(0)
        c.set_graphs(False)
        m = c.register(desc)
        c.load_layers(m, desc.num_layers)
        ref[desc.name] = _run(c, m, desc, batch, 6, 3)
        c.close()
    # one context, graphs on: small (capture), large (workspace grows), small again
    ctx = eeb.Context(0)
    try:
        ms = ctx.register(SMALL)
        ml = ctx.register(LARGE)
        ctx.load_layers(ms, SMALL.num_layers)
        ctx.load_layers(ml, LARGE.num_layers)
        first = _run(ctx, ms, SMALL, 8, 3, 3)                  # positions 0..2, graphs captured
        large = _run(ctx, ml, LARGE, 24, 6, 3)                 # grows every shared buffer
        rng = np.random.default_rng(3)
        toks = [rng.integers(0, SMALL.vocab, 8).astype(np.int32) for _ in range(6)]
        again = [ctx.decode_step(ms, 0, eeb.INTROSPECTIVE, 0.7, np.arange(8), toks[t], np.full(8, t))
                 for t in range(3, 6)]                         # the small model's graph replayed after growth
        _same(first, ref[SMALL.name][:3])
        _same(large, ref[LARGE.name])
        _same(again, ref[SMALL.name][3:])
    finally:
        ctx.close()


def test_kv_paging_after_capture_drops_graphs():
    desc = eeb.PRESETS["opt-1.3b-4x"].replace(num_layers=4, exit_layers=(2, 4), max_slots=8, max_seq_len=128,
                                               name="paging-after-capture")
    ctx = eeb.Context(0)
    try:
        m = ctx.register(desc)
        ctx.load_layers(m, desc.num_layers)
        _run(ctx, m, desc, 4, 2, 5)  # graph captured on the unpaged pool
        ctx.kv_configure_pages(m, 64, 16)
        for s in range(4):
            ctx.kv_reserve(m, s, 8)
        out = _run(ctx, m, desc, 4, 4, 6)
        c2 = eeb.Context(0)
        c2.set_graphs(False)
        m2 = c2.register(desc)
        c2.load_layers(m2, desc.num_layers)
        c2.kv_configure_pages(m2, 64, 16)
        for s in range(4):
            c2.kv_reserve(m2, s, 8)
        _same(out, _run(c2, m2, desc, 4, 4, 6))
        c2.close()
    finally:
        ctx.close()
