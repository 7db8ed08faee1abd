"""GPU checks of the greedy layer loader over a pinned host tier
(eeb_host_stage / eeb_load_layers_async / eeb_load_wait ↔ do_load,
engine.hpp:197-216, and apply_load, memory_model.hpp:86-105).

A model loaded layer by layer from host memory (async H2D on the load
stream, overlapped with decode at the old depth) must decode bit-identically
to the same model materialised on device; the measured transfer must move
exactly the layers' bytes.
"""
import numpy as np
import pytest

from paper_2504_10724_b200 import eeb

pytestmark = pytest.mark.gpu

TH = 0.7


@pytest.fixture(scope="module")
def ctx():
    c = eeb.Context(0)
    yield c
    c.close()


def _desc(name):
    return eeb.PRESETS["tiny"].replace(dtype=eeb.BF16, name=name, max_slots=16, max_seq_len=64)


def _same(a, b):
    for k in ("exit_layer", "token_id", "confidence", "logprob", "hist"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


def test_async_load_matches_device_materialised(ctx):
    ref_m = ctx.register(_desc("tiny-ref"))
    ctx.load_layers(ref_m, 12)
    m = ctx.register(_desc("tiny-host"))
    ctx.host_stage(m, 12)
    assert ctx.loaded_depth(m) == 0
    ctx.load_layers_async(m, 6)      # greedy first-k: base weights + layers 1..6
    rng = np.random.default_rng(3)
    B = 16
    slots = np.arange(B)
    for pos in range(3):             # flat decode at depth 6 while nothing deeper exists
        toks = rng.integers(0, 512, B)
        _same(ctx.decode_step(m, 6, eeb.FLAT, TH, slots, toks, np.full(B, pos)),
              ctx.decode_step(ref_m, 6, eeb.FLAT, TH, slots, toks, np.full(B, pos)))
    sec, nbytes = ctx.load_wait(m)
    assert nbytes == ctx.weight_bytes(m, 6) and sec > 0
    # load-more to full depth, overlapped with flat steps at the old depth;
    # the full-depth step waits on the in-flight layers' events
    ctx.load_layers_async(m, 12)
    toks = rng.integers(0, 512, B)
    _same(ctx.decode_step(m, 6, eeb.FLAT, TH, slots, toks, np.full(B, 3)),
          ctx.decode_step(ref_m, 6, eeb.FLAT, TH, slots, toks, np.full(B, 3)))
    for pos in range(4, 7):
        toks = rng.integers(0, 512, B)
        _same(ctx.decode_step(m, 0, eeb.FULL_DEPTH, TH, slots, toks, np.full(B, pos)),
              ctx.decode_step(ref_m, 0, eeb.FULL_DEPTH, TH, slots, toks, np.full(B, pos)))
    sec, nbytes = ctx.load_wait(m)
    assert nbytes == ctx.weight_bytes(m, 12) - ctx.weight_bytes(m, 6)
    for pos in range(7, 9):
        toks = rng.integers(0, 512, B)
        _same(ctx.decode_step(m, 0, eeb.INTROSPECTIVE, TH, slots, toks, np.full(B, pos)),
              ctx.decode_step(ref_m, 0, eeb.INTROSPECTIVE, TH, slots, toks, np.full(B, pos)))
    # shrink (evict deeper layers) and regrow from the host tier
    ctx.load_layers_async(m, 6)
    assert ctx.loaded_depth(m) == 6
    ctx.load_layers_async(m, 12)
    toks = rng.integers(0, 512, B)
    _same(ctx.decode_step(m, 0, eeb.FULL_DEPTH, TH, slots, toks, np.full(B, 9)),
          ctx.decode_step(ref_m, 0, eeb.FULL_DEPTH, TH, slots, toks, np.full(B, 9)))
    ctx.evict(m)
    ctx.evict(ref_m)


def test_async_load_needs_host_tier(ctx):
    m = ctx.register(_desc("tiny-nohost"))
    ctx.host_stage(m, 4)
    with pytest.raises(eeb.EebError) as e:
        ctx.load_layers_async(m, 8)
    assert e.value.kind == "CapacityError"
    ctx.load_layers_async(m, 4)
    ctx.load_wait(m)
    assert ctx.loaded_depth(m) == 4
    ctx.evict(m)


def test_host_stage_from_resident_layers(ctx):
    """Staging a model whose layers are already on device copies them out (D2H)."""
    a = ctx.register(_desc("tiny-res"))
    ctx.load_layers(a, 12)
    ctx.host_stage(a, 12)
    ctx.evict(a)
    ctx.load_layers_async(a, 12)
    b = ctx.register(_desc("tiny-res-ref"))
    ctx.load_layers(b, 12)
    rng = np.random.default_rng(4)
    toks = rng.integers(0, 512, 8)
    _same(ctx.decode_step(a, 0, eeb.FULL_DEPTH, TH, np.arange(8), toks, np.zeros(8)),
          ctx.decode_step(b, 0, eeb.FULL_DEPTH, TH, np.arange(8), toks, np.zeros(8)))
    ctx.evict(a)
    ctx.evict(b)
