"""GPU parity of the prefill path (eeb_prefill ↔ serve_one's prefill phase,
engine.hpp:333-341): a prompt prefilled in chunks on the GPU must leave the
same KV (and therefore the same next decode step) as the oracle decoding the
prompt token by token at the same depth.

Bars as in test_gpu_parity.py: f32 — K/V within 1e-3 relative, next-step
tokens equal, exit layers equal except rows within 1e-4 of th; bf16 — K/V
within bf16 rounding, next-step token agreement >= 99 %.
"""
import numpy as np
import pytest

from oracle.oracle import OracleModel
from paper_2504_10724_b200 import eeb

from test_gpu_parity import MINI, TH, _compare_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = eeb.Context(0)
    yield c
    c.close()


def _tokenwise(step, slots, prompts, start):
    """Feed prompts one position at a time: step k carries every sequence that has a k-th token."""
    for k in range(max(len(p) for p in prompts)):
        rows = [i for i, p in enumerate(prompts) if k < len(p)]
        step(np.array([slots[i] for i in rows]), np.array([prompts[i][k] for i in rows]),
             np.array([start[i] + k for i in rows]))


@pytest.mark.parametrize("depth_policy", ["full", "flat4"])
def test_prefill_matches_oracle_tokenwise(ctx, depth_policy):
    desc = MINI
    m = ctx.register(desc)
    ctx.load_layers(m, desc.num_layers)
    ref = OracleModel(desc)
    ref.load(desc.num_layers)
    rng = np.random.default_rng(11)
    slots = np.array([3, 0, 7])
    lens = [5, 9, 1]
    start = np.array([0, 0, 2])
    prompts = [rng.integers(0, desc.vocab, n) for n in lens]
    if depth_policy == "full":
        depth, pol, dec_depth = desc.num_layers, eeb.FULL_DEPTH, 0
    else:
        depth, pol, dec_depth = 4, eeb.FLAT, 4
    # sequence 2 starts at position 2: give it a real history first (both sides)
    hist = rng.integers(0, desc.vocab, 2)
    for p in range(2):
        ctx.decode_step(m, dec_depth, pol, TH, [slots[2]], [hist[p]], [p])
        ref.decode_step(dec_depth, pol, TH, [slots[2]], [hist[p]], [p])
    ctx.prefill(m, depth, slots, prompts, start)
    _tokenwise(lambda s, t, p: ref.decode_step(dec_depth, pol, TH, s, t, p), slots, prompts, start)
    # K/V of every prompt position at every layer <= depth
    for i, s in enumerate(slots):
        for k in range(lens[i]):
            for layer in range(1, depth + 1):
                gk, gv = ctx.read_kv(m, layer, int(s), int(start[i] + k))
                rk, rv = ref.read_kv(layer, int(s), int(start[i] + k))
                for g_, r_ in ((gk, rk), (gv, rv)):
                    np.testing.assert_allclose(g_, r_, atol=1e-3 * max(1.0, np.abs(r_).max()), rtol=0)
    # the next decode step sees identical context
    nxt = rng.integers(0, desc.vocab, 3)
    pos = start + np.array(lens)
    policy = eeb.INTROSPECTIVE if depth_policy == "full" else eeb.FLAT
    g = ctx.decode_step(m, dec_depth, policy, TH, slots, nxt, pos)
    r = ref.decode_step(dec_depth, policy, TH, slots, nxt, pos)
    _compare_rows(g, r, TH)
    ref.close() if hasattr(ref, "close") else None


HD128 = eeb.ModelDesc("pf-gqa-hd128", 4, 1024, 8, 2, 1024, 1000, (2, 4), dtype=eeb.BF16, max_slots=8,
                      max_seq_len=160)


# OPT-2.7B's head_dim 80 (C3): padded 128-wide attention tiles, the KV maps'
# dims 80..127 read as TMA out-of-bounds zeros
HD80 = eeb.ModelDesc("pf-mha-hd80", 4, 1280, 16, 16, 1024, 1000, (2, 4), dtype=eeb.BF16, max_slots=8,
                     max_seq_len=160)


@pytest.mark.parametrize("which", ["tiny", "gqa-hd128", "mha-hd80", "paged-hd80", "paged", "history"])
def test_prefill_bf16_chunk_boundary(ctx, which):
    """bf16, > 256 prompt tokens: two chunks, one sequence split across them;
    the tensor-core prefill attention (64-row query blocks, causal within the
    chunk) on MHA head_dim 64, GQA head_dim 128, a paged pool, and prompts
    that continue a sequence with decoded history (start position > 0)."""
    if which == "gqa-hd128":
        desc = HD128
    elif which.endswith("hd80"):
        desc = HD80.replace(name="pf-" + which)
    else:
        desc = eeb.PRESETS["tiny"].replace(dtype=eeb.BF16, name="tiny-bf16-pf-" + which, max_slots=8,
                                           max_seq_len=192)
    m = ctx.register(desc)
    ctx.load_layers(m, desc.num_layers)
    if which.startswith("paged"):
        ctx.kv_configure_pages(m, 64, 20)
        ctx.kv_reserve(m, 7, 64)  # page 0 taken: the sequences' pages differ from their slots
    ref = OracleModel(desc)
    ref.load(desc.num_layers)
    rng = np.random.default_rng(5)
    slots = np.array([0, 1, 2])
    lens = [150, 90, 40]  # 280 tokens: chunk 0 = seq 0 + 106 tokens of seq 1
    start = np.zeros(3, np.int32)
    if which == "history":  # 7 decoded tokens before slot 1's prompt (its blocks start at position 7)
        hist = rng.integers(0, desc.vocab, 7)
        for p in range(7):
            ctx.decode_step(m, 0, eeb.FULL_DEPTH, TH, [1], [hist[p]], [p])
            ref.decode_step(0, eeb.FULL_DEPTH, TH, [1], [hist[p]], [p])
        start[1] = 7
    prompts = [rng.integers(0, desc.vocab, n) for n in lens]
    ctx.prefill(m, desc.num_layers, slots, prompts, start)
    _tokenwise(lambda s, t, p: ref.decode_step(0, eeb.FULL_DEPTH, TH, s, t, p), slots, prompts, start)
    worst = 0.0
    for i, s in enumerate(slots):
        for k in (0, lens[i] // 2, lens[i] - 1):
            for layer in (1, desc.num_layers):
                gk, gv = ctx.read_kv(m, layer, int(s), int(start[i] + k))
                rk, rv = ref.read_kv(layer, int(s), int(start[i] + k))
                for g_, r_ in ((gk, rk), (gv, rv)):
                    worst = max(worst, float(np.abs(g_ - r_).max() / max(1e-6, np.abs(r_).max())))
    assert worst < 0.05, worst  # bf16 activations through 12 layers
    agree = []
    for step in range(4):
        nxt = rng.integers(0, desc.vocab, 3)
        pos = start + np.array(lens) + step
        g = ctx.decode_step(m, 0, eeb.INTROSPECTIVE, TH, slots, nxt, pos)
        r = ref.decode_step(0, eeb.INTROSPECTIVE, TH, slots, nxt, pos)
        agree.extend(g["token_id"] == r["token_id"])
    assert np.mean(agree) >= 0.99, np.mean(agree)


def test_prefill_validation(ctx):
    desc = MINI.replace(name="mini-pf-val")
    m = ctx.register(desc)
    ctx.load_layers(m, 4)
    with pytest.raises(eeb.EebError) as e:
        ctx.prefill(m, 6, [0], [[1, 2]])
    assert e.value.kind == "CapacityError"
    with pytest.raises(eeb.EebError) as e:
        ctx.prefill(m, 4, [0], [np.zeros(desc.max_seq_len + 1, np.int32)])
    assert e.value.kind == "DomainError"
    with pytest.raises(eeb.EebError) as e:
        ctx.prefill(m, 4, [0, 0], [[1], [2]])
    assert e.value.kind == "ValidationError"


def test_prefill_bf16_long_context(ctx):
    """A 1100-token prompt (max_seq_len 2048): the tensor-core prefill
    attention past the 1024 positions whose KV depth it stages in shared
    memory (the rest read from global), against the oracle."""
    desc = eeb.PRESETS["tiny"].replace(dtype=eeb.BF16, name="tiny-bf16-long", max_slots=2, max_seq_len=2048)
    m = ctx.register(desc)
    ctx.load_layers(m, desc.num_layers)
    ref = OracleModel(desc)
    ref.load(desc.num_layers)
    rng = np.random.default_rng(17)
    slots = np.array([0, 1])
    lens = [1100, 30]
    start = np.zeros(2, np.int32)
    prompts = [rng.integers(0, desc.vocab, n) for n in lens]
    ctx.prefill(m, desc.num_layers, slots, prompts, start)
    for k in range(max(lens)):  # the oracle decodes the prompts token by token
        live = np.array([i for i in range(2) if k < lens[i]])
        ref.decode_step(0, eeb.FULL_DEPTH, TH, slots[live], np.array([prompts[i][k] for i in live]), np.full(len(live), k))
    agree = []
    for step in range(3):
        nxt = rng.integers(0, desc.vocab, 2)
        pos = np.array(lens) + step
        g = ctx.decode_step(m, 0, eeb.INTROSPECTIVE, TH, slots, nxt, pos)
        r = ref.decode_step(0, eeb.INTROSPECTIVE, TH, slots, nxt, pos)
        agree.extend(g["token_id"] == r["token_id"])
    assert np.mean(agree) >= 0.99, np.mean(agree)

