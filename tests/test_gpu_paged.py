"""Paged KV pool (eeb_kv_configure_pages / eeb_kv_reserve / eeb_kv_release,
SURVEY §8f rank 4) on the GPU.

A paged model and an unpaged model with the same descriptor (same seed, so
the same weights) are driven through the same prefill + decode schedule —
with the paged pool's pages handed out in a scrambled order and a slot
released and reused mid-run (continuous batching).  The arithmetic is the
same, only KV addresses differ, so every output must be bit-identical; the
unpaged path is itself checked against the oracle (test_gpu_parity.py).
"""
import numpy as np
import pytest

from paper_2504_10724_b200 import eeb

pytestmark = pytest.mark.gpu

TH = 0.7
# bf16, head_dim 64 (8 x 64 = 512), GQA 2 KV heads; 256 positions = 4 pages of 64
DESC = eeb.ModelDesc("paged-mini", 4, 512, 8, 2, 1024, 1000, (2, 4), dtype=eeb.BF16, max_slots=8,
                     max_seq_len=256)
DESC128 = eeb.ModelDesc("paged-hd128", 4, 1024, 8, 2, 1024, 1000, (2, 4), dtype=eeb.BF16, max_slots=8,
                        max_seq_len=256)


@pytest.fixture(scope="module")
def ctx():
    c = eeb.Context(0)
    yield c
    c.close()


def _same(a, b, exact, stats):
    """Bit-identical when both pools use the same attention kernel (head_dim 64).
    Head_dim 128 unpaged runs the pipelined kernel (another summation order, so
    bf16 roundings differ), paged the one-item kernel: the bf16 bars of
    test_gpu_parity.py apply — token agreement >= 99 % over the run, exit
    layers equal except rows within 1e-3 of th, confidences within 1e-3."""
    if exact:
        for k in ("token_id", "exit_layer", "breached", "hist", "confidence", "logprob"):
            np.testing.assert_array_equal(np.asarray(a[k]), np.asarray(b[k]), err_msg=k)
        return
    ca, cb = np.asarray(a["confidence"]), np.asarray(b["confidence"])
    np.testing.assert_allclose(ca, cb, rtol=0, atol=1e-3)
    near = np.abs(ca - TH) <= 1e-3
    assert (np.asarray(a["exit_layer"]) == np.asarray(b["exit_layer"]))[~near].all()
    stats[0] += int((np.asarray(a["token_id"]) == np.asarray(b["token_id"])).sum())
    stats[1] += len(ca)


DESC_MHA = eeb.ModelDesc("paged-mha", 4, 512, 8, 8, 1024, 1000, (2, 4), dtype=eeb.BF16, max_slots=8,
                         max_seq_len=256)


@pytest.mark.parametrize("desc", [DESC, DESC128, DESC_MHA], ids=["hd64", "hd128", "hd64-mha"])
def test_paged_equals_unpaged(ctx, desc):
    mu = ctx.register(desc)
    mp = ctx.register(desc.replace(name=desc.name + "-p"))
    for m in (mu, mp):
        ctx.load_layers(m, desc.num_layers)
    ctx.kv_configure_pages(mp, 64, 24)
    assert ctx.kv_pages(mp) == (64, 24, 24)
    # slot 7 holds the first two pages throughout, so no slot's pages start at
    # its unpaged offset; decode growth then interleaves the slots' pages
    ctx.kv_reserve(mp, 7, 128)
    rng = np.random.default_rng(5)
    slots = np.array([0, 3, 5, 6])
    lens = [70, 1, 130, 64]  # page-crossing, single token, 3 pages, exactly one page
    prompts = [rng.integers(0, desc.vocab, n) for n in lens]
    for m in (mu, mp):
        ctx.prefill(m, desc.num_layers, slots, prompts)
    pos = np.array(lens)
    exact = desc.d_model // desc.n_heads == 64
    stats = [0, 0]
    for step in range(70):  # crosses page boundaries (64, 128, 192) for several rows
        toks = rng.integers(0, desc.vocab, len(slots))
        pol = eeb.INTROSPECTIVE if step % 3 else eeb.FULL_DEPTH
        a = ctx.decode_step(mu, 0, pol, TH, slots, toks, pos)
        b = ctx.decode_step(mp, 0, pol, TH, slots, toks, pos)
        _same(a, b, exact, stats)
        pos = pos + 1
        if step == 30:  # request in slot 3 finishes; a new one takes the slot (continuous batching)
            free_before = ctx.kv_pages(mp)[2]
            ctx.kv_release(mp, 3)
            assert ctx.kv_pages(mp)[2] == free_before + 1
            newp = [rng.integers(0, desc.vocab, 20)]
            for m in (mu, mp):
                ctx.reset_slots(m, [3])
                ctx.prefill(m, desc.num_layers, [3], newp)
            pos[1] = 20
    if not exact:
        assert stats[0] >= 0.99 * stats[1], stats
    # KV reads agree position by position (layer 1 and the last layer)
    for s, p in ((0, 5), (5, 150), (3, 10)):
        for layer in (1, desc.num_layers):
            ku, vu = ctx.read_kv(mu, layer, s, p)
            kp, vp = ctx.read_kv(mp, layer, s, p)
            np.testing.assert_allclose(ku, kp, rtol=1e-2, atol=1e-2)  # bf16 K/V (exact for head_dim 64)
            np.testing.assert_allclose(vu, vp, rtol=1e-2, atol=1e-2)


def test_paged_capacity_and_release(ctx):
    m = ctx.register(DESC.replace(name="paged-cap"))
    ctx.load_layers(m, DESC.num_layers)
    ctx.kv_configure_pages(m, 64, 3)
    ctx.kv_reserve(m, 0, 128)  # 2 pages
    ctx.kv_reserve(m, 1, 64)   # 1 page
    assert ctx.kv_pages(m)[2] == 0
    with pytest.raises(eeb.EebError) as e:
        ctx.decode_step(m, 0, eeb.FULL_DEPTH, TH, [2], [1], [0])  # slot 2 needs a page
    assert e.value.kind == "CapacityError"
    ctx.kv_release(m, 0)
    assert ctx.kv_pages(m)[2] == 2
    r = ctx.decode_step(m, 0, eeb.FULL_DEPTH, TH, [2], [1], [0])
    assert r["exit_layer"][0] == DESC.num_layers
    with pytest.raises(eeb.EebError):
        ctx.kv_configure_pages(m, 48, 3)  # not a multiple of 64
