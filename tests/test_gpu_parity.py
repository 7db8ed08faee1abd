"""GPU parity: the sm_100a decode step (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north star):
  * f32 model: logits within 1e-3 relative (|gpu - ref| <= 1e-3 * max|ref| per row),
    token ids equal, exit layers equal except rows whose confidence lies
    within 1e-4 of the threshold;
  * bf16 model: token agreement >= 99 %;
  * integer outputs (histogram, breach count, exit layers) bit-exact
    wherever the per-row decisions agree.
"""
import numpy as np
import pytest

from oracle.oracle import OracleModel
from paper_2504_10724_b200 import eeb

pytestmark = pytest.mark.gpu

TH = 0.7
LOGIT_RTOL = 1e-3      # north star: fp32 logits within 1e-3 relative
CONF_BAND = 1e-4       # exit mismatches allowed only within 1e-4 of th
BF16_AGREE = 0.99      # bf16 token agreement


MINI = eeb.ModelDesc("mini-gqa", 6, 512, 8, 2, 1024, 1000, (2, 4, 6), dtype=eeb.F32,
                     mlp_kind=eeb.MLP_SWIGLU, max_slots=16, max_seq_len=64, seed=99)


@pytest.fixture(scope="module")
def ctx():
    c = eeb.Context(0)
    yield c
    c.close()


def _pair(ctx, desc, depth=None):
    m = ctx.register(desc)
    ctx.load_layers(m, depth or desc.num_layers)
    ref = OracleModel(desc)
    ref.load(depth or desc.num_layers)
    return m, ref


def _compare_rows(g, r, th, strict_tokens=True):
    near = np.abs(r["confidence"] - th) <= CONF_BAND
    ok_exit = (g["exit_layer"] == r["exit_layer"]) | near
    assert ok_exit.all(), (g["exit_layer"], r["exit_layer"], r["confidence"])
    same = g["exit_layer"] == r["exit_layer"]
    if strict_tokens:
        assert (g["token_id"][same] == r["token_id"][same]).all()
        np.testing.assert_allclose(g["confidence"][same], r["confidence"][same], atol=2e-4, rtol=2e-3)
        np.testing.assert_allclose(g["logprob"][same], r["logprob"][same], atol=2e-3, rtol=2e-3)
    return same


def _logit_check(glog, rlog):
    for row_g, row_r in zip(glog, rlog):
        if np.isnan(row_r).any():
            continue
        scale = np.max(np.abs(row_r))
        err = np.max(np.abs(row_g - row_r))
        assert err <= LOGIT_RTOL * scale, (err, scale)


@pytest.mark.parametrize("desc", [eeb.PRESETS["tiny"], MINI], ids=["tiny", "mini-gqa-swiglu"])
def test_weights_bit_exact(ctx, desc):
    m, ref = _pair(ctx, desc)
    rng = np.random.default_rng(1)
    D = desc.d_model
    for tensor, layer, n in [(1, 1, (desc.n_heads + 2 * desc.n_kv_heads) * desc.head_dim * D),
                             (2, 2, D * D), (4, desc.num_layers, D * desc.d_ffn), (5, 1, D * desc.d_ffn),
                             (0, 3, D), (100, 0, desc.vocab * D), (200, 0, desc.vocab * D),
                             (201, 0, desc.vocab * D), (300, 0, D)]:
        idx = np.sort(rng.choice(n, size=min(n, 64), replace=False))
        for i in idx:
            gv = ctx.read_weight(m, tensor, layer, int(i), 1)[0]
            rv = ref.weight(tensor, layer, int(i))
            assert gv == rv or (np.isnan(gv) and np.isnan(rv)), (tensor, layer, i, gv, rv)


@pytest.mark.parametrize("desc", [eeb.PRESETS["tiny"], MINI], ids=["tiny", "mini-gqa-swiglu"])
def test_f32_step_parity_all_policies(ctx, desc):
    """Prefill 6 positions through profile steps, then every policy at 3 more."""
    m, ref = _pair(ctx, desc)
    ctx.retain_logits(True)
    rng = np.random.default_rng(3)
    B = 8
    slots = np.arange(B)
    L = desc.num_layers
    for pos in range(9):
        toks = rng.integers(0, desc.vocab, B)
        policy = eeb.PROFILE if pos < 6 else [eeb.INTROSPECTIVE, eeb.FLAT, eeb.FULL_DEPTH][pos - 6]
        depth = desc.exit_layers[0] if policy == eeb.FLAT else 0
        g = ctx.decode_step(m, depth, policy, TH, slots, toks, np.full(B, pos))
        r = ref.decode_step(depth, policy, TH, slots, toks, np.full(B, pos), want_logits=True)
        same = _compare_rows(g, r, TH)
        if same.all():
            assert (g["hist"] == r["hist"]).all()
            assert g["n_breached"][0] == r["n_breached"][0]
            assert (g["breached"] == r["breached"]).all()
            assert (g["unchanged"] == r["unchanged"]).all()
        if policy == eeb.PROFILE:
            np.testing.assert_array_equal(g["head_token"], r["head_token"])
            np.testing.assert_allclose(g["head_confidence"], r["head_confidence"], atol=2e-4, rtol=2e-3)
        # logits of every head that ran on every row (profile) / the final head (full depth)
        heads = range(len(desc.exit_layers)) if policy == eeb.PROFILE else (
            [len(desc.exit_layers) - 1] if policy == eeb.FULL_DEPTH else [])
        for e in heads:
            _logit_check(ctx.last_logits(e, B, desc.vocab), r["logits"][e])
        # KV written at this position matches (layer 1 and the deepest computed layer)
        for layer in (1, L if policy != eeb.FLAT else depth):
            for b in (0, B - 1):
                if policy == eeb.INTROSPECTIVE and g["exit_layer"][b] < layer:
                    continue
                gk, gv = ctx.read_kv(m, layer, int(slots[b]), pos)
                rk, rv = ref.read_kv(layer, int(slots[b]), pos)
                where = f"pos {pos} policy {policy} layer {layer} row {b}"
                np.testing.assert_allclose(gk, rk, atol=1e-4, rtol=1e-3, err_msg="K " + where)
                np.testing.assert_allclose(gv, rv, atol=1e-4, rtol=1e-3, err_msg="V " + where)
    ctx.retain_logits(False)


def test_introspective_compaction_and_masking(ctx):
    """Rows exit at different heads; survivors are compacted; later steps attend
    over positions whose deeper KV is missing (masked) exactly like the oracle."""
    desc = eeb.PRESETS["tiny"]
    m, ref = _pair(ctx, desc)
    rng = np.random.default_rng(11)
    B = 8
    slots = np.arange(B)
    exits = []
    for pos in range(10):
        toks = rng.integers(0, desc.vocab, B)
        g = ctx.decode_step(m, 0, eeb.INTROSPECTIVE, TH, slots, toks, np.full(B, pos))
        r = ref.decode_step(0, eeb.INTROSPECTIVE, TH, slots, toks, np.full(B, pos))
        _compare_rows(g, r, TH)
        exits.append(g["exit_layer"].copy())
        np.testing.assert_array_equal(g["hist"], np.bincount(
            [desc.exit_layers.index(x) for x in g["exit_layer"]], minlength=len(desc.exit_layers)))
    exits = np.concatenate(exits)
    assert len(set(exits.tolist())) == 2, "both heads must see exits for the test to mean anything"


MINI128 = eeb.ModelDesc("mini-hd128", 4, 1024, 8, 2, 1024, 1000, (2, 4), dtype=eeb.BF16,
                        mlp_kind=eeb.MLP_SWIGLU, max_slots=16, max_seq_len=320, seed=7)


# MHA (one query head per kv head, head_dim 64): the OPT shapes' CUDA-core
# decode attention (attention_mha_kernel); 300 positions = ten 32-position chunks
MINI_MHA = eeb.ModelDesc("mini-mha", 4, 512, 8, 8, 1024, 1000, (2, 4), dtype=eeb.BF16,
                         max_slots=16, max_seq_len=320, seed=13)
MINI_MHA128 = eeb.ModelDesc("mini-mha128", 4, 1024, 8, 8, 1024, 1000, (2, 4), dtype=eeb.BF16,
                            max_slots=16, max_seq_len=320, seed=17)
MINI_MHA80 = eeb.ModelDesc("mini-mha80", 4, 1280, 16, 16, 1024, 1000, (2, 4), dtype=eeb.BF16,
                           max_slots=16, max_seq_len=320, seed=19)


@pytest.mark.parametrize("desc,npos", [(MINI.replace(dtype=eeb.BF16, name="mini-bf16"), 8), (MINI128, 300),
                                       (MINI_MHA, 300), (MINI_MHA128, 300), (MINI_MHA80, 300)],
                         ids=["hd64-gqa4", "hd128-gqa4-2chunks", "hd64-mha-10chunks", "hd128-mha", "hd80-mha"])
def test_bf16_token_agreement(ctx, desc, npos):
    """bf16 tensor-core path (mma.sync flash-decode attention, tcgen05 GEMMs at
    B=16) against the oracle; npos=300 crosses the 128-position attention chunk."""
    m, ref = _pair(ctx, desc)
    rng = np.random.default_rng(5)
    B = 16
    slots = np.arange(B)
    agree = total = 0
    conf_err = 0.0
    for pos in range(npos):
        if npos > 8 and pos not in (0, 1, 127, 128, 129, 255, 256, 299) and pos % 37:
            # fast-forward: both sides must still write the KV of every position
            toks = rng.integers(0, desc.vocab, B)
            ctx.decode_step(m, 0, eeb.FULL_DEPTH, TH, slots, toks, np.full(B, pos))
            ref.decode_step(0, eeb.FULL_DEPTH, TH, slots, toks, np.full(B, pos))
            continue
        toks = rng.integers(0, desc.vocab, B)
        g = ctx.decode_step(m, 0, eeb.PROFILE, TH, slots, toks, np.full(B, pos))
        r = ref.decode_step(0, eeb.PROFILE, TH, slots, toks, np.full(B, pos))
        agree += int((g["head_token"] == r["head_token"]).sum())
        total += g["head_token"].size
        conf_err = max(conf_err, float(np.abs(g["head_confidence"] - r["head_confidence"]).max()))
    assert agree / total >= BF16_AGREE, agree / total
    assert conf_err < 0.05, conf_err


def test_bf16_large_batch_two_row_blocks(ctx):
    """200 rows: every GEMM (layer, fused up + activation, exit head) runs two
    128-row CTAs per weight tile (the second block ragged, 72 rows) — against
    the oracle for PROFILE (every head) and INTROSPECTIVE (compaction) steps."""
    desc = MINI_MHA.replace(name="mini-mha-b200", max_slots=200, max_seq_len=64)
    m, ref = _pair(ctx, desc)
    rng = np.random.default_rng(23)
    B = 200
    slots = np.arange(B)
    agree = total = 0
    for pos in range(6):
        toks = rng.integers(0, desc.vocab, B)
        policy = eeb.PROFILE if pos % 2 == 0 else eeb.INTROSPECTIVE
        g = ctx.decode_step(m, 0, policy, TH, slots, toks, np.full(B, pos))
        r = ref.decode_step(0, policy, TH, slots, toks, np.full(B, pos))
        if policy == eeb.PROFILE:
            agree += int((g["head_token"] == r["head_token"]).sum())
            total += g["head_token"].size
            assert np.abs(g["head_confidence"] - r["head_confidence"]).max() < 0.05
        else:
            same = g["exit_layer"] == r["exit_layer"]
            assert same.mean() >= 0.97, same.mean()
            agree += int((g["token_id"][same] == r["token_id"][same]).sum())
            total += int(same.sum())
    assert agree / total >= BF16_AGREE, agree / total


def test_graph_replay_matches_eager(ctx):
    desc = eeb.PRESETS["tiny"].replace(dtype=eeb.BF16, name="tiny-bf16")
    m = ctx.register(desc)
    ctx.load_layers(m, desc.num_layers)
    rng = np.random.default_rng(9)
    B = 4
    toks = [rng.integers(0, desc.vocab, B) for _ in range(4)]
    outs = {}
    for graphs in (False, True):
        ctx.set_graphs(graphs)
        ctx.reset_slots(m, np.arange(B))
        res = []
        for pos in range(4):
            res.append(ctx.decode_step(m, 0, eeb.INTROSPECTIVE, TH, np.arange(B), toks[pos], np.full(B, pos)))
        outs[graphs] = res
    ctx.set_graphs(True)
    for a, b in zip(outs[False], outs[True]):
        for k in ("exit_layer", "token_id", "confidence", "hist"):
            np.testing.assert_array_equal(a[k], b[k])


def test_error_codes(ctx):
    desc = eeb.PRESETS["tiny"]
    m = ctx.register(desc)
    ctx.load_layers(m, 6)
    one = np.zeros(1, np.int32)
    with pytest.raises(eeb.EebError) as e:  # full depth needs all layers resident
        ctx.decode_step(m, 0, eeb.PROFILE, TH, one, one, one)
    assert e.value.kind == "CapacityError"
    with pytest.raises(eeb.EebError) as e:  # observation_for_depth below every head
        ctx.decode_step(m, 3, eeb.FLAT, TH, one, one, one)
    assert e.value.kind == "DomainError"
    g = ctx.decode_step(m, 6, eeb.FLAT, TH, one, one, one)
    assert g["exit_layer"][0] == 6
    with pytest.raises(eeb.EebError) as e:
        ctx.decode_step(m, 6, eeb.FLAT, TH, np.array([0, 0], np.int32), np.array([1, 2], np.int32),
                        np.zeros(2, np.int32))
    assert e.value.kind == "ValidationError"
    bad = eeb.PRESETS["tiny"].replace(exit_layers=(6, 11))
    with pytest.raises(eeb.EebError) as e:  # last exit must equal num_layers (model_spec.hpp:73-74)
        ctx.register(bad)
    assert e.value.kind == "ValidationError"


def test_opt13b_shape_bf16_agreement(ctx):
    """C2 shape (OPT-1.3B dims, exits 6/12/18/24) at a small batch: bf16 GPU vs oracle."""
    desc = eeb.PRESETS["opt-1.3b-4x"].replace(max_slots=8, max_seq_len=16)
    m, ref = _pair(ctx, desc)
    rng = np.random.default_rng(13)
    B = 4
    slots = np.arange(B)
    agree = total = 0
    for pos in range(2):
        toks = rng.integers(0, desc.vocab, B)
        g = ctx.decode_step(m, 0, eeb.PROFILE, TH, slots, toks, np.full(B, pos))
        r = ref.decode_step(0, eeb.PROFILE, TH, slots, toks, np.full(B, pos))
        agree += int((g["head_token"] == r["head_token"]).sum())
        total += g["head_token"].size
        near = np.abs(r["confidence"] - TH) <= 1e-2
        assert ((g["exit_layer"] == r["exit_layer"]) | near).all()
    assert agree / total >= BF16_AGREE


def test_all_rows_exit_early_bf16(ctx):
    """Every row exits at the first head (th = 0): the deeper layers' tcgen05
    GEMMs see no live row and stream no weights; the steps that follow (th
    0.7, rows reaching deeper layers whose older positions have no KV there)
    must still agree with the oracle at the bf16 bar."""
    desc = MINI.replace(dtype=eeb.BF16, name="mini-bf16-allexit")
    m, ref = _pair(ctx, desc)
    rng = np.random.default_rng(9)
    B = 8
    slots = np.arange(B)
    agree = total = 0
    for pos in range(12):
        th = 0.0 if pos % 3 != 2 else TH
        toks = rng.integers(0, desc.vocab, B)
        g = ctx.decode_step(m, 0, eeb.INTROSPECTIVE, th, slots, toks, np.full(B, pos))
        r = ref.decode_step(0, eeb.INTROSPECTIVE, th, slots, toks, np.full(B, pos))
        if th == 0.0:
            assert (g["exit_layer"] == desc.exit_layers[0]).all()
        near = np.abs(r["confidence"] - th) <= 1e-3
        assert ((g["exit_layer"] == r["exit_layer"]) | near).all(), (g["exit_layer"], r["exit_layer"])
        agree += int((g["token_id"] == r["token_id"]).sum())
        total += B
    assert agree / total >= BF16_AGREE, agree / total


@pytest.mark.parametrize("B", [1, 2])
def test_conditional_skip_small_batch(ctx, B):
    """Batches of <= 2 rows capture the layers after each non-final head as a
    conditional graph body that decide switches off when no row survives.
    Graph replay must equal eager launches (same kernels, all rows exited or
    not) and the oracle at the bf16 bar, over steps of both kinds."""
    desc = MINI.replace(dtype=eeb.BF16, name=f"mini-bf16-cond{B}")
    mg, ref = _pair(ctx, desc)
    me = ctx.register(desc.replace(name=f"mini-bf16-cond{B}-eager"))
    ctx.load_layers(me, desc.num_layers)
    rng = np.random.default_rng(21 + B)
    slots = np.arange(B)
    exits = set()
    agree = total = 0
    for pos in range(24):
        toks = rng.integers(0, desc.vocab, B)
        ctx.set_graphs(True)
        g = ctx.decode_step(mg, 0, eeb.INTROSPECTIVE, TH, slots, toks, np.full(B, pos))
        ctx.set_graphs(False)
        e = ctx.decode_step(me, 0, eeb.INTROSPECTIVE, TH, slots, toks, np.full(B, pos))
        ctx.set_graphs(True)
        r = ref.decode_step(0, eeb.INTROSPECTIVE, TH, slots, toks, np.full(B, pos))
        for k in ("token_id", "exit_layer", "confidence", "hist"):
            np.testing.assert_array_equal(np.asarray(g[k]), np.asarray(e[k]), err_msg=k)
        near = np.abs(r["confidence"] - TH) <= 1e-3
        assert ((g["exit_layer"] == r["exit_layer"]) | near).all()
        agree += int((g["token_id"] == r["token_id"]).sum())
        total += B
        exits.add(int(max(g["exit_layer"])))
    assert agree / total >= BF16_AGREE, agree / total
    assert len(exits) >= 2, exits  # both skipped and full steps were exercised


@pytest.mark.parametrize("dtype", [eeb.F32, eeb.BF16], ids=["f32", "bf16"])
def test_head_dim_80(ctx, dtype):
    """OPT-2.7B's head geometry (2560 = 32 heads x 80): the generic attention
    kernel (P.V thread groups that do not divide the CTA) against the oracle,
    prefill then decode."""
    desc = eeb.ModelDesc("mini-hd80", 4, 1280, 16, 16, 1024, 1000, (2, 4), dtype=dtype, max_slots=4,
                         max_seq_len=96)
    m, ref = _pair(ctx, desc)
    rng = np.random.default_rng(80)
    slots = np.arange(4)
    prompts = [rng.integers(0, desc.vocab, n) for n in (20, 7, 33, 1)]
    ctx.prefill(m, desc.num_layers, slots, prompts)
    for i, p in enumerate(prompts):
        for k, t in enumerate(p):
            ref.decode_step(0, eeb.FULL_DEPTH, TH, [slots[i]], [t], [k])
    pos = np.array([len(p) for p in prompts])
    agree = total = 0
    for step in range(6):
        toks = rng.integers(0, desc.vocab, 4)
        g = ctx.decode_step(m, 0, eeb.INTROSPECTIVE, TH, slots, toks, pos + step)
        r = ref.decode_step(0, eeb.INTROSPECTIVE, TH, slots, toks, pos + step)
        if dtype == eeb.F32:
            _compare_rows(g, r, TH)
        agree += int((g["token_id"] == r["token_id"]).sum())
        total += 4
    assert agree / total >= BF16_AGREE, agree / total


def test_bf16_gqa_large_batch_staging():
    """34B-style GQA (8 query heads per kv head, head_dim 128) at 256 rows:
    1024 (row, kv head) items, 7 per CTA — the streaming decode attention's
    per-CTA prologue staging no longer fits beside 3-deep rings, so it runs
    2-deep rings (the C4 batch-256 configuration); d_ffn 8192 puts the down
    projection (K = 8192) on the long-K one-tile-per-weight-tile GEMM path —
    against the oracle."""
    desc = eeb.ModelDesc("mini-gqa8-b256", 2, 4096, 32, 4, 8192, 1000, (1, 2), dtype=eeb.BF16,
                         mlp_kind=eeb.MLP_SWIGLU, max_slots=256, max_seq_len=64, seed=29)
    c = eeb.Context(0)
    try:
        m, ref = _pair(c, desc)
        rng = np.random.default_rng(31)
        B = 256
        slots = np.arange(B)
        agree = total = 0
        for pos in range(3):
            toks = rng.integers(0, desc.vocab, B)
            g = c.decode_step(m, 0, eeb.PROFILE, TH, slots, toks, np.full(B, pos))
            r = ref.decode_step(0, eeb.PROFILE, TH, slots, toks, np.full(B, pos))
            agree += int((g["head_token"] == r["head_token"]).sum())
            total += g["head_token"].size
            assert np.abs(g["head_confidence"] - r["head_confidence"]).max() < 0.05
        assert agree / total >= BF16_AGREE, agree / total
    finally:
        c.close()
