"""GPU parity of the persistent decode-step kernel (eeb_set_gemm_tier(ctx, 3),
csrc/step_mk.cu) against the CPU oracle, every token policy, MHA/ReLU and
GQA/SwiGLU configurations, introspective compaction over several steps.

Bars as in test_gpu_parity.py (bf16 model): token agreement >= 99 %, exit
layers equal except rows whose oracle confidence is within the bf16 band of
th, histogram / breach count consistent with the per-row outputs."""
import numpy as np
import pytest

from oracle.oracle import OracleModel
from paper_2504_10724_b200 import eeb

pytestmark = pytest.mark.gpu

TH = 0.7
BF16_AGREE = 0.99
BAND = 1e-2  # bf16 confidences near th may flip the exit decision

MHA = eeb.ModelDesc("mk-mha-relu", 4, 512, 8, 8, 1024, 1000, (2, 4), dtype=eeb.BF16, max_slots=64,
                    max_seq_len=64, seed=5)
GQA = eeb.ModelDesc("mk-gqa-swiglu", 4, 512, 8, 2, 1024, 1000, (1, 2, 4), dtype=eeb.BF16,
                    mlp_kind=eeb.MLP_SWIGLU, max_slots=64, max_seq_len=64, seed=6)


@pytest.fixture(scope="module")
def ctx():
    c = eeb.Context(0)
    c.set_gemm_tier(3)
    yield c
    c.close()


def _check(g, r, desc):
    near = np.abs(r["confidence"] - TH) <= BAND
    assert ((g["exit_layer"] == r["exit_layer"]) | near).all(), (g["exit_layer"], r["exit_layer"])
    same = g["exit_layer"] == r["exit_layer"]
    agree = (g["token_id"][same] == r["token_id"][same]).mean() if same.any() else 1.0
    assert g["hist"].sum() == len(g["token_id"])
    assert g["n_breached"][0] == g["breached"].sum()
    assert g["sum_logprob"][0] == pytest.approx(float(g["logprob"].astype(np.float64).sum()), rel=1e-6)
    return agree


@pytest.mark.parametrize("desc", [MHA, GQA], ids=["mha-relu", "gqa-swiglu"])
@pytest.mark.parametrize("B", [16, 64])
def test_persistent_kernel_matches_oracle(ctx, desc, B):
    m = ctx.register(desc)
    ctx.load_layers(m, desc.num_layers)
    ref = OracleModel(desc)
    ref.load(desc.num_layers)
    rng = np.random.default_rng(B)
    slots = np.arange(B)
    agrees = []
    for pos in range(6):
        toks = rng.integers(0, desc.vocab, B)
        g = ctx.decode_step(m, 0, eeb.PROFILE, TH, slots, toks, np.full(B, pos))
        r = ref.decode_step(0, eeb.PROFILE, TH, slots, toks, np.full(B, pos))
        agrees.append((g["head_token"] == r["head_token"]).mean())
        _check(g, r, desc)
    for pos, (pol, depth) in enumerate([(eeb.INTROSPECTIVE, 0), (eeb.FULL_DEPTH, 0), (eeb.FLAT, 2),
                                        (eeb.INTROSPECTIVE, 0)], start=6):
        toks = rng.integers(0, desc.vocab, B)
        g = ctx.decode_step(m, depth, pol, TH, slots, toks, np.full(B, pos))
        r = ref.decode_step(depth, pol, TH, slots, toks, np.full(B, pos))
        agrees.append(_check(g, r, desc))
        if pol == eeb.FLAT:
            assert (g["exit_layer"] == depth).all()
        if pol == eeb.FULL_DEPTH:
            assert (g["exit_layer"] == desc.num_layers).all() and not g["breached"].any()
    assert np.mean(agrees) >= BF16_AGREE, agrees


def test_persistent_kernel_is_deterministic(ctx):
    desc = MHA.replace(name="mk-det")
    B = 32
    outs = []
    for _ in range(2):
        m = ctx.register(desc)
        ctx.load_layers(m, desc.num_layers)
        rng = np.random.default_rng(4)
        res = []
        for pos in range(4):
            res.append(ctx.decode_step(m, 0, eeb.INTROSPECTIVE, TH, np.arange(B), rng.integers(0, desc.vocab, B),
                                       np.full(B, pos)))
        outs.append(res)
    for a, b in zip(*outs):
        for k in ("exit_layer", "token_id", "confidence", "logprob", "hist"):
            np.testing.assert_array_equal(a[k], b[k])


def test_persistent_kernel_refuses_unsupported(ctx):
    desc = eeb.PRESETS["tiny"]  # f32 parity model: not on the persistent path
    m = ctx.register(desc)
    ctx.load_layers(m, desc.num_layers)
    one = np.zeros(1, np.int32)
    with pytest.raises(eeb.EebError) as e:
        ctx.decode_step(m, 0, eeb.PROFILE, TH, one, one, one)
    assert e.value.kind == "DomainError"
