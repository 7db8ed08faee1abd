"""CPU checks of the oracle (oracle/eeb_oracle.c) — the checker every GPU
parity test trusts, so it is pinned here first:

* its decision layer against the reference's own KATs (test_trace.cpp:39-63,
  SPEC.md:159-161) and against vectors produced by the compiled reference
  (tests/golden/decision_vectors.json, tools/make_golden.py);
* its tensor arithmetic against a second, independent restatement in numpy
  (the reference computes no logits, so this is a cross-check, not a pin —
  DESIGN.md "parity unpinned" for logits);
* the internal consistency of its policies (the introspective / flat / full
  decisions equal the reference rule applied to the all-heads profile record);
* the biased exit heads: the exit distribution tracks the stated coverage.
"""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import OracleModel, decide
from paper_2504_10724_b200 import eeb

GOLDEN = Path(__file__).resolve().parent / "golden" / "decision_vectors.json"
FLAT, INTRO, FULL, PROF = eeb.FLAT, eeb.INTROSPECTIVE, eeb.FULL_DEPTH, eeb.PROFILE


# ---------------------------------------------------------------------------
# decision layer
# ---------------------------------------------------------------------------
def test_exit_rule_reference_kats():
    # test_trace.cpp:39-47: confidences (0.2, 0.6, 0.97) at heads 6/12/24
    layers, toks, confs = [6, 12, 24], [1, 2, 3], [0.2, 0.6, 0.97]
    assert decide(INTRO, layers, toks, confs, 0.5)[1] == 12
    assert decide(INTRO, layers, toks, confs, 0.7)[1] == 24
    assert decide(INTRO, layers, toks, confs, 0.1)[1] == 6
    assert decide(INTRO, layers, toks, confs, 0.99)[1] == 24  # forced exit at the final head
    i, _, _, _ = decide(INTRO, layers, toks, confs, 0.5)
    assert toks[i] == 2
    # test_trace.cpp:53-63: observation_for_depth falls back to the deepest head below
    layers, toks, confs = [6, 12, 24], [4, 7, 9], [0.3, 0.8, 0.99]
    assert toks[decide(FLAT, layers, toks, confs, 0.5, depth=12)[0]] == 7
    assert layers[decide(FLAT, layers, toks, confs, 0.5, depth=17)[0]] == 12
    assert layers[decide(FLAT, layers, toks, confs, 0.5, depth=30)[0]] == 24
    with pytest.raises(ValueError):
        decide(FLAT, layers, toks, confs, 0.5, depth=3)  # DomainError in the reference


def test_flags_follow_engine_semantics():
    layers, toks, confs = [6, 12, 24], [5, 5, 9], [0.4, 0.7, 0.9]
    # introspective: >= is an exit (trace.hpp:74), breached is strict < (engine.hpp:358)
    assert decide(INTRO, layers, toks, confs, 0.7) == (1, 12, False, False)
    assert decide(INTRO, layers, toks, confs, 0.95) == (2, 24, True, True)  # forced, breached
    # flat: exit = depth, breached on the head's confidence (engine.hpp:350-354)
    assert decide(FLAT, layers, toks, confs, 0.5, depth=6) == (0, 6, True, False)
    # full depth never breaches (engine.hpp:360-364)
    assert decide(FULL, layers, toks, confs, 0.95, num_layers=24) == (2, 24, False, True)


def test_exit_rules_match_compiled_reference_vectors():
    g = json.loads(GOLDEN.read_text())
    assert len(g["exit_rules"]) >= 400
    for r in g["exit_rules"]:
        L, T, Cf, th = r["layers"], r["tokens"], r["confidences"], r["th"]
        i, layer, _, _ = decide(INTRO, L, T, Cf, th)
        assert [layer, T[i]] == r["introspective"], r
        for depth, want in r["flat"].items():
            if want == "DomainError":
                with pytest.raises(ValueError):
                    decide(FLAT, L, T, Cf, th, depth=int(depth))
            else:
                i, layer, _, _ = decide(FLAT, L, T, Cf, th, depth=int(depth))
                assert [L[i], T[i]] == want and layer == int(depth), (r, depth)


def test_exit_rules_match_live_reference_randomized():
    from oracle.oracle import REF_LIB

    if not REF_LIB.exists():
        pytest.skip("compiled reference absent (built only where /root/reference exists)")
    import ctypes as C

    L = C.CDLL(str(REF_LIB))
    i32p, f64p = C.POINTER(C.c_int), C.POINTER(C.c_double)
    L.ref_earliest_confident.argtypes = [C.c_int, i32p, i32p, f64p, f64p, C.c_double, i32p]
    rng = np.random.default_rng(5)
    for _ in range(3000):
        n = int(rng.integers(1, 8))
        layers = np.cumsum(rng.integers(1, 6, n)).astype(np.int32)
        toks = rng.integers(0, 4, n).astype(np.int32)
        confs = rng.choice(np.float32([0.1, 0.25, 0.5, 0.7, 0.7000001, 0.9, 1.0]), n)
        th = float(rng.choice(np.float32([0.0, 0.25, 0.5, 0.7, 0.9, 1.0])))
        t = C.c_int()
        want = L.ref_earliest_confident(n, (C.c_int * n)(*layers), (C.c_int * n)(*toks),
                                        (C.c_double * n)(*confs.astype(np.float64)), (C.c_double * n)(*([0.0] * n)),
                                        th, C.byref(t))
        i, layer, _, _ = decide(INTRO, layers, toks, confs, th)
        assert (layer, int(toks[i])) == (want, t.value)


# ---------------------------------------------------------------------------
# tensor arithmetic: an independent numpy restatement of the synthetic model
# ---------------------------------------------------------------------------
M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _fin64(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _draw(seed, tid, idx):
    with np.errstate(over="ignore"):
        h = _fin64(np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15) * np.uint64(tid + 1))
        h = _fin64(h ^ (np.asarray(idx, np.uint64) * np.uint64(0xD1B54A32D192ED03) + np.uint64(0x632BE59BD9B4E019)))
    return (h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24) - np.float32(0.5)


class NumpyModel:
    """Second restatement of DESIGN.md §3 (weights) and §4 (the step), f64 math."""

    U, SIG, A, B, BETA, JIT, LV = np.float32(3.46410161513775), np.float32(0.02), np.float32(0.25), \
        np.float32(1.0), np.float32(0.02), np.float32(0.1), 2e-3

    def __init__(self, d):
        assert d.dtype == eeb.F32
        self.d = d
        D, F, V = d.d_model, d.d_ffn, d.vocab
        self.hd = d.head_dim
        unit = lambda tid, n: _draw(d.seed, tid, np.arange(n, dtype=np.uint64)) * self.U
        gain = lambda tid: np.float32(1.0) + _draw(d.seed, tid, np.arange(D, dtype=np.uint64)) * np.float32(0.2)
        var_h = float(D) * float(self.SIG) * float(self.SIG) / 2.0
        rsig = np.float32(np.sqrt(self.LV / (F * var_h)))

        def lin(tid, rows, cols, scale, zero_sig):
            w = (unit(tid, rows * cols) * np.float32(scale)).reshape(rows, cols)
            if zero_sig:
                w[: D // 2] = 0
            return w

        z = _draw(d.seed, 8192 + 64, np.arange(V, dtype=np.uint64)) + np.float32(0.5)
        G = unit(8192, V * D).reshape(V, D)
        amp = np.concatenate([np.repeat((self.A * (np.float32(1) - z))[:, None], D // 2, 1),
                              np.full((V, D - D // 2), self.B, np.float32)], 1)
        self.emb = G * amp
        th = float(np.float32(d.design_th))
        C0 = np.log(V - 1.0) + float(self.BETA) ** 2 * D / 2.0 + np.log(th / (1.0 - th))
        k = 1.0 - np.sqrt(max(1.0 - 4.0 * C0 / D, 0.05))
        pmul = next(p for p in range(7919, 10 ** 6) if np.gcd(p, V) == 1)
        src = (np.arange(V, dtype=np.uint64) * np.uint64(pmul) + np.uint64(17)) % np.uint64(V)
        self.heads, self.head_norms = [], []
        for e, (layer, c) in enumerate(zip(d.exit_layers, d.coverage())):
            c = min(max(float(np.float32(c)), 0.01), 0.99)
            a_star = float(self.A) * (1.0 - c)
            rms = np.sqrt((a_star ** 2 + float(self.B) ** 2 + self.LV * layer) / 2.0)
            alpha = np.float32(k * rms / a_star)
            h = unit(8192 + 2 * 64 + e, V * D).reshape(V, D) * self.BETA
            h[:, : D // 2] += G[src.astype(np.int64), : D // 2] * alpha
            self.heads.append(h)
            self.head_norms.append(gain(8192 + 3 * 64 + e))
        hd, dq, dkv = self.hd, d.n_heads * self.hd, d.n_kv_heads * self.hd
        up = 2 * F if d.mlp_kind == eeb.MLP_SWIGLU else F
        self.layers = []
        for l in range(1, d.num_layers + 1):
            t = lambda kind: l * 16 + kind
            self.layers.append(dict(an=gain(t(0)), mn=gain(t(3)), wqkv=lin(t(1), dq + 2 * dkv, D, self.SIG, False),
                                    wo=lin(t(2), D, dq, rsig, True), wup=lin(t(4), up, D, self.SIG, False),
                                    wdown=lin(t(5), D, F, rsig, True)))
        half = hd // 2
        inv = float(d.rope_theta) ** (-2.0 * np.arange(half) / hd)
        ang = np.arange(d.max_seq_len)[:, None] * inv[None, :]
        self.cos, self.sin = np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)
        self.kv = {}  # (layer, slot, pos) -> (k, v)
        self.depth = {}  # (slot, pos) -> layers computed

    def _norm(self, x, g):
        inv = np.float32(1.0 / np.sqrt(np.dot(x.astype(np.float64), x) / len(x) + float(np.float32(self.d.norm_eps))))
        return x * inv * g

    def _rope(self, v, pos):
        h = len(v) // 2
        c, s = self.cos[pos], self.sin[pos]
        return np.concatenate([v[:h] * c - v[h:] * s, v[:h] * s + v[h:] * c]).astype(np.float32)

    def logits_all_heads(self, slot, tok, pos):
        """Full-depth pass of one row (teacher forced); returns {exit layer: logits}."""
        d, hd = self.d, self.hd
        H, Hkv = d.n_heads, d.n_kv_heads
        dq, dkv = H * hd, Hkv * hd
        x = self.emb[tok].copy()
        out = {}
        for l, W in enumerate(self.layers, 1):
            qkv = (W["wqkv"].astype(np.float64) @ self._norm(x, W["an"]).astype(np.float64)).astype(np.float32)
            att = np.zeros(dq, np.float32)
            for g in range(Hkv):
                k = self._rope(qkv[dq + g * hd: dq + (g + 1) * hd], pos)
                v = qkv[dq + dkv + g * hd: dq + dkv + (g + 1) * hd]
                self.kv[(l, slot, pos, g)] = (k, v)
                ps = [p for p in range(pos + 1) if p == pos or self.depth.get((slot, p), 0) >= l]
                K = np.stack([self.kv[(l, slot, p, g)][0] for p in ps]).astype(np.float64)
                Vv = np.stack([self.kv[(l, slot, p, g)][1] for p in ps]).astype(np.float64)
                for h in range(g * H // Hkv, (g + 1) * H // Hkv):
                    q = self._rope(qkv[h * hd:(h + 1) * hd], pos).astype(np.float64)
                    s = K @ q / np.sqrt(hd)
                    p_ = np.exp(s - s.max())
                    att[h * hd:(h + 1) * hd] = (p_ @ Vv / p_.sum()).astype(np.float32)
            x = x + (W["wo"].astype(np.float64) @ att).astype(np.float32)
            u = (W["wup"].astype(np.float64) @ self._norm(x, W["mn"]).astype(np.float64)).astype(np.float32)
            if d.mlp_kind == eeb.MLP_SWIGLU:
                gt, up = u[0::2].astype(np.float64), u[1::2]
                hmid = (gt / (1 + np.exp(-gt))).astype(np.float32) * up
            else:
                hmid = np.maximum(u, 0)
            x = x + (W["wdown"].astype(np.float64) @ hmid.astype(np.float64)).astype(np.float32)
            if l in d.exit_layers:
                e = d.exit_layers.index(l)
                hn = self._norm(x, self.head_norms[e]).astype(np.float64)
                out[l] = (self.heads[e].astype(np.float64) @ hn).astype(np.float32)
        self.depth[(slot, pos)] = d.num_layers
        return out


SMALL = eeb.ModelDesc("small-cpu", 4, 256, 4, 2, 512, 384, (2, 4), dtype=eeb.F32, mlp_kind=eeb.MLP_SWIGLU,
                      max_slots=4, max_seq_len=16, seed=4242)


@pytest.mark.parametrize("desc", [SMALL, SMALL.replace(name="small-relu-mha", n_kv_heads=4, mlp_kind=eeb.MLP_RELU,
                                                       exit_layers=(1, 3, 4), seed=77)], ids=["gqa-swiglu", "mha-relu"])
def test_oracle_logits_match_independent_numpy_restatement(desc):
    orc = OracleModel(desc, threads=2)
    orc.load(desc.num_layers)
    npm = NumpyModel(desc)
    for e in range(len(desc.exit_layers)):  # weights: spot-check the head tensor bit-for-bit
        for v in (0, 1, desc.vocab - 1):
            for i in (0, desc.d_model // 2 - 1, desc.d_model // 2, desc.d_model - 1):
                assert orc.weight(200 + e, 0, v * desc.d_model + i) == npm.heads[e][v, i]
    rng = np.random.default_rng(3)
    slots = np.arange(3)
    for pos in range(4):
        toks = rng.integers(0, desc.vocab, 3)
        r = orc.decode_step(0, PROF, 0.7, slots, toks, np.full(3, pos), want_logits=True)
        for b in range(3):
            ref = npm.logits_all_heads(int(slots[b]), int(toks[b]), pos)
            for e, layer in enumerate(desc.exit_layers):
                got = r["logits"][e, b]
                scale = np.abs(ref[layer]).max()
                assert np.abs(got - ref[layer]).max() <= 1e-5 * scale, (pos, b, layer)
                assert r["head_token"][b, e] == int(np.argmax(ref[layer]))
    orc.close()


# ---------------------------------------------------------------------------
# policy consistency and calibration of the biased exit heads
# ---------------------------------------------------------------------------
def test_policies_agree_with_rule_on_profile_record():
    d = eeb.PRESETS["tiny"]
    th = 0.7
    results = {}
    for pol in (PROF, INTRO, FULL, FLAT):
        o = OracleModel(d, threads=4)
        o.load(d.num_layers)
        rng = np.random.default_rng(11)
        B = 6
        for pos in range(3):
            toks = rng.integers(0, d.vocab, B)
            depth = 6 if pol == FLAT else 0
            results[(pol, pos)] = o.decode_step(depth, pol, th, np.arange(B), toks, np.full(B, pos))
        o.close()
    # position 0 has no history: every policy sees identical hidden states at
    # the heads it evaluates, so the profile record decides all of them.
    prof = results[(PROF, 0)]
    for b in range(6):
        rec = (list(d.exit_layers), prof["head_token"][b], prof["head_confidence"][b])
        for pol in (INTRO, FULL, FLAT):
            got = results[(pol, 0)]
            i, layer, br, un = decide(pol, *rec, th, depth=6, num_layers=d.num_layers)
            assert got["exit_layer"][b] == layer
            assert got["token_id"][b] == rec[1][i]
            assert got["confidence"][b] == rec[2][i]
            assert bool(got["breached"][b]) == br
        assert prof["unchanged"][b] == (prof["token_id"][b] == prof["head_token"][b][-1])
    for pol in (PROF, INTRO, FULL, FLAT):
        r = results[(pol, 0)]
        assert r["hist"].sum() == 6 and r["n_breached"][0] == r["breached"].sum()
        assert r["sum_logprob"][0] == pytest.approx(float(np.sum(r["logprob"].astype(np.float64))))


def test_biased_exit_heads_reproduce_stated_coverage():
    d = eeb.PRESETS["tiny"].replace(max_slots=64)
    o = OracleModel(d, threads=8)
    o.load(d.num_layers)
    toks = np.arange(d.vocab)
    first = 0
    for lo in range(0, d.vocab, 64):
        t = toks[lo:lo + 64]
        r = o.decode_step(0, INTRO, d.design_th, np.arange(len(t)), t, np.zeros(len(t), np.int32))
        first += int((r["exit_layer"] == d.exit_layers[0]).sum())
    frac = first / d.vocab
    assert abs(frac - d.coverage()[0]) < 0.05, frac  # 73 % at the first head (FIXTURES.md:47-55)
    o.close()


def test_kv_import_reproduces_the_oracles_own_state():
    """orc_write_kv (the bench-config parity test seeds the oracle from the
    GPU's prefilled KV): an oracle seeded with another oracle's KV takes the
    same decode step bit for bit."""
    for desc in (eeb.PRESETS["tiny"], eeb.PRESETS["tiny"].replace(dtype=eeb.BF16, name="tiny-bf16")):
        d = desc.replace(max_slots=3, max_seq_len=16)
        a, b = OracleModel(d), OracleModel(d)
        a.load(d.num_layers)
        b.load(d.num_layers)
        rng = np.random.default_rng(5)
        slots = np.arange(3)
        for p in range(4):
            a.decode_step(0, eeb.FULL_DEPTH, 0.7, slots, rng.integers(0, d.vocab, 3), np.full(3, p))
        hd = d.n_kv_heads * d.head_dim
        for layer in range(1, d.num_layers + 1):
            for s in range(3):
                kv = [a.read_kv(layer, s, p) for p in range(4)]
                b.write_kv(layer, s, 0, np.stack([x[0] for x in kv]), np.stack([x[1] for x in kv]))
                assert np.array_equal(b.read_kv(layer, s, 2)[0], kv[2][0])
        toks = rng.integers(0, d.vocab, 3)
        for policy in (eeb.INTROSPECTIVE, eeb.PROFILE):
            ra = a.decode_step(0, policy, 0.7, slots, toks, np.full(3, 4))
            rb = b.decode_step(0, policy, 0.7, slots, toks, np.full(3, 4))
            for k in ("exit_layer", "token_id", "confidence", "logprob", "hist", "head_confidence"):
                assert np.array_equal(ra[k], rb[k]), k
        assert hd == a.read_kv(1, 0, 0)[0].size
        a.close()
        b.close()


def test_synthetic_kv_fill_is_deterministic_and_rounded():
    d = eeb.PRESETS["tiny"].replace(dtype=eeb.BF16, max_slots=2, max_seq_len=16)
    a, b = OracleModel(d), OracleModel(d)
    a.fill_kv_synthetic(1, 10, 3)
    b.fill_kv_synthetic(1, 10, 3)
    k1, v1 = a.read_kv(5, 1, 7)
    k2, v2 = b.read_kv(5, 1, 7)
    assert np.array_equal(k1, k2) and np.array_equal(v1, v2)
    assert np.all(np.abs(k1) <= 1) and np.abs(k1).max() > 0
    assert np.array_equal(eeb.bf16_round(k1), k1)  # bf16 model: values on the bf16 grid
    assert not np.array_equal(k1, v1)
    with pytest.raises(RuntimeError):
        a.fill_kv_synthetic(2, 4)
    a.close()
    b.close()
