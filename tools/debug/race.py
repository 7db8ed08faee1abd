"""Debug: after the async-loader scenario, does the f32 introspective step's KV
still match the oracle, and do two GPU contexts agree with each other?"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[2] / "tests"))
from oracle.oracle import OracleModel  # noqa: E402
from paper_2504_10724_b200 import eeb  # noqa: E402

TH = 0.7


def loader_scenario():
    import test_gpu_loader as T
    c = eeb.Context(0)
    T.test_async_load_matches_device_materialised(c)
    c.close()


def parity_scenario(tag):
    desc = eeb.PRESETS["tiny"]
    c = eeb.Context(0)
    m = c.register(desc)
    c.load_layers(m, desc.num_layers)
    ref = OracleModel(desc)
    ref.load(desc.num_layers)
    c.retain_logits(True)
    rng = np.random.default_rng(3)
    B = 8
    slots = np.arange(B)
    kv = {}
    for pos in range(7):
        toks = rng.integers(0, desc.vocab, B)
        policy = eeb.PROFILE if pos < 6 else eeb.INTROSPECTIVE
        g = c.decode_step(m, 0, policy, TH, slots, toks, np.full(B, pos))
        r = ref.decode_step(0, policy, TH, slots, toks, np.full(B, pos), want_logits=True)
        snap = {}
        for layer in (6, 7, 8):
            for b in range(B):
                for pp in range(pos + 1):
                    snap[(pos, layer, b, pp)] = c.read_kv(m, layer, b, pp)[1]
        kv.setdefault("snaps", {}).update(snap)
        if pos == 6:
            print(tag, "exit", g["exit_layer"], r["exit_layer"])
            for layer in range(1, 13):
                bad = []
                for b in range(B):
                    gk, _ = c.read_kv(m, layer, b, pos)
                    rk, _ = ref.read_kv(layer, b, pos)
                    kv[(layer, b)] = gk
                    if g["exit_layer"][b] >= layer and not np.allclose(gk, rk, atol=1e-4, rtol=1e-3):
                        bad.append(b)
                if bad:
                    print(tag, "layer", layer, "bad rows", bad)
    c.close()
    return kv


if __name__ == "__main__":
  a = parity_scenario("fresh")
  loader_scenario()
  b = parity_scenario("after-loader")
  sa, sb = a.pop("snaps"), b.pop("snaps")
  vd = sorted(k for k in sa if not np.array_equal(sa[k], sb[k]))
  print("V history differing (step pos, layer, row, position):", vd[:30], len(vd))
  diff = [k for k in a if not np.array_equal(a[k], b[k])]
  print("gpu-vs-gpu differing (layer,row):", diff[:20], len(diff))
