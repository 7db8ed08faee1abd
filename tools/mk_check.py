"""GPU check: persistent step kernel vs the multi-kernel path vs the CPU oracle."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle.oracle import OracleModel  # noqa: E402
from paper_2504_10724_b200 import eeb  # noqa: E402

desc = eeb.ModelDesc("mk-small", 4, 512, 8, 8, 1024, 1000, (2, 4), dtype=eeb.BF16, max_slots=32, max_seq_len=64, seed=5)
if len(sys.argv) > 1 and sys.argv[1] == "gqa":
    desc = desc.replace(name="mk-gqa", n_kv_heads=2, mlp_kind=eeb.MLP_SWIGLU, exit_layers=(1, 2, 4))
B = int(os.environ.get("B", "16"))
ctxs = {}
for mode in ("1", "0"):
    c = eeb.Context(0)
    c.set_gemm_tier(3 if mode == "1" else 2)
    m = c.register(desc)
    c.load_layers(m, desc.num_layers)
    ctxs[mode] = (c, m)
orc = OracleModel(desc)
orc.load(desc.num_layers)
rng = np.random.default_rng(3)
slots = np.arange(B)
agree = tot = 0
for pos in range(6):
    toks = rng.integers(0, desc.vocab, B)
    for pol, depth in ((eeb.PROFILE, 0), (eeb.INTROSPECTIVE, 0), (eeb.FULL_DEPTH, 0), (eeb.FLAT, 2)):
        if pol != eeb.PROFILE and pos < 5:
            continue
        res = {k: c.decode_step(m, depth, pol, 0.7, slots, toks, np.full(B, pos)) for k, (c, m) in ctxs.items()}
        r = orc.decode_step(depth, pol, 0.7, slots, toks, np.full(B, pos))
        a, b = res["1"], res["0"]
        same_tok = (a["token_id"] == r["token_id"]).mean()
        print(f"pos {pos} policy {pol}: mk/oracle tok {same_tok:.3f} exit {(a['exit_layer'] == r['exit_layer']).mean():.3f} | "
              f"mk/multi tok {(a['token_id'] == b['token_id']).mean():.3f} | multi/oracle tok {(b['token_id'] == r['token_id']).mean():.3f} "
              f"| conf maxdiff mk {np.abs(a['confidence'] - r['confidence']).max():.2e} multi {np.abs(b['confidence'] - r['confidence']).max():.2e} "
              f"| hist mk {a['hist']} oracle {r['hist']}", flush=True)
        agree += (a["token_id"] == r["token_id"]).sum()
        tot += B
    # keep the three KV caches in step: full-depth prefill already applied above via PROFILE at every position
print(f"mk token agreement with the oracle: {agree}/{tot}")
prof = ctxs["1"][0]
prof.profile_enable(True)
prof.decode_step(ctxs["1"][1], 0, eeb.INTROSPECTIVE, 0.7, slots, rng.integers(0, desc.vocab, B), np.full(B, 6))
print(prof.profile_read())
