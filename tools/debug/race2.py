import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import race  # noqa: E402  (runs its own scenario once at import; ignore)
from paper_2504_10724_b200 import eeb  # noqa: E402


def variant(name, fn):
    a = race.parity_scenario("a")
    fn()
    b = race.parity_scenario("b")
    a.pop("snaps"); b.pop("snaps")
    diff = [k for k in a if not np.array_equal(a[k], b[k])]
    print("VARIANT", name, "differs:", len(diff), flush=True)


def bf16_steps(graphs=True, B=16):
    c = eeb.Context(0)
    d = eeb.PRESETS["tiny"].replace(dtype=eeb.BF16, name="t", max_slots=16, max_seq_len=64)
    m = c.register(d)
    c.load_layers(m, 12)
    c.set_graphs(graphs)
    rng = np.random.default_rng(0)
    for pos in range(4):
        c.decode_step(m, 0, eeb.FULL_DEPTH, 0.7, np.arange(B), rng.integers(0, 512, B), np.full(B, pos))
    c.close()


def stage_only():
    c = eeb.Context(0)
    d = eeb.PRESETS["tiny"].replace(dtype=eeb.BF16, name="t", max_slots=16, max_seq_len=64)
    m = c.register(d)
    c.host_stage(m, 12)
    c.close()


variant("nothing", lambda: None)
variant("bf16_steps_graphs", lambda: bf16_steps(True))
variant("bf16_steps_eager", lambda: bf16_steps(False))
variant("bf16_steps_b8", lambda: bf16_steps(True, 8))
variant("stage_only", stage_only)
