"""Generate tests/golden/decision_vectors.json from the compiled reference.

Runs the UNMODIFIED reference headers (oracle/_ref/libeeref.so, built by
`make -C oracle ref` from /root/reference/proj/include) on seeded random
records and stores the reference's answers, so the CPU tests can pin the
oracle's decision layer without /root/reference (it does not exist on the GPU
box).  Re-run here after changing the generator:

    python tools/make_golden.py

Entry points exercised (oracle/ref_driver.cpp):
  earliest_confident_obs  trace.hpp:69-76
  observation_for_depth   trace.hpp:86-97
  observe_token           policy.hpp:147-156
  choose_depth            pht.hpp:119-126
"""
from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden" / "decision_vectors.json"
LADDERS = [[6, 12, 24], [6, 12, 18, 24], [9, 17, 32], [12, 16, 24, 48], [8, 10, 20, 40, 80], [6, 12]]


def ref_lib() -> C.CDLL:
    path = ROOT / "oracle" / "_ref" / "libeeref.so"
    if not path.exists():
        sys.exit(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
    L = C.CDLL(str(path))
    i32p, f64p = C.POINTER(C.c_int), C.POINTER(C.c_double)
    L.ref_earliest_confident.argtypes = [C.c_int, i32p, i32p, f64p, f64p, C.c_double, i32p]
    L.ref_observation_for_depth.argtypes = [C.c_int, i32p, i32p, f64p, f64p, C.c_int, i32p]
    L.ref_observe_tokens.argtypes = [C.c_int, C.POINTER(C.c_uint8), C.c_int, C.c_int, C.POINTER(C.c_uint8)]
    L.ref_choose_depth.argtypes = [C.c_int, i32p, C.POINTER(C.c_int64), C.c_int, C.c_double]
    return L


def arr(t, xs):
    return (t * len(xs))(*xs)


def main() -> None:
    L = ref_lib()
    rng = np.random.default_rng(20260819)
    records = []
    for i in range(400):
        layers = LADDERS[i % len(LADDERS)]
        n = len(layers)
        # confidences on an f32 grid so the f32 (device) and f64 (reference)
        # comparisons agree exactly; every 5th record plants an exact tie with th.
        confs = [float(np.float32(c)) for c in np.round(rng.uniform(0.0, 1.0, n), 3)]
        toks = [int(t) for t in rng.integers(0, 8, n)]
        th = float(np.float32(np.round(rng.choice([0.1, 0.5, 0.7, 0.8, 0.9, 0.95, rng.uniform()]), 3)))
        if i % 5 == 0:
            confs[rng.integers(0, n)] = th
        logps = [float(np.log(max(c, 1e-6))) for c in confs]
        out_tok = C.c_int(-1)
        layer = L.ref_earliest_confident(n, arr(C.c_int, layers), arr(C.c_int, toks), arr(C.c_double, confs),
                                         arr(C.c_double, logps), th, C.byref(out_tok))
        flat = {}
        for depth in sorted({1, layers[0] - 1, *layers, layers[0] + 1, layers[-1] - 1}):
            if depth < 1:
                continue
            t = C.c_int(-1)
            fl = L.ref_observation_for_depth(n, arr(C.c_int, layers), arr(C.c_int, toks), arr(C.c_double, confs),
                                             arr(C.c_double, logps), depth, C.byref(t))
            flat[str(depth)] = "DomainError" if fl == -3 else [fl, t.value]
        records.append({"layers": layers, "tokens": toks, "confidences": confs, "th": th,
                        "introspective": [layer, out_tok.value], "flat": flat})

    breach = []
    for i in range(40):
        n = int(rng.integers(50, 600))
        p = float(rng.choice([0.05, 0.3, 0.5, 0.6, 0.9]))
        seq = (rng.uniform(size=n) < p).astype(np.uint8)
        cbc_max, window = [(50, 100), (5, 20), (0, 1), (10, 10)][i % 4]
        trig = (C.c_uint8 * n)()
        fired = L.ref_observe_tokens(n, arr(C.c_uint8, seq.tolist()), cbc_max, window, trig)
        breach.append({"breached": seq.tolist(), "cbc_max": cbc_max, "window": window,
                       "triggers": list(trig), "fired": fired})

    depths = []
    for i in range(120):
        layers = LADDERS[i % len(LADDERS)]
        counts = [int(c) for c in rng.integers(0, 1000, len(layers))]
        if sum(counts) == 0:
            counts[-1] = 1
        cov = float(rng.choice([0.5, 0.7, 0.73, 0.74, 0.78, 0.79, 0.9, 1.0, rng.uniform()]))
        d = L.ref_choose_depth(len(layers), arr(C.c_int, layers), arr(C.c_int64, counts), layers[-1], cov)
        depths.append({"layers": layers, "counts": counts, "coverage": cov, "depth": d})

    OUT.write_text(json.dumps({"generator": "tools/make_golden.py (compiled reference, oracle/_ref/libeeref.so)",
                               "exit_rules": records, "breach": breach, "choose_depth": depths},
                              separators=(",", ":")))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
