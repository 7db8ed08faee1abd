"""Static check of the built kernels (CPU, cuobjdump): no kernel of the PDL
chain may load global memory before `griddepcontrol.wait` (SASS ACQBULK).

A `const T* __restrict__` kernel parameter lets the compiler treat its loads
as invariant and hoist them above the wait, so a kernel reads its
predecessor's output (e.g. the compacted row count) before the predecessor
has written it — a race that only shows under particular timings.  Weight
streams (TMA, UTMALDG) are allowed before the wait: weights never change
inside a step.  A volatile load (LDG.E.STRONG.SYS) is the one deliberate
exception: the tcgen05 GEMM reads the live-row count before the wait only as
a hint whether to prefetch weights (a stale value costs a useless or a missed
prefetch; the count read after the wait decides what is computed) — plain
(hoistable) loads stay forbidden.  The launch-timeline stamp (REDG.E.MIN.64,
common.cuh StampScope) writes only its own diagnostics buffer.  The row-norm
kernels load their RMSNorm gains (weights) with explicit __ldg before the wait
(LDG.E.128.CONSTANT), in those kernels only.
"""
import re
import subprocess

import pytest

from paper_2504_10724_b200 import eeb

ALLOWED_PRE_WAIT = ("UTMALDG", "LDG.E.STRONG.SYS", "REDG.E.MIN.64")  # TMA weight prefetch; live-count hint; stamp
NO_PDL_KERNELS = ("synth",)  # standalone launches (weight synthesis)
GAIN_PRELOAD_KERNELS = ("residual_norm_kernel", "tp_norm_kernel", "embed_norm_kernel")  # norm gains before the wait


def _functions(sass: str):
    cur, body = None, []
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
        elif cur:
            ins = re.search(r"/\*[0-9a-f]{4,}\*/\s+(.*?);", line)
            if ins:
                body.append(ins.group(1))
    if cur:
        yield cur, body


def test_no_global_load_before_griddepcontrol_wait():
    try:
        sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(eeb.LIB_PATH)], capture_output=True,
                              text=True, check=True).stdout
    except (FileNotFoundError, subprocess.CalledProcessError) as e:
        pytest.skip(f"cuobjdump unavailable: {e}")
    checked, bad = 0, []
    for name, body in _functions(sass):
        if any(k in name for k in NO_PDL_KERNELS) or not any("ACQBULK" in i for i in body):
            continue
        checked += 1
        for ins in body:
            if "ACQBULK" in ins:
                break
            op = ins.split()[0] if not ins.startswith("@") else ins.split()[1]
            if op.startswith("LDG.E.128.CONSTANT") and any(k in name for k in GAIN_PRELOAD_KERNELS):
                continue
            if op.startswith(("LDG", "LD.", "ATOMG", "REDG", "STG", "ST.")) and not op.startswith(ALLOWED_PRE_WAIT):
                bad.append((name, ins))
                break
    assert checked >= 10, checked
    assert not bad, bad
