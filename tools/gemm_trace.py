"""Per-CTA timeline of two consecutive mid-chain tcgen05 GEMM launches
(EEB_GEMM_TRACE stamps, see gemm_tc.cu): where a launch's time goes.
Needs libeeb built with -DEEB_GEMM_TRACE:
  EEB_NVCC_EXTRA=-DEEB_GEMM_TRACE python -c "from paper_2504_10724_b200 import build as b; b.build_eeb()"
Run on the GPU box:  python tools/gemm_trace.py N K [B]
(EEB_BENCH_ACT=1|2: the fused up projection with its activation epilogue)"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    n, k = int(sys.argv[1]), int(sys.argv[2])
    b = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    path = f"/tmp/gemm_trace_{n}_{k}.bin"
    os.environ["EEB_GEMM_TRACE"] = path
    from paper_2504_10724_b200 import eeb

    ctx = eeb.Context(0)
    for _ in range(3):  # ~clocks up: a short chain alone would run at whatever clock the GPU idles at
        ctx.bench_gemm(2, n, k, b, 400)
    ms = ctx.bench_gemm(2, n, k, b, 40)
    t = np.fromfile(path, dtype=np.uint64).reshape(2, -1, 8).astype(np.int64)
    names = ["start", "init", "pdl_wait", "1st stage", "acc done", "epi done", "dealloc", "cl. sync"]
    print(f"N={n} K={k} B={b}: {ms*1e3:.2f} us per launch (chain of 40)")
    t0 = None
    for li in range(2):
        live = t[li][t[li][:, 0] > 0]
        if t0 is None:
            t0 = live[:, 0].min()
        rel = (live[:, :8] - t0) / 1e3
        print(f" launch {li}: {len(live)} CTAs")
        for j, nm in enumerate(names):
            c = rel[:, j]
            c = c[live[:, j] > 0]
            if len(c):
                print(f"   {nm:10s} min {c.min():7.2f}  med {np.median(c):7.2f}  max {c.max():7.2f} us")
        for r in list(range(0, len(live), max(1, len(live) // 6)))[:6]:
            print("   cta", r, " ".join(f"{x:7.2f}" for x in rel[r]))


if __name__ == "__main__":
    main()
