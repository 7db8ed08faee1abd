"""Sweep the large-batch decode GEMM decomposition (row halves x split count
x pipeline stages) over the 34B and C2 layer shapes; one subprocess per
setting (the knobs are read once per process).  Run on the GPU box:
  B=128,256 python tools/gemm_split_sweep.py > gpurun_out/split_sweep.txt"""
import itertools
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
Bs = os.environ.get("B", "128,256")
rows = []
for rh, st, sp in itertools.product(("1", "0"), ("0", "4"), ("1", "2", "3", "4", "5", "6", "8", "10", "12")):
    if rh == "1" and st == "4":
        continue
    env = dict(os.environ, EEB_TC_RHALF=rh, EEB_TC_STAGES=st, EEB_TC_SPLITS=sp, B=Bs, ITERS="30")
    r = subprocess.run([sys.executable, str(ROOT / "tools/gemm_big.py")], env=env, capture_output=True, text=True,
                       timeout=300)
    for line in r.stdout.splitlines():
        if " us " in line and "layer" not in line:
            f = line.split()
            rows.append((f[0], f[1] + f[2] if f[1] == "B=" else f[1], f[-9] if False else line.split(" us")[0].split()[-1],
                         rh, st, sp, line))
            print(f"rh={rh} st={st} sp={sp:>2s} {line}", flush=True)
