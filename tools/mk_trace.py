"""Summarise a persistent-kernel phase trace (EEB_MK_TRACE=<file>).

Stamps per (CTA, phase): 0 barrier passed, 1 last X issued, 2 epilogue done,
3 phase done, 4 W first issue, 5 W last issue, 6 MMA first k-block, 7 MMA last."""
import sys

import numpy as np

path, G = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 148
names = sys.argv[3].split(",") if len(sys.argv) > 3 else None
t = np.fromfile(path, dtype=np.uint64).astype(np.int64).reshape(G, -1, 8)
P = t.shape[1]
t0 = t[:, 0, 0].min()
rel = (t - t0) / 1e3
print("per-phase medians over CTAs (us, relative to the phase's barrier-passed stamp):")
print(" phase  start   Wfirst  Wlast  MMA1st MMAlast Xlast  epi   done  | Wlead(us ahead of barrier)")
for p in list(range(min(P, 12))):
    st = rel[:, p, 0]
    f = lambda k: np.median(rel[:, p, k] - st)
    nm = names[p % len(names)] if names else str(p)
    print(f"{nm:>6s} {np.median(st):7.1f} {f(4):7.2f} {f(5):7.2f} {f(6):7.2f} {f(7):7.2f} {f(1):6.2f} {f(2):6.2f} {f(3):6.2f}")
print(f"total {(t[:, -1, 3].max() - t0)/1e3:.1f} us over {P} phases")
