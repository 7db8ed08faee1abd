"""Per-phase-kind time of one persistent step (EEB_MK_TRACE dump)."""
import collections
import sys

import numpy as np

path, G = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 148
kinds = [int(x) for x in open(path + ".kinds").read().split()]
t = np.fromfile(path, dtype=np.uint64).astype(np.int64).reshape(G, len(kinds), 8)
names = {0: "gemm", 1: "norm", 2: "attn", 3: "act", 4: "head_reduce", 5: "decide", 6: "finalize"}
start = t[:, :, 0].astype(np.float64)
start[start == 0] = np.nan
begin = np.nanmin(start, axis=0)
begin[0] = t[t > 0].min()  # phase 0 has no barrier stamp: first stamp of the launch
last = t[:, -1, :].max()  # the final phase's end: its latest stamp
end = np.append(begin[1:], max(last, begin[-1]))
agg = collections.defaultdict(lambda: [0, 0.0])
for p, k in enumerate(kinds):
    agg[names[k]][0] += 1
    agg[names[k]][1] += (end[p] - begin[p]) / 1e3
tot = sum(v[1] for v in agg.values())
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:12s} n={n:4d} total {us:8.1f} us  avg {us / n:6.2f} us  share {us / tot:5.1%}")
print(f"step {tot:.1f} us, {len(kinds)} phases")
