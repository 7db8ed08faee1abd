import sys, json, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2504_10724_b200 import eeb
import bench
class A: prompt=128; policy="introspective"; th=0.7; depth=6
ctx = eeb.Context(0)
stream = torch.cuda.ExternalStream(ctx.stream())
print(json.dumps(bench.batch_sweep(ctx, eeb, eeb.PRESETS["opt-1.3b-4x"], A, stream, batches=(1, 2, 4, 8, 16))))
