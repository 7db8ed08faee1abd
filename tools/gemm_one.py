import sys
sys.path.insert(0, '.')
from paper_2504_10724_b200 import eeb
ctx = eeb.Context(0)
print(ctx.bench_gemm(2, 2048, 2048, 64, 5))
