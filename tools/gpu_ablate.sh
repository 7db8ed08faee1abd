mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
for sk in none gemm attn norm head gemm,attn,norm,head; do
  EEB_SKIP=$sk timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('skip=$sk', round(d['ms_per_step'],3), 'ms/step')"
done > gpurun_out/ablate.log 2>&1
cat gpurun_out/ablate.log
