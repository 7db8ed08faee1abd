export EEB_SKIP_BUILD=1
mkdir -p gpurun_out
for w in 148 296 444 592; do EEB_TC_WAVE=$w timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bw.log 2>&1; tail -1 gpurun_out/bw.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('wave=$w', round(d['value']), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"; done
