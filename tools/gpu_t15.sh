export EEB_SKIP_BUILD=1
mkdir -p gpurun_out
for w in 5 30; do timeout 600 python bench.py --no-cpu-baseline --no-secondary --warmup $w > gpurun_out/bw.log 2>&1; tail -1 gpurun_out/bw.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('warmup=$w', round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']))"; done
