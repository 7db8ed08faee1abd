export EEB_SKIP_BUILD=1
mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
free -g | head -2
timeout 900 python bench.py --no-cpu-baseline --model codellama-34b --policy flat --depth 12 --batch 64 > gpurun_out/b34.log 2>&1; tail -3 gpurun_out/b34.log | cut -c1-1800
timeout 900 python bench.py --no-cpu-baseline --batch 256 > gpurun_out/b256.log 2>&1; tail -1 gpurun_out/b256.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('b256', round(d['value']), round(d['ms_per_step'],3), d['roofline']['frac'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
