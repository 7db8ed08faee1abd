mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_mk.log 2>&1; tail -1 gpurun_out/bench_mk.log | cut -c1-2500
timeout 600 python bench.py --no-cpu-baseline --tier 2 > gpurun_out/bench_chain.log 2>&1; tail -1 gpurun_out/bench_chain.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('chain', d['value'], d['ms_per_step'])"
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
