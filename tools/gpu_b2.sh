mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
timeout 300 python -m pytest tests/test_gpu_gemm.py -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_chain.log 2>&1; tail -1 gpurun_out/bench_chain.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('chain', d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernel_ms_per_step'])"
timeout 120 python tools/gemm_sweep.py
