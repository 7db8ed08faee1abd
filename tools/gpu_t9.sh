export EEB_SKIP_BUILD=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
for cs in 1 8; do EEB_TC_CLUSTER=$cs TAG="cs=$cs" timeout 120 python tools/gemm_sweep.py | tail -6; done
for cs in 1 8; do EEB_TC_CLUSTER=$cs timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_cs$cs.log 2>&1; tail -1 gpurun_out/bench_cs$cs.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cs=$cs', round(d['value']), d['ms_per_step'], d['kernel_ms_per_step'])"; done
