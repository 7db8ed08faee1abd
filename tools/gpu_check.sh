# GPU-box check: tests, smoke, bench (each bounded by its own timeout).
mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.log
timeout 300 python -m pytest tests/test_gpu_gemm.py -m gpu -x -q > gpurun_out/pytest_gemm.log 2>&1
tail -30 gpurun_out/pytest_gemm.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
tail -40 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; tail -3 gpurun_out/bench.log
