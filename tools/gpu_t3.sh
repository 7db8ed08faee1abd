export EEB_SKIP_BUILD=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mk.py -m gpu -q -x 2>&1 | tail -5
