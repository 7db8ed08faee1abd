export EEB_SKIP_BUILD=1
TAG=hbm timeout 120 python tools/gemm_sweep.py
EEB_BENCH_L2=1 TAG=l2 timeout 120 python tools/gemm_sweep.py
