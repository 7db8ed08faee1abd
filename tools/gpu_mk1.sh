mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
timeout 120 python tools/mk_bench.py 2>&1 | tail -5
for st in 4 6 8; do EEB_MK_WSTAGES=$st TAG="wst=$st" BS=64 timeout 120 python tools/mk_bench.py 2>&1 | tail -1; done
BS=16,32,128 timeout 120 python tools/mk_bench.py 2>&1 | tail -3
