mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
for l2 in 0 16 24 32 48 64; do EEB_MK_L2=$l2 TAG="l2=$l2" timeout 120 python tools/mk_bench.py 2>&1 | tail -1; done
EEB_MK_L2=32 EEB_MK_XSTAGES=8 TAG="l2=32 xs=8" timeout 120 python tools/mk_bench.py 2>&1 | tail -1
EEB_MK_L2=32 EEB_MK_XSTAGES=8 EEB_MK_WSTAGES=6 TAG="l2=32 xs=8 ws=6" timeout 120 python tools/mk_bench.py 2>&1 | tail -1
EEB_MK_L2=32 EEB_MK_TRACE=gpurun_out/mk_trace.bin timeout 120 python tools/mk_bench.py 2>&1 | tail -1
python tools/mk_trace.py gpurun_out/mk_trace.bin 148 qkv,o,up,down
