mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
for dbg in 0 4; do EEB_MK_DBG=$dbg TAG="dbg=$dbg" timeout 120 python tools/mk_bench.py 2>&1 | tail -1; done
EEB_MK_L2=16 TAG="l2=16" timeout 120 python tools/mk_bench.py 2>&1 | tail -1
EEB_MK_XSTAGES=8 TAG="xs=8" timeout 120 python tools/mk_bench.py 2>&1 | tail -1
EEB_MK_TRACE=gpurun_out/mk_trace.bin timeout 120 python tools/mk_bench.py 2>&1 | tail -1
python tools/mk_trace.py gpurun_out/mk_trace.bin 148 qkv,o,up,down
BS=16,32,128 timeout 120 python tools/mk_bench.py 2>&1 | tail -3
