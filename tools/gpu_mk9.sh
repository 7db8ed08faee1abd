mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
export EEB_MK_L2=0
for dbg in 14 15; do EEB_MK_DBG=$dbg TAG="dbg=$dbg" timeout 120 python tools/mk_bench.py 2>&1 | tail -1; done
for xs in 4 16; do EEB_MK_XSTAGES=$xs EEB_MK_DBG=14 TAG="dbg=14 xs=$xs" timeout 120 python tools/mk_bench.py 2>&1 | tail -1; done
EEB_MK_DBG=14 EEB_MK_XSTAGES=16 EEB_MK_TRACE=gpurun_out/mk_trace.bin timeout 120 python tools/mk_bench.py 2>&1 | tail -1
python tools/mk_trace.py gpurun_out/mk_trace.bin 148 qkv,o,up,down
EEB_MK_DBG=15 EEB_MK_TRACE=gpurun_out/mk_trace2.bin timeout 120 python tools/mk_bench.py 2>&1 | tail -1
python tools/mk_trace.py gpurun_out/mk_trace2.bin 148 qkv,o,up,down
