mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
for dbg in 0 16; do for xs in 4 12; do EEB_MK_DBG=$dbg EEB_MK_XSTAGES=$xs TAG="dbg=$dbg xs=$xs" timeout 120 python tools/mk_bench.py 2>&1 | tail -1; done; done
EEB_MK_DBG=16 EEB_MK_L2=16 TAG="bulk l2=16" timeout 120 python tools/mk_bench.py 2>&1 | tail -1
EEB_MK_DBG=16 EEB_MK_TRACE=gpurun_out/mk_trace.bin timeout 120 python tools/mk_bench.py 2>&1 | tail -1
python tools/mk_trace.py gpurun_out/mk_trace.bin 148 qkv,o,up,down
