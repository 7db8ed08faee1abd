mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
for dbg in 1 5 7; do EEB_MK_DBG=$dbg EEB_MK_TRACE=gpurun_out/mk_trace$dbg.bin TAG="dbg=$dbg" timeout 120 python tools/mk_bench.py 2>&1 | tail -1; python tools/mk_trace.py gpurun_out/mk_trace$dbg.bin 148 qkv,o,up,down | sed -n 7,10p; done
