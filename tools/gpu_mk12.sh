mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
for dbg in 7 39 32 15; do EEB_MK_DBG=$dbg TAG="dbg=$dbg" timeout 120 python tools/mk_bench.py 2>&1 | tail -1; done
EEB_MK_DBG=7 EEB_MK_TRACE=gpurun_out/mk_trace.bin timeout 120 python tools/mk_bench.py 2>&1 | tail -1
python tools/mk_trace.py gpurun_out/mk_trace.bin 148 qkv,o,up,down
for b in 16 128; do EEB_MK_DBG=7 BS=$b TAG="dbg=7" timeout 120 python tools/mk_bench.py 2>&1 | tail -1; done
