mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
EEB_MK_TRACE=gpurun_out/mk_trace.bin timeout 120 python tools/mk_bench.py 2>&1 | tail -1
python tools/mk_trace.py gpurun_out/mk_trace.bin 148 qkv,o,up,down
for xs in 8 12; do EEB_MK_XSTAGES=$xs TAG="xs=$xs" timeout 120 python tools/mk_bench.py 2>&1 | tail -1; done
