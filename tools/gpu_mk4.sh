mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
for xs in 4 8 12 16 20; do EEB_MK_XSTAGES=$xs TAG="xs=$xs" timeout 120 python tools/mk_bench.py 2>&1 | tail -1; done
EEB_MK_XSTAGES=16 EEB_MK_WSTAGES=4 TAG="xs=16 ws=4" timeout 120 python tools/mk_bench.py 2>&1 | tail -1
EEB_MK_XSTAGES=16 EEB_MK_TRACE=gpurun_out/mk_trace16.bin timeout 120 python tools/mk_bench.py 2>&1 | tail -1
python tools/mk_trace.py gpurun_out/mk_trace16.bin 148 qkv,o,up,down
