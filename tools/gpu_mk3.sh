mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
for bm in 0 1 2; do EEB_MK_BAR=$bm TAG="bar=$bm" timeout 120 python tools/mk_bench.py 2>&1 | tail -1; done
EEB_MK_TRACE=gpurun_out/mk_trace.bin timeout 120 python tools/mk_bench.py 2>&1 | tail -1
python tools/mk_trace.py gpurun_out/mk_trace.bin 148 qkv,o,up,down
EEB_MK_HEADONLY=1 TAG=headonly timeout 120 python tools/mk_bench.py 2>&1 | tail -1
EEB_MK_HEADONLY=1 EEB_MK_BAR=2 TAG=headonly-nobar timeout 120 python tools/mk_bench.py 2>&1 | tail -1
