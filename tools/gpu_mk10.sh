mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
for l2 in 0 16 32; do for ws in 4 8 0; do EEB_MK_L2=$l2 EEB_MK_WSTAGES=$ws TAG="l2=$l2 ws=$ws" timeout 120 python tools/mk_bench.py 2>&1 | tail -1; done; done
EEB_MK_DBG=4 TAG="noW" timeout 120 python tools/mk_bench.py 2>&1 | tail -1
EEB_MK_L2=16 EEB_MK_TRACE=gpurun_out/mk_trace.bin timeout 120 python tools/mk_bench.py 2>&1 | tail -1
python tools/mk_trace.py gpurun_out/mk_trace.bin 148 qkv,o,up,down
