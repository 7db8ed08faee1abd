mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
for dbg in 0 1 2 3; do EEB_MK_DBG=$dbg TAG="dbg=$dbg" timeout 120 python tools/mk_bench.py 2>&1 | tail -1; done
EEB_MK_DBG=3 EEB_MK_BAR=2 TAG="dbg=3 nobar" timeout 120 python tools/mk_bench.py 2>&1 | tail -1
for k in 0 1 2 3; do EEB_MK_ONLY=$k TAG="only=$k" timeout 120 python tools/mk_bench.py 2>&1 | tail -1; done
for k in 0 1 2 3; do EEB_MK_ONLY=$k EEB_MK_BAR=2 EEB_MK_DBG=3 TAG="only=$k raw" timeout 120 python tools/mk_bench.py 2>&1 | tail -1; done
