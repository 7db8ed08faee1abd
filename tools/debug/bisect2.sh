export EEB_SKIP_BUILD=1
TAG=default timeout 300 python tools/debug/race3.py 2>&1 | grep RESULT
TAG=noretain RETAIN=0 timeout 300 python tools/debug/race3.py 2>&1 | grep RESULT
TAG=nopdl EEB_NO_PDL=1 timeout 300 python tools/debug/race3.py 2>&1 | grep RESULT
for k in gemm_cc attention residual_norm gather head_reduce decide finalize; do
  TAG=$k EEB_NO_PDL_K=$k timeout 300 python tools/debug/race3.py 2>&1 | grep RESULT
done
