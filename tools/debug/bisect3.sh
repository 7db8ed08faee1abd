export EEB_SKIP_BUILD=1
export RETAIN=0
TAG=graph timeout 300 python tools/debug/race3.py 2>&1 | grep RESULT
TAG=graph-poison EEB_DEBUG_POISON=1 timeout 300 python tools/debug/race3.py 2>&1 | grep RESULT
TAG=graph-eager-modules CUDA_MODULE_LOADING=EAGER timeout 300 python tools/debug/race3.py 2>&1 | grep RESULT
TAG=graph-nopdl EEB_NO_PDL=1 timeout 300 python tools/debug/race3.py 2>&1 | grep RESULT
