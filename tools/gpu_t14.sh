export EEB_SKIP_BUILD=1
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
