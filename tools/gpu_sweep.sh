mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
for st in 0 2 3 4 6 8; do
  for wv in 0 74 296; do
    EEB_TC_STAGES=$st EEB_TC_WAVE=$wv TAG="st=$st wave=$wv" timeout 120 python tools/gemm_sweep.py
  done
done > gpurun_out/sweep.log 2>&1
cat gpurun_out/sweep.log | grep layer
