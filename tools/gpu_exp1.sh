mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
for cfg in "0 0" "148 0" "148 8" "296 3" "444 0"; do
  set -- $cfg
  EEB_TC_WAVE=$1 EEB_TC_STAGES=$2 TAG="wave=$1 st=$2" timeout 120 python tools/gemm_sweep.py
done > gpurun_out/sweep.log 2>&1
cat gpurun_out/sweep.log
bash tools/gpu_ablate.sh
