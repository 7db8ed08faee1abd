# Large-batch GEMM experiment: parity of the GEMM tiers, 34B / C2 shapes at
# B=128/256, the fused SwiGLU up projection at 256 rows (row halves vs one tile).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -m gpu -x -q > gpurun_out/ge_pytest.txt 2>&1; tail -2 gpurun_out/ge_pytest.txt
timeout 300 python tools/gemm_big.py > gpurun_out/ge_big.txt 2>&1; grep layer gpurun_out/ge_big.txt
for v in "rh:EEB_BENCH_ACT=2" "one:EEB_BENCH_ACT=2,EEB_TC_RHALF=0" "one4:EEB_BENCH_ACT=2,EEB_TC_RHALF=0,EEB_ACT_STAGES=4"; do
  env $(echo ${v#*:} | tr "," " ") MODEL=34b B=256 ONLY=up timeout 120 python tools/gemm_big.py 2>&1 | sed "s/^/${v%%:*} /" | head -1
done
