export EEB_SKIP_BUILD=1
export RETAIN=0 RUNS=2
for k in gemm_cc attention residual_norm act_kernel gather head_reduce decide finalize embed; do
  TAG=$k EEB_NO_PDL_K=$k timeout 300 python tools/debug/race3.py 2>&1 | grep RESULT
done
