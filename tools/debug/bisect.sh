export EEB_SKIP_BUILD=1
for k in gemm_cc attention residual_norm act_kernel gather head_reduce decide embed finalize; do
  r=$(EEB_NO_PDL_K=$k timeout 300 python tools/debug/race.py 2>&1 | tail -1)
  echo "$k: $r"
done
