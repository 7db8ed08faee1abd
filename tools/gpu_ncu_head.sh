# ncu --set full of the first exit-head GEMM (25th tcgen05 GEMM of a C2 step) at head cluster sizes 1 and 2.
mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
for cs in 1 2; do
  EEB_HEAD_CS=$cs timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:gemm_tc_kernel --launch-skip 24 --launch-count 1 -o gpurun_out/head_cs$cs python tools/profile_step.py --steps 1 > gpurun_out/ncu_head_cs$cs.log 2>&1
  tail -2 gpurun_out/ncu_head_cs$cs.log
done
