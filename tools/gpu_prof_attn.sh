# ncu full capture of the first attention launch, pipelined vs one-item-per-CTA
mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for v in pipe one; do
  if [ $v = one ]; then export EEB_ATTN_ONE=1; fi
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attention -c 2 -o gpurun_out/attn_$v python tools/profile_step.py --steps 1 > gpurun_out/attn_$v.log 2>&1
  tail -2 gpurun_out/attn_$v.log
done
