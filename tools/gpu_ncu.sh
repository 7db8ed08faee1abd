# ncu --set full of selected kernels of one C2 decode step (stream launches;
# profile_step.py brackets the step with cudaProfilerStart/Stop).
#   TAG=name KREGEX="attention_dec|residual_norm" SKIP=0 COUNT=4 bash tools/gpu_ncu.sh
mkdir -p gpurun_out
TAG=${TAG:-ncu}
timeout ${NCU_TIMEOUT:-900} ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"${KREGEX:-attention_dec}" -s ${SKIP:-0} -c ${COUNT:-3} -o gpurun_out/${TAG} -f \
  python tools/profile_step.py --steps 1 --graphs 0 ${PARGS:-} > gpurun_out/${TAG}.log 2>&1
tail -3 gpurun_out/${TAG}.log
