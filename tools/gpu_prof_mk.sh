export EEB_SKIP_BUILD=1
mkdir -p gpurun_out
EEB_MK=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:step_kernel -c 1 -o gpurun_out/prof_mk python tools/profile_step.py --steps 1 > gpurun_out/prof_mk.log 2>&1
tail -3 gpurun_out/prof_mk.log
