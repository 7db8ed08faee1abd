export EEB_SKIP_BUILD=1
mkdir -p gpurun_out
EEB_MK_TRACE=gpurun_out/step_trace.bin timeout 300 python tools/profile_step.py --steps 1 > /dev/null 2>&1
python tools/mk_trace_step.py gpurun_out/step_trace.bin
