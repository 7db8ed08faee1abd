export EEB_SKIP_BUILD=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mk.py -m gpu -q -x 2>&1 | tail -3
EEB_MK=1 EEB_MK_TRACE=gpurun_out/step_trace.bin timeout 300 python tools/profile_step.py --steps 1 > /dev/null 2>&1
python tools/mk_trace_step.py gpurun_out/step_trace.bin 2>/dev/null
EEB_MK=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_mk.log 2>&1; tail -1 gpurun_out/bench_mk.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('mk', d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_step'], d['roofline']['frac'], d['e2e'])"
