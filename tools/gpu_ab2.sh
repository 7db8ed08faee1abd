# A/B of kernel variants on the C2 bench (env toggles) after the GPU parity tests,
# then the serialised ncu launch list of one step.
mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
run() {  # label, env...
  local label=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_ARGS:---no-secondary} > gpurun_out/ab_$label.log 2>&1
  tail -1 gpurun_out/ab_$label.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$label', round(d['ms_per_step'],3), 'ms/step', round(d['value']), 'tok/s', 'e2e', round(d['e2e']['value']), 'gemm_frac', round(d['roofline']['frac'],3), d.get('kernel_ms_per_step'), d.get('secondary_c4',{}).get('ms_per_step'))" || tail -3 gpurun_out/ab_$label.log
}
for v in ${AB_VARIANTS:-new:X=1}; do run ${v%%:*} $(echo ${v#*:} | tr "," " "); done
if [ -n "$LAUNCHES" ]; then
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 1 --graphs 0 > gpurun_out/prof_launch.log 2>&1
  python tools/launch_summary.py gpurun_out/launches.csv
fi
