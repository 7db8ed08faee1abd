# One GPU call: GPU tests, the in-graph timeline, a short bench (and optional A/B env variants).
#   TAG=name TESTS="tests/..." AB_VARIANTS="label:ENV=1,ENV2=2 ..." bash tools/gpu_check.sh
mkdir -p gpurun_out
TAG=${TAG:-chk}
if [ "${TESTS:-all}" != "none" ]; then
  timeout 1200 python -m pytest ${TESTS:-tests} -m gpu -x -q -rs > gpurun_out/${TAG}_pytest.txt 2>&1; tail -3 gpurun_out/${TAG}_pytest.txt
fi
timeout 300 python tools/step_timeline.py --steps 5 --top ${TOP:-50} --json gpurun_out/${TAG}_tl.json > gpurun_out/${TAG}_tl.txt 2>&1; head -8 gpurun_out/${TAG}_tl.txt
for v in ${AB_VARIANTS:-base:X=1}; do
  label=${v%%:*}
  env $(echo ${v#*:} | tr "," " ") timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-secondary > gpurun_out/${TAG}_ab_$label.log 2>&1
  tail -1 gpurun_out/${TAG}_ab_$label.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$label', round(d['ms_per_step'],4), 'ms/step', round(d['value']), 'tok/s e2e', round(d['e2e']['value']))" || tail -3 gpurun_out/${TAG}_ab_$label.log
done
