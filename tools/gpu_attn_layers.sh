mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
for v in one pipe; do
  EEB_ATTN=$v timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$v.csv python tools/profile_step.py --steps 1 > /dev/null 2>&1
  python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/launches_$v.csv')))
hi=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
hdr=rows[hi]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value')
att=[int(float(r[vi])) for r in rows[hi+1:] if 'attention' in r[ki]]
print('$v', sum(att)/1000, [a//1000 for a in att])
PY
  EEB_ATTN=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-secondary 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3))"
done
