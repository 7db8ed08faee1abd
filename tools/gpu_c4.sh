mkdir -p gpurun_out
for v in "deep:EEB_TC_DEEP=1" "nodeep:EEB_TC_DEEP=0"; do
env $(echo ${v#*:} | tr "," " ") timeout 600 python bench.py --model codellama-34b --policy flat --depth 12 --sweep --no-secondary --no-cpu-baseline --no-parity > gpurun_out/c4_${v%%:*}.log 2>&1
tail -1 gpurun_out/c4_${v%%:*}.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('${v%%:*}', d['value'], d['ms_per_step'], d['clocks'])
for b in d['batch_sweep']: print(b)"
done
