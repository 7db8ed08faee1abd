# C4 (34B, greedy depth 12) batch sweep A/B: VARIANTS="label:ENV=1,ENV2=2 ..."
mkdir -p gpurun_out
for v in ${VARIANTS:-base:X=1}; do
env $(echo ${v#*:} | tr "," " ") timeout 600 python bench.py --model codellama-34b --policy flat --depth 12 --sweep --no-secondary --no-cpu-baseline --no-parity > gpurun_out/c4_${v%%:*}.log 2>&1
tail -1 gpurun_out/c4_${v%%:*}.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('${v%%:*}', round(d['value']), round(d['ms_per_step'],3), d['clocks'])
for b in d['batch_sweep'][-3:]: print('  ', b['batch'], round(b['ms_per_step'],3), round(b['tokens_per_s']), {k: round(v,3) for k,v in b.items() if 'frac' in k})"
done
