# Prefill wall time per env variant: VARIANTS="label:ENV=1 ..."
for v in ${VARIANTS:-base:X=1}; do
  echo "${v%%:*}: $(env $(echo ${v#*:} | tr "," " ") timeout 300 python tools/prefill_time.py ${PARGS:-} 2>&1 | tail -1)"
done
