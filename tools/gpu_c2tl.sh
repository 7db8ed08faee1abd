# C2 attention per-CTA timeline per env variant: VARIANTS="label:ENV=1 ..."
mkdir -p gpurun_out
for v in ${VARIANTS:-base:X=1}; do
  env $(echo ${v#*:} | tr "," " ") timeout 300 python tools/step_timeline.py --steps 3 --top 0 --cta ${CTA:-2,47} > gpurun_out/tlc2_${v%%:*}.txt 2>&1
  echo "== ${v%%:*}"; grep -A4 "^launch" gpurun_out/tlc2_${v%%:*}.txt | grep -v start; grep "unstamped\|attention " gpurun_out/tlc2_${v%%:*}.txt
done
