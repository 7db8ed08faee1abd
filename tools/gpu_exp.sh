mkdir -p gpurun_out
T=${TAG:-exp}
for v in ${VARIANTS:-base:X=1}; do
  label=${v%%:*}
  env $(echo ${v#*:} | tr "," " ") timeout 300 python tools/step_timeline.py --steps 3 --top ${TOP:-8} ${TLARGS:-} > gpurun_out/${T}_tl_$label.txt 2>&1
  echo "== $label"; sed -n 2,5p gpurun_out/${T}_tl_$label.txt; grep -A4 "^launch" gpurun_out/${T}_tl_$label.txt | head -40
done
