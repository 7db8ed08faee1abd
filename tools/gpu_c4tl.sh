# C4 (34B flat-12) attention timeline per env variant: VARIANTS="label:ENV=1 ..." BS="64 256"
mkdir -p gpurun_out
for v in ${VARIANTS:-base:X=1}; do for B in ${BS:-64 256}; do
  env $(echo ${v#*:} | tr "," " ") timeout 300 python tools/step_timeline.py --model codellama-34b --policy flat --depth 12 --batch $B --steps 3 --top 3 --cta 2 > gpurun_out/tlv_${v%%:*}_$B.txt 2>&1
  echo "${v%%:*} B=$B $(sed -n 3p gpurun_out/tlv_${v%%:*}_$B.txt) $(sed -n 5p gpurun_out/tlv_${v%%:*}_$B.txt) | $(grep 'unstamped' gpurun_out/tlv_${v%%:*}_$B.txt)"
done; done
