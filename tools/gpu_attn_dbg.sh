# MHA decode attention: where the time goes at a fixed row count (flat policy,
# no exits, so garbage outputs cannot change the rows): EEB_ATTN_DBG 0 / 1 (no
# compute) / 2 (no K/V loads) / 3 (neither).  BS="18 64"
mkdir -p gpurun_out
for B in ${BS:-18 64}; do for d in 0 1 2 3; do
  EEB_ATTN_DBG=$d timeout 300 python tools/step_timeline.py --policy flat --depth 24 --batch $B --steps 3 --top 0 --cta 2,9 > gpurun_out/ad_${B}_$d.txt 2>&1
  echo "B=$B dbg=$d $(grep -A4 '^launch 9' gpurun_out/ad_${B}_$d.txt | grep -E 'mark|end' | tr -s ' ' | tr '\n' ' ') $(grep 'attention ' gpurun_out/ad_${B}_$d.txt)"
done; done
