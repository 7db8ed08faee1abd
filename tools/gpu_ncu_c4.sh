# ncu --set full of the 34B batch-256 kernels changed in session 6: the deep
# (one 256-row tile) QKV GEMM and the GQA decode attention (helper warps).
mkdir -p gpurun_out
MODEL=34b B=256 ONLY=qkv ITERS=2 timeout 600 ncu --set full --clock-control none -k regex:gemm_tc -s 2 -c 1 \
  -o gpurun_out/c4_qkv256 -f python tools/gemm_big.py > gpurun_out/c4_qkv256.log 2>&1; tail -1 gpurun_out/c4_qkv256.log
TAG=c4_attn256 KREGEX=attention_dec SKIP=1 COUNT=1 PARGS="--model codellama-34b --policy flat --depth 12 --batch 256" bash tools/gpu_ncu.sh
for f in c4_qkv256 c4_attn256; do ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null; done
