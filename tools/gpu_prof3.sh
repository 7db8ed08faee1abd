mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"attention_mma" -s 8 -c 1 -o gpurun_out/prof_attn_mma python tools/profile_step.py --steps 1 > gpurun_out/prof_attn.log 2>&1
tail -3 gpurun_out/prof_attn.log
