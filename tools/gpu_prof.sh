# ncu: launch list of one decode step + full capture of the top kernels.
mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 1 > gpurun_out/prof_launch.log 2>&1
tail -3 gpurun_out/prof_launch.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tc -c 4 -o gpurun_out/prof_gemm python tools/profile_step.py --steps 1 > gpurun_out/prof_gemm.log 2>&1
tail -3 gpurun_out/prof_gemm.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attention -c 2 -o gpurun_out/prof_attn python tools/profile_step.py --steps 1 > gpurun_out/prof_attn.log 2>&1
tail -3 gpurun_out/prof_attn.log
