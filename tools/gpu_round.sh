# One GPU call: parity tests, smoke, bench (with clocks), ncu launch list + full capture of the top kernels.
mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/nvsmi.log
nproc > gpurun_out/nproc.log; lscpu | head -20 >> gpurun_out/nproc.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -25 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-1500
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-600
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 1 --graphs 0 > gpurun_out/prof_launch.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"gemm|attention|exit_head|head_" -c 12 -o gpurun_out/prof_full python tools/profile_step.py --steps 1 --graphs 0 > gpurun_out/prof_full.log 2>&1
tail -3 gpurun_out/prof_full.log
