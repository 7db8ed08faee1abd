# quick GPU check: parity tests + bench + launch list (bounded)
mkdir -p gpurun_out
export EEB_SKIP_BUILD=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -2 gpurun_out/bench.log | cut -c1-400
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 1 > gpurun_out/prof_launch.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv
