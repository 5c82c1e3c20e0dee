set -x
mkdir -p gpurun_out/r02b
timeout 400 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/r02b/bench.json 2> gpurun_out/r02b/bench.err
tail -c 600 gpurun_out/r02b/bench.json
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b/launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r02b/ncu_bench.log 2>&1
python scripts/launch_summary.py gpurun_out/r02b/launches.csv > gpurun_out/r02b/launches_summary.txt
head -40 gpurun_out/r02b/launches_summary.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02b/pytest_gpu.log 2>&1; tail -5 gpurun_out/r02b/pytest_gpu.log
