# Round-2 closing bench refresh after the late SCW / eigensolver changes (1 x B200): bench line, launch lists of
# the step / eigensolver / SCW, C5 bench line.  Outputs under gpurun_out/r02y/.
set -x
mkdir -p gpurun_out/r02y
timeout 600 python bench.py > gpurun_out/r02y/bench_1gpu.json 2> gpurun_out/r02y/bench_1gpu.err
tail -c 400 gpurun_out/r02y/bench_1gpu.json
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02y/bench_launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r02y/ncu_bench.log 2>&1
python scripts/launch_summary.py gpurun_out/r02y/bench_launches.csv > gpurun_out/r02y/bench_launches_summary.txt
PROFILE=1 timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02y/eig_c4_launches.csv python scripts/eig_bench.py C4 > gpurun_out/r02y/eig_c4.log 2>&1
python scripts/launch_summary.py gpurun_out/r02y/eig_c4_launches.csv > gpurun_out/r02y/eig_c4_launches_summary.txt
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02y/scw_c4_launches.csv python scripts/scw_prof.py C4 > gpurun_out/r02y/scw_c4.log 2>&1
python scripts/launch_summary.py gpurun_out/r02y/scw_c4_launches.csv > gpurun_out/r02y/scw_c4_launches_summary.txt
timeout 900 python bench.py --config C5 --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r02y/bench_c5_1gpu.json 2> gpurun_out/r02y/bench_c5.err
tail -c 300 gpurun_out/r02y/bench_c5_1gpu.json
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02y/smoke.log 2>&1; tail -2 gpurun_out/r02y/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02y/pytest_gpu.log 2>&1; tail -2 gpurun_out/r02y/pytest_gpu.log
