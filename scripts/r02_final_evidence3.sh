# Round-2 closing evidence (1 x B200): bench line, launch lists of the step / eigensolver / SCW, C5 bench line, smoke, GPU tests, random sweeps.  Outputs under gpurun_out/r02z/.
set -x
mkdir -p gpurun_out/r02z
timeout 600 python bench.py > gpurun_out/r02z/bench_1gpu.json 2> gpurun_out/r02z/bench_1gpu.err
tail -c 400 gpurun_out/r02z/bench_1gpu.json
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z/bench_launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r02z/ncu_bench.log 2>&1
python scripts/launch_summary.py gpurun_out/r02z/bench_launches.csv > gpurun_out/r02z/bench_launches_summary.txt
PROFILE=1 timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z/eig_c4_launches.csv python scripts/eig_bench.py C4 > gpurun_out/r02z/eig_c4.log 2>&1
python scripts/launch_summary.py gpurun_out/r02z/eig_c4_launches.csv > gpurun_out/r02z/eig_c4_launches_summary.txt
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z/scw_c4_launches.csv python scripts/scw_prof.py C4 > gpurun_out/r02z/scw_c4.log 2>&1
python scripts/launch_summary.py gpurun_out/r02z/scw_c4_launches.csv > gpurun_out/r02z/scw_c4_launches_summary.txt
timeout 900 python bench.py --config C5 --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r02z/bench_c5_1gpu.json 2> gpurun_out/r02z/bench_c5.err
tail -c 300 gpurun_out/r02z/bench_c5_1gpu.json
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02z/smoke.log 2>&1; tail -2 gpurun_out/r02z/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02z/pytest_gpu.log 2>&1; tail -2 gpurun_out/r02z/pytest_gpu.log
for s in core spectra; do timeout 600 python scripts/random_sweep.py $s > gpurun_out/r02z/random_sweep_$s.log 2>&1; tail -3 gpurun_out/r02z/random_sweep_$s.log; done
