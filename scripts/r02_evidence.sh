set -x
mkdir -p gpurun_out/r02
timeout 400 python bench.py > gpurun_out/r02/bench_1gpu.json 2> gpurun_out/r02/bench_1gpu.err
tail -c 300 gpurun_out/r02/bench_1gpu.json
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/bench_launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r02/ncu_bench.log 2>&1
python scripts/launch_summary.py gpurun_out/r02/bench_launches.csv > gpurun_out/r02/bench_launches_summary.txt
head -12 gpurun_out/r02/bench_launches_summary.txt
[ -n "$GRAM_NCU" ] && timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_pair_kernel -c 1 -o gpurun_out/r02/gram_pair_c4 python scripts/gram_one.py 2000 0 4 > gpurun_out/r02/ncu_gram.log 2>&1
timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tf32x3_ts_kernel -s 0 -c 1 -o gpurun_out/r02/scw_sa_c4 python scripts/scw_prof.py > gpurun_out/r02/ncu_sa.log 2>&1
timeout 300 python bench.py --impl reference > gpurun_out/r02/reference_arm.json 2> gpurun_out/r02/reference_arm.err
tail -c 300 gpurun_out/r02/reference_arm.json
timeout 900 python bench.py --config C5 --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r02/bench_c5_1gpu.json 2> gpurun_out/r02/bench_c5.err
tail -c 400 gpurun_out/r02/bench_c5_1gpu.json
