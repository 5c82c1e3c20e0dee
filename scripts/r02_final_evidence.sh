# Round-2 closing evidence (1 x B200): bench line, launch list of the timed steps, ncu --set full of the pair
# Gram and of the SCW SA product, the reference arm, the C5 bench line.  Outputs under gpurun_out/r02z/.
set -x
mkdir -p gpurun_out/r02z
timeout 600 python bench.py > gpurun_out/r02z/bench_1gpu.json 2> gpurun_out/r02z/bench_1gpu.err
tail -c 400 gpurun_out/r02z/bench_1gpu.json
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z/bench_launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r02z/ncu_bench.log 2>&1
python scripts/launch_summary.py gpurun_out/r02z/bench_launches.csv > gpurun_out/r02z/bench_launches_summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_pair_kernel -c 1 -o gpurun_out/r02z/gram_pair_c4 python scripts/gram_one.py 2000 0 4 > gpurun_out/r02z/ncu_gram.log 2>&1
timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tf32x3_ts_kernel -s 0 -c 1 -o gpurun_out/r02z/scw_sa_c4 python scripts/scw_prof.py > gpurun_out/r02z/ncu_sa.log 2>&1
PROFILE=1 timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z/eig_c4_launches.csv python scripts/eig_bench.py C4 > gpurun_out/r02z/eig_c4.log 2>&1
python scripts/launch_summary.py gpurun_out/r02z/eig_c4_launches.csv > gpurun_out/r02z/eig_c4_launches_summary.txt
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z/scw_c4_launches.csv python scripts/scw_prof.py C4 > gpurun_out/r02z/scw_c4.log 2>&1
python scripts/launch_summary.py gpurun_out/r02z/scw_c4_launches.csv > gpurun_out/r02z/scw_c4_launches_summary.txt
timeout 400 python bench.py --impl reference > gpurun_out/r02z/reference_arm.json 2> gpurun_out/r02z/reference_arm.err
timeout 900 python bench.py --config C5 --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r02z/bench_c5_1gpu.json 2> gpurun_out/r02z/bench_c5.err
tail -c 300 gpurun_out/r02z/bench_c5_1gpu.json
