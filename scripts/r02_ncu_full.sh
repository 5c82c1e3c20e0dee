# Round-2 closing ncu --set full captures on the final code (1 x B200): the pair Gram at full C4 and the SCW SA
# product (one scw_error at C4).  Each command runs once without ncu first (exit 0) as the profiling recipe asks.
# Outputs under gpurun_out/r02n/.
set -x
mkdir -p gpurun_out/r02n
timeout 300 python scripts/gram_one.py 2000 0 4 > gpurun_out/r02n/plain_gram.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_pair_kernel -c 1 -o gpurun_out/r02n/gram_pair_c4 python scripts/gram_one.py 2000 0 4 > gpurun_out/r02n/ncu_gram.log 2>&1
timeout 300 python scripts/scw_prof.py > gpurun_out/r02n/plain_sa.log 2>&1 && \
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tf32x3_ts_kernel -s 0 -c 1 -o gpurun_out/r02n/scw_sa_c4 python scripts/scw_prof.py > gpurun_out/r02n/ncu_sa.log 2>&1
ls -la gpurun_out/r02n
