# eigensolver kernels at C4 under ncu (one launch each) + SCW timing
mkdir -p gpurun_out/r02c
timeout 200 python scripts/scw_prof.py C4 > gpurun_out/r02c/scw_time.log 2>&1; cat gpurun_out/r02c/scw_time.log
for k in gq_f64_kernel trd_kernel chol_scale_kernel trsm2_kernel tev_kernel gemm_tn_f64_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 6 -c 1 -o gpurun_out/r02c/$k python scripts/eig_bench.py C4 > gpurun_out/r02c/ncu_$k.log 2>&1
done
ls gpurun_out/r02c
