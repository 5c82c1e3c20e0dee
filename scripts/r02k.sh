for v in "" "TSK_TN_CLUSTER=16" "TSK_TN_SPLIT=1"; do echo "== $v"; env $v timeout 200 python scripts/eig_bench.py C4 C3 2>&1 | grep topk | awk 'NR%3==0'; done
PROFILE=1 timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/eigl.csv python scripts/eig_bench.py C4 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/eigl.csv > gpurun_out/eigl.txt 2>/dev/null; head -12 gpurun_out/eigl.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_shapes.py tests/test_gpu_full_size.py tests/test_gpu_matrix_free.py tests/test_gpu_end_to_end.py -x -q 2>&1 | tail -1
timeout 300 python scripts/random_sweep.py spectra 30 59 2>&1 | tail -1; timeout 300 python scripts/random_sweep.py f_rows 12 61 2>&1 | tail -1
