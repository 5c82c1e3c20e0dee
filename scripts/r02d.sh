mkdir -p gpurun_out/r02d
timeout 200 python scripts/eig_bench.py C4 C3 C5 2>&1 | grep topk | awk 'NR%3==0'
TSK_GQ_DFMA=1 timeout 200 python scripts/eig_bench.py C4 C3 C5 2>&1 | grep topk | awk 'NR%3==0'
PROFILE=1 timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02d/eig_launches.csv python scripts/eig_bench.py C4 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/r02d/eig_launches.csv > gpurun_out/r02d/eig_launches.txt; head -8 gpurun_out/r02d/eig_launches.txt
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_shapes.py tests/test_gpu_full_size.py -x -q 2>&1 | tail -2
