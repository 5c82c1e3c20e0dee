python scripts/gram_pair_time.py 1080,1920,2000 "0:4:0:,0:4:0:,0:4:0:" 2>&1 | grep mode
timeout 300 python scripts/gram_fold.py C4 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py tests/test_gpu_streaming.py -x -q 2>&1 | tail -1
