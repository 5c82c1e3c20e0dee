for R in 1e7 1e8 1e9 1e10; do for O in 16 24 32; do echo "R=$R OS=$O"; TSK_EIG_RANGE=$R OVERSAMPLE=$O timeout 200 python scripts/eig_bench.py C4 C3 C5 2>&1 | grep topk | awk 'NR%3==0'; done; done
