for rep in 1 2; do for F in 64 512 2048 8192 100000; do TSK_PAIR_FOLD=$F timeout 300 python scripts/gram_fold.py C4 2>&1 | tail -1; done; done
