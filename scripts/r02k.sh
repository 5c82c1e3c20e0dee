timeout 200 python scripts/scw_prof.py C4 2>&1
TSK_SCW_CHOL1=1 timeout 200 python scripts/scw_prof.py C4 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/scwl.csv python scripts/scw_prof.py C4 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/scwl.csv | head -9
timeout 900 python -m pytest tests -m gpu -x -q -k "scw or SCW or end_to_end or two_sided or parity or random or c5 or full" 2>&1 | tail -2
timeout 300 python scripts/random_sweep.py core 40 13 2>&1 | tail -1; timeout 300 python scripts/random_sweep.py limits 30 17 2>&1 | tail -1; timeout 300 python scripts/random_sweep.py api 30 19 2>&1 | tail -1
