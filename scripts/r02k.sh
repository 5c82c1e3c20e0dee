timeout 200 python scripts/scw_prof.py C4 2>&1 | grep scw_error
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/scwl.csv python scripts/scw_prof.py C4 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/scwl.csv > gpurun_out/scwl.txt 2>/dev/null; head -8 gpurun_out/scwl.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "scw or SCW or end_to_end or parity or c5 or full" 2>&1 | tail -1
