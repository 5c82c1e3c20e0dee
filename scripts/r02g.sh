mkdir -p gpurun_out/r02g
timeout 200 python scripts/scw_prof.py C4 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02g/scw_launches.csv python scripts/scw_prof.py C4 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/r02g/scw_launches.csv > gpurun_out/r02g/scw_launches.txt; head -8 gpurun_out/r02g/scw_launches.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02g/pytest.log 2>&1; tail -2 gpurun_out/r02g/pytest.log
timeout 400 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/r02g/bench.json 2> gpurun_out/r02g/bench.err
python -c "import json;d=json.load(open('gpurun_out/r02g/bench.json'));print(d['value'],d['ms_per_step'],d['phases_ms'],d['clocks'])"
