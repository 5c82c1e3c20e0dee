mkdir -p gpurun_out/r02e
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02e/pytest_gpu.log 2>&1; tail -2 gpurun_out/r02e/pytest_gpu.log
for i in 1 2; do timeout 400 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/r02e/bench$i.json 2> gpurun_out/r02e/bench$i.err
python -c "import json;d=json.load(open('gpurun_out/r02e/bench$i.json'));print(d['value'],d['ms_per_step'],d['phases_ms'],d['roofline']['frac'],d['clocks'])"; done
