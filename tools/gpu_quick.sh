python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>gpurun_out/b.err
python -c "import json;d=json.load(open('gpurun_out/b.json'));print(round(d['value'],1),d['kernel_ms_per_step'])"
