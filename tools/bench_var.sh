# bench value + per-class kernel ms under compile-time variants (SS_NVCC_EXTRA -D overrides)
for v in "$@"; do
  SS_NVCC_EXTRA="$v" python -c "from paper_2604_02851_b200 import _build; _build.build(force=True)" > /dev/null
  python bench.py --no-cpu-baseline --no-e2e --step-only --steps 10 > gpurun_out/bv.json 2>gpurun_out/bv.err
  echo "$v"; python -c "import json;d=json.load(open('gpurun_out/bv.json'));print(round(d['value'],1),d['kernel_ms_per_step'])"
done
