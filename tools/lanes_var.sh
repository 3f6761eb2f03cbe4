# bench value (step only) for each SS_VIEW_LANES value given
for v in "$@"; do
  SS_VIEW_LANES=$v python bench.py --no-cpu-baseline --no-e2e --step-only --steps 10 > gpurun_out/lv.json 2>gpurun_out/lv.err
  echo "lanes=$v"; python -c "import json;d=json.load(open('gpurun_out/lv.json'));print(round(d['value'],1),d['kernel_ms_per_step'])" || tail -5 gpurun_out/lv.err
done
