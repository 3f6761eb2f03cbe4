# bench value (step only) for each "lanes:x" argument (x ignored; SS_VIEW_LANES = lanes)
for v in "$@"; do
  SS_VIEW_LANES=${v%%:*} SS_CHAIN_EVERY=${v##*:} python bench.py --no-cpu-baseline --no-e2e --step-only --steps 20 > gpurun_out/lv.json 2>gpurun_out/lv.err
  echo "lanes:chain=$v"; python -c "import json;d=json.load(open('gpurun_out/lv.json'));print(round(d['value'],1),d['kernel_ms_per_step']['chain_rule'])" || tail -5 gpurun_out/lv.err
done
