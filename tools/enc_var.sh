# delta tick + snapshot (bench records) under compile-time variants
for v in "$@"; do
  SS_NVCC_EXTRA="$v" python -c "from paper_2604_02851_b200 import _build; _build.build(force=True)" > /dev/null
  echo "$v: $(python tools/enc_bench.py 2>&1 | tail -1)"
done
