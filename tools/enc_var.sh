# delta tick device time under compile-time variants (SS_NVCC_EXTRA -D overrides)
for v in "$@"; do
  SS_NVCC_EXTRA="$v" python -c "from paper_2604_02851_b200 import _build; _build.build(force=True)" > /dev/null
  echo "$v: $(python tools/enc_time.py) | $(python tools/enc_time.py --sparse)"
done
