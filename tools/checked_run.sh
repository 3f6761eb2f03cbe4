# the bounds-checked build (-DSS_CHECKS) through the GPU suite, the sanitizer target and a short bench
set -x
SS_NVCC_EXTRA=-DSS_CHECKS python -m paper_2604_02851_b200._build --force > gpurun_out/checked_build.log 2>&1
python -m pytest tests -m gpu -q 2>&1 | tail -2
python tools/sanitize_target.py 2>&1 | tail -1
python bench.py --step-only --steps 3 --no-cpu-baseline > gpurun_out/checked_bench.json 2>gpurun_out/checked_bench.err; echo bench_rc=$?
