# Round-2 evidence: launch list of the step-only bench (same command as the
# bench, K=2, W=1) and ncu --set full of the step's kernels (one launch each).
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r02_launches_step.csv \
    python bench.py --step-only --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none \
    -k regex:"k_blend_bwd|k_blend_fwd2|k_chain_views|k_sh_grad_rows|k_sum_partials|k_adam<|k_preprocess|k_onesweep|k_emit_warp" \
    -s 40 -c 12 -o gpurun_out/r02_step_full -f python tools/profile_step.py --steps 1 > gpurun_out/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_tick_fused|k_snap_body" -c 2 \
    -o gpurun_out/r02_codec_full -f python tools/enc_bench.py > gpurun_out/ncu_codec.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/r02_launches_step.csv
