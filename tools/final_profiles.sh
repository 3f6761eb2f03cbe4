# Round-end evidence: full bench line, ncu launch list of the same command,
# ncu --set full of the step's kernels.  Outputs in gpurun_out/.
set -x
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/profile_step.py --steps 1 > gpurun_out/pstep.log 2>&1 && \
ncu --set full --import-source on --clock-control none \
    -k regex:"k_blend_bwd|k_blend_fwd2|k_chain|k_sum_partials|k_sh_grad|k_emit_warp|k_adam" \
    -c 14 -o gpurun_out/step_full -f python tools/profile_step.py --steps 1 > gpurun_out/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_preprocess|k_onesweep" \
    -c 8 -o gpurun_out/step_full2 -f python tools/profile_step.py --steps 1 > gpurun_out/ncu_full2.log 2>&1
ls -la gpurun_out/
