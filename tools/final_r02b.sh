set -x
ncu --set full --import-source on --clock-control none -k regex:"k_blend_bwd" -c 1 -o gpurun_out/r02_bwd_full -f python tools/profile_step.py --steps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_chain_views|k_sh_grad_rows|k_adam" -c 4 -o gpurun_out/r02_tail_full -f python tools/profile_step.py --steps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_sum_partials" -c 1 -o gpurun_out/r02_sump_full -f python tools/profile_step.py --steps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_snap_body" -c 1 -o gpurun_out/r02_snap_full -f python tools/snap_profile.py > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
