# L2 reuse of the delta tick's residual inputs: application replay (no
# save/restore between passes, no cache flush), bench-like L2 flush per tick
python tools/enc_profile.py --flush --ticks 2 > gpurun_out/e.log 2>&1 && \
ncu --replay-mode application --cache-control none --clock-control none -k regex:k_tick -s 3 -c 2 --csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum \
  python tools/enc_profile.py --flush --ticks 2 > gpurun_out/ncu_l2.csv 2>&1
python tools/ncu_metrics.py gpurun_out/ncu_l2.csv
