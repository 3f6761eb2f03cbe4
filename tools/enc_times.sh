# per-launch device times of the delta tick (warm, serialised) for dense and sparse baselines
python tools/enc_profile.py --ticks 2 > gpurun_out/e.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:k_tick -s 6 -c 4 --csv python tools/enc_profile.py --ticks 2 > gpurun_out/ncu_t.csv 2>&1
python tools/enc_profile.py --sparse --ticks 2 > gpurun_out/e2.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:k_tick -s 6 -c 4 --csv python tools/enc_profile.py --sparse --ticks 2 > gpurun_out/ncu_ts.csv 2>&1
python tools/ncu_csv_times.py gpurun_out/ncu_t.csv gpurun_out/ncu_ts.csv
