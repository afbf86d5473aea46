LP_DEBUG_ROUNDS=1 python scripts/ab_time.py --config rmat22 --batches 0 --runs 1 > gpurun_out/g21_dbg.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/g21_launches_b0.csv \
   python scripts/prof_run.py --batches 0 --runs 1 --no-calibrate > /dev/null 2>&1
