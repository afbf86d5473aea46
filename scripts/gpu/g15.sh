M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/g15_launches_b0.csv \
   python scripts/prof_run.py --batches 0 --runs 1 --no-calibrate > /dev/null 2>&1; echo ncu rc $?
