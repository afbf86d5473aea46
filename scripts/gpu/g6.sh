# fused gather A/B + parity
O=gpurun_out/g6_ab.log; : > $O
LP_FUSED=0 python scripts/ab_time.py --tag two-phase >> $O 2>&1
python scripts/ab_time.py --tag fused >> $O 2>&1
LP_FUSED=0 python scripts/ab_time.py --config grid --tag two-phase >> $O 2>&1
python scripts/ab_time.py --config grid --tag fused >> $O 2>&1
LP_FUSED=0 python scripts/ab_time.py --config planted --tag two-phase >> $O 2>&1
python scripts/ab_time.py --config planted --tag fused >> $O 2>&1
timeout 900 python -m pytest tests/test_rak_gpu.py tests/test_fullsize_gpu.py -x -q -k "rak or rmat22 or planted or grid or nonstrict or Reference or exact" > gpurun_out/g6_tests.log 2>&1; echo tests rc $? >> $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/g6_launches_b1.csv \
   python scripts/prof_run.py --batches 1 --runs 1 --no-calibrate > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/g6_launches_b0.csv \
   python scripts/prof_run.py --batches 0 --runs 1 --no-calibrate > /dev/null 2>&1
