# gpu tests, full bench line, ncu launch lists of one exact / one synchronous detection
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g3_tests.log 2>&1; echo tests rc $?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/g3_bench.json 2> gpurun_out/g3_bench.err; echo bench rc $?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
for b in 0 1; do
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/g3_launches_b$b.csv \
   python scripts/prof_run.py --batches $b --runs 2 --no-calibrate > gpurun_out/g3_ncu_b$b.log 2>&1; echo ncu $b rc $?
done
python scripts/prof_run.py --batches 1 --runs 3 > gpurun_out/g3_calib.log 2>&1
