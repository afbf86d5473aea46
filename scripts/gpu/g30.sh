# per-round launch lists for the slow configs (weighted, non-strict, planted)
O=gpurun_out/g30
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
for c in rmat22w planted; do
  python scripts/prof_run.py --config $c --runs 3 --no-calibrate > ${O}_prof_$c.log 2>&1
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file ${O}_launches_$c.csv \
      python scripts/prof_run.py --config $c --runs 1 --no-calibrate > ${O}_ncu_$c.log 2>&1
  python scripts/launch_rounds.py ${O}_launches_$c.csv > ${O}_rounds_$c.txt
  gzip -f ${O}_launches_$c.csv
done
python scripts/prof_run.py --config rmat22 --non-strict --runs 3 --no-calibrate > ${O}_prof_ns.log 2>&1
timeout 900 ncu --metrics $M --clock-control none --csv --log-file ${O}_launches_ns.csv \
    python scripts/prof_run.py --config rmat22 --non-strict --runs 1 --no-calibrate > ${O}_ncu_ns.log 2>&1
python scripts/launch_rounds.py ${O}_launches_ns.csv > ${O}_rounds_ns.txt
gzip -f ${O}_launches_ns.csv
python scripts/bench_mlp.py > ${O}_copra_slpa.jsonl 2> ${O}_copra_slpa.err
tail -3 ${O}_prof_*.log
