# Round measurement (run on a B200 via gpurun; plain runs first, ncu afterwards):
#   bench lines (ours with parity/modes/configs, the reference arm), COPRA / SLPA lines,
#   the ncu launch list of one exact and one synchronous R-MAT-22 detection (time, DRAM
#   bytes, L2 hit rate, occupancy per launch), ncu_traffic.json, and --set full captures of
#   the tally / gather kernels for rmat22, rmat22w, planted and grid.
#   Usage: bash scripts/round_measure.sh TAG
TAG=${1:-r2c}
mkdir -p gpurun_out
O=gpurun_out/${TAG}
timeout 900 python bench.py --steps 20 --warmup 5 > ${O}_bench_line.json 2> ${O}_bench.err || exit 1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > ${O}_bench_reference.json 2> ${O}_bench_reference.err
timeout 1200 python scripts/bench_mlp.py > ${O}_copra_slpa.jsonl 2> ${O}_copra_slpa.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
for b in 0 1; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file ${O}_launches_b$b.csv \
      python scripts/prof_run.py --batches $b --runs 1 --no-calibrate > ${O}_ncu_launches_b$b.log 2>&1
  python scripts/launch_table.py ${O}_launches_b$b.csv > ${O}_launch_table_b$b.txt
  python scripts/launch_rounds.py ${O}_launches_b$b.csv > ${O}_launch_rounds_b$b.txt
done
python scripts/traffic_json.py ${O}_launches_b0.csv rmat22 > ${O}_ncu_traffic.json
for c in rmat22 rmat22w planted grid; do
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"k_team|k_warp|k_gather|k_small|k_mid|k_first_round" -s 0 -c 14 \
      -o ${O}_full_$c python scripts/prof_run.py --config $c --batches 0 --runs 1 --no-calibrate > ${O}_ncu_full_$c.log 2>&1
  ncu -i ${O}_full_$c.ncu-rep --page details --csv > ${O}_full_details_$c.csv 2>/dev/null
  python scripts/ncu_summary.py ${O}_full_details_$c.csv > ${O}_ncu_full_summary_$c.txt
  python scripts/ncu_lines.py ${O}_full_$c.ncu-rep 12 > ${O}_hot_lines_$c.txt 2>/dev/null
  gzip -f ${O}_full_details_$c.csv
  rm -f ${O}_full_$c.ncu-rep  # (gpurun copies back <= 64 MiB; the summaries above are kept)
done
gzip -f ${O}_launches_b0.csv ${O}_launches_b1.csv
ls -la gpurun_out/ | grep ${TAG}
