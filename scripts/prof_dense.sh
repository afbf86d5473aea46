set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-modes"
$B > gpurun_out/p1_bench_plain.json 2> gpurun_out/p1_bench_plain.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none --csv --log-file gpurun_out/p1_launches.csv $B > gpurun_out/p1_ncu_launches.log 2>&1
python scripts/launch_table.py gpurun_out/p1_launches.csv > gpurun_out/p1_launch_table.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_team|k_warp" -s 0 -c 5 \
    -o gpurun_out/p1_tally python scripts/prof_run.py --runs 1 --no-calibrate > gpurun_out/p1_ncu_tally.log 2>&1
ncu -i gpurun_out/p1_tally.ncu-rep --page details --csv > gpurun_out/p1_tally_details.csv 2>/dev/null
python scripts/ncu_summary.py gpurun_out/p1_tally_details.csv > gpurun_out/p1_tally_summary.txt
for k in "k_team<0, 0, 1024" "k_team<0, 0, 256" "k_team<0, 0, 512" "k_warp<0, 0, 1>" "k_warp<0, 0, 0>"; do
  echo "== $k" >> gpurun_out/p1_tally_lines.txt
  python scripts/ncu_srclines.py gpurun_out/p1_tally.ncu-rep "$k" 25 >> gpurun_out/p1_tally_lines.txt 2>&1
done
du -sh gpurun_out/*
