# Round measurement: bench lines for every BASELINE RAK config, COPRA/SLPA lines,
# then the ncu launch list (+DRAM bytes) and --set full captures of the dominant
# kernels of the default bench command.  Usage: bash scripts/round_measure.sh TAG
TAG=${1:-r04}
mkdir -p gpurun_out
O=gpurun_out/${TAG}
timeout 600 python bench.py > ${O}_bench_line.json 2> ${O}_bench.err || exit 1
for c in rmat22w planted grid; do
  timeout 900 python bench.py --config $c --steps 5 > ${O}_bench_$c.json 2> ${O}_bench_$c.err
done
timeout 900 python bench.py --non-strict --steps 5 --no-modes > ${O}_bench_nonstrict.json 2> ${O}_bench_nonstrict.err
timeout 900 python bench.py --batches 1 --steps 10 --no-modes > ${O}_bench_sync.json 2> ${O}_bench_sync.err
timeout 1200 python scripts/bench_mlp.py > ${O}_copra_slpa.jsonl 2> ${O}_copra_slpa.err
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-modes"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none --csv --log-file ${O}_launches.csv $B > ${O}_ncu_launches.log 2>&1
python scripts/launch_table.py ${O}_launches.csv > ${O}_launch_table.txt
python scripts/traffic_json.py ${O}_launches.csv rmat22 > ${O}_ncu_traffic.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_team|k_warp|k_gather" -s 0 -c 7 \
    -o ${O}_full python scripts/prof_run.py --runs 1 --no-calibrate > ${O}_ncu_full.log 2>&1
ncu -i ${O}_full.ncu-rep --page details --csv > ${O}_full_details.csv 2>/dev/null
python scripts/ncu_summary.py ${O}_full_details.csv > ${O}_ncu_full_summary.txt
gzip -f ${O}_launches.csv
ls -la gpurun_out/ | grep ${TAG}
