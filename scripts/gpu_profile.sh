# Round profile: plain bench (must exit 0 first), then under ncu: the launch
# list with DRAM bytes per launch (one step), and --set full captures of the
# dominant kernels (exported to CSV on the box; the .ncu-rep files are kept
# only while they fit the 64 MiB return limit).
# Usage: bash scripts/gpu_profile.sh TAG [bench args]
TAG=${1:-r01}; shift
set -x
mkdir -p gpurun_out
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-modes $*"
$B > gpurun_out/${TAG}_bench_plain.json 2> gpurun_out/${TAG}_bench_plain.err || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_ncu_launches.log 2>&1
python scripts/launch_table.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launch_table.txt
N=$(python -c "import json; print(json.load(open('gpurun_out/${TAG}_bench_plain.json'))['rounds'])")
# first dense + first frontier gather of the timed step; one launch of each tally kernel
ncu --set full --clock-control none --import-source on -k regex:k_gather -s $((N*3)) -c 2 \
    -o gpurun_out/${TAG}_gather $B > gpurun_out/${TAG}_ncu_gather.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_warp|k_team|k_small" -s 0 -c 5 \
    -o gpurun_out/${TAG}_tally $B > gpurun_out/${TAG}_ncu_tally.log 2>&1
for r in gather tally; do
  ncu -i gpurun_out/${TAG}_${r}.ncu-rep --page details --csv > gpurun_out/${TAG}_${r}_details.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_${r}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${r}_raw.csv 2>/dev/null
done
du -sh gpurun_out/*
SZ=$(du -sm gpurun_out | cut -f1)
if [ "$SZ" -gt 60 ]; then rm -f gpurun_out/${TAG}_tally.ncu-rep; fi
SZ=$(du -sm gpurun_out | cut -f1)
if [ "$SZ" -gt 60 ]; then rm -f gpurun_out/${TAG}_gather.ncu-rep gpurun_out/*_raw.csv; fi
tail -12 gpurun_out/${TAG}_launch_table.txt
