set -x
mkdir -p gpurun_out
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
python scripts/prof_run.py --no-calibrate > gpurun_out/p2_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_warp|k_team|k_mark|k_small" -s 0 -c 12 -o gpurun_out/p2 python scripts/prof_run.py --no-calibrate > gpurun_out/p2_ncu.log 2>&1
ncu -i gpurun_out/p2.ncu-rep --page details --csv > gpurun_out/p2_details.csv
python scripts/ncu_summary.py gpurun_out/p2_details.csv | grep -E "==|Duration|Achieved Occ|Issue Slots|Eligible Warps|Threads Per"
python scripts/ncu_srclines.py gpurun_out/p2.ncu-rep "" 14 > gpurun_out/p2_lines.txt
