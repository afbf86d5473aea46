set -x
mkdir -p gpurun_out
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
python scripts/prof_run.py --no-calibrate > gpurun_out/pr_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_warp|k_team" -s 12 -c 4 -o gpurun_out/pr python scripts/prof_run.py --no-calibrate > gpurun_out/pr_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_warp|k_team" -s 0 -c 4 -o gpurun_out/pr1 python scripts/prof_run.py --no-calibrate > gpurun_out/pr1_ncu.log 2>&1
ncu -i gpurun_out/pr.ncu-rep --page details --csv > gpurun_out/pr_details.csv
ncu -i gpurun_out/pr1.ncu-rep --page details --csv > gpurun_out/pr1_details.csv
python scripts/ncu_summary.py gpurun_out/pr_details.csv | grep -E "==|Duration|Occupancy|Issue|Eligible|L1/TEX Cache|Threads Per"
python scripts/ncu_summary.py gpurun_out/pr1_details.csv | grep -E "==|Duration|Occupancy|Issue|Eligible|L1/TEX Cache|Threads Per"
for i in 0 1 2 3; do python scripts/ncu_hot.py gpurun_out/pr.ncu-rep $i 30 > gpurun_out/pr_hot$i.txt; python scripts/ncu_hot.py gpurun_out/pr1.ncu-rep $i 30 > gpurun_out/pr1_hot$i.txt; done
