set -x
mkdir -p gpurun_out
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
python scripts/prof_mlp.py copra 1 1 > gpurun_out/pc_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_copra -s 3 -c 3 -o gpurun_out/pc python scripts/prof_mlp.py copra 1 1 > gpurun_out/pc_ncu.log 2>&1
ncu -i gpurun_out/pc.ncu-rep --page details --csv > gpurun_out/pc_details.csv
python scripts/ncu_summary.py gpurun_out/pc_details.csv
for i in 0 1 2; do python scripts/ncu_hot.py gpurun_out/pc.ncu-rep $i 25 > gpurun_out/pc_hot$i.txt; done
ls -la gpurun_out
