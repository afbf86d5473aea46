mkdir -p gpurun_out
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
python scripts/prof_mlp.py copra 8 0 > gpurun_out/pc2_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_copra" -s 3 -c 6 -o gpurun_out/pc2 python scripts/prof_mlp.py copra 8 0 > gpurun_out/pc2_ncu.log 2>&1
ncu -i gpurun_out/pc2.ncu-rep --page details --csv > gpurun_out/pc2_details.csv
python scripts/ncu_summary.py gpurun_out/pc2_details.csv | grep -E "==|Duration|Achieved Occ|Issue Slots|Eligible Warps"
python scripts/ncu_srclines.py gpurun_out/pc2.ncu-rep "k_copra_team" 25
