mkdir -p gpurun_out
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
python scripts/prof_run.py --batches 1 > gpurun_out/prof5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_team -s 0 -c 1 -o gpurun_out/prof5_team python scripts/prof_run.py --batches 1 > gpurun_out/ncu5a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_team -s 4 -c 1 -o gpurun_out/prof5_team_s3 python scripts/prof_run.py --batches 1 > gpurun_out/ncu5b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_warp -s 2 -c 1 -o gpurun_out/prof5_warp_s3 python scripts/prof_run.py --batches 1 > gpurun_out/ncu5c.log 2>&1
ls gpurun_out/prof5*
