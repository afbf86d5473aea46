mkdir -p gpurun_out
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
python scripts/prof_run.py --batches 1 > gpurun_out/prof4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_team -s 0 -c 2 -o gpurun_out/prof4_team python scripts/prof_run.py --batches 1 > gpurun_out/ncu4a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_warp -s 0 -c 1 -o gpurun_out/prof4_warp python scripts/prof_run.py --batches 1 > gpurun_out/ncu4b.log 2>&1
ls -la gpurun_out/prof4*
