mkdir -p gpurun_out
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
python scripts/prof_run.py --batches 1 > gpurun_out/prof6_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_warp -s 0 -c 2 -o gpurun_out/prof6_warp_s1 python scripts/prof_run.py --batches 1 > gpurun_out/ncu6a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_warp -s 4 -c 2 -o gpurun_out/prof6_warp_s3 python scripts/prof_run.py --batches 1 > gpurun_out/ncu6b.log 2>&1
ls gpurun_out/prof6*
