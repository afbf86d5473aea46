set -x
mkdir -p gpurun_out
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
timeout 900 python -m pytest tests/test_rak_gpu.py -x -q 2>&1 | tail -3
python scripts/prof_run.py --batches 1 > gpurun_out/prof3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_warp -s 3 -c 1 -o gpurun_out/prof3_warp python scripts/prof_run.py --batches 1 > gpurun_out/ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_small -s 9 -c 3 -o gpurun_out/prof3_small python scripts/prof_run.py --batches 1 > gpurun_out/ncu4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_team -s 6 -c 2 -o gpurun_out/prof3_team python scripts/prof_run.py --batches 1 > gpurun_out/ncu5.log 2>&1
tail -2 gpurun_out/ncu*.log
