set -x
mkdir -p gpurun_out
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
python scripts/prof_run.py --batches 1 > gpurun_out/prof2_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rmat22_sync_v2.csv python scripts/prof_run.py --batches 1 > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_team -s 2 -c 4 -o gpurun_out/prof2_team python scripts/prof_run.py --batches 1 > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_warp -s 1 -c 2 -o gpurun_out/prof2_warp python scripts/prof_run.py --batches 1 > gpurun_out/ncu3.log 2>&1
cat gpurun_out/prof2_plain.log
