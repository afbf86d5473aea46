set -x
mkdir -p gpurun_out
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
python scripts/prof_run.py --runs 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rmat22_exact.csv python scripts/prof_run.py > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_block -s 1 -c 2 -o gpurun_out/prof_block python scripts/prof_run.py > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_warp -c 1 -s 1 -o gpurun_out/prof_warp python scripts/prof_run.py > gpurun_out/ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_small -c 1 -s 1 -o gpurun_out/prof_small python scripts/prof_run.py > gpurun_out/ncu4.log 2>&1
cat gpurun_out/prof_plain.log; tail -3 gpurun_out/ncu*.log
