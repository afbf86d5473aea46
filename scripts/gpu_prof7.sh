mkdir -p gpurun_out
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
python scripts/prof_run.py --batches 1 > gpurun_out/prof7_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sync_v5.csv python scripts/prof_run.py --batches 1 > gpurun_out/ncu7l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_team -s 0 -c 4 -o gpurun_out/prof7_team python scripts/prof_run.py --batches 1 > gpurun_out/ncu7a.log 2>&1
python scripts/launch_table.py gpurun_out/launches_sync_v5.csv all | grep -v "cub\|k_plan\|k_iota\|k_i64\|k_nbr\|k_degree\|k_gtab\|k_set\|k_init\|k_reset\|k_calib"
