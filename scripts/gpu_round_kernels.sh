make -s -C paper_2301_09125_b200/csrc >/dev/null
python scripts/prof_run.py --no-calibrate --runs 1 > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rk.csv python scripts/prof_run.py --no-calibrate --runs 1 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/rk.csv all | tail -150 | awk '{printf "%s %s | ", $1, $2} END {print ""}' | fold -w 240
