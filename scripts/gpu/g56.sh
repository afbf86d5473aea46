LP_DEBUG_ROUNDS=1 timeout 300 python scripts/ab_time.py --config rmat22 --non-strict --runs 1 --batches 0 2>&1 | tail -48 > gpurun_out/g56_dbg_ns.log
timeout 300 python scripts/prof_run.py --config rmat22 --non-strict --runs 3 --no-calibrate 2>&1 | cut -c1-330 > gpurun_out/g56_prof_ns.log
cat gpurun_out/g56_prof_ns.log; grep "dense\|first\|frontier)" gpurun_out/g56_dbg_ns.log | tail -24
