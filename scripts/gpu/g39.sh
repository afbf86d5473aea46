O=gpurun_out/g39_knobs.log; : > $O
run() { env "$@" timeout 300 python scripts/ab_time.py --config rmat22w --runs 7 --batches 0 --tag "$*" >> $O 2>&1; 
        env "$@" timeout 300 python scripts/ab_time.py --config rmat22 --non-strict --runs 7 --batches 0 --tag "$*" >> $O 2>&1; }
run LP_NONE=1
run LP_WAVES_MID=1
run LP_WAVES_MID=2
run LP_WAVES_MID=4
run LP_WAVES_MID=8
cat $O
LP_WAVES_MID=1 LP_DEBUG_ROUNDS=1 timeout 300 python scripts/ab_time.py --config rmat22w --runs 1 --batches 0 2>&1 | tail -60 > gpurun_out/g39_dbg_w.log
