O=gpurun_out/g40_knobs.log; : > $O
run() { env "$@" timeout 300 python scripts/ab_time.py --config rmat22w --runs 9 --batches 0 --tag "$*" >> $O 2>&1; 
        env "$@" timeout 300 python scripts/ab_time.py --config rmat22 --non-strict --runs 5 --batches 0 --tag "$*" >> $O 2>&1; }
run LP_HUB_ORDER=0
run LP_HUB_ORDER=1
run LP_HUB_ORDER=2
cat $O
for o in 1 2; do LP_HUB_ORDER=$o LP_DEBUG_ROUNDS=1 timeout 300 python scripts/ab_time.py --config rmat22w --runs 2 --batches 0 2>&1 | grep "dense\|first\|strict" | tail -30 > gpurun_out/g40_dbg_w$o.log; done
