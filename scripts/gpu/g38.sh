O=gpurun_out/g38_knobs.log; : > $O
run() { env "$@" timeout 300 python scripts/ab_time.py --config rmat22w --runs 3 --batches 0 --tag "$*" >> $O 2>&1; 
        env "$@" timeout 300 python scripts/ab_time.py --config rmat22 --non-strict --runs 3 --batches 0 --tag "$*" >> $O 2>&1; }
run LP_FUSE_MAXD=-1
run LP_FUSE_MAXD=-1 LP_DENSE_FRAC=0.25
run LP_FUSE_MAXD=-1 LP_DENSE_FRAC=0.45
run LP_FUSE_MAXD=-1 LP_ID_SINGLE_W=0 LP_ID_SINGLE_RANDOM=0
run LP_FUSE_MAXD=-1 LP_TWO_TEAM_W=0
run LP_FUSE_MAXD=-1 LP_FIRST_ROUND=0
run LP_FUSE_MAXD=-1 LP_MID_MAX=0
run LP_FUSE_MAXD=-1 LP_L2_PERSIST=0
run LP_FUSE_MAXD=-1 LP_CARRY_FRAC=0.7
run LP_FUSE_MAXD=-1 LP_LOOP_ROWS=0
LP_FUSE_MAXD=-1 timeout 300 python scripts/ab_time.py --config rmat22 --runs 5 --tag "fuse all" >> $O 2>&1
LP_FUSE_MAXD=-1 timeout 300 python scripts/ab_time.py --config grid --runs 3 --batches 0 --tag "fuse all" >> $O 2>&1
LP_FUSE_MAXD=-1 timeout 300 python scripts/ab_time.py --config planted --non-strict --runs 3 --batches 0 --tag "fuse all" >> $O 2>&1
cat $O
LP_FUSE_MAXD=-1 LP_DEBUG_ROUNDS=1 timeout 300 python scripts/ab_time.py --config rmat22w --runs 1 --batches 0 2>&1 | tail -60 > gpurun_out/g38_dbg_w.log
