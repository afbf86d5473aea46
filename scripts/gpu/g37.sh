O=gpurun_out/g37_knobs.log; : > $O
run() { env "$@" timeout 300 python scripts/ab_time.py --config rmat22w --runs 3 --batches 0 --tag "$*" >> $O 2>&1; 
        env "$@" timeout 300 python scripts/ab_time.py --config rmat22 --non-strict --runs 3 --batches 0 --tag "$*" >> $O 2>&1; }
run LP_NONE=1
run LP_DENSE_FRAC=0.2
run LP_DENSE_FRAC=0.5
run LP_DENSE_FRAC=0.7
run LP_DENSE_FRAC=1.01
run LP_FUSE_MAXD=-1
run LP_FUSE_MAXD=-1 LP_DENSE_FRAC=0.7
run LP_FUSE_MAXD=64
run LP_PULL_ROUNDS=1
run LP_ID_SINGLE_W=0 LP_ID_SINGLE_RANDOM=0
run LP_MARGIN=0
run LP_FIRST_ROUND=0
cat $O
