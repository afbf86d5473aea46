O=gpurun_out/g42_knobs.log; : > $O
run() { env "$@" timeout 300 python scripts/ab_time.py --config rmat22w --runs 15 --batches 0 --tag "$*" >> $O 2>&1; }
run LP_DENSE_FRAC=0.35
run LP_DENSE_FRAC=0.5
run LP_DENSE_FRAC=0.7
run LP_DENSE_FRAC=1.01
run LP_DENSE_FRAC=0.35 LP_MID_MAX=0
run LP_DENSE_FRAC=0.35 LP_ID_SINGLE_W=0
run LP_DENSE_FRAC=0.35 LP_FIRST_ROUND=0
cat $O
