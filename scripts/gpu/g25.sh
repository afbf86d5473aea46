# re-tune policy knobs after the round-2 changes (exact + synchronous R-MAT-22)
O=gpurun_out/g25_knobs.log; : > $O
run() { env "$@" python scripts/ab_time.py --config rmat22 --runs 5 --tag "$*" >> $O 2>&1; }
run LP_NONE=1
run LP_REG_EST=32
run LP_REG_EST=24
run LP_FIRST_EST_DIV=8
run LP_FIRST_EST_DIV=2
run LP_FIRST_EST_MIN=64
run LP_DENSE_FRAC=0.25
run LP_DENSE_FRAC=0.5
run LP_CARRY_FRAC=0.7
run LP_PUSH_DIV=6
run LP_MARK_SCAN_DIV=4
run LP_WARP0_MAXD=1024
run LP_MID_MAX=32
run LP_NONE=2
