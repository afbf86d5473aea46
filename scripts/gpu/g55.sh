O=gpurun_out/g55_knobs.log; : > $O
run() { env "$@" timeout 300 python scripts/ab_time.py --config rmat22 --runs 7 --batches 0 --tag "$*" >> $O 2>&1; 
        env "$@" timeout 300 python scripts/ab_time.py --config grid --runs 5 --batches 0 --tag "$*" >> $O 2>&1; }
run LP_NONE=1
run LP_LOOP_ROWS=32768 LP_LOOP_MAX_QUEUE=262144
run LP_LOOP_ROWS=131072 LP_LOOP_MAX_QUEUE=1000000
run LP_LOOP_ROWS=2048
run LP_LOOP_BLOCKS=2
cat $O
