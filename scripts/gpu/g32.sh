# frontier loop: parity + timing
O=gpurun_out/g32
timeout 900 python -m pytest tests/test_rak_gpu.py -x -q -m gpu > ${O}_pytest_rak.log 2>&1; echo "pytest rak rc=$?" 
for c in planted grid rmat22 rmat22w; do
  for L in 0 8192; do
    LP_LOOP_ROWS=$L timeout 600 python scripts/ab_time.py --config $c --runs 5 --batches 0 --tag "loop=$L" >> ${O}_time.log 2>&1
  done
done
LP_LOOP_ROWS=0 timeout 600 python scripts/ab_time.py --config planted --non-strict --runs 5 --batches 0 --tag "loop=0" >> ${O}_time.log 2>&1
timeout 600 python scripts/ab_time.py --config planted --non-strict --runs 5 --batches 0 --tag "loop=8192" >> ${O}_time.log 2>&1
LP_DEBUG_ROUNDS=1 timeout 300 python scripts/ab_time.py --config planted --runs 1 --batches 0 > ${O}_dbg_planted.log 2>&1
cat ${O}_time.log; tail -5 ${O}_pytest_rak.log
timeout 1500 python -m pytest tests/test_fullsize_gpu.py -x -q -m gpu > ${O}_pytest_full.log 2>&1; echo "pytest full rc=$?"; tail -3 ${O}_pytest_full.log
