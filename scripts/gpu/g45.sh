O=gpurun_out/g45
timeout 1200 python -m pytest tests/test_rak_gpu.py tests/test_slpa_gpu.py -x -q -m gpu > ${O}_pytest_rak.log 2>&1; echo "pytest rak rc=$?"; tail -3 ${O}_pytest_rak.log
: > ${O}_time.log
timeout 600 python scripts/ab_time.py --config rmat22 --runs 9 >> ${O}_time.log 2>&1
for c in planted grid; do
  timeout 600 python scripts/ab_time.py --config $c --runs 9 --batches 0 >> ${O}_time.log 2>&1
done
timeout 600 python scripts/ab_time.py --config rmat22 --non-strict --runs 7 --batches 0 >> ${O}_time.log 2>&1
timeout 600 python scripts/ab_time.py --config rmat22w --runs 15 --batches 0 >> ${O}_time.log 2>&1
cat ${O}_time.log
LP_DEBUG_ROUNDS=1 timeout 300 python scripts/ab_time.py --config rmat22 --runs 1 --batches 0 2>&1 | tail -22 > ${O}_dbg_rmat22.log
cat ${O}_dbg_rmat22.log
timeout 1500 python -m pytest tests/test_fullsize_gpu.py -x -q -m gpu > ${O}_pytest_full.log 2>&1; echo "pytest full rc=$?"; tail -3 ${O}_pytest_full.log
