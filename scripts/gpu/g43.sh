O=gpurun_out/g43
timeout 1200 python -m pytest tests/test_rak_gpu.py -x -q -m gpu > ${O}_pytest_rak.log 2>&1; echo "pytest rak rc=$?"; tail -3 ${O}_pytest_rak.log
: > ${O}_time.log
for S in 1 0; do
LP_STAGED=$S timeout 300 python scripts/ab_time.py --config rmat22w --runs 15 --batches 0 --tag "staged=$S" >> ${O}_time.log 2>&1
LP_STAGED=$S timeout 300 python scripts/ab_time.py --config rmat22 --non-strict --runs 9 --batches 0 --tag "staged=$S" >> ${O}_time.log 2>&1
done
LP_FUSE_MAXD=-1 timeout 300 python scripts/ab_time.py --config rmat22 --runs 7 --batches 0 --tag "staged fused strict" >> ${O}_time.log 2>&1
cat ${O}_time.log
LP_DEBUG_ROUNDS=1 timeout 300 python scripts/ab_time.py --config rmat22w --runs 2 --batches 0 2>&1 | tail -45 > ${O}_dbg_w.log
timeout 1500 python -m pytest tests/test_fullsize_gpu.py -x -q -m gpu > ${O}_pytest_full.log 2>&1; echo "pytest full rc=$?"; tail -3 ${O}_pytest_full.log
