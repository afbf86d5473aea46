O=gpurun_out/g44
timeout 1200 python -m pytest tests/test_rak_gpu.py tests/test_slpa_gpu.py -x -q -m gpu > ${O}_pytest_rak.log 2>&1; echo "pytest rak rc=$?"; tail -3 ${O}_pytest_rak.log
: > ${O}_time.log
for c in rmat22 planted grid; do
  timeout 600 python scripts/ab_time.py --config $c --runs 9 --batches 0 >> ${O}_time.log 2>&1
done
timeout 600 python scripts/ab_time.py --config rmat22 --non-strict --runs 7 --batches 0 >> ${O}_time.log 2>&1
timeout 600 python scripts/ab_time.py --config rmat22w --runs 15 --batches 0 >> ${O}_time.log 2>&1
cat ${O}_time.log
