O=gpurun_out/g47
timeout 1200 python -m pytest tests/test_rak_gpu.py -x -q -m gpu > ${O}_pytest_rak.log 2>&1; echo "pytest rak rc=$?"; tail -3 ${O}_pytest_rak.log
: > ${O}_time.log
timeout 600 python scripts/ab_time.py --config rmat22 --runs 9 >> ${O}_time.log 2>&1
for c in planted grid; do
  timeout 600 python scripts/ab_time.py --config $c --runs 9 --batches 0 >> ${O}_time.log 2>&1
done
cat ${O}_time.log
