O=gpurun_out/g53
: > ${O}_ab.log
for rep in 1 2; do
for lib in paper_2301_09125_b200/liblabelprop_cuda.so build/carry.so; do
  LP_LIB_PATH=$lib timeout 600 python scripts/ab_time.py --config rmat22 --runs 7 --tag "$lib" >> ${O}_ab.log 2>&1
  LP_LIB_PATH=$lib timeout 600 python scripts/ab_time.py --config planted --runs 7 --batches 0 --tag "$lib" >> ${O}_ab.log 2>&1
  LP_LIB_PATH=$lib timeout 600 python scripts/ab_time.py --config grid --runs 5 --batches 0 --tag "$lib" >> ${O}_ab.log 2>&1
done
done
cat ${O}_ab.log
LP_LIB_PATH=build/carry.so timeout 1200 python -m pytest tests/test_rak_gpu.py -x -q -m gpu > ${O}_pytest_rak.log 2>&1; echo "pytest rak rc=$?"; tail -3 ${O}_pytest_rak.log
LP_LIB_PATH=build/carry.so timeout 1500 python -m pytest tests/test_fullsize_gpu.py -x -q -m gpu > ${O}_pytest_full.log 2>&1; echo "pytest full rc=$?"; tail -3 ${O}_pytest_full.log
