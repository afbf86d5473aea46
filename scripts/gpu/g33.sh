O=gpurun_out/g33
: > ${O}_ab.log
for rep in 1 2; do
for lib in build/j2_1.so paper_2301_09125_b200/liblabelprop_cuda.so; do
  LP_LIB_PATH=$lib timeout 600 python scripts/ab_time.py --config rmat22 --runs 7 --tag "$lib" >> ${O}_ab.log 2>&1
done
done
timeout 600 python scripts/ab_time.py --config planted --runs 7 --batches 0 >> ${O}_ab.log 2>&1
timeout 600 python scripts/ab_time.py --config planted --non-strict --runs 7 --batches 0 >> ${O}_ab.log 2>&1
LP_LIB_PATH=build/j2_1.so timeout 600 python scripts/ab_time.py --config rmat22w --runs 3 --batches 0 --tag j2_1 >> ${O}_ab.log 2>&1
timeout 600 python scripts/ab_time.py --config rmat22w --runs 3 --batches 0 --tag j2_4 >> ${O}_ab.log 2>&1
cat ${O}_ab.log
LP_DEBUG_ROUNDS=1 timeout 300 python scripts/ab_time.py --config rmat22 --runs 1 --batches 0 2>&1 | tail -40 > ${O}_dbg_rmat22.log
timeout 600 python scripts/prof_mlp.py copra 8 0 20 > ${O}_copra8.log 2>&1
timeout 600 python scripts/prof_mlp.py copra 8 1 20 >> ${O}_copra8.log 2>&1
cat ${O}_copra8.log
