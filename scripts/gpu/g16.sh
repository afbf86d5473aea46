CONFIGS="rmat22w rmat22" bash scripts/gpu/ab.sh gpurun_out/g16_ab.log paper_2301_09125_b200/liblabelprop_cuda.so build/lib_wchain.so
LP_LIB_PATH=build/lib_wchain.so LP_DEBUG_ROUNDS=1 python scripts/ab_time.py --config rmat22w --batches 0 --runs 1 > gpurun_out/g16_dbg.log 2>&1
LP_LIB_PATH=build/lib_wchain.so timeout 900 python -m pytest tests/test_rak_gpu.py tests/test_fullsize_gpu.py -x -q -k "weight or rmat22 or exact" > gpurun_out/g16_tests.log 2>&1; echo tests rc $? >> gpurun_out/g16_ab.log
