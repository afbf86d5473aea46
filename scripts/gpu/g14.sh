CONFIGS="rmat22 planted grid" bash scripts/gpu/ab.sh gpurun_out/g14_ab.log paper_2301_09125_b200/liblabelprop_cuda.so build/lib_chain.so
LP_LIB_PATH=build/lib_chain.so LP_DEBUG_ROUNDS=1 python scripts/ab_time.py --batches 0 --runs 1 > gpurun_out/g14_dbg.log 2>&1
LP_LIB_PATH=build/lib_chain.so timeout 900 python -m pytest tests/test_rak_gpu.py tests/test_fullsize_gpu.py tests/test_integration_binding.py -x -q > gpurun_out/g14_tests.log 2>&1; echo tests rc $? >> gpurun_out/g14_ab.log
