LP_LIB_PATH=build/lib_upl.so python scripts/e2e_parts.py > gpurun_out/g24_e2e_upl.log 2>&1
python scripts/e2e_parts.py > gpurun_out/g24_e2e_base.log 2>&1
LP_LIB_PATH=build/lib_upl.so timeout 900 python -m pytest tests/test_host_abi.py tests/test_rak_gpu.py tests/test_integration_binding.py -x -q > gpurun_out/g24_tests.log 2>&1; echo tests rc $? >> gpurun_out/g24_e2e_upl.log
LP_LIB_PATH=build/lib_upl.so timeout 900 python -m pytest tests/test_fullsize_gpu.py -x -q -k "float32 or grid" >> gpurun_out/g24_tests.log 2>&1; echo tests2 rc $? >> gpurun_out/g24_e2e_upl.log
