CONFIGS="rmat22 planted grid" bash scripts/gpu/ab.sh gpurun_out/g22_ab.log paper_2301_09125_b200/liblabelprop_cuda.so build/lib_hubp2.so
LP_LIB_PATH=build/lib_hubp2.so timeout 900 python -m pytest tests/test_rak_gpu.py tests/test_fullsize_gpu.py -x -q -k "rak or rmat22 or exact or planted or grid or polic" > gpurun_out/g22_tests.log 2>&1; echo tests rc $? >> gpurun_out/g22_ab.log
