CONFIGS="rmat22 planted grid" bash scripts/gpu/ab.sh gpurun_out/g20_ab.log paper_2301_09125_b200/liblabelprop_cuda.so build/lib_wgrid.so build/lib_hubp.so
LP_LIB_PATH=build/lib_hubp.so timeout 900 python -m pytest tests/test_rak_gpu.py tests/test_fullsize_gpu.py tests/test_slpa_gpu.py -x -q > gpurun_out/g20_tests.log 2>&1; echo tests rc $? >> gpurun_out/g20_ab.log
