CONFIGS="rmat22 planted" bash scripts/gpu/ab.sh gpurun_out/g12_ab.log build/lib_teampf.so build/lib_mid16.so
LP_LIB_PATH=build/lib_mid16.so timeout 900 python -m pytest tests/test_rak_gpu.py tests/test_fullsize_gpu.py tests/test_slpa_gpu.py -x -q > gpurun_out/g12_tests.log 2>&1; echo tests rc $? >> gpurun_out/g12_ab.log
