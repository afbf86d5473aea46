O=gpurun_out/g19_ab.log; : > $O
for rep in 1 2; do
python scripts/ab_time.py --config rmat22 --tag base >> $O 2>&1
LP_LIB_PATH=build/lib_few.so python scripts/ab_time.py --config rmat22 --tag few >> $O 2>&1
LP_HUB_BUCKET=1 LP_LIB_PATH=build/lib_few.so python scripts/ab_time.py --config rmat22 --tag few+bucket >> $O 2>&1
done
LP_LIB_PATH=build/lib_few.so python scripts/ab_time.py --config planted --tag few >> $O 2>&1
python scripts/ab_time.py --config planted --tag base >> $O 2>&1
LP_LIB_PATH=build/lib_few.so timeout 900 python -m pytest tests/test_rak_gpu.py tests/test_fullsize_gpu.py -x -q -k "rak or rmat22 or exact or planted or grid" > gpurun_out/g19_tests.log 2>&1; echo tests rc $? >> $O
