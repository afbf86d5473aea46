CONFIGS="rmat22 grid planted" bash scripts/gpu/ab.sh gpurun_out/g18_ab.log paper_2301_09125_b200/liblabelprop_cuda.so build/lib_ppw.so
LP_LIB_PATH=build/lib_ppw.so timeout 900 python -m pytest tests/test_rak_gpu.py tests/test_fullsize_gpu.py tests/test_slpa_gpu.py -x -q > gpurun_out/g18_tests.log 2>&1; echo tests rc $? >> gpurun_out/g18_ab.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
LP_LIB_PATH=build/lib_ppw.so timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/g18_launches_b0.csv \
   python scripts/prof_run.py --batches 0 --runs 1 --no-calibrate > /dev/null 2>&1
