# A/B: round-1 build vs streaming hints vs hints + persisting L2 window; LP_WAVES for the exact schedule
O=gpurun_out/g5_ab.log; : > $O
LP_LIB_PATH=build/lib_base.so python scripts/ab_time.py >> $O 2>&1
LP_LIB_PATH=build/lib_nohints.so LP_L2_PERSIST=0 python scripts/ab_time.py --tag nohints-nowindow >> $O 2>&1
LP_LIB_PATH=build/lib_nohints.so python scripts/ab_time.py --tag nohints-window >> $O 2>&1
LP_L2_PERSIST=0 python scripts/ab_time.py --tag hints-nowindow >> $O 2>&1
python scripts/ab_time.py --tag hints-window >> $O 2>&1
for w in 2 4 8 16; do LP_WAVES=$w python scripts/ab_time.py --batches 0 --tag "hints-window waves=$w" >> $O 2>&1; done
python -c "
import ctypes; c=ctypes.CDLL('libcudart.so') if False else None
import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size)" >> $O 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/g5_launches_b1.csv \
   python scripts/prof_run.py --batches 1 --runs 1 --no-calibrate > /dev/null 2>&1
