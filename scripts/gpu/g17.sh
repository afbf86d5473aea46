O=gpurun_out/g17_ab.log; : > $O
for w in 1 4 16 64; do
  for c in rmat22 rmat22w; do LP_WAVES1=$w LP_LIB_PATH=build/lib_waves1.so python scripts/ab_time.py --config $c --batches 0 --tag "waves1=$w" >> $O 2>&1; done
done
LP_WAVES1=16 LP_LIB_PATH=build/lib_waves1.so LP_DEBUG_ROUNDS=1 python scripts/ab_time.py --config rmat22w --batches 0 --runs 1 > gpurun_out/g17_dbg.log 2>&1
