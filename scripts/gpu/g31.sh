# position-ordered waves for mid-sweep dense rounds (LP_WAVES_MID)
O=gpurun_out/g31_waves.log; : > $O
for W in 1 4 8 16 32; do
  LP_WAVES_MID=$W python scripts/ab_time.py --config rmat22w --runs 3 --batches 0 --tag "W=$W" >> $O 2>&1
  LP_WAVES_MID=$W python scripts/ab_time.py --config rmat22 --non-strict --runs 3 --batches 0 --tag "W=$W" >> $O 2>&1
  LP_WAVES_MID=$W python scripts/ab_time.py --config rmat22 --runs 3 --batches 0 --tag "W=$W" >> $O 2>&1
  LP_WAVES_MID=$W python scripts/ab_time.py --config planted --runs 3 --batches 0 --tag "W=$W" >> $O 2>&1
done
cat $O
