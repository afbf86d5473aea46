# fused small rows (no phase-1 pieces for them) + random-tie sweep frontier; full gpu tests
O=gpurun_out/g8_ab.log; : > $O
for c in rmat22 grid planted; do
for f in 0 16 -1; do LP_FUSE_MAXD=$f python scripts/ab_time.py --config $c --tag "fuse<=$f" >> $O 2>&1; done
done
python scripts/ab_time.py --config rmat22 --non-strict --tag "nonstrict" >> $O 2>&1
LP_SWEEP_FRONTIER=0 python scripts/ab_time.py --config rmat22 --non-strict --batches 0 --tag "nonstrict no-frontier" >> $O 2>&1
python scripts/ab_time.py --config planted --non-strict --tag "nonstrict" >> $O 2>&1
LP_DEBUG_ROUNDS=1 python scripts/ab_time.py --config rmat22 --non-strict --batches 0 --runs 1 > gpurun_out/g8_dbg_nonstrict.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g8_tests.log 2>&1; echo tests rc $? >> $O
