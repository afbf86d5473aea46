# partial fusion A/B (LP_FUSE_MAXD) + parity
O=gpurun_out/g7_ab.log; : > $O
for c in rmat22 grid planted; do
for f in 0 16 64 -1; do LP_FUSE_MAXD=$f python scripts/ab_time.py --config $c --tag "fuse<=$f" >> $O 2>&1; done
done
LP_FUSE_MAXD=64 python scripts/ab_time.py --config rmat22 --non-strict --batches 0 --tag "fuse<=64" >> $O 2>&1
LP_FUSE_MAXD=0 python scripts/ab_time.py --config rmat22 --non-strict --batches 0 --tag "fuse<=0" >> $O 2>&1
timeout 900 python -m pytest tests/test_rak_gpu.py tests/test_fullsize_gpu.py tests/test_slpa_gpu.py -x -q > gpurun_out/g7_tests.log 2>&1; echo tests rc $? >> $O
