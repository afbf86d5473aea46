O=gpurun_out/g59
timeout 900 python -m pytest tests/test_copra_gpu.py -x -q -m gpu > ${O}_pytest_copra.log 2>&1; echo "pytest copra rc=$?"; tail -3 ${O}_pytest_copra.log
: > ${O}_copra.log
for V in 1 0; do
for K in 1 8 16; do
  echo "== bitmap=$V K=$K" >> ${O}_copra.log
  LP_COPRA_BITMAP=$V timeout 600 python scripts/prof_mlp.py copra $K 0 20 2>&1 | tail -1 >> ${O}_copra.log
done
done
cat ${O}_copra.log | cut -c1-260
timeout 900 python -m pytest tests/test_fullsize_gpu.py -x -q -m gpu -k "copra or COPRA" > ${O}_pytest_full.log 2>&1; echo "pytest full rc=$?"; tail -3 ${O}_pytest_full.log
