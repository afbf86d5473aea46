O=gpurun_out/g49
timeout 1200 python -m pytest tests/test_slpa_gpu.py tests/test_rak_gpu.py -x -q -m gpu > ${O}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 ${O}_pytest.log
for A in 16777216 100000000; do
for T in 10 20; do
  echo "== LP_LOOP_DENSE_ARCS=$A T=$T" >> ${O}_slpa.log
  LP_LOOP_DENSE_ARCS=$A timeout 300 python scripts/prof_mlp.py slpa $T 0 >> ${O}_slpa.log 2>&1
done
done
echo "== loop off" >> ${O}_slpa.log
LP_LOOP_ROWS=0 timeout 300 python scripts/prof_mlp.py slpa 20 0 >> ${O}_slpa.log 2>&1
cat ${O}_slpa.log | cut -c1-250
timeout 900 python -m pytest tests/test_fullsize_gpu.py -x -q -m gpu -k "slpa or SLPA" > ${O}_pytest_full.log 2>&1; echo "pytest full rc=$?"; tail -3 ${O}_pytest_full.log
