O=gpurun_out/g34
gcc -O3 -march=native -fopenmp -o /tmp/narrow scripts/bench_host/narrow.c && /tmp/narrow > ${O}_narrow.log 2>&1; cat ${O}_narrow.log
for W in 0 256 4096 65536; do
  echo "== WAVE0=$W" >> ${O}_copra.log
  LP_COPRA_WAVE0=$W LP_DEBUG_ROUNDS=1 timeout 600 python scripts/prof_mlp.py copra 8 0 20 >> ${O}_copra.log 2>&1
done
grep -v "^\[lp\]" ${O}_copra.log
LP_COPRA_WAVE0=64 timeout 900 python -m pytest tests/test_copra_gpu.py -x -q -m gpu > ${O}_pytest_copra.log 2>&1; echo "pytest copra waves rc=$?"; tail -3 ${O}_pytest_copra.log
timeout 600 python scripts/e2e_parts.py > ${O}_e2e.log 2>&1; cat ${O}_e2e.log
