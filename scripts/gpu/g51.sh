O=gpurun_out/g51
LP_COPRA_WAVE0=16 LP_COPRA_WAVE_MAX=256 LP_COPRA_LONG=64 timeout 900 python -m pytest tests/test_copra_gpu.py -x -q -m gpu > ${O}_pytest_copra.log 2>&1; echo "pytest copra waves rc=$?"; tail -3 ${O}_pytest_copra.log
: > ${O}_copra.log
run() { echo "== $*" >> ${O}_copra.log; env "$@" timeout 600 python scripts/prof_mlp.py copra 8 0 20 2>&1 | grep -v "^\[lp\]" | tail -1 >> ${O}_copra.log; }
run LP_COPRA_LONG=0
run LP_COPRA_LONG=8192
run LP_COPRA_LONG=2048
run LP_COPRA_LONG=32768
run LP_COPRA_LONG=8192 LP_COPRA_WAVE0=1024 LP_COPRA_WAVE_MAX=65536
run LP_COPRA_LONG=8192 LP_COPRA_WAVE0=1024 LP_COPRA_WAVE_MAX=262144
run LP_COPRA_LONG=2048 LP_COPRA_WAVE0=1024 LP_COPRA_WAVE_MAX=65536
run LP_COPRA_LONG=8192 LP_COPRA_WAVE0=4096 LP_COPRA_WAVE_MAX=131072
echo "== sync" >> ${O}_copra.log
timeout 600 python scripts/prof_mlp.py copra 8 1 20 2>&1 | tail -1 >> ${O}_copra.log
cat ${O}_copra.log | cut -c1-260
