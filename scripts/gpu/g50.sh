O=gpurun_out/g50
LP_COPRA_WAVE0=16 LP_COPRA_WAVE_MAX=256 timeout 900 python -m pytest tests/test_copra_gpu.py -x -q -m gpu > ${O}_pytest_copra.log 2>&1; echo "pytest copra waves rc=$?"; tail -3 ${O}_pytest_copra.log
: > ${O}_copra.log
run() { echo "== $*" >> ${O}_copra.log; env "$@" timeout 600 python scripts/prof_mlp.py copra 8 0 20 2>&1 | grep -v "^\[lp\]" | tail -1 >> ${O}_copra.log; }
run LP_COPRA_WAVE0=0
run LP_COPRA_WAVE0=1024 LP_COPRA_WAVE_MAX=16384
run LP_COPRA_WAVE0=1024 LP_COPRA_WAVE_MAX=65536
run LP_COPRA_WAVE0=1024 LP_COPRA_WAVE_MAX=262144
run LP_COPRA_WAVE0=256 LP_COPRA_WAVE_MAX=65536
run LP_COPRA_WAVE0=8192 LP_COPRA_WAVE_MAX=32768
cat ${O}_copra.log | cut -c1-260
LP_COPRA_WAVE0=1024 LP_COPRA_WAVE_MAX=65536 LP_DEBUG_ROUNDS=1 timeout 600 python scripts/prof_mlp.py copra 8 0 20 2>&1 | grep "^\[lp\]" | head -150 > ${O}_dbg.log
