# A/B timing of engine knobs on R-MAT-22 (exact strict + synchronous), then the GPU parity suite.
# Usage: bash scripts/ab.sh "ENV1=.. ENV2=.." "ENV..." ...
mkdir -p gpurun_out
for cfg in "$@"; do
  echo "== $cfg" >> gpurun_out/ab.log
  env $cfg timeout 300 python scripts/prof_run.py --runs 4 --no-calibrate --config ${CONFIG:-rmat22} 2>&1 | grep -o "run 3: iterations.*kernel_ms [0-9.]*" >> gpurun_out/ab.log
  env $cfg timeout 300 python scripts/prof_run.py --runs 4 --no-calibrate --batches 1 2>&1 | grep -o "run 3: iterations.*kernel_ms [0-9.]*" >> gpurun_out/ab.log
  [ -n "$NONSTRICT" ] && env $cfg timeout 300 python scripts/prof_run.py --runs 3 --no-calibrate --non-strict 2>&1 | grep -o "run 2: iterations.*kernel_ms [0-9.]*" >> gpurun_out/ab.log
done
if [ -z "$SKIP_TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab.log; tail -3 gpurun_out/ab_pytest.log >> gpurun_out/ab.log; fi
cat gpurun_out/ab.log
