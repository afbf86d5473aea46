timeout 600 python scripts/prof_run.py --config rmat22w --runs 12 --no-calibrate > gpurun_out/g41_prof_w.log 2>&1
cat gpurun_out/g41_prof_w.log | cut -c1-330
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv
