# tests + exact/sync profile runs + a short bench
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
timeout 900 python -m pytest tests/test_rak_gpu.py -x -q 2>&1 | tail -15
timeout 300 python scripts/prof_run.py 2>&1 | tail -40
timeout 300 python scripts/prof_run.py --batches 1 2>&1 | tail -25
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
