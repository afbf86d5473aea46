set -x
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
timeout 900 python -m pytest tests/test_rak_gpu.py -x -q 2>&1 | tail -3
timeout 300 python scripts/prof_run.py --no-calibrate --runs 2 2>&1 | tail -5
timeout 300 python scripts/prof_run.py --no-calibrate --batches 1 2>&1 | tail -5
